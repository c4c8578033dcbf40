#!/bin/bash
# GPU suite + a sweep file on C5 (one gpurun call): bash tools/gpu_r2e.sh TAG SWEEPFILE
TAG=${1:-r2e}; SW=${2:-tools/sweep_r2e.txt}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/$TAG/pytest_gpu.log
timeout 900 python tools/amg_sweep.py $SW c5 > gpurun_out/$TAG/sweep.jsonl 2> gpurun_out/$TAG/sweep.err
