#!/bin/bash
TAG=${1:-r2h}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf  > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_r2h.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
