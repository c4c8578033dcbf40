#!/bin/bash
TAG=${1:-r2i}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg or programmatic or multislice or pressure_solve"  > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_r2i.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
