#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_piso.py -q -rf -x -k "momentum or bicg or cavity or pipe" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_cfg7.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
