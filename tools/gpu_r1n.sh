#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -x -k "amg or pressure or htree or next4 or graph or timing" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_cfg9.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
