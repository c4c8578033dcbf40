#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg or pressure or piso or multirank or adjoint or graph" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python tools/amg_sweep.py tools/sweep_cfg2.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
