#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg or pressure or piso_steps or multirank or adjoint or htree or c3" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
DFVM_AMG_VERBOSE=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 1200 python tools/amg_sweep.py tools/sweep_cfg.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
