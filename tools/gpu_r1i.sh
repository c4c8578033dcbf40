#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_piso.py tests/test_gpu_next4.py tests/test_gpu_multirank.py -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python tools/amg_sweep.py tools/sweep_cfg6.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo done
