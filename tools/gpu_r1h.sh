#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_piso.py tests/test_gpu_next4.py -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_cfg5.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
echo done
