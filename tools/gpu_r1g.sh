#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_piso.py tests/test_gpu_next4.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_cg_spmv|k_bi_t|k_amg_smooth|k_amg_resid$' \
  --launch-skip 30 --launch-count 4 -o $O/ncu_full_step -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/ncu_full.log 2>&1
echo done
