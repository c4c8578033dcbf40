#!/bin/bash
# Launch list of one timed step + ncu --set full of the roofline kernels (the
# last two passes of gpu_final.sh), for refreshing profiles/ at a new head.
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
DFVM_GRAPHS=0 timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_cg_spmv|k_amg_smooth|k_bi_t|k_grad|k_amg_prolong_smooth' --launch-skip 2 --launch-count 6 -o $O/ncu_full_step -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/ncu_full.log 2>&1
echo done
