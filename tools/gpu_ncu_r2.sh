#!/bin/bash
# ncu evidence of round 2 (one gpurun call):
#  1. launch list of one timed C5 step (gpu__time_duration per launch,
#     cold-cache serialised; DFVM_GRAPHS=0 so every kernel is a plain launch)
#  2. ncu --set full of the kernels the per-kernel table ranks highest:
#     k_cg_spmv, k_amg_smooth_dot, k_amg_resid (level 0), k_amg_prolong_smooth /
#     k_amg_pre_resid (levels 1-2), k_bi_v / k_bi_t / k_bi_x
TAG=${1:-ncu}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py $ARGS > $O/launches.log 2>&1
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_cg_spmv|k_amg_smooth_dot|k_amg_prolong_smooth|k_amg_pre_resid|k_bi_v|k_bi_t|k_bi_x|k_amg_resid' \
  --launch-count 24 -o $O/ncu_full -f python bench.py $ARGS > $O/ncu_full.log 2>&1
$NCU -i $O/ncu_full.ncu-rep --page raw --csv > $O/ncu_full_raw.csv 2>/dev/null
echo done
