#!/bin/bash
# ncu evidence of round 2 (one gpurun call; big files stay in /tmp on the box,
# compact summaries come back in gpurun_out/TAG):
#  1. launch list of one timed C5 step (gpu__time_duration per launch,
#     cold-cache serialised; DFVM_GRAPHS=0 so every kernel is a plain launch),
#     summed per kernel name + grid (launches_summary.csv) and gzipped raw
#  2. ncu --set full of the kernels the per-kernel table ranks highest
#     (k_cg_spmv, k_amg_smooth_dot, k_amg_resid / k_amg_smooth (levels 0-2),
#     k_bi_v / k_bi_t / k_bi_x), selected metrics exported per launch
TAG=${1:-ncu}
O=gpurun_out/$TAG
T=/tmp/ncu_$TAG
mkdir -p $O $T
NCU=/usr/local/cuda/bin/ncu
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
DFVM_GRAPHS=0 timeout 1200 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches.csv python bench.py $ARGS > $O/launches.log 2>&1
python tools/ncu_summarize.py launches $T/launches.csv $O/launches_summary.csv
gzip -c $T/launches.csv > $O/launches.csv.gz
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_cg_spmv|k_amg_smooth_dot|k_amg_resid|k_amg_smooth|k_bi_v|k_bi_t|k_bi_x' \
  --launch-count 16 -o $T/ncu_full -f python bench.py $ARGS > $O/ncu_full.log 2>&1
$NCU -i $T/ncu_full.ncu-rep --page raw --csv > $T/ncu_full_raw.csv 2>/dev/null
python tools/ncu_summarize.py full $T/ncu_full_raw.csv $O/ncu_full_summary.csv
ls -la $O
echo done
