#!/bin/bash
# bench line with per-kernel profile, then ncu --set full of the coarse AMG
# kernels (levels 1-2: one thread per row), the BiCGStab kernels and k_prhs
# inside one timed C5 step (big files stay in /tmp on the box)
TAG=${1:-ncu2}
O=gpurun_out/$TAG
T=/tmp/ncu_$TAG
mkdir -p $O $T
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  --kernel-name-base demangled \
  -k regex:'k_amg_resid<1, float, float>|k_amg_smooth<1, float, float, float>|k_bi_t|k_bi_v|k_bi_x|k_prhs|k_amg_pre_resid<4|k_amg_prolong_smooth<4' \
  --launch-count 24 -o $T/ncu_full -f python bench.py $ARGS > $O/ncu_full.log 2>&1
$NCU -i $T/ncu_full.ncu-rep --page raw --csv > $T/ncu_full_raw.csv 2>/dev/null
python tools/ncu_summarize.py full $T/ncu_full_raw.csv $O/ncu_full_summary.csv
gzip -c $T/ncu_full_raw.csv > $O/ncu_full_raw.csv.gz
ls -la $O
echo done
