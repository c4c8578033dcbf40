#!/bin/bash
TAG=${1:-r2f}
O=gpurun_out/$TAG; T=/tmp/ncu_$TAG
mkdir -p $O $T
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q -rf -k "sigma_storage or amg_kernel_variants or amg_coarsest or graph_replay or multislice" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_r2f.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
for spec in "resid:k_amg_resid:8" "smooth:k_amg_smooth:6"; do
  IFS=: read nm rx cnt <<< "$spec"
  DFVM_GRAPHS=0 timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
    -k regex:"$rx" --launch-count $cnt -o $T/ncu_$nm -f python bench.py $ARGS > $O/ncu_$nm.log 2>&1
  $NCU -i $T/ncu_$nm.ncu-rep --page raw --csv > $T/ncu_${nm}_raw.csv 2>/dev/null
  python tools/ncu_summarize.py full $T/ncu_${nm}_raw.csv $O/ncu_${nm}_summary.csv
  gzip -c $T/ncu_${nm}_raw.csv > $O/ncu_${nm}_raw.csv.gz
done
echo done
