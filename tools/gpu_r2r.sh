#!/bin/bash
O=gpurun_out/r2r; mkdir -p $O
DFVM_AMG_COARSE=4000 DFVM_AMG_DIRECT=4000 timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_blk|k_dense_rows|k_negate' --launch-count 220 --log-file $O/blk.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile > $O/blk.log 2>&1
python tools/ncu_summarize.py launches $O/blk.csv $O/blk_summary.csv
