#!/bin/bash
O=gpurun_out/r2bb; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "large_coarsest or amg_kernel_variants or overlap or pressure_solve" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_blk|k_dense_rows|k_mirror' --launch-count 230 --log-file $O/blk.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile > $O/blk.log 2>&1
python tools/ncu_summarize.py launches $O/blk.csv $O/blk_summary.csv
