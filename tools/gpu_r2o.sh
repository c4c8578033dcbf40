#!/bin/bash
TAG=${1:-r2o}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "large_coarsest or amg_coarsest or amg_kernel_variants" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python tools/amg_sweep.py tools/sweep_r2m.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
DFVM_AMG_COARSE=4000 DFVM_AMG_DIRECT=4000 timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > $O/bench_lvl4.json 2> $O/bench_lvl4.err
