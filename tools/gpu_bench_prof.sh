#!/bin/bash
# default bench line (C5 fp64) with its per-kernel profile table, optional extra env per run
TAG=${1:-bp}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/smi.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
DFVM_BI_T=2 timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > gpurun_out/$TAG/bench_bit2.json 2> gpurun_out/$TAG/bench_bit2.err
