#!/bin/bash
TAG=${1:-r2n}
O=gpurun_out/$TAG
mkdir -p $O
DFVM_AMG_COARSE=4000 DFVM_AMG_DIRECT=4000 timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > $O/bench_lvl4.json 2> $O/bench_lvl4.err
