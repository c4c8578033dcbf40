#!/bin/bash
TAG=${1:-r2j}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for c in c2 c3; do timeout 600 python tools/amg_sweep.py tools/sweep_r2j.txt $c > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; done
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
