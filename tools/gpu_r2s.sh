#!/bin/bash
TAG=${1:-r2s}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python tools/amg_sweep.py tools/sweep_r2s.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
