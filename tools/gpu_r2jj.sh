#!/bin/bash
O=gpurun_out/r2jj; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
