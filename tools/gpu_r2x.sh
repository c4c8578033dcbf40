#!/bin/bash
O=gpurun_out/r2x; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "piso or momentum or transport or next1 or adjoint or cavity or multirank" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > $O/bench.json 2> $O/bench.err
