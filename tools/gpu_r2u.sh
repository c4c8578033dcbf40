#!/bin/bash
O=gpurun_out/r2u; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "large_coarsest or amg_kernel_variants" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python tools/amg_sweep.py tools/sweep_r2u.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
