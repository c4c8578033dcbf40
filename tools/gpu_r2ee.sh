#!/bin/bash
O=gpurun_out/r2ee; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg_kernel_variants or large_coarsest or pressure_solve" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1500 python tools/amg_sweep.py tools/sweep_r2ee.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
