#!/bin/bash
TAG=${1:-r2m}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg or pressure_solve or cavity" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python tools/amg_sweep.py tools/sweep_r2m.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
timeout 600 python tools/amg_sweep.py tools/sweep_r2m.txt c4 > $O/sweep_c4.jsonl 2> $O/sweep_c4.err
