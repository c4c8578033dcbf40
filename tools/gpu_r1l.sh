#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 python tools/amg_sweep.py tools/sweep_cfg8.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
