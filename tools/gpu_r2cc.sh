#!/bin/bash
O=gpurun_out/r2cc; mkdir -p $O
timeout 1500 python tools/amg_sweep.py tools/sweep_r2cc.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
