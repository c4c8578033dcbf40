#!/bin/bash
O=gpurun_out/r2dd; mkdir -p $O
timeout 1500 python tools/amg_sweep.py tools/sweep_r2dd.txt c5 > $O/sweep.jsonl 2> $O/sweep.err
timeout 600 python tools/amg_sweep.py tools/sweep_r2dd.txt c3 > $O/sweep_c3.jsonl 2> $O/sweep_c3.err
