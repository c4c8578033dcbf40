mkdir -p gpurun_out/r2l
timeout 1500 python tools/amg_sweep.py tools/sweep_r2l.txt c5 > gpurun_out/r2l/sweep.jsonl 2> gpurun_out/r2l/sweep.err
