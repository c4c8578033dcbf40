mkdir -p gpurun_out/r2d
timeout 1200 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r2d/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2d/pytest_gpu.log
timeout 900 python tools/amg_sweep.py tools/sweep_r2d.txt c5 > gpurun_out/r2d/sweep.jsonl 2> gpurun_out/r2d/sweep.err
