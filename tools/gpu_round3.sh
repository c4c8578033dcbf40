#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_piso.py -q -x -k "tail_bitwise and amg32" > $O/sanitizer.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -k "amg or pressure_solve or tail or coarsest or transport or piso_steps" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --precond amg32 > $O/bench_amg32.json 2> $O/bench_amg32.err
DFVM_AMG_DIRECT=0 timeout 600 python bench.py --precond amg32 --no-cpu-baseline --no-e2e --no-operators > $O/bench_amg32_sweeps.json 2> $O/bench_amg32_sweeps.err
timeout 600 python bench.py --precond amg --no-cpu-baseline --no-operators > $O/bench_amg.json 2> $O/bench_amg.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline --no-operators > $O/bench_f32.json 2> $O/bench_f32.err
echo done
