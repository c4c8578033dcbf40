#!/bin/bash
# tests touched this round + benches + ncu captures of the operator kernels
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q -rf -k "tail or pressure_solve or parity or c3 or htree" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --precond amg32 > $O/bench_amg32.json 2> $O/bench_amg32.err
timeout 600 python bench.py --precond amg --no-cpu-baseline > $O/bench_amg.json 2> $O/bench_amg.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_grad|k_lap|k_div|k_interp' \
  --launch-skip 5 --launch-count 5 -o $O/ncu_full_ops -f python tools/op_profile.py c5 f64 > $O/ncu_ops.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_amg_tail|k_amg_pre_resid' \
  --launch-skip 10 --launch-count 4 -o $O/ncu_full_tail -f \
  python bench.py --precond amg32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/ncu_tail.log 2>&1
echo done
