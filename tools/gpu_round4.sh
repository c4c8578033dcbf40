#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
DFVM_AMG_VERBOSE=1 timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_grad|k_lap' \
  --launch-skip 5 --launch-count 4 -o $O/ncu_full_ops -f python tools/op_profile.py c5 f64 > $O/ncu_ops.log 2>&1
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
echo done
