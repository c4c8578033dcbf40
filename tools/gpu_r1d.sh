#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_piso.py tests/test_gpu_next4.py -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/op_ab.py c5 f64 > $O/op_ab.json 2> $O/op_ab.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:'k_grad|k_lap' \
  --launch-count 3 -o $O/ncu_ops -f python tools/op_profile.py c5 f64 > $O/ncu_ops.log 2>&1
echo done
