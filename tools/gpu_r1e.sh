#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python tools/op_ab.py c5 f64 DFVM_OPS_VARIANT 0 1 2 3 4 0 > $O/op_var.json 2> $O/op_var.err
DFVM_OPS_VARIANT=3 timeout 600 python tools/op_ab.py c5 f64 DFVM_LD3 1 0 1 > $O/op_ld3_v3.json 2> $O/op_ld3.err
timeout 1500 python tools/amg_sweep.py tools/sweep_cfg3.txt c5 - amg32 > $O/sweep.txt 2> $O/sweep.err
echo done
