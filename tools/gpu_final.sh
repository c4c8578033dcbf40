#!/bin/bash
# Full round-end evidence in one gpurun call: GPU suite, smoke, bench lines,
# launch list of one timed step, ncu --set full of the roofline kernels.
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
DFVM_GRAPHS=0 timeout 1500 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
DFVM_GRAPHS=0 timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_cg_spmv|k_amg_smooth|k_bi_t|k_grad|k_amg_prolong_smooth' --launch-skip 2 --launch-count 6 -o $O/ncu_full_step -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/ncu_full.log 2>&1
echo done
