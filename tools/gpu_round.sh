#!/bin/bash
# One gpurun call: GPU tests, bench lines, ncu full capture of the level-0
# kernels, optional launch list.  Usage (on the box):
#   bash tools/gpu_round.sh TAG [launches]
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_amg.json 2> $O/bench_amg.err
timeout 600 python bench.py --precond amg32 --no-cpu-baseline > $O/bench_amg32.json 2> $O/bench_amg32.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_amg_smooth|k_cg_spmv' \
  --launch-skip 20 --launch-count 4 -o $O/ncu_full_l0 -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/ncu_full.log 2>&1
if [ "$2" = "launches" ]; then
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
fi
echo done
