#!/bin/bash
# One gpurun call: GPU tests, default bench lines, ncu launch list + full
# capture of the dominant kernels.  Usage (on the box): bash tools/gpu_round.sh TAG
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_amg.json 2> $O/bench_amg.err
timeout 600 python bench.py --precision f32 --no-cpu-baseline > $O/bench_amg_f32.json 2> $O/bench_amg_f32.err
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:'k_amg_smooth|k_amg_resid|k_cg_spmv' \
  --launch-skip 60 --launch-count 9 -o $O/ncu_full_top -f \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches.log 2>&1
echo done
