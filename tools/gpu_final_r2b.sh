#!/bin/bash
# Round-2 evidence in one gpurun call: GPU suite, smoke, the default bench
# line (C5 fp64) and the other bench lines, the reference arm, the launch
# list of one timed step, ncu --set full of the roofline kernel (traffic)
TAG=${1:-final}
O=gpurun_out/$TAG; T=/tmp/ncu_$TAG
mkdir -p $O $T
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/host.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
for c in c4 c3 c2 c1; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
DFVM_GRAPHS=0 timeout 1200 $NCU --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $T/launches.csv python bench.py $ARGS > $O/launches.log 2>&1
python tools/ncu_summarize.py launches $T/launches.csv $O/launches_summary.csv
gzip -c $T/launches.csv > $O/launches.csv.gz
DFVM_GRAPHS=0 timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_cg_spmv|k_amg_smooth_dot' --launch-count 4 -o $T/ncu_spmv -f python bench.py $ARGS > $O/ncu_spmv.log 2>&1
$NCU -i $T/ncu_spmv.ncu-rep --page raw --csv > $T/ncu_spmv_raw.csv 2>/dev/null
python tools/ncu_summarize.py full $T/ncu_spmv_raw.csv $O/ncu_spmv_summary.csv
echo done
