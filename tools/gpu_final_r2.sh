#!/bin/bash
# Round-2 evidence in one gpurun call: GPU suite, smoke, the default bench
# line (C5 fp64), fp32, the reference arm, and the other BASELINE configs.
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/host.txt
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --precision f32 --no-cpu-baseline > $O/bench_f32.json 2> $O/bench_f32.err
for c in c4 c3 c2 c1; do
  timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
echo done
