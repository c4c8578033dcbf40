#!/bin/bash
# Round-2 GPU check in one gpurun call:
#   bash tools/gpu_r2.sh TAG [tests|notests] [VAR=VAL ... bench variants, ';'-separated]
# GPU suite (unless notests), smoke, the default bench line, then one bench
# line (no cpu baseline / e2e / operators) per variant environment.
TAG=${1:-r}
MODE=${2:-tests}
VARIANTS=${3:-}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
if [ "$MODE" = "tests" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rf -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
fi
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
i=0
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  i=$((i+1))
  env $v timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-operators > $O/bench_v$i.json 2> $O/bench_v$i.err
  echo "$v" > $O/bench_v$i.env
done
echo done
