#!/bin/bash
# One gpurun call: full GPU test suite, smoke(), default bench line, launch list.
#   bash tools/gpu_check.sh TAG [launches]
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
if [ "$2" = "launches" ]; then
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators > $O/launches.log 2>&1
fi
echo done
