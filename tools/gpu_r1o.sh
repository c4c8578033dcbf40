#!/bin/bash
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
for c in c4 c3 c2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --config c4 --precond jacobi --no-cpu-baseline --no-operators --no-e2e > $O/bench_c4_jacobi.json 2> $O/bench_c4_jacobi.err
echo done
