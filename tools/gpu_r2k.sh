#!/bin/bash
# GPU subset tests, bench line with profile, ncu --set full of the face-pass kernels
TAG=${1:-r2k}
O=gpurun_out/$TAG; T=/tmp/ncu_$TAG
mkdir -p $O $T
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -q -rf -k "piso or momentum or amg or next1 or transport" > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
ARGS="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-operators --no-profile"
DFVM_GRAPHS=0 timeout 900 $NCU --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:'k_transport_assemble|k_prhs|k_pcoef|k_Ucorr|k_HbyA' --launch-count 6 -o $T/ncu_face -f python bench.py $ARGS > $O/ncu_face.log 2>&1
$NCU -i $T/ncu_face.ncu-rep --page raw --csv > $T/ncu_face_raw.csv 2>/dev/null
python tools/ncu_summarize.py full $T/ncu_face_raw.csv $O/ncu_face_summary.csv
echo done
