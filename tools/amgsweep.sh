mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py 2>&1 | tail -6 > gpurun_out/tests.log
run() { tag=$1; shift; env "$@" timeout 400 python bench.py --config c5 --nz $NZ --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --precond amg > gpurun_out/sw_${NZ}_$tag.json 2> gpurun_out/sw_${NZ}_$tag.err; python -c "
import json; d=json.loads(open('gpurun_out/sw_${NZ}_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$NZ $tag', 'ms/step %.1f'%d['ms_per_step'], 'its %.1f'%d['krylov']['pcg_iterations_per_solve'], 'it_ms %.3f'%r['pcg_iteration_ms'], 'launches', d['gpu_launches'], r['kernel'].split()[0], 'GB/s %.0f'%r['achieved'], 'lv', r['amg_levels'])" >> gpurun_out/sweep3.txt 2>&1; }
for NZ in 102 814; do
run V18 DFVM_AMG_CYCLE=V DFVM_AMG_COARSE=2048 DFVM_AMG_SWEEPS=24 DFVM_AMG_OMEGA=1.8
run W4w15 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=4 DFVM_AMG_COARSE=256 DFVM_AMG_OMEGA=1.5
run W4w17 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=4 DFVM_AMG_COARSE=256 DFVM_AMG_OMEGA=1.7
run W4w19 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=4 DFVM_AMG_COARSE=256 DFVM_AMG_OMEGA=1.9
run W2w17 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=2 DFVM_AMG_COARSE=256 DFVM_AMG_OMEGA=1.7
done
cat gpurun_out/tests.log gpurun_out/sweep3.txt
