mkdir -p gpurun_out
run() { tag=$1; shift; env "$@" timeout 400 python bench.py --config c5 --nz $NZ --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --precond amg > gpurun_out/sw_${NZ}_$tag.json 2> gpurun_out/sw_${NZ}_$tag.err; python -c "
import json; d=json.loads(open('gpurun_out/sw_${NZ}_$tag.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$NZ $tag', 'ms/step %.1f'%d['ms_per_step'], 'its %.1f'%d['krylov']['pcg_iterations_per_solve'], 'it_ms %.3f'%r['pcg_iteration_ms'], 'launches', d['gpu_launches'])" >> gpurun_out/sweep2.txt 2>&1; }
NZ=102
run V2048w15 DFVM_AMG_CYCLE=V DFVM_AMG_COARSE=2048 DFVM_AMG_SWEEPS=24 DFVM_AMG_OMEGA=1.5
run V2048w18 DFVM_AMG_CYCLE=V DFVM_AMG_COARSE=2048 DFVM_AMG_SWEEPS=24 DFVM_AMG_OMEGA=1.8
NZ=814
run V2048 DFVM_AMG_CYCLE=V DFVM_AMG_COARSE=2048 DFVM_AMG_SWEEPS=24
run V2048w15 DFVM_AMG_CYCLE=V DFVM_AMG_COARSE=2048 DFVM_AMG_SWEEPS=24 DFVM_AMG_OMEGA=1.5
run W4 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=4 DFVM_AMG_COARSE=256
run W5 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=5 DFVM_AMG_COARSE=256
run W4w15 DFVM_AMG_CYCLE=W DFVM_AMG_WMAX=4 DFVM_AMG_COARSE=256 DFVM_AMG_OMEGA=1.5
cat gpurun_out/sweep2.txt
