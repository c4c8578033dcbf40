import os, sys, ctypes
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2603_15920_b200 as dfvm
from test_gpu_piso import pipe_case, initial_state, TIGHT
raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
U0, p0, phi0 = initial_state(mo)
s = torch.cuda.Stream(); sp = ctypes.c_void_p(s.cuda_stream)
envs = [("P0F1", {"DFVM_AMG_PERM": "0", "DFVM_AMG_FUSED_FROM": "1"}), ("P0F1b", {"DFVM_AMG_PERM": "0", "DFVM_AMG_FUSED_FROM": "1"}),
        ("P1F1", {"DFVM_AMG_PERM": "1", "DFVM_AMG_FUSED_FROM": "1"}), ("P0F3", {"DFVM_AMG_PERM": "0", "DFVM_AMG_FUSED_FROM": "3"}),
        ("P1F3", {"DFVM_AMG_PERM": "1", "DFVM_AMG_FUSED_FROM": "3"})]
for prec in ("amg", "amg32"):
    out = {}
    for tag, env in envs:
        os.environ.update(env)
        S = dfvm.Solver(mg, bg, p_precond=prec, **kw, **TIGHT)
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [S.step(Ug, pg, phig, sp) for _ in range(2)]
        out[tag] = (pg.get(sp), [r["it"] for rep in reps for r in rep["p"]])
    for tag in out:
        print(prec, tag, out[tag][1], np.abs(out[tag][0] - out["P0F1"][0]).max())
