"""AMG parameter sweep on one mesh in one process (the mesh is built once;
AmgParams are read from the environment when a solver builds its
hierarchy).  Times `steps` PISO steps after `warmup` per configuration.
usage: python tools/amg_sweep.py CONFIG_FILE [c5] [nz] [precond]
CONFIG_FILE lines: tag VAR=VALUE VAR=VALUE ..."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import cases  # noqa: E402
import paper_2603_15920_b200 as dfvm  # noqa: E402

cfgfile = sys.argv[1]
cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
nz = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
precond = sys.argv[4] if len(sys.argv) > 4 else "amg32"
steps, warmup = 3, 2
case = cases.c5(n_z=nz) if (cfg == "c5" and nz) else cases.CONFIGS[cfg]()
mesh = dfvm.Mesh(case.raw)
geo = mesh.export_geometry()
U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
B = case.apply_bcs(dfvm.BCs(mesh))
stream = torch.cuda.Stream()          # non-default: the library replays CUDA graphs there
torch.cuda.set_stream(stream)
import ctypes as C  # noqa: E402
sp = C.c_void_p(stream.cuda_stream)
keys = ["DFVM_AMG_COARSE", "DFVM_AMG_SWEEPS", "DFVM_AMG_CYCLE", "DFVM_AMG_WMAX", "DFVM_AMG_OMEGA",
        "DFVM_AMG_TAIL", "DFVM_AMG_DIRECT", "DFVM_AMG_SIGMA", "DFVM_AMG_GROUP", "DFVM_GRAPHS"]
for line in open(cfgfile):
    parts = line.split()
    if not parts or parts[0].startswith("#"):
        continue
    for k in [k for k in os.environ if k.startswith("DFVM_")]:
        os.environ.pop(k, None)
    for kv in parts[1:]:
        k, v = kv.split("=")
        os.environ[k] = v
    t0 = time.time()
    S = dfvm.Solver(mesh, B, **dict(case.solver, p_precond=precond))
    U, p, phi = mesh.field("cells", 3, U0, sp), mesh.field("cells", 1, p0, sp), mesh.field("flux", 1, phi0, sp)
    for _ in range(warmup):
        S.step(U, p, phi, sp)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    reps = [S.step(U, p, phi, sp) for _ in range(steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    its = [r["it"] for rep in reps for r in rep["p"]]
    bits = [r["it"] for rep in reps for r in rep["U"]]
    print(json.dumps({"tag": parts[0], "ms_per_step": round(ms, 2), "pcg_its": float(np.mean(its)),
                      "bicgstab_its": float(np.mean(bits)) if bits else None,
                      "levels": S.amg_levels(), "wall_s": round(time.time() - t0, 1)}), flush=True)
    del S, U, p, phi
