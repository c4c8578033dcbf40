"""PCG iterations per pressure solve at P = 1, 2, 4, 8 ranks on ONE GPU
(VERDICT round 1, item 6): the partitioned solver path through the
library's in-process communicator (ranks = host threads, same kernels, halo
slices and rank-order reductions as the NCCL path).  Timings here are not
scaling numbers (the ranks share one GPU); the iteration counts are what
strong scaling depends on.

    python tools/scale_iters.py [n_z] [precond] [P ...]
"""
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cases  # noqa: E402
import paper_2603_15920_b200 as dfvm  # noqa: E402


def run(case, P, precond, steps=3):
    import torch
    torch.cuda.set_device(0)
    comms = dfvm.Comm.local_group(P) if P > 1 else [None]
    ms = [dfvm.Mesh(case.raw, n_parts=P, rank=r, comm=comms[r]) for r in range(P)]
    geo = ms[0].export_geometry()
    U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
    st = []
    for m in ms:
        B = case.apply_bcs(dfvm.BCs(m))
        S = dfvm.Solver(m, B, **dict(case.solver, p_precond=precond))
        st.append((B, S, m.field("cells", 3, U0), m.field("cells", 1, p0), m.field("flux", 1, phi0)))
    streams = [torch.cuda.Stream() for _ in range(P)]
    sp = [dfvm.C.c_void_p(s.cuda_stream) for s in streams]
    reps = [[] for _ in range(P)]
    errs = []

    def work(r):
        try:
            for _ in range(steps):
                reps[r].append(st[r][1].step(st[r][2], st[r][3], st[r][4], stream=sp[r]))
        except Exception as e:
            errs.append(e)
    t0 = time.time()
    ts = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    its = [x["it"] for rep in reps[0] for x in rep["p"]]
    lv = st[0][1].amg_levels() if precond != "jacobi" else []
    return dict(P=P, pcg_its=its, mean=float(np.mean(its)), bicgstab=[x["it"] for x in reps[0][-1]["U"]],
                amg_levels_rank0=lv, wall_s=time.time() - t0, cont=reps[0][-1]["cont_err_max"])


def main():
    n_z = int(sys.argv[1]) if len(sys.argv) > 1 else 204
    precond = sys.argv[2] if len(sys.argv) > 2 else "amg32"
    Ps = [int(x) for x in sys.argv[3:]] or [1, 2, 4, 8]
    case = cases.c5(n_z=n_z)
    out = {"case": case.name, "cells": case.raw.n_cells, "precond": precond, "runs": []}
    for P in Ps:
        r = run(case, P, precond)
        print(json.dumps(r), flush=True)
        out["runs"].append(r)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
