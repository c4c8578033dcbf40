"""Writes tests/golden/c5_nz12_mid.npz: oracle-only expected values of the
mid-size parity tier: the C5 generator
at n_z = 12 (737,280 tets), where the CUDA path runs production grid shapes
(~23k SELL slices, every warp over several slices, a >= 4-level AMG W-cycle).

Calls only oracle/ (and the seeded generators of synth/ / cases.py): no value
here comes from the CUDA path.  The oracle needs ~6 minutes per tight PISO
step at this size, so the expected values are computed once by this script
and sampled (every 97th cell, every 197th face) plus global norms.

    python tools/gen_golden_mid.py        # ~15 min, single core
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import cases  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c5_nz12_mid.npz")
TIGHT = dict(p_tol=1e-13, U_tol=1e-13, p_rel_tol=0.0, p_rel_tol_final=0.0, p_maxit=20000, U_maxit=2000)
CS, FS = 97, 197     # cell / face sampling strides


def main():
    t0 = time.time()
    case = cases.c5(n_z=12)
    m = oracle.Mesh(case.raw)
    b = case.apply_bcs(oracle.BCs(m))
    kw = dict(case.solver)
    kw.update(TIGHT)
    S = oracle.Solver(m, b, **kw)
    out = dict(N=m.N, NF=m.NF, cell_stride=CS, face_stride=FS)
    # pressure solve with seeded rAU / rhs / warm start (test_gpu_midsize.py uses the same recipe)
    rAU = 1e-3 * (1.5 + 0.5 * synth.cell_field(60, m.N))
    rhs = 1e-6 * synth.cell_field(61, m.N)
    p0 = synth.cell_field(62, m.N)
    ps, rep = S.pressure_solve(rAU, rhs, p0=p0, tol=1e-13)
    assert rep["converged"], rep
    out.update(psolve_p=ps[::CS], psolve_norm=np.linalg.norm(ps), psolve_it=rep["it"])
    print("pressure solve", rep, time.time() - t0, flush=True)
    # two PISO steps from the C5 initial condition
    U, p, phi = case.initial_state(m.xc, m.xf, m.Sf)
    for k in range(2):
        r = S.step(U, p, phi)
        print("step", k + 1, [x["it"] for x in r["p"]], [x["it"] for x in r["U"]], r["cont_err_max"],
              time.time() - t0, flush=True)
        out[f"step{k + 1}_U"] = U[::CS].copy()
        out[f"step{k + 1}_p"] = p[::CS].copy()
        out[f"step{k + 1}_phi"] = phi[::FS].copy()
        out[f"step{k + 1}_norms"] = np.array([np.linalg.norm(U), np.linalg.norm(p), np.linalg.norm(phi)])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, time.time() - t0)


if __name__ == "__main__":
    main()
