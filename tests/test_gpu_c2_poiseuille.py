"""C2 (BASELINE configs[1]: laminar pipe Poiseuille on the ~200k-cell
unstructured tet mesh "vs analytic profile"; SURVEY §8(c) pin (iv)
parabolic inlet): the CUDA path marched towards steady state, the axial
velocity profile and the pressure gradient compared with the analytic
Hagen-Poiseuille solution u_z = U_max (1 - r^2 / R^2), dp/dz = -4 nu U_max / R^2
(= -3.2 for U_max = 2, nu = 0.1, R = 0.5).  On skewed tets the scheme has no
convergence order (A-32), so the numbers are reported with bounds, not an
order; the measured values are written to gpurun_out/c2_poiseuille.json."""
import json
import os

import numpy as np
import pytest

import cases
import paper_2603_15920_b200 as dfvm

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c2_poiseuille_vs_analytic():
    case = cases.c2()
    mg = dfvm.Mesh(case.raw)
    g = mg.export_geometry()
    U0, p0, phi0 = case.initial_state(g["xc"], g["xf"], g["Sf"])
    B = case.apply_bcs(dfvm.BCs(mg))
    kw = dict(case.solver, p_precond="amg", p_tol=1e-10, p_rel_tol=0.0, U_tol=1e-10)
    S = dfvm.Solver(mg, B, **kw)
    U, p, phi = mg.field("cells", 3, U0), mg.field("cells", 1, p0), mg.field("flux", 1, phi0)
    dt = case.solver["dt"]
    prev = U0
    for n in range(1, 401):
        r = S.step(U, p, phi)
        assert not r["nonfinite"]
        if n % 100 == 0:
            cur = U.get()
            change = np.abs(cur - prev).max() / (100 * dt)
            prev = cur
    xc = g["xc"]
    Uh, ph = U.get(), p.get()
    R, umax, nu = 0.5, 2.0, 0.1
    rr = np.hypot(xc[:, 0], xc[:, 1])
    mid = (xc[:, 2] > 0.5) & (xc[:, 2] < 2.1)
    ua = umax * (1 - rr ** 2 / R ** 2)
    prof_rms = float(np.sqrt(np.mean((Uh[mid, 2] - ua[mid]) ** 2)) / umax)
    prof_max = float(np.abs(Uh[mid, 2] - ua[mid]).max() / umax)
    dpdz = float(np.polyfit(xc[mid, 2], ph[mid], 1)[0])
    exact = -4 * nu * umax / R ** 2
    flux_in = -sum(phi.get()[pt.start:pt.start + pt.n].sum() for pt in case.raw.patches if pt.name == "inlet")
    out = dict(cells=int(mg.N), steps=400, t=400 * dt, dpdz=dpdz, dpdz_exact=exact, dpdz_rel_err=abs(dpdz / exact - 1),
               profile_rms_rel=prof_rms, profile_max_rel=prof_max, final_dU_dt_inf=float(change),
               inlet_flux=float(flux_in), cont_err_max=r["cont_err_max"])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "c2_poiseuille.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(out)
    assert out["dpdz_rel_err"] <= 0.15, out
    assert prof_rms <= 0.05, out
    assert r["cont_err_max"] <= 1e-8
