"""Mid-size parity tier: the C5
generator at n_z = 12 (737,280 tets, ~23k SELL slices, a 5-level AMG
hierarchy), i.e. the production grid shapes of the C5 bench (every warp over
several slices, full one-wave grids, the deep AMG W-cycle), against the
oracle:

* every operator (f64 and f32) and the momentum apply: live oracle applies;
* the pressure solve (Jacobi and amg32) and two PISO steps: the oracle needs
  ~6 minutes per tight step at this size, so its values were computed once by
  tools/gen_golden_mid.py (oracle only) and sampled into
  tests/golden/c5_nz12_mid.npz (every 97th cell, every 197th face, plus
  global norms); the comparison is relative L2 over the samples and of the
  norms, at the §8(c) converged-field bound 1e-8.
"""
import os

import numpy as np
import pytest

import cases
import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import TOL_OP, grad_scale, rel_l2, rel_op_err

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "c5_nz12_mid.npz")
TIGHT = dict(p_tol=1e-13, U_tol=1e-13, p_rel_tol=0.0, p_rel_tol_final=0.0, p_maxit=20000, U_maxit=2000)

_c = {}


def mid():
    if "case" not in _c:
        case = cases.c5(n_z=12)
        _c["case"] = case
        _c["mo"] = oracle.Mesh(case.raw)
    return _c["case"], _c["mo"]


def gpu_mesh(precision):
    key = "mg_" + precision
    if key not in _c:
        case, _ = mid()
        _c[key] = dfvm.Mesh(case.raw, precision=precision)
    return _c[key]


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_mid_operators(precision):
    case, mo = mid()
    mg = gpu_mesh(precision)
    raw = case.raw
    assert mg.info["sell_slices"] >= 20000
    tol = TOL_OP[precision]
    # gradients (scalar fixed / zeroGradient, vector)
    for fld, nc, kind in (("s", 1, oracle.BC_FIXED), ("U", 3, oracle.BC_FIXED), ("s", 1, oracle.BC_ZEROGRAD)):
        bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
        for p in raw.patches:
            bo.set(p.name, fld, kind, (0.3, -0.2, 0.1)); bg.set(p.name, fld, kind, (0.3, -0.2, 0.1))
        x = synth.cell_field(100, mo.N, nc)
        ref = mo.grad(bo, fld, x)
        G = mg.field("cells", 3 * nc)
        dfvm.grad(mg, mg.field("cells", nc, x), bg, fld, G)
        assert rel_op_err(G.get().reshape(ref.shape), ref, grad_scale(mo, mo.interpolate(bo, fld, x), nc)) <= tol
    # divergence
    F = synth.face_field(300, mo.NF)
    out = mg.field("cells", 1)
    dfvm.div(mg, mg.field("flux", 1, F), out)
    scale = np.zeros(mo.N)
    np.add.at(scale, mo.owner, np.abs(F)); np.add.at(scale, mo.neighbour, np.abs(F[:mo.F]))
    assert rel_op_err(out.get(), mo.div(F), scale) <= tol
    # interpolation
    bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
    for p in raw.patches:
        bo.set(p.name, "U", oracle.BC_FIXED, (1.0, 2.0, 3.0)); bg.set(p.name, "U", oracle.BC_FIXED, (1.0, 2.0, 3.0))
    x3 = synth.cell_field(100, mo.N, 3)
    ref = mo.interpolate(bo, "U", x3)
    xf = mg.field("faces", 3)
    dfvm.interpolate(mg, mg.field("cells", 3, x3), bg, "U", xf)
    assert np.abs(xf.get() - ref).max() <= (1e-14 if precision == "f64" else 1e-6) * np.abs(ref).max()
    # Laplacian with gamma, fixed + zeroGradient patches
    bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
    for i, p in enumerate(raw.patches):
        k = oracle.BC_FIXED if i != 2 else oracle.BC_ZEROGRAD
        bo.set(p.name, "s", k, (0.7, 0, 0)); bg.set(p.name, "s", k, (0.7, 0, 0))
    x = synth.cell_field(100, mo.N)
    gam = 1.0 + 0.5 * synth.cell_field(200, mo.N)
    y, ya = mo.laplacian(bo, "s", x, gamma=gam)
    out = mg.field("cells", 1)
    dfvm.laplacian(mg, bg, "s", mg.field("cells", 1, x), out, gamma=mg.field("cells", 1, gam))
    assert rel_op_err(out.get(), y, ya) <= tol


def test_mid_momentum_apply():
    case, mo = mid()
    mg = gpu_mesh("f64")
    So = oracle.Solver(mo, case.apply_bcs(oracle.BCs(mo)), **case.solver)
    Sg = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), **case.solver)
    U = synth.cell_field(40, mo.N, 3)
    phi = 0.01 * synth.face_field(41, mo.NF)
    diag, lo, up, b = So.momentum_assemble(U, phi)
    dg, bgf = mg.field("cells", 1), mg.field("cells", 3)
    Sg.momentum_assemble(mg.field("cells", 3, U), mg.field("flux", 1, phi), dg, bgf)
    assert rel_l2(dg.get(), diag) <= 1e-13 and rel_l2(bgf.get(), b) <= 1e-12
    x = synth.cell_field(50, mo.N, 3)
    y = mg.field("cells", 3)
    Sg.momentum_apply(mg.field("cells", 3, x), y)
    ref = np.stack([mo.ldu_apply(diag, lo, up, x[:, k]) for k in range(3)], 1)
    scale = np.stack([mo.ldu_apply(np.abs(diag), np.abs(lo), np.abs(up), np.abs(x[:, k])) for k in range(3)], 1)
    assert rel_op_err(y.get(), ref, scale) <= 1e-12


@pytest.mark.parametrize("precond", ["jacobi", "amg32"])
def test_mid_pressure_solve(precond):
    case, mo = mid()
    g = np.load(GOLD)
    mg = gpu_mesh("f64")
    Sg = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), p_precond=precond, **dict(case.solver, **TIGHT))
    N = mo.N
    rAU = 1e-3 * (1.5 + 0.5 * synth.cell_field(60, N))
    rhs = 1e-6 * synth.cell_field(61, N)
    pg = mg.field("cells", 1, synth.cell_field(62, N))
    r = Sg.pressure_solve(mg.field("cells", 1, rAU), mg.field("cells", 1, rhs), pg, tol=1e-13)
    assert r["converged"], r
    p = pg.get()
    cs = int(g["cell_stride"])
    assert rel_l2(p[::cs], g["psolve_p"]) <= 1e-8
    assert abs(np.linalg.norm(p) / float(g["psolve_norm"]) - 1) <= 1e-8
    if precond == "amg32":
        assert len(Sg.amg_levels()) >= 4, Sg.amg_levels()
        assert r["it"] < int(g["psolve_it"]) / 10


def test_mid_piso_two_steps():
    case, mo = mid()
    g = np.load(GOLD)
    mg = gpu_mesh("f64")
    Sg = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), **dict(case.solver, p_precond="amg32", **TIGHT))
    geo = mg.export_geometry()
    U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
    U, p, phi = mg.field("cells", 3, U0), mg.field("cells", 1, p0), mg.field("flux", 1, phi0)
    cs, fs = int(g["cell_stride"]), int(g["face_stride"])
    for k in (1, 2):
        r = Sg.step(U, p, phi)
        assert r["cont_err_max"] <= 1e-10
        Uh, ph, fh = U.get(), p.get(), phi.get()
        assert rel_l2(Uh[::cs], g[f"step{k}_U"]) <= 1e-8
        assert rel_l2(ph[::cs], g[f"step{k}_p"]) <= 1e-8
        assert rel_l2(fh[::fs], g[f"step{k}_phi"]) <= 1e-8
        nrm = np.array([np.linalg.norm(Uh), np.linalg.norm(ph), np.linalg.norm(fh)])
        assert np.abs(nrm / g[f"step{k}_norms"] - 1).max() <= 1e-8
