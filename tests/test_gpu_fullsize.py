"""Full-size checks at BASELINE.json's C5 size (50 012 160 tets, the mesh
bench.py times), in the same launch configuration:

* sampled operator parity: the oracle cannot hold the 50M-cell mesh, but the
  first axial layers of C5 are geometrically identical to those of a short
  pipe with the same cross-section and axial spacing.  Gradient and Laplacian
  of a smooth field are compared cell by cell on the first layers (matched
  by centroid, away from the short pipe's outlet) at the operator tolerance.
* properties that hold at any size: the uniform-flow PISO fixed point and
  discrete continuity after a PISO step.
"""
import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import rel_op_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NZ_SHORT = 6
R, L_FULL, NZ_FULL = 0.5, 10.0, 814


@pytest.fixture(scope="module")
def c5():
    raw = synth.pipe_c5()
    assert raw.n_cells == 50012160
    return raw, dfvm.Mesh(raw)


def _field(xc):
    return np.sin(7.0 * xc[:, 0]) * np.cos(5.0 * xc[:, 1]) + 0.3 * xc[:, 2]


def _bcs_pair(raw_o, mo, mg):
    bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
    for b in (bo, bg):
        b.set("inlet", "s", 0, 0.5)
        b.set("wall", "s", 1)
        b.set("outlet", "s", 0, 0.0)
    return bo, bg


def test_sampled_operator_parity_first_layers(c5):
    raw, mg = c5
    short = synth.pipe(64, 32, NZ_SHORT, R, L_FULL * NZ_SHORT / NZ_FULL, tets=True, scramble=3)
    mo = oracle.Mesh(short)
    bo, bg = _bcs_pair(short, mo, mg)
    geo = mg.export_geometry()
    xg = geo["xc"]
    dz = L_FULL / NZ_FULL
    zmax = (NZ_SHORT - 3) * dz            # two layers clear of the short pipe's outlet
    sel_g = np.nonzero(xg[:, 2] < zmax)[0]
    sel_o = np.nonzero(mo.xc[:, 2] < zmax)[0]
    assert len(sel_g) == len(sel_o) > 100000
    # match cells by centroid (nearest neighbour; rounding-to-grid keys can
    # split two sides' 1e-16-different centroids across a grid line)
    from scipy.spatial import cKDTree
    dist, j = cKDTree(mo.xc[sel_o]).query(xg[sel_g])
    og, oo = sel_g, sel_o[j]
    assert len(np.unique(j)) == len(sel_o)
    assert dist.max() <= 1e-12
    # gradient
    Go = mo.grad(bo, "s", _field(mo.xc))
    xf = mg.field("cells", 1, _field(xg))
    Gg = mg.field("cells", 3)
    dfvm.grad(mg, xf, bg, "s", Gg)
    Gg = Gg.get()
    scale = np.abs(Go[oo]).max() + 1.0
    assert np.abs(Gg[og] - Go[oo]).max() <= 1e-11 * scale
    # Laplacian (over-relaxed correction with the Gauss gradient)
    yo, yabs = mo.laplacian(bo, "s", _field(mo.xc))
    yg = mg.field("cells", 1)
    dfvm.laplacian(mg, bg, "s", xf, yg)
    assert rel_op_err(yg.get()[og], yo[oo], yabs[oo]) <= 1e-11


def test_uniform_flow_fixed_point_full_size(c5):
    raw, mg = c5
    U0 = np.array([0.0, 0.0, 1.0])
    b = dfvm.BCs(mg)
    b.set("inlet", "U", dfvm.BC_FIXED, U0); b.set("wall", "U", dfvm.BC_FIXED, U0)
    b.set("outlet", "U", dfvm.BC_ZEROGRAD)
    b.set("inlet", "p", dfvm.BC_ZEROGRAD); b.set("wall", "p", dfvm.BC_ZEROGRAD)
    b.set("outlet", "p", dfvm.BC_FIXED, 0.0)
    S = dfvm.Solver(mg, b, nu=0.01, dt=0.001, n_corr=2, n_nonorth=1, p_precond="amg", p_tol=1e-10, U_tol=1e-10,
                    p_maxit=2000, U_maxit=200)
    geo = mg.export_geometry()
    U = mg.field("cells", 3, np.tile(U0, (raw.n_cells, 1)))
    p = mg.field("cells", 1)
    phi = mg.field("flux", 1, geo["Sf"] @ U0)
    r = S.step(U, p, phi)
    assert np.abs(U.get() - U0).max() <= 1e-10 and np.abs(p.get()).max() <= 1e-10
    assert not r["nonfinite"]


def test_piso_step_continuity_full_size(c5):
    import cases
    raw, mg = c5
    case = cases.c5()
    geo = mg.export_geometry()
    U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
    S = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), **dict(case.solver, p_precond="amg"))
    U, p, phi = mg.field("cells", 3, U0), mg.field("cells", 1, p0), mg.field("flux", 1, phi0)
    r = S.step(U, p, phi)
    assert not r["nonfinite"] and all(x["converged"] for x in r["p"])
    # final corrector solved to 1e-6 ||b||: per-cell continuity far below the flux scale
    flux_scale = np.abs(phi0).max()
    assert r["cont_err_max"] <= 1e-6 * flux_scale
