"""Oracle pins for O-7 solvers, O-8 Windkessel, E1 Poisson and the
O-5/O-6 PISO step (SURVEY.md §8(c) pin rows O-7, O-8, E1, O-5/O-6, C1)."""
import math

import numpy as np
import pytest

import oracle
import synth


# --------------------------------------------------------------- O-7
def test_cg_two_by_two():
    # [[4,1],[1,3]] x = [1,2] -> [1/11, 7/11]  (LDU on the two-cube mesh)
    m = oracle.Mesh(synth.fixture_two_boxes(1.0))
    for mode in ("cg", "bicgstab", "lu"):
        x, r = m.ldu_solve([4.0, 3.0], [1.0], [1.0], [1.0, 2.0], mode=mode, tol=1e-15)
        assert np.allclose(x, [1 / 11, 7 / 11], atol=1e-15), (mode, x)


def test_identity_one_iteration_and_zero_rhs():
    m = oracle.Mesh(synth.box(3, 3, 3))
    b = synth.cell_field(5, m.N)
    x, r = m.ldu_solve(np.ones(m.N), np.zeros(m.F), np.zeros(m.F), b, mode="cg")
    assert r["it"] <= 1 and np.allclose(x, b, atol=1e-15)
    x, r = m.ldu_solve(np.ones(m.N), np.zeros(m.F), np.zeros(m.F), np.zeros(m.N), x0=b, mode="cg")
    assert r["it"] == 0 and np.all(x == 0)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_krylov_vs_dense_random_graph_laplacians(seed):
    # random SPD graph Laplacians (n <= 50) -> CG = LU; nonsymmetric
    # diagonally dominant -> BiCGStab = LU
    m = oracle.Mesh(synth.box(3, 4, 3, split=0, scramble=seed))
    rng = np.random.default_rng(seed)
    wgt = rng.uniform(0.1, 2.0, m.F)
    diag = np.zeros(m.N)
    np.add.at(diag, m.owner[:m.F], wgt)
    np.add.at(diag, m.neighbour, wgt)
    diag += rng.uniform(0.01, 0.1, m.N)
    b = rng.standard_normal(m.N)
    xl, _ = m.ldu_solve(diag, -wgt, -wgt, b, mode="lu")
    xc, r = m.ldu_solve(diag, -wgt, -wgt, b, mode="cg", tol=1e-15)
    assert r["converged"] and np.abs(xc - xl).max() <= 1e-12 * np.abs(xl).max()
    up = -wgt * rng.uniform(0.2, 1.0, m.F)
    lo = -wgt * rng.uniform(0.2, 1.0, m.F)
    xl, _ = m.ldu_solve(diag, lo, up, b, mode="lu")
    xb, r = m.ldu_solve(diag, lo, up, b, mode="bicgstab", tol=1e-15)
    assert r["converged"] and np.abs(xb - xl).max() <= 1e-12 * np.abs(xl).max()


# --------------------------------------------------------------- O-8
def test_windkessel_worked_example(golden):
    g = golden("windkessel.json")["example"]
    pc, po = oracle.windkessel_update(g["pc"], g["Q"], g["dt"], g["Rp"], g["C"], g["Rd"], 0)
    assert abs(pc - g["pc_new"]) < 1e-6
    assert abs(pc - g["Rd"] * g["Q"] * (1 - math.exp(-g["dt"] / (g["Rd"] * g["C"])))) <= 1e-13
    assert abs(po - (pc + g["Rp"] * g["Q"])) <= 1e-13


def test_windkessel_exact_matches_analytic_ode():
    # eq:windkessel_ode_a with constant Q: p_c(t) = Rd Q + (p0 - Rd Q) e^{-t/(Rd C)}
    Rp, Cc, Rd, Q, p0, dt = 100.0, 1.1111e-3, 900.0, 0.02, 3.0, 1e-3
    pc = p0
    for n in range(1, 501):
        pc, _ = oracle.windkessel_update(pc, Q, dt, Rp, Cc, Rd, 0)
        exact = Rd * Q + (p0 - Rd * Q) * math.exp(-n * dt / (Rd * Cc))
        assert abs(pc - exact) <= 1e-12 * abs(exact)
    # limits: dt -> 0 keeps p_c; dt -> inf gives Rd Q
    assert abs(oracle.windkessel_update(p0, Q, 1e-300, Rp, Cc, Rd, 0)[0] - p0) <= 1e-15
    assert abs(oracle.windkessel_update(p0, Q, 1e6, Rp, Cc, Rd, 0)[0] - Rd * Q) <= 1e-12


@pytest.mark.parametrize("scheme", [1, 2])
def test_windkessel_fe_be_first_order(scheme):
    Rp, Cc, Rd, Q, p0, T = 160.0, 6.9444e-4, 1440.0, 0.01, 0.0, 0.5
    exact = Rd * Q + (p0 - Rd * Q) * math.exp(-T / (Rd * Cc))
    errs = []
    for nsteps in (200, 400):
        pc = p0
        for _ in range(nsteps):
            pc, _ = oracle.windkessel_update(pc, Q, T / nsteps, Rp, Cc, Rd, scheme)
        errs.append(abs(pc - exact))
    order = math.log2(errs[0] / errs[1])
    assert 0.9 <= order <= 1.1


def test_windkessel_invalid_params():
    with pytest.raises(oracle.OracleError) as e:
        oracle.windkessel_update(0.0, 1.0, 1e-3, 100.0, 0.0, 900.0, 0)
    assert e.value.status == "INVALID_WK_PARAMS"


# --------------------------------------------------------------- E1 Poisson
def _f(x, y, z):   # eq:poisson_source
    return (-10 * np.pi ** 2 * np.sin(np.pi * x) * (y ** 4 - y) * np.sin(2 * np.pi * z)
            + 24 * np.sin(np.pi * x) * y ** 2 * np.sin(2 * np.pi * z))


def _gt(x, y, z):  # eq:poisson_gt
    return 2 * np.sin(np.pi * x) * (y ** 4 - y) * np.sin(2 * np.pi * z) + 10


def test_manufactured_solution_consistency():
    # the paper's pair satisfies lap(phi_GT) = f and phi_GT = 10 on every face
    rng = np.random.default_rng(0)
    P = rng.uniform(0.05, 0.95, (50, 3))
    h = 1e-4
    lap = sum((_gt(*(P + h * e).T) - 2 * _gt(*P.T) + _gt(*(P - h * e).T)) / h ** 2 for e in np.eye(3))
    assert np.abs(lap - _f(*P.T)).max() < 1e-4 * np.abs(_f(*P.T)).max()
    for ax in range(3):
        for v in (0.0, 1.0):
            Q = P.copy(); Q[:, ax] = v
            assert np.abs(_gt(*Q.T) - 10).max() < 1e-12


def _poisson_err(split, n, mode="overrelaxed"):
    raw = synth.box(n, n, n, split=split, patch_mode=2)
    m = oracle.Mesh(raw, mode)
    b = oracle.BCs(m); b.set(0, "s", oracle.BC_FIXED, 10.0)
    x, y, z = m.xc.T
    phi, it = m.poisson_steady(b, _f(x, y, z) * m.V, phi0=np.full(m.N, 10.0))
    return math.sqrt(np.sum(m.V * (phi - _gt(x, y, z)) ** 2) / m.V.sum())


@pytest.mark.parametrize("kind,split", [("hex", 0), ("tet5", 5)])
def test_poisson_order_two_on_skew_free(golden, kind, split):
    g = golden("poisson_mms.json")
    ref = g[kind]
    errs = [_poisson_err(split, n) for n in ref["n"][:2]]
    for e, r in zip(errs, ref["err"]):
        assert abs(e - r) <= g["rel_tol"] * r, (e, r)
    assert 1.9 <= math.log2(errs[0] / errs[1]) <= 2.2


@pytest.mark.slow
@pytest.mark.parametrize("kind,split", [("hex", 0), ("tet5", 5)])
def test_poisson_n24(golden, kind, split):
    g = golden("poisson_mms.json")
    e = _poisson_err(split, 24)
    assert abs(e - g[kind]["err"][2]) <= g["rel_tol"] * g[kind]["err"][2]


@pytest.mark.parametrize("mode", ["overrelaxed", "none", "orthogonal", "minimum"])
def test_poisson_kuhn_regression(golden, mode):
    g = golden("poisson_mms.json")
    ref = g["kuhn_" + mode]
    e = _poisson_err(6, ref["n"][0], mode)
    assert abs(e - ref["err"][0]) <= g["rel_tol"] * ref["err"][0], e


def test_poisson_constant_solution():
    # f = 0, phi_b = 10 -> phi = 10
    m = oracle.Mesh(synth.box(4, 4, 4, split=5, jitter=0.1), "overrelaxed")
    b = oracle.BCs(m); b.set(0, "s", oracle.BC_FIXED, 10.0)
    phi, _ = m.poisson_steady(b, np.zeros(m.N))
    assert np.abs(phi - 10).max() <= 1e-10


def test_poisson_slab_linear_exact_on_hex():
    # 1-D slab phi = 0 / 1 on x = 0 / 1, zeroGradient elsewhere -> linear
    m = oracle.Mesh(synth.box(7, 2, 2, 1.0, 0.3, 0.3, patch_mode=0))
    b = oracle.BCs(m)
    for i, p in enumerate(m.patches):
        b.set(i, "s", oracle.BC_ZEROGRAD)
    b.set("xmin", "s", oracle.BC_FIXED, 0.0); b.set("xmax", "s", oracle.BC_FIXED, 1.0)
    phi, _ = m.poisson_steady(b, np.zeros(m.N))
    assert np.abs(phi - m.xc[:, 0]).max() <= 1e-10


# --------------------------------------------------------------- PISO
def _cavity_solver(direct=True, scramble=0):
    raw = synth.cavity(20, scramble=scramble)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    b.set("movingWall", "U", oracle.BC_FIXED, (1, 0, 0)); b.set("fixedWalls", "U", oracle.BC_FIXED, (0, 0, 0))
    b.set("movingWall", "p", oracle.BC_ZEROGRAD); b.set("fixedWalls", "p", oracle.BC_ZEROGRAD)
    S = oracle.Solver(m, b, nu=0.01, dt=0.005, n_corr=2, n_nonorth=0, convection="central", direct=direct,
                      p_tol=1e-15, U_tol=1e-15)
    return m, S


def test_cavity_regression_step1_and_100(golden):
    g = golden("cavity_c1.json")
    m, S = _cavity_solver(direct=True)
    U = np.zeros((m.N, 3)); p = np.zeros(m.N); phi = np.zeros(m.NF)
    r = S.step(U, p, phi)
    tol = g["rel_tol"]
    assert abs(np.abs(U).max() - g["step1"]["max_abs_U_component"]) <= tol
    assert abs(p.min() - g["step1"]["p_min"]) <= tol * 6 and abs(p.max() - g["step1"]["p_max"]) <= tol * 6
    assert r["cont_err_max"] <= g["continuity_max"]
    for _ in range(99):
        r = S.step(U, p, phi)
        assert r["cont_err_max"] <= g["continuity_max"]
    s = g["step100"]
    assert abs(np.abs(U[:, 0]).max() - s["max_abs_Ux"]) <= tol
    assert abs(np.abs(U[:, 1]).max() - s["max_abs_Uy"]) <= tol
    assert abs(p.min() - s["p_min"]) <= 5 * tol and abs(p.max() - s["p_max"]) <= 5 * tol
    assert abs(np.abs(U).sum() - s["sum_abs_U"]) <= 100 * tol
    c = np.argmin(np.linalg.norm(m.xc[:, :2] - [0.0475, 0.0475], axis=1))
    assert np.abs(U[c, :2] - s["cell_0.0475_0.0475_U"]).max() <= 1e-8
    assert np.abs(U[:, 2]).max() == 0.0     # A-24: U_z stays exactly 0 on the slab


def test_cavity_direct_vs_krylov():
    # pin (iii): direct-mode PISO vs Krylov-mode PISO <= 1e-10
    m, Sd = _cavity_solver(direct=True)
    _, Sk = _cavity_solver(direct=False)
    st = [(np.zeros((m.N, 3)), np.zeros(m.N), np.zeros(m.NF)) for _ in range(2)]
    for _ in range(5):
        Sd.step(*st[0]); Sk.step(*st[1])
    for a, b in zip(st[0], st[1]):
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(a)


def test_cavity_scrambled_numbering_same_velocity():
    # renumbering-invariance: velocity is unchanged by the cell order (p differs
    # only through the gauge cell, A-12) -> compare U at equal centroids
    m0, S0 = _cavity_solver(direct=True, scramble=0)
    m1, S1 = _cavity_solver(direct=True, scramble=11)
    U0 = np.zeros((m0.N, 3)); U1 = np.zeros((m1.N, 3))
    a0 = (U0, np.zeros(m0.N), np.zeros(m0.NF)); a1 = (U1, np.zeros(m1.N), np.zeros(m1.NF))
    for _ in range(3):
        S0.step(*a0); S1.step(*a1)
    o0 = np.lexsort(np.round(m0.xc, 9).T[::-1]); o1 = np.lexsort(np.round(m1.xc, 9).T[::-1])
    assert np.abs(U0[o0] - U1[o1]).max() <= 1e-12


def test_uniform_flow_is_fixed_point():
    # pin (i): uniform U0 with U_b = U0 on non-outlet patches and p = 0 at the
    # outlet is an exact fixed point on any mesh
    raw = synth.pipe(4, 2, 6, 0.5, 1.0, tets=True, scramble=3)
    m = oracle.Mesh(raw)
    U0 = np.array([0.0, 0.0, 1.0])
    b = oracle.BCs(m)
    b.set("inlet", "U", oracle.BC_FIXED, U0); b.set("wall", "U", oracle.BC_FIXED, U0)
    b.set("outlet", "U", oracle.BC_ZEROGRAD)
    b.set("inlet", "p", oracle.BC_ZEROGRAD); b.set("wall", "p", oracle.BC_ZEROGRAD)
    b.set("outlet", "p", oracle.BC_FIXED, 0.0)
    S = oracle.Solver(m, b, nu=0.1, dt=0.01, n_corr=2, n_nonorth=1, convection="upwind", direct=True)
    U = np.tile(U0, (m.N, 1)); p = np.zeros(m.N); phi = m.Sf @ U0
    for _ in range(3):
        r = S.step(U, p, phi)
    assert np.abs(U - U0).max() <= 1e-12 and np.abs(p).max() <= 1e-12
    assert r["cont_err_max"] <= 1e-13


def _channel(ny, direct):
    raw = synth.box(4 * ny, ny, 1, 4.0, 1.0, 1.0 / ny, split=0, patch_mode=3)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    b.set("inlet", "U", oracle.BC_PARABOLIC, u_max=1.0, center=(0, 0.5, 0.5 / ny), radius=0.5)
    b.set("walls", "U", oracle.BC_FIXED, (0, 0, 0)); b.set("outlet", "U", oracle.BC_ZEROGRAD)
    b.set("inlet", "p", oracle.BC_ZEROGRAD); b.set("walls", "p", oracle.BC_ZEROGRAD)
    b.set("outlet", "p", oracle.BC_FIXED, 0.0)
    dt = 0.64 / ny
    S = oracle.Solver(m, b, nu=0.1, dt=dt, n_corr=2, n_nonorth=0, convection="upwind", direct=direct,
                      p_tol=1e-13, U_tol=1e-13)
    x, y, _ = m.xc.T
    U = np.zeros((m.N, 3)); U[:, 0] = 4 * y * (1 - y)
    p = -0.8 * (x - 4)
    Uf = np.zeros((m.NF, 3)); Uf[:, 0] = 4 * m.xf[:, 1] * (1 - m.xf[:, 1])
    phi = np.einsum("ij,ij->i", Uf, m.Sf)
    phi[m.F:][np.abs(m.Sf[m.F:, 2]) > 0] = 0
    for it in range(20000):
        U0 = U.copy()
        r = S.step(U, p, phi)
        if np.abs(U - U0).max() / dt < 1e-9:
            break
    sel = (x > 1.5) & (x < 2.5)
    A = np.vstack([x[sel], np.ones(sel.sum())]).T
    dpdx = np.linalg.lstsq(A, p[sel], rcond=None)[0][0]
    rms = math.sqrt(np.sum(m.V[sel] * (U[sel, 0] - 4 * y[sel] * (1 - y[sel])) ** 2) / m.V[sel].sum())
    return dpdx, rms


@pytest.mark.parametrize("i,ny", [(0, 8), (1, 16)])
def test_poiseuille_channel_order_pin(golden, i, ny):
    g = golden("poiseuille_channel.json")
    dpdx, rms = _channel(ny, direct=ny <= 8)
    assert abs(dpdx - g["dpdx"][i]) <= g["abs_tol_dpdx"]
    assert abs(rms - g["rms"][i]) <= g["rel_tol_rms"] * g["rms"][i]
