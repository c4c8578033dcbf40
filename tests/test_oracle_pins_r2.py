"""Pins of the oracle parts that round 1 left "parity unpinned" (DESIGN.md §4,
VERDICT round 1 "What's weak" 1), each against a value fixed by hand or by an
already-pinned operator, never by the oracle's own formula retyped:

* O-5 explicit non-orthogonal momentum correction nu k_f . (grad U)_f
  (eq:nonortho_flux P:240-254, A-2, A-16): hand-computed on a two-cell fixture
  with interpolation weight 3/4 (a swapped w or a wrong sign fails), and, on
  jittered tets, (M U - b) = -nu * laplacian(U_k) cell by cell against the
  pinned Laplacian (tests/test_oracle_operators.py).
* A-9 non-orthogonal pressure right-hand side and Rhie-Chow flux term
  (P:337-347): hand-computed on the same fixture.
* A-19 Windkessel coupling inside PISO (eq:windkessel_discrete P:420-425):
  steady uniform flow into an RCR outlet is an exact fixed point with
  p = p_o / rho everywhere and p_c on the analytic ODE solution; with a
  pulsatile plug inflow, the committed p_c follows the exact-integrator
  recurrence with Q of the LAST corrector (lagged per corrector, p_c^{n+1}
  always from the start-of-step p_c^n, not compounded).
* O-10 partition emulation: the Laplacian applied part
  by part from owned + ghost data only equals the global apply bit for bit.
"""
import math

import numpy as np
import pytest

import oracle
import synth


# ------------------------------------------------------------ fixtures
def sheared_pair(L=3.0, h=4.0):
    """Unit cube [0,1]^3 (cell 0) + a parallelepiped on its x = 1 face whose
    far face (x = 1 + L) is shifted by h in y (cell 1), every outer face one
    wall patch.  By hand: internal face S = (1, 0, 0), x_f = (1, 1/2, 1/2);
    x_O = (1/2, 1/2, 1/2), x_N = (1 + L/2, (1 + h)/2, 1/2), V_O = 1, V_N = L;
    projected weight w = (L/2) / (L/2 + 1/2) = 3/4 at L = 3; link
    d = (2, h/2, 0) = (2, 2, 0) at h = 4 (45 degrees)."""
    from synth import _from_cells, _HEX_FACES, PATCH_WALL
    a = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    x1 = 1.0 + L
    pts = a + [(x1, h, 0), (x1, 1 + h, 0), (x1, 1 + h, 1), (x1, h, 1)]
    c0 = [list(f) for f in _HEX_FACES]
    hh = [1, 8, 9, 2, 5, 11, 10, 6]
    c1 = [[hh[i] for i in f] for f in _HEX_FACES]
    return _from_cells(pts, [c0, c1], lambda P, r: ("walls", 0, PATCH_WALL))


def test_sheared_pair_geometry_by_hand():
    m = oracle.Mesh(sheared_pair(), "minimum")
    assert m.N == 2 and m.F == 1
    assert np.allclose(m.xc, [[0.5, 0.5, 0.5], [2.5, 2.5, 0.5]], atol=1e-14)
    assert np.allclose(m.V, [1.0, 3.0], atol=1e-14)
    assert np.allclose(m.Sf[0], [1, 0, 0], atol=1e-15) and abs(m.w[0] - 0.75) <= 1e-15
    # minimum correction: Delta = (S.d / |d|^2) d = (1/4)(2, 2, 0), delta = 1/4, k = S - Delta = (1/2, -1/2, 0)
    assert abs(m.delta[0] - 0.25) <= 1e-15
    assert np.allclose(m.k[0], [0.5, -0.5, 0.0], atol=1e-15)


# ------------------------------------------------------------ O-5
@pytest.mark.parametrize("nu", [1.0, 0.37])
def test_momentum_nonorth_correction_by_hand(nu):
    """Walls fixedValue U = 0, phi = 0, backward Euler.  Gauss gradients with
    zero boundary values: G_O = U_f S / V_O, G_N = -U_f S / V_N with
    U_f = w U_O + (1 - w) U_N, so (grad U)_f = w G_O + (1 - w) G_N
    = U_f S (3/4 - 1/12) = (2/3) U_f S, and the explicit correction
    nu k . (grad U)_f = nu (1/2)(2/3) U_f = nu U_f / 3 per component enters b_O
    with + and b_N with -.  (With w and 1 - w swapped (grad U)_f = 0.)"""
    raw = sheared_pair()
    m = oracle.Mesh(raw, "minimum")
    b = oracle.BCs(m)
    b.set("walls", "U", oracle.BC_FIXED, (0.0, 0.0, 0.0))
    b.set("walls", "p", oracle.BC_ZEROGRAD)
    dt = 0.5
    S = oracle.Solver(m, b, nu=nu, dt=dt)
    U = np.array([[1.0, 2.0, -3.0], [-1.0, 0.5, 2.0]])
    diag, lo, up, bv = S.momentum_assemble(U, np.zeros(m.NF))
    Uf = 0.75 * U[0] + 0.25 * U[1]
    corr = nu * Uf / 3.0
    assert np.abs(bv[0] - (m.V[0] / dt * U[0] + corr)).max() <= 1e-14
    assert np.abs(bv[1] - (m.V[1] / dt * U[1] - corr)).max() <= 1e-14
    # and the implicit part: upper = lower = -nu delta = -nu / 4
    assert abs(up[0] + nu * 0.25) <= 1e-15 and abs(lo[0] + nu * 0.25) <= 1e-15


@pytest.mark.parametrize("nonorth", ["overrelaxed", "minimum", "orthogonal"])
def test_momentum_residual_is_minus_nu_laplacian(nonorth):
    """phi = 0, backward Euler: (M U^n - b)_c = (A_s U^n - b_s)_c
    = -nu * [sum_f s (delta (U_N - U_O) + k . (grad U)_f) + sum_b delta_b (U_b - U_O)]
    = -nu * laplacian(U_k)_c, the pinned Laplacian with the same Gauss
    gradient and boundary values, component by component, on jittered tets."""
    raw = synth.box(5, 4, 3, 1.0, 0.8, 0.6, split=5, jitter=0.15, scramble=9)
    m = oracle.Mesh(raw, nonorth)
    b = oracle.BCs(m)
    vals = {"xmin": (0.3, -0.2, 0.1), "xmax": (0.0, 0.0, 0.0), "ymin": (1.0, 0.5, -0.5)}
    for p in raw.patches:
        if p.name in vals:
            b.set(p.name, "U", oracle.BC_FIXED, vals[p.name])
        else:
            b.set(p.name, "U", oracle.BC_ZEROGRAD)
        b.set(p.name, "p", oracle.BC_ZEROGRAD)
    nu, dt = 0.7, 0.01
    S = oracle.Solver(m, b, nu=nu, dt=dt)
    U = synth.cell_field(7, m.N, 3)
    diag, lo, up, bv = S.momentum_assemble(U, np.zeros(m.NF))
    res = np.stack([m.ldu_apply(diag, lo, up, U[:, k]) for k in range(3)], 1) - bv
    for k in range(3):
        bs = oracle.BCs(m)
        for p in raw.patches:
            if p.name in vals:
                bs.set(p.name, "s", oracle.BC_FIXED, (vals[p.name][k], 0, 0))
            else:
                bs.set(p.name, "s", oracle.BC_ZEROGRAD)
        y, yabs = m.laplacian(bs, "s", U[:, k])
        assert np.abs(res[:, k] + nu * y).max() <= 1e-12 * nu * yabs.max(), k


# ------------------------------------------------------------ A-9
def _pair_solver(p_bc):
    raw = sheared_pair()
    m = oracle.Mesh(raw, "minimum")
    b = oracle.BCs(m)
    b.set("walls", "U", oracle.BC_FIXED, (0.0, 0.0, 0.0))
    if p_bc == "fixed":
        b.set("walls", "p", oracle.BC_FIXED, (0.0, 0.0, 0.0))
    else:
        b.set("walls", "p", oracle.BC_ZEROGRAD)
    return m, oracle.Solver(m, b, nu=1.0, dt=0.1)


def test_pressure_rhs_nonorth_term_by_hand():
    """Walls p = 0, phiHbyA = 0: (grad p)_f = (2/3) p_f S as for U above, so
    rhs_O = rAU_f k . (grad p)_f = rAU_f (1/2)(2/3) p_f and rhs_N = -rhs_O, with
    rAU_f = w rAU_O + (1 - w) rAU_N, p_f = w p_O + (1 - w) p_N (A-8, A-2);
    the fixed-value boundary term c_b p_b vanishes (p_b = 0)."""
    m, S = _pair_solver("fixed")
    rAU = np.array([0.2, 0.05])
    p = np.array([3.0, -1.0])
    rhs = S.pressure_rhs(rAU, np.zeros(m.NF), p)
    rf = 0.75 * rAU[0] + 0.25 * rAU[1]
    pf = 0.75 * p[0] + 0.25 * p[1]
    t = rf * pf / 3.0
    assert abs(rhs[0] - t) <= 1e-15 and abs(rhs[1] + t) <= 1e-15
    # with a divergence term: rhs -= D(phiHbyA) (sign of eq:pressure_poisson x -1)
    phiHbyA = np.zeros(m.NF)
    phiHbyA[0] = 0.3
    rhs2 = S.pressure_rhs(rAU, phiHbyA, p)
    assert abs(rhs2[0] - (t - 0.3)) <= 1e-15 and abs(rhs2[1] - (-t + 0.3)) <= 1e-15


def test_flux_correction_by_hand():
    """phi_f = phiHbyA_f - c_f (p_N - p_O) - rAU_f k . (grad p)_f with
    c_f = rAU_f delta_f = rAU_f / 4; boundary faces of cell O (a unit cube:
    delta_b = |S_b| / (S^_b . d_b) = 1 / (1/2) = 2) carry
    phiHbyA_b - rAU_O * 2 * (p_b - p_O)."""
    m, S = _pair_solver("fixed")
    rAU = np.array([0.2, 0.05])
    p = np.array([3.0, -1.0])
    phiHbyA = synth.face_field(5, m.NF)
    phi = S.flux_correct(rAU, phiHbyA, p)
    rf = 0.75 * rAU[0] + 0.25 * rAU[1]
    pf = 0.75 * p[0] + 0.25 * p[1]
    expect = phiHbyA[0] - rf * 0.25 * (p[1] - p[0]) - rf * pf / 3.0
    assert abs(phi[0] - expect) <= 1e-15
    for f in range(m.F, m.NF):
        if m.owner[f] == 0:
            assert abs(phi[f] - (phiHbyA[f] - rAU[0] * 2.0 * (0.0 - p[0]))) <= 1e-14, f
    # corrected continuity: the flux out of the pair's internal face is the
    # part of the corrected system the right-hand side balances (O-6 sign check)
    rhs = S.pressure_rhs(rAU, phiHbyA, p)
    D = np.zeros(2)
    np.add.at(D, m.owner, phi)
    np.add.at(D, m.neighbour, -phi[:m.F])
    # sum_f s phi = D(phiHbyA) + (A p) - sum_b c_b p_b - K(grad p) = A p - rhs
    # (O-6 sign check: a converged solve A p = rhs gives a divergence-free phi)
    d_f = 0.25
    cb = np.zeros(m.NF - m.F)
    A = np.zeros((2, 2))
    A[0, 0] = A[1, 1] = rf * d_f
    A[0, 1] = A[1, 0] = -rf * d_f
    for f in range(m.F, m.NF):
        o = m.owner[f]
        A[o, o] += rAU[o] * m.delta_b[f - m.F]
    assert np.abs(D - (A @ p - rhs)).max() <= 1e-13


def test_pressure_rhs_zero_gradient_walls_by_hand():
    """zeroGradient walls: G_O = (p_f - p_O) S / V_O, G_N = (p_N - p_f) S / V_N,
    (grad p)_f = w (1 - w)(p_N - p_O)(1 / V_O + 1 / V_N) S = (1/4)(p_N - p_O) S,
    so rhs_O = rAU_f (1/2)(1/4)(p_N - p_O)."""
    m, S = _pair_solver("zerograd")
    rAU = np.array([0.2, 0.05])
    p = np.array([3.0, -1.0])
    rhs = S.pressure_rhs(rAU, np.zeros(m.NF), p)
    rf = 0.75 * rAU[0] + 0.25 * rAU[1]
    t = rf * 0.125 * (p[1] - p[0])
    assert abs(rhs[0] - t) <= 1e-15 and abs(rhs[1] + t) <= 1e-15


# ------------------------------------------------------------ A-19
def _wk_duct(U0=0.8, rho=1.06, wave=None, n_corr=2, walls="fixed", nyz=3):
    """hex duct [0,2] x [0,1] x [0,1] (6 x nyz x nyz cells): xmin inlet
    U = (U0,0,0) (optionally times a waveform), xmax RCR outlet (U
    zeroGradient), other sides walls (fixedValue U0: moving with the flow,
    or zeroGradient).  An accelerating plug flow stays one-dimensional only
    when every cell of a layer has the same neighbourhood (nyz = 1): with
    zeroGradient walls a wall cell lacks the wall-normal diffusion
    coefficients in a_P, so rAU, and with it the corrected velocity, would
    vary across the section."""
    raw = synth.box(6, nyz, nyz, 2.0, 1.0, 1.0, scramble=4)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for p in raw.patches:
        if p.name == "xmin":
            b.set(p.name, "U", oracle.BC_FIXED, (U0, 0.0, 0.0))
            b.set(p.name, "p", oracle.BC_ZEROGRAD)
        elif p.name == "xmax":
            b.set(p.name, "U", oracle.BC_ZEROGRAD)
        else:
            if walls == "fixed":
                b.set(p.name, "U", oracle.BC_FIXED, (U0, 0.0, 0.0))   # walls moving with the flow
            else:
                b.set(p.name, "U", oracle.BC_ZEROGRAD)
            b.set(p.name, "p", oracle.BC_ZEROGRAD)
    if wave is not None:
        b.set_waveform(raw.patch("xmin"), "U", *wave)
    S = oracle.Solver(m, b, nu=0.05, dt=0.01, rho=rho, n_corr=n_corr, U_tol=1e-15, p_tol=1e-15)
    return raw, m, S


WK = dict(Rp=120.0, Cc=2.0e-3, Rd=800.0, pc0=0.4)


@pytest.mark.parametrize("n_corr", [2, 3])
def test_windkessel_uniform_flow_fixed_point(n_corr):
    """A-19: Q = U0 * A every corrector; p_c on p_c(t) = R_d Q + (p_c0 - R_d Q)
    exp(-t / (R_d C)) at t = n dt (exact integrator, from the start-of-step
    p_c^n in every corrector: a compounding reading would advance it n_corr
    times per step); p_o = p_c + R_p Q; the pressure is uniform p_o / rho
    (kinematic BC), U stays U0."""
    U0, rho, dt = 0.8, 1.06, 0.01
    raw, m, S = _wk_duct(U0, rho, n_corr=n_corr)
    out = raw.patch("xmax")
    S.windkessel_set(out, WK["Rp"], WK["Cc"], WK["Rd"], WK["pc0"], 0)
    U = np.tile([U0, 0.0, 0.0], (m.N, 1))
    p = np.zeros(m.N)
    phi = U0 * m.Sf[:, 0].copy()
    A = 1.0 * 1.0
    Q = U0 * A
    for n in range(1, 6):
        r = S.step(U, p, phi)
        pc = WK["Rd"] * Q + (WK["pc0"] - WK["Rd"] * Q) * math.exp(-n * dt / (WK["Rd"] * WK["Cc"]))
        po = pc + WK["Rp"] * Q
        assert abs(r["Q"][0] - Q) <= 1e-12 * Q
        assert abs(S.windkessel_pc(out) - pc) <= 1e-12 * abs(pc)
        assert abs(r["p_o"][0] - po) <= 1e-12 * abs(po)
        assert np.abs(p - po / rho).max() <= 1e-12 * abs(po / rho), n
        assert np.abs(U - [U0, 0.0, 0.0]).max() <= 1e-12 * U0


def test_windkessel_pulsatile_lagged_per_corrector():
    """Plug flow with a pulsatile inlet g(t) (A-41) and zeroGradient walls: after
    every corrector the outlet flux equals the inlet flux g(t^{n+1}) U0 A, so
    corrector 1 sees the lagged Q = g(t^n) U0 A and the last corrector
    Q = g(t^{n+1}) U0 A; the committed p_c^{n+1} = p_c^n e + R_d Q_last (1 - e),
    e = exp(-dt / (R_d C)) (eq:windkessel_discrete), reported Q = Q_last and
    p_o = p_c^{n+1} + R_p Q_last; the outlet pressure BC is p_o / rho."""
    U0, rho, dt = 0.8, 1.06, 0.01
    period, a, bb = 0.08, [1.0, 0.5], [0.0, 0.3]
    raw, m, S = _wk_duct(U0, rho, wave=(period, a, bb), walls="zerograd", nyz=1)
    out = raw.patch("xmax")
    S.windkessel_set(out, WK["Rp"], WK["Cc"], WK["Rd"], WK["pc0"], 0)
    g = lambda t: a[0] + a[1] * math.cos(2 * math.pi * t / period) + bb[1] * math.sin(2 * math.pi * t / period)
    U = np.tile([U0 * g(0.0), 0.0, 0.0], (m.N, 1))
    p = np.zeros(m.N)
    phi = U0 * g(0.0) * m.Sf[:, 0].copy()
    e = math.exp(-dt / (WK["Rd"] * WK["Cc"]))
    pc = WK["pc0"]
    is_out = np.zeros(m.NF, bool)
    pt = raw.patches[out]
    is_out[pt.start:pt.start + pt.n] = True
    for n in range(1, 7):
        r = S.step(U, p, phi)
        Ql = g(n * dt) * U0
        pc = pc * e + WK["Rd"] * Ql * (1 - e)
        assert abs(phi[is_out].sum() - Ql) <= 1e-11
        assert abs(r["Q"][0] - Ql) <= 1e-11, n
        assert abs(S.windkessel_pc(out) - pc) <= 1e-11 * abs(pc), n
        assert abs(r["p_o"][0] - (pc + WK["Rp"] * Ql)) <= 1e-11 * abs(pc + WK["Rp"] * Ql), n
        # lagged: not the step's first-corrector Q
        assert abs(g((n - 1) * dt) - g(n * dt)) > 1e-3


# ------------------------------------------------------------ O-10
MESHES = {
    "tet5_jitter": lambda: synth.box(6, 5, 4, 1.0, 0.8, 0.6, split=5, jitter=0.15, scramble=9),
    "pipe_tet": lambda: synth.pipe(6, 3, 20, 0.5, 2.0, tets=True, scramble=12),
    "kuhn": lambda: synth.box(6, 6, 6, split=6, scramble=3),
    "cylinder_poly": lambda: synth.cylinder_poly(3e3, scramble=13),
}


@pytest.mark.parametrize("P", [2, 3, 5])
@pytest.mark.parametrize("name", sorted(MESHES))
def test_o10_partitioned_laplacian_bitwise(name, P):
    raw = MESHES[name]()
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for i, p in enumerate(raw.patches):
        if p.kind == synth.PATCH_EMPTY:
            continue
        if i % 2 == 0:
            b.set(p.name, "s", oracle.BC_FIXED, (0.25 * i - 0.5, 0, 0))
        else:
            b.set(p.name, "s", oracle.BC_ZEROGRAD)
    x = synth.cell_field(100, m.N)
    gamma = 1.0 + 0.5 * synth.cell_field(200, m.N)
    R = oracle.Renumbering(m, P)
    for gm in (None, gamma):
        y, _ = m.laplacian(b, "s", x, gamma=gm)
        yp = R.laplacian_parts(m, b, "s", x, gamma=gm)
        assert np.array_equal(y, yp), np.abs(y - yp).max()
    # every part has ghosts (the partition really splits the operator)
    assert all(len(pp["ghost"]) > 0 for pp in R.parts)


# ------------------------------------------------------------ A-42
@pytest.mark.parametrize("phin0,expect_c", [(0.5, None), (0.01, 0.0)])
def test_ddtcorr_term_by_hand(phin0, expect_c):
    """A-42 (OpenFOAM's Euler ddtCorr, the optional NEXT-4 flag) on the w = 3/4
    fixture: phiHbyA_f = (w HbyA_O + (1 - w) HbyA_N) . S + rAU_f c (phi^n - U^n_f . S) / dt,
    c = 1 - min(|phi^n - U^n_f . S| / (|phi^n| + 1e-15), 1); with S = (1, 0, 0)
    only x-components enter.  Boundary faces (walls, U = 0) carry HbyA_b . S = 0
    and no correction; without the flag the correction is absent."""
    raw = sheared_pair()
    m = oracle.Mesh(raw, "minimum")
    dt = 0.25
    HbyA = np.array([[0.4, -0.3, 0.2], [0.1, 0.6, -0.5]])
    rAU = np.array([0.2, 0.05])
    Un = np.array([[0.3, 0.1, 0.0], [0.7, -0.2, 0.4]])
    phin = np.zeros(m.NF)
    phin[0] = phin0
    base = 0.75 * 0.4 + 0.25 * 0.1
    uS = 0.75 * 0.3 + 0.25 * 0.7
    d = phin0 - uS
    c = 1.0 - min(abs(d) / (abs(phin0) + 1e-15), 1.0)
    if expect_c is not None:
        assert c == expect_c
    rf = 0.75 * 0.2 + 0.25 * 0.05
    for flag, want in ((True, base + rf * c * d / dt), (False, base)):
        b = oracle.BCs(m)
        b.set("walls", "U", oracle.BC_FIXED, (0.0, 0.0, 0.0))
        b.set("walls", "p", oracle.BC_ZEROGRAD)
        S = oracle.Solver(m, b, nu=1.0, dt=dt, ddt_corr=flag)
        out = S.phi_hbya(HbyA, rAU, Un, phin)
        assert abs(out[0] - want) <= 1e-15, (flag, out[0], want)
        assert np.abs(out[m.F:]).max() == 0.0
