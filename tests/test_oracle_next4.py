"""Oracle pins for NEXT-4: the time schemes of Table 1
(forward Euler, backward Euler, Crank-Nicolson; reading A-40, the
theta method on the spatial operator) and the time-varying inflow boundary
condition ("time-varying inflow profiles", "pulsatile parabolic
velocity profile"; reading A-41).

Pins:
* theta: a shear mode U = (0, 0, cos(k pi x/L)) in a 1-D slab (z sides
  empty, x ends and y sides zero-gradient) is an eigenvector of the cell-centred Neumann
  Laplacian (DCT-II) with eigenvalue lam = (4 nu/h^2) sin^2(k pi/(2n)); the
  flux is zero so a PISO step is exactly the theta-method on that mode:
  amplification G = (1 - (1 - theta) dt lam)/(1 + theta dt lam) per step.
* waveform: a unit waveform reproduces the steady BC bitwise; in a 1-D slab
  with a uniform time-varying inflow, continuity forces every x-face flux to
  equal the inlet flux g(t^{n+1}) A after each step (Fourier series closed
  form evaluated here independently).
"""
import math

import numpy as np
import pytest

import oracle
import synth


def _slab(n, L=1.0, A=0.1):
    raw = synth.box(n, 1, 1, L, A, A, scramble=3)
    for p in raw.patches:
        if p.name in ("zmin", "zmax"):
            p.kind = synth.PATCH_EMPTY
    return raw


def _patch(raw, name):
    return raw.patch(name)


@pytest.mark.parametrize("theta", [1.0, 0.5, 0.0])
@pytest.mark.parametrize("k", [1, 3])
def test_theta_shear_mode_amplification(theta, k):
    n, L, nu, dt, steps = 32, 1.0, 0.01, 0.02, 10
    raw = _slab(n, L)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for i, p in enumerate(raw.patches):
        if p.kind != synth.PATCH_EMPTY:
            b.set(i, "U", oracle.BC_ZEROGRAD)
            b.set(i, "p", oracle.BC_ZEROGRAD)
    S = oracle.Solver(m, b, nu=nu, dt=dt, n_corr=2, theta=theta, U_tol=1e-15, p_tol=1e-15)
    h = L / n
    U = np.zeros((m.N, 3))
    U[:, 2] = np.cos(k * math.pi * m.xc[:, 0] / L)
    u0 = U[:, 2].copy()
    p = np.zeros(m.N)
    phi = np.zeros(m.NF)
    lam = 4.0 * nu / h ** 2 * math.sin(k * math.pi / (2 * n)) ** 2
    G = (1.0 - (1.0 - theta) * dt * lam) / (1.0 + theta * dt * lam)
    for s in range(1, steps + 1):
        S.step(U, p, phi)
        assert np.abs(U[:, 2] - G ** s * u0).max() <= 1e-12, (s, np.abs(U[:, 2] - G ** s * u0).max())
    assert np.abs(U[:, :2]).max() <= 1e-14 and np.abs(phi).max() <= 1e-14


def test_theta_schemes_differ_and_order():
    # CN's amplification matches exp(-lam dt) to O((lam dt)^3), BE/FE to O((lam dt)^2)
    x = 0.05
    G = {t: (1 - (1 - t) * x) / (1 + t * x) for t in (1.0, 0.5, 0.0)}
    e = {t: abs(G[t] - math.exp(-x)) for t in G}
    assert e[0.5] < 0.02 * e[1.0] and e[0.5] < 0.02 * e[0.0]


def _plug_case(n=16, L=1.0, A=0.1, dt=0.01, wave=None, theta=1.0):
    raw = _slab(n, L, A)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    i_in, i_out = raw.patch("xmin"), raw.patch("xmax")
    for i, p in enumerate(raw.patches):
        if p.kind == synth.PATCH_EMPTY:
            continue
        if i == i_in:
            b.set(i, "U", oracle.BC_FIXED, (1.0, 0.0, 0.0))
            b.set(i, "p", oracle.BC_ZEROGRAD)
        elif i == i_out:
            b.set(i, "U", oracle.BC_ZEROGRAD)
            b.set(i, "p", oracle.BC_FIXED, (0.0, 0.0, 0.0))
        else:
            b.set(i, "U", oracle.BC_ZEROGRAD)
            b.set(i, "p", oracle.BC_ZEROGRAD)
    if wave is not None:
        b.set_waveform(i_in, "U", *wave)
    S = oracle.Solver(m, b, nu=0.01, dt=dt, n_corr=2, theta=theta, U_tol=1e-15, p_tol=1e-15)
    return raw, m, S


def _g(t, period, a, bb):
    return a[0] + sum(a[k] * math.cos(2 * math.pi * k * t / period) + bb[k] * math.sin(2 * math.pi * k * t / period)
                      for k in range(1, len(a)))


@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_pulsatile_plug_flow_flux(theta):
    # 1-D continuity: every x-face flux equals the inlet flux g(t^{n+1}) A
    period, a, bb = 0.08, [1.0, 0.5, -0.2], [0.0, 0.3, 0.1]
    raw, m, S = _plug_case(wave=(period, a, bb), theta=theta)
    U, p, phi = np.zeros((m.N, 3)), np.zeros(m.N), np.zeros(m.NF)
    xf = np.abs(m.Sf[:, 0]) > 0.5 * np.abs(m.Sf).max()
    yf = np.abs(m.Sf[:, 1]) > 0.5 * np.abs(m.Sf).max()
    dt = 0.01
    for s in range(1, 9):
        S.step(U, p, phi)
        g = _g(s * dt, period, a, bb)
        assert np.abs(phi[xf] / m.Sf[xf, 0] - g).max() <= 1e-11 * max(1.0, abs(g)), s
        assert np.abs(phi[yf]).max() <= 1e-14
        # and not the start-of-step value
        assert abs(_g((s - 1) * dt, period, a, bb) - g) > 1e-3


def test_unit_waveform_is_steady_bitwise():
    import cases
    outs = []
    for wave in (False, True):
        case = cases.c1(scramble=11)
        mo = oracle.Mesh(case.raw)
        b = case.apply_bcs(oracle.BCs(mo))
        if wave:
            b.set_waveform(case.raw.patch("movingWall"), "U", 1.0, [1.0, 0.0], [0.0, 0.0])
        S = oracle.Solver(mo, b, **case.solver)
        U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
        for _ in range(2):
            S.step(U, p, phi)
        outs.append((U, p, phi))
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_waveform_rejected_on_zero_gradient_patch():
    raw, m, S = _plug_case()
    S.bcs.set_waveform(raw.patch("xmax"), "U", 1.0, [1.0])
    U, p, phi = np.zeros((m.N, 3)), np.zeros(m.N), np.zeros(m.NF)
    with pytest.raises(oracle.OracleError) as e:
        S.step(U, p, phi)
    assert e.value.status == "INVALID_ARG"


# ---------------------------------------------------------------- ddtCorr (A-42)
def _cavity(ddt_corr):
    import cases
    case = cases.c1(scramble=11)
    mo = oracle.Mesh(case.raw)
    b = case.apply_bcs(oracle.BCs(mo))
    return mo, oracle.Solver(mo, b, **dict(case.solver, ddt_corr=ddt_corr))


def test_ddtcorr_vanishes_on_a_consistent_start():
    # phi^n = interp(U^n).S on every internal face (the cavity from rest) ->
    # d = 0, the term is exactly zero: step 1 bitwise equal; later steps differ
    runs = []
    for flag in (False, True):
        mo, S = _cavity(flag)
        U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
        S.step(U, p, phi)
        first = (U.copy(), p.copy(), phi.copy())
        S.step(U, p, phi)
        runs.append((first, (U, p, phi)))
    for x, y in zip(runs[0][0], runs[1][0]):
        assert np.array_equal(x, y)
    assert not np.array_equal(runs[0][1][2], runs[1][1][2])
    # a small correction: the two fluxes agree to O(dt) of the flux scale
    assert np.abs(runs[0][1][2] - runs[1][1][2]).max() <= 0.05 * np.abs(runs[0][1][2]).max()


def test_ddtcorr_keeps_uniform_flow_fixed_point():
    raw = synth.box(6, 5, 4, 1.0, 1.0, 1.0, split=5, jitter=0.15, scramble=9)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    u = np.array([0.7, -0.3, 0.2])
    xmin = raw.patch("xmin")
    for i, pt in enumerate(raw.patches):
        b.set(i, "U", oracle.BC_FIXED, tuple(u))
        b.set(i, "p", oracle.BC_FIXED if i == xmin else oracle.BC_ZEROGRAD, (0.0, 0.0, 0.0))
    S = oracle.Solver(m, b, nu=0.01, dt=0.01, n_corr=2, n_nonorth=1, ddt_corr=True, U_tol=1e-15, p_tol=1e-15)
    U = np.tile(u, (m.N, 1))
    p = np.zeros(m.N)
    phi = m.Sf @ u
    for _ in range(3):
        S.step(U, p, phi)
    assert np.abs(U - u).max() <= 1e-11 and np.abs(phi - m.Sf @ u).max() <= 1e-11 * np.abs(m.Sf).max()
