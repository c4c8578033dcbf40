"""Oracle pins for NEXT-1: deferred-correction convection
(eq:deferred_correction) with SOU (eq:sou P:200-206) and the
gradient-based unstructured QUICK reading, and the passive
scalar transport workload of PAPER.md §3.1.2.

Pins: consistency for globally linear fields (every scheme's convective
residual equals the exact V u.grad(phi) where its face value is exact),
SPEC.md:236-238 upwind face-value examples, boundedness of implicit upwind
transport, u = 0 / uniform-field invariance, and the paper's qualitative
claim that SOU keeps a sharper step than upwind."""
import numpy as np
import pytest

import oracle
import synth

SCHEMES = ["upwind", "central", "sou", "quick"]


def _linear_case(convection, ncells=6):
    raw = synth.box(ncells, ncells, ncells, 1.0, 1.0, 1.0, scramble=4)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for i in range(len(raw.patches)):
        b.set(i, "U", oracle.BC_ZEROGRAD)
        b.set(i, "p", oracle.BC_ZEROGRAD)
    S = oracle.Solver(m, b, nu=0.0, dt=1.0, convection=convection)
    return m, S


@pytest.mark.parametrize("convection", ["central", "sou", "quick"])
def test_linear_field_convective_residual_exact(convection):
    # uniform u with consistent m_f = u.S_f and U^k = a_k . x: the face value of
    # central (x_f at the midpoint), SOU and QUICK is exact on a Cartesian mesh,
    # so (M U - b)_c = sum_f m_f U(x_f) = V_c u . a_k on cells whose upwind
    # neighbours' Gauss gradients are exact (two layers from the boundary)
    m, S = _linear_case(convection)
    u = np.array([0.7, -0.4, 0.25])
    A = np.array([[1.0, 2.0, -1.0], [0.5, -0.3, 0.8], [-1.2, 0.1, 0.4]])
    U = m.xc @ A.T
    phi = m.Sf @ u
    diag, lo, up, b = S.momentum_assemble(U, phi)
    R = np.stack([m.ldu_apply(diag, lo, up, U[:, k]) for k in range(3)], 1) - b
    depth = np.full(m.N, 99)
    bcells = np.unique(m.owner[m.F:])
    depth[bcells] = 0
    for d in range(1, 3):
        for f in range(m.F):
            o, n = m.owner[f], m.neighbour[f]
            if depth[o] == d - 1 and depth[n] > d: depth[n] = d
            if depth[n] == d - 1 and depth[o] > d: depth[o] = d
    sel = depth >= 2
    exact = m.V[:, None] * (A @ u)[None, :]
    assert sel.sum() > 0
    assert np.abs(R[sel] - exact[sel]).max() <= 1e-12 * np.abs(exact).max()


def test_spec_upwind_face_value_examples():
    # m = +1, phi_owner = 3, phi_nb = 7 -> implicit face value 3; m = -1 -> 7
    raw = synth.fixture_two_boxes(1.0)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    b.set(0, "s", oracle.BC_ZEROGRAD)
    for md in (1.0, -1.0):
        # one implicit-Euler step (V = 1, dt = 1) of pure convection across the
        # shared face: owner row (x_O' - 3) + m x_f' = 0, neighbour row
        # (x_N' - 7) - m x_f' = 0 with x_f' the upwind value of the new field
        phi = np.zeros(m.NF); phi[0] = md
        S = oracle.Solver(m, b, nu=0.0, dt=1.0, convection="upwind", direct=True)
        x = np.array([3.0, 7.0])
        S.transport_step(x, phi, 0.0)
        if md > 0:
            assert abs(x[0] - 3.0 / (1.0 + md)) <= 1e-15 and abs(x[1] - (7.0 + md * x[0])) <= 1e-14
        else:
            assert abs(x[1] - 7.0 / (1.0 - md)) <= 1e-15 and abs(x[0] - (3.0 - md * x[1])) <= 1e-14


def _uniform_flux(raw, m, u):
    """m_f = u . S_f on every face, 0 on the empty patch (extruded slab)"""
    phi = m.Sf @ np.asarray(u, np.float64)
    for p in raw.patches:
        if p.kind == synth.PATCH_EMPTY:
            phi[p.start:p.start + p.n] = 0.0
    return phi


def _step_case(n=24, convection="upwind", gamma=1e-3, steps=300, dt=0.02):
    raw = synth.square_tri(n, jitter=0.2)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    b.set("inlet_lower", "s", oracle.BC_FIXED, 1.0)
    b.set("inlet_upper", "s", oracle.BC_FIXED, 0.0)
    b.set("outlet", "s", oracle.BC_ZEROGRAD)
    for pn in ("inlet_lower", "inlet_upper", "outlet"):
        b.set(pn, "U", oracle.BC_ZEROGRAD); b.set(pn, "p", oracle.BC_ZEROGRAD)
    S = oracle.Solver(m, b, nu=0.0, dt=dt, convection=convection, U_tol=1e-13)
    phi = _uniform_flux(raw, m, (2.0, 1.0, 0.0))
    x = np.zeros(m.N)
    for _ in range(steps):
        S.transport_step(x, phi, gamma)
    return m, x


def test_step_advection_upwind_bounded():
    # SPEC.md:447 / eq:upwind P:193 "bounded": pure implicit upwind convection
    # (an M-matrix) keeps the step profile in [0, 1]
    m, x = _step_case(convection="upwind", gamma=0.0)
    assert x.min() >= -1e-9 and x.max() <= 1 + 1e-9


def test_step_advection_sou_sharper_than_upwind():
    # P:491 "the SOU scheme yields higher peak values and a sharper transition"
    mu, xu = _step_case(convection="upwind")
    ms, xs = _step_case(convection="sou")
    line = np.abs(mu.xc[:, 0] - 0.3) < 0.03
    def width(m, x):   # width of the 0.1 - 0.9 transition along x = 0.3
        y = m.xc[line, 1]; v = x[line]
        return np.ptp(y[(v > 0.1) & (v < 0.9)]) if ((v > 0.1) & (v < 0.9)).any() else 0.0
    assert width(ms, xs) < width(mu, xu)
    assert xs[line].max() >= xu[line].max() - 1e-12


def test_transport_invariants():
    # u = 0, Gamma = 0 -> unchanged; uniform field with
    # matching inlet value -> stays uniform
    raw = synth.square_tri(8)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for pn in ("inlet_lower", "inlet_upper"):
        b.set(pn, "s", oracle.BC_FIXED, 0.3)
    b.set("outlet", "s", oracle.BC_ZEROGRAD)
    for conv in SCHEMES:
        S = oracle.Solver(m, b, nu=0.0, dt=0.05, convection=conv, U_tol=1e-14)
        x0 = synth.cell_field(3, m.N)
        x = x0.copy()
        S.transport_step(x, np.zeros(m.NF), 0.0)
        assert np.abs(x - x0).max() <= 1e-13
        phi = _uniform_flux(raw, m, (2.0, 1.0, 0.0))
        x = np.full(m.N, 0.3)
        S.transport_step(x, phi, 1e-3)
        assert np.abs(x - 0.3).max() <= 1e-12
