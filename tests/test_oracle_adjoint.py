"""Oracle pins for NEXT-3: the transposed LDU apply behind
the VJP (eq:vjp P:352-358) and the implicit differentiation of the pressure
solve (eq:implicit_diff P:366-370).

Pins: adjointness <A x, y> = <x, A^T y> against the independent forward
apply (random nonsymmetric LDU and the assembled momentum matrix); A^T = A
for the symmetric pressure matrix; the adjoint solve equals the dense
solution of the explicitly transposed system; dL/drAU from the VJP agrees
with central finite differences of L(rAU) = g . p(rAU) through dense LU
solves, with and without the A-12 gauge."""
import numpy as np
import pytest

import oracle
import synth


def _mesh():
    return oracle.Mesh(synth.box(5, 4, 3, 1.0, 0.8, 0.6, split=5, jitter=0.15, scramble=9))


def test_transpose_adjointness_random_ldu():
    m = _mesh()
    diag = 1.0 + synth.cell_field(1, m.N)
    lo, up = synth.face_field(2, m.F), synth.face_field(3, m.F)
    x, y = synth.cell_field(4, m.N), synth.cell_field(5, m.N)
    Ax = m.ldu_apply(diag, lo, up, x)
    Aty = m.ldu_apply_transpose(diag, lo, up, y)
    assert abs(Ax @ y - x @ Aty) <= 1e-13 * (np.abs(Ax) @ np.abs(y))
    # swapping lower/upper in the forward apply is the transpose
    assert np.abs(m.ldu_apply(diag, up, lo, y) - Aty).max() <= 1e-14 * np.abs(Aty).max()
    # symmetric -> A^T = A
    assert np.abs(m.ldu_apply_transpose(diag, lo, lo, x) - m.ldu_apply(diag, lo, lo, x)).max() <= 1e-15


def test_transpose_of_momentum_matrix():
    raw = synth.pipe(4, 2, 6, 0.5, 1.0, tets=True, scramble=21)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    b.set("inlet", "U", oracle.BC_PARABOLIC, u_max=2.0, center=(0, 0, 0), radius=0.5)
    b.set("wall", "U", oracle.BC_FIXED, value=(0, 0, 0))
    b.set("outlet", "U", oracle.BC_ZEROGRAD)
    for pn in ("inlet", "wall"):
        b.set(pn, "p", oracle.BC_ZEROGRAD)
    b.set("outlet", "p", oracle.BC_FIXED, value=0.0)
    S = oracle.Solver(m, b, nu=0.1, dt=0.01, convection="upwind")
    U = np.zeros((m.N, 3)); U[:, 2] = 1.0
    U += 0.1 * synth.cell_field(7, m.N, 3)
    phi = m.Sf @ np.array([0.0, 0.0, 1.0])
    diag, lo, up, _ = S.momentum_assemble(U, phi)
    assert np.abs(lo - up).max() > 0            # convection makes it nonsymmetric
    x, y = synth.cell_field(8, m.N), synth.cell_field(9, m.N)
    assert abs(m.ldu_apply(diag, lo, up, x) @ y - x @ m.ldu_apply_transpose(diag, lo, up, y)) <= 1e-12


def _pressure_case(fixed):
    raw = synth.pipe(4, 2, 6, 0.5, 1.0, tets=True, scramble=21)
    m = oracle.Mesh(raw)
    b = oracle.BCs(m)
    for pn in ("inlet", "wall", "outlet"):
        b.set(pn, "U", oracle.BC_ZEROGRAD)
        b.set(pn, "p", oracle.BC_ZEROGRAD)
    if fixed:
        b.set("outlet", "p", oracle.BC_FIXED, value=0.3)
    S = oracle.Solver(m, b, nu=0.1, dt=0.01, p_ref_cell=5)
    rAU = 0.01 * (1.5 + 0.5 * synth.cell_field(60, m.N))
    rhs = 1e-3 * synth.cell_field(61, m.N)
    g = synth.cell_field(63, m.N)
    return m, S, rAU, rhs, g


@pytest.mark.parametrize("fixed", [True, False])
def test_adjoint_solve_matches_forward_of_transpose(fixed):
    m, S, rAU, rhs, g = _pressure_case(fixed)
    lam_cg, rep = S.pressure_adjoint(rAU, g, tol=1e-14)
    lam_lu, _ = S.pressure_adjoint(rAU, g, direct=True)
    assert rep["converged"]
    assert np.linalg.norm(lam_cg - lam_lu) <= 1e-9 * np.linalg.norm(lam_lu)
    if fixed:
        # the pressure matrix is symmetric: adjoint solve = forward solve with rhs g
        p_g, _ = S.pressure_solve(rAU, g, direct=True)
        assert np.linalg.norm(p_g - lam_lu) <= 1e-11 * np.linalg.norm(lam_lu)


@pytest.mark.parametrize("fixed", [True, False])
def test_pressure_vjp_finite_differences(fixed):
    m, S, rAU, rhs, g = _pressure_case(fixed)
    p, _ = S.pressure_solve(rAU, rhs, direct=True)
    lam, _ = S.pressure_adjoint(rAU, g, direct=True)
    grad = S.pressure_vjp(rAU, p, lam)

    def L(r):
        return g @ S.pressure_solve(r, rhs, direct=True)[0]
    cells = [0, 5, 17, m.N // 2, m.N - 1]
    for c in cells:
        h = 1e-4 * rAU[c]           # (1e-6 is already rounding-limited: |lambda| ~ 1e4 in the gauged case)
        rp, rm = rAU.copy(), rAU.copy()
        rp[c] += h; rm[c] -= h
        fd = (L(rp) - L(rm)) / (2 * h)
        assert abs(grad[c] - fd) <= 2e-6 * max(abs(fd), 1e-3 * np.abs(grad).max()), (c, grad[c], fd)
