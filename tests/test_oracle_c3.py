"""Oracle pins on the C3 mesh family (configs[2]): the
polygon dual of a Delaunay triangulation around a cylinder, extruded one
layer with empty front/back (A-24).

Pins: SURVEY §8 size relations (E = 2N, F/N ~ 3), per-cell closedness, the
exact domain volume (channel minus the polygon the cylinder ring spans,
shoelace formula, times dz), exact Gauss gradient of a linear field with exact
face values on polygon prisms, and PISO invariants on the C3 recipe
(continuity at the solver tolerance, U_z stays at round-off on a 2-D slab)."""
import numpy as np
import pytest

import cases
import oracle
import synth


@pytest.fixture(scope="module")
def c3small():
    raw = synth.cylinder_poly(2e4, scramble=13)
    return raw, oracle.Mesh(raw)


def test_sizes_and_patches(c3small):
    raw, m = c3small
    E = [p.n for p in raw.patches if p.kind == synth.PATCH_EMPTY][0]
    assert E == 2 * m.N
    assert 2.8 <= m.F / m.N <= 3.2
    assert {p.name for p in raw.patches} == {"inlet", "outlet", "sides", "cylinder", "frontAndBack"}
    assert (m.V > 0).all()


def test_cell_closedness(c3small):
    raw, m = c3small
    acc = np.zeros((m.N, 3))
    np.add.at(acc, m.owner, m.Sf)
    np.add.at(acc, m.neighbour, -m.Sf[:m.F])
    A = np.linalg.norm(m.Sf, axis=1).max()
    assert np.abs(acc).max() <= 1e-13 * A


def test_total_volume_exact(c3small):
    # channel [-1,3]x[-1,1] minus the polygon through the cylinder ring's
    # vertices (r = 0.1 exactly), times dz
    raw, m = c3small
    P = raw.points
    r = np.hypot(P[:, 0], P[:, 1])
    ring = P[(np.abs(r - 0.1) < 1e-13) & (P[:, 2] == 0.0)]
    ring = ring[np.argsort(np.arctan2(ring[:, 1], ring[:, 0]))]
    x, y = ring[:, 0], ring[:, 1]
    area = 0.5 * abs(np.dot(x, np.roll(y, -1)) - np.dot(y, np.roll(x, -1)))
    assert len(ring) == raw.meta["n_theta"]
    exact = (8.0 - area) * raw.meta["dz"]
    assert abs(m.V.sum() - exact) <= 1e-12 * exact


def test_linear_gradient_exact_with_exact_face_values(c3small):
    raw, m = c3small
    a = np.array([0.7, -1.3, 0.0])
    fv = m.xf @ a + 0.25
    G = m.grad_faces(fv)
    assert np.abs(G - a[None, :]).max() <= 1e-10


def test_c3_piso_invariants():
    case = cases.c3(target_cells=2e4)
    m = oracle.Mesh(case.raw)
    S = oracle.Solver(m, case.apply_bcs(oracle.BCs(m)), **dict(case.solver, p_tol=1e-12, p_rel_tol=0.0))
    U, p, phi = case.initial_state(m.xc, m.xf, m.Sf)
    assert np.abs(U[:, 2]).max() == 0.0
    for _ in range(3):
        r = S.step(U, p, phi)
        assert r["cont_err_max"] <= 1e-10 and not r["nonfinite"]
    assert np.abs(U[:, 2]).max() <= 1e-13
    # no-slip cylinder: the wall faces carry no flux
    cyl = [pt for pt in case.raw.patches if pt.name == "cylinder"][0]
    assert np.abs(phi[cyl.start:cyl.start + cyl.n]).max() <= 1e-15
