"""Oracle pins for O-0 validation, O-1 geometry, O-2 connectivity and O-3
coefficients (SURVEY.md §8(c) pin table rows O-1, O-2/O-9, O-3).
Every pin is fixed by closed forms or invariants, not by the oracle itself."""
import math

import numpy as np
import pytest

import oracle
import synth


def test_unit_cube_fixture():
    # S:66 unit cube -> V = 1, |S_f| = 1, centroid (1/2, 1/2, 1/2); S:48 N=1, F=0, B=6
    raw = synth.fixture_unit_cube()
    m = oracle.Mesh(raw)
    assert (m.N, m.F, m.NF) == (1, 0, 6)
    assert abs(m.V[0] - 1.0) <= 1e-14
    assert np.allclose(np.linalg.norm(m.Sf, axis=1), 1.0, rtol=0, atol=1e-14)
    assert np.allclose(m.xc[0], 0.5, atol=1e-14)


def test_unit_tet_volume():
    # S:67 reference tetrahedron V = 1/6; centroid = vertex mean = 1/4
    m = oracle.Mesh(synth.fixture_unit_tet())
    assert abs(m.V[0] - 1.0 / 6.0) <= 1e-14
    assert np.allclose(m.xc[0], 0.25, atol=1e-14)
    # face centroid of a triangle = vertex mean; |S| of the slanted face = sqrt(3)/2
    assert np.isclose(np.linalg.norm(m.Sf, axis=1).max(), math.sqrt(3) / 2, atol=1e-15)


def test_two_cubes_fixture():
    # two unit cubes sharing a face: F=1, owner 0, neighbour 1, w = 0.5
    raw = synth.fixture_two_boxes(1.0)
    m = oracle.Mesh(raw)
    assert (m.N, m.F, m.NF) == (2, 1, 11)
    assert raw.owner[0] == 0 and raw.neighbour[0] == 1
    assert abs(m.w[0] - 0.5) <= 1e-15
    # S_f points out of the owner: +x
    assert np.allclose(m.Sf[0], [1, 0, 0], atol=1e-15)


def test_weight_one_to_three_boxes():
    # SURVEY.md §4 correction of S:138: 1x1x1 + 1x3 boxes (along x) -> centroid
    # distances 0.5 and 1.5 from the shared face -> w = 1.5 / 2.0 = 0.75
    m = oracle.Mesh(synth.fixture_two_boxes(3.0))
    assert abs(m.w[0] - 0.75) <= 1e-15
    assert abs(m.V[1] - 3.0) <= 1e-14


def test_out_of_range_point_is_reported():
    raw = synth.fixture_two_boxes(1.0)
    raw.face_points = raw.face_points.copy()
    raw.face_points[raw.face_offsets[3]] = len(raw.points)   # face 3 -> point n_points
    with pytest.raises(oracle.OracleError) as e:
        oracle.Mesh(raw)
    assert e.value.status == "MESH_CONSISTENCY" and e.value.index == 3


def test_owner_not_less_than_neighbour_is_reported():
    raw = synth.fixture_two_boxes(1.0)
    raw.owner = raw.owner.copy(); raw.neighbour = raw.neighbour.copy()
    raw.owner[0], raw.neighbour[0] = 1, 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.Mesh(raw)
    assert e.value.status == "MESH_CONSISTENCY" and e.value.index == 0


def _sheared_pair(shift):
    """unit cube + parallelepiped on its x=1 face whose far face is shifted by
    `shift` in y: centroid link d = (1, shift, 0)."""
    from synth import _from_cells, _HEX_FACES, PATCH_WALL
    a = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
    # second cell VTK order: x=1 face corners then x=2 (shifted) corners
    pts = a + [(2, shift, 0), (2, 1 + shift, 0), (2, 1 + shift, 1), (2, shift, 1)]
    c0 = [list(f) for f in _HEX_FACES]
    # cell 1 corners: 0:(1,0,0)=1, 1:(2,s,0)=8, 2:(2,1+s,0)=9, 3:(1,1,0)=2, 4:(1,0,1)=5, 5:(2,s,1)=11, 6:(2,1+s,1)=10, 7:(1,1,1)=6
    h = [1, 8, 9, 2, 5, 11, 10, 6]
    c1 = [[h[i] for i in f] for f in _HEX_FACES]
    return _from_cells(pts, [c0, c1], lambda P, r: ("walls", 0, PATCH_WALL))


@pytest.mark.parametrize("mode,delta_mag", [("overrelaxed", math.sqrt(2.0)), ("minimum", 1 / math.sqrt(2.0)),
                                            ("orthogonal", 1.0)])
def test_45_degree_face_delta(mode, delta_mag):
    # S:246 / P:251-254: d at 45 deg to S (A = 1): over-relaxed |Delta| = A sqrt2,
    # minimum A / sqrt2, orthogonal A; k = S - Delta
    m = oracle.Mesh(_sheared_pair(2.0), mode)
    d = np.array([1.0, 1.0, 0.0])
    assert np.allclose(m.xc[1], [1.5, 1.5, 0.5], atol=1e-14)
    Delta = m.delta[0] * d
    assert abs(np.linalg.norm(Delta) - delta_mag) <= 1e-14
    assert np.allclose(m.k[0], m.Sf[0] - Delta, atol=1e-15)
    assert abs(m.w[0] - 0.5) <= 1e-15


@pytest.mark.parametrize("mode", ["none", "minimum", "orthogonal", "overrelaxed"])
def test_orthogonal_faces_have_no_correction(mode):
    m = oracle.Mesh(synth.box(3, 4, 2, 1.0, 2.0, 0.5), mode)
    assert np.abs(m.k).max() <= 1e-15
    # every mode gives |S|/|d| on orthogonal faces
    d = m.xc[m.neighbour] - m.xc[m.owner[:m.F]]
    assert np.allclose(m.delta, np.linalg.norm(m.Sf[:m.F], axis=1) / np.linalg.norm(d, axis=1), rtol=1e-14)


@pytest.mark.parametrize("split", [0, 5, 6])
def test_closedness_and_total_volume_box(split):
    # S:32-34 / S:68: per-cell closedness and sum V = domain volume
    raw = synth.box(4, 3, 5, 1.0, 0.7, 1.3, split=split, jitter=0.2 if split else 0.0, scramble=3)
    m = oracle.Mesh(raw)
    assert abs(m.V.sum() - 1.0 * 0.7 * 1.3) <= 1e-12
    acc = np.zeros((m.N, 3))
    np.add.at(acc, m.owner, m.Sf)
    np.add.at(acc, m.neighbour, -m.Sf[:m.F])
    area = np.zeros(m.N)
    np.add.at(area, m.owner, np.linalg.norm(m.Sf, axis=1))
    np.add.at(area, m.neighbour, np.linalg.norm(m.Sf[:m.F], axis=1))
    assert (np.linalg.norm(acc, axis=1) <= 1e-12 * area).all()
    assert m.n_bad_pyramids == 0


@pytest.mark.parametrize("n,tets", [(6, True), (6, False), (12, True)])
def test_pipe_volume_inscribed_polygon(n, tets):
    # SURVEY.md §8(c) O-1 pin: the O-grid cross-section is the inscribed 4n-gon,
    # sum V = 2 n R^2 sin(pi / (2n)) L exactly.  Prototype: 1.552914 (n=6), 1.566314 (n=12)
    R, L = 0.5, 2.0
    raw = synth.pipe(n, 3 if n == 6 else 6, 8, R, L, tets=tets, scramble=5)
    m = oracle.Mesh(raw)
    exact = 2 * n * R * R * math.sin(math.pi / (2 * n)) * L
    assert abs(m.V.sum() - exact) <= 1e-12 * exact
    assert abs(exact - {6: 1.552914, 12: 1.566314}[n]) < 1e-6


def test_pipe_patch_counts():
    # SURVEY.md §8 "Config sizes": inlet = outlet = 2(n^2 + 4 n m_r), wall = 8 n n_z, F = (4N - B)/2
    raw = synth.pipe(6, 3, 20, 0.5, 2.0, tets=True)
    assert raw.n_cells == 10800
    sizes = {p.name: p.n for p in raw.patches}
    assert sizes == {"inlet": 216, "outlet": 216, "wall": 960}
    B = sum(sizes.values())
    assert raw.n_internal == (4 * raw.n_cells - B) // 2


def test_cavity_sizes():
    raw = synth.cavity(20)
    assert raw.n_cells == 400 and raw.n_internal == 760
    assert {p.name: p.n for p in raw.patches} == {"movingWall": 20, "fixedWalls": 60, "frontAndBack": 800}


def test_empty_patch_on_tet_slab_rejected():
    # O-0 rule 5: a one-layer tet slab with empty front/back is invalid
    raw = synth.box(3, 3, 1, 1.0, 1.0, 0.1, split=5, patch_mode=1)
    with pytest.raises(oracle.OracleError) as e:
        oracle.Mesh(raw)
    assert e.value.status == "MESH_CONSISTENCY"


def test_interpolation_weight_on_segment_matches_euclidean():
    # A-1: projected weight equals the Euclidean one when x_f lies on segment O-N
    m = oracle.Mesh(synth.box(5, 1, 1, 1.0, 1.0, 1.0))
    d0 = np.linalg.norm(m.xf[:m.F] - m.xc[m.owner[:m.F]], axis=1)
    d1 = np.linalg.norm(m.xc[m.neighbour] - m.xf[:m.F], axis=1)
    assert np.allclose(m.w, d1 / (d0 + d1), atol=1e-15)


def test_overrelaxed_clamp_on_extreme_faces():
    """A-4: on faces beyond ~87.1 deg the over-relaxed denominator S^.d is
    clamped at 0.05 |d|, delta = |S| / (0.05 |d|), and every clamped face is
    counted.  Sheared lattice (x, y + 25 x, z), h = 1/6 in x: x-faces have
    S = (A, 0, 0), A = h_y h_z, d = (h, 25 h, 0), S^.d = h < 0.05 |d| = 0.05 h sqrt(626)."""
    raw = synth.sheared_box(6, 5, 3, 25.0, scramble=0)
    m = oracle.Mesh(raw, "overrelaxed")
    # x-faces (5*5*3) and y-faces (6*4*3, normal ~ (-25, 1, 0) against d = (0, h_y, 0))
    # are clamped; the z-faces (6*5*2) are orthogonal
    assert m.F == 75 + 72 + 60 and m.n_clamped == 75 + 72
    hx, hy, hz = 1 / 6, 1 / 5, 1 / 3
    d = m.xc[m.neighbour] - m.xc[m.owner[:m.F]]
    xf = np.abs(d[:, 0]) > 0.5 * hx
    A = hy * hz
    assert np.allclose(m.delta[xf], A / (0.05 * hx * math.sqrt(626.0)), rtol=1e-13)
    assert np.allclose(np.linalg.norm(m.Sf[:m.F][xf], axis=1), A, rtol=1e-13)
