"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY.md §8(c) tolerances): integer maps bit-exact,
geometry <= 1e-14, operator applies <= 1e-12 (fp64) / 1e-5 (fp32) relative to
the absolute-term scale, converged fields <= 1e-8 relative L2 (fp64)."""
import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import MESHES, TOL_OP, all_patches, grad_scale, make_bcs, rel_l2, rel_op_err

pytestmark = pytest.mark.gpu

_cache = {}


def pair(name, nonorth="overrelaxed", precision="f64"):
    key = (name, nonorth, precision)
    if key not in _cache:
        raw = MESHES[name]()
        _cache[key] = (raw, oracle.Mesh(raw, nonorth), dfvm.Mesh(raw, nonorth=nonorth, precision=precision))
    return _cache[key]


# ------------------------------------------------------------ maps, geometry
@pytest.mark.parametrize("name", list(MESHES))
def test_integer_maps_bit_exact(name):
    raw, mo, mg = pair(name)
    R = mo.renumber(1)
    g = mg.export_maps()
    assert np.array_equal(g["cell_new_of_old"], R.cell_new_of_old)
    assert np.array_equal(g["face_new_of_old"], R.face_new_of_old)
    assert np.array_equal(g["face_flip"], R.flip_of_old)
    assert np.array_equal(g["row_ptr"], R.row_ptr)
    assert np.array_equal(g["inc_face"], R.inc_face)
    assert np.array_equal(g["inc_nb"], R.inc_nb)
    assert mg.info["bandwidth_after"] == R.bw_after and mg.info["bandwidth_before"] == R.bw_before


@pytest.mark.parametrize("name", list(MESHES))
@pytest.mark.parametrize("mode", ["overrelaxed", "minimum", "none"])
def test_geometry_and_coefficients(name, mode):
    raw, mo, mg = pair(name, mode)
    g = mg.export_geometry()
    L = np.abs(mo.xc).max() + 1.0
    A = np.linalg.norm(mo.Sf, axis=1).max()
    assert np.abs(g["Sf"] - mo.Sf).max() <= 1e-14 * A
    assert np.abs(g["xf"] - mo.xf).max() <= 1e-14 * L
    assert np.abs(g["xc"] - mo.xc).max() <= 1e-14 * L
    assert np.abs(g["V"] - mo.V).max() <= 1e-14 * mo.V.max()
    assert np.abs(g["w"] - mo.w).max() <= 1e-14
    assert np.abs(g["delta"] - mo.delta).max() <= 1e-14 * np.abs(mo.delta).max()
    assert np.abs(g["k"] - mo.k).max() <= 1e-14 * A
    assert np.abs(g["delta_b"] - mo.delta_b).max() <= 1e-14 * np.abs(mo.delta_b).max()
    assert mg.info["n_clamped"] == mo.n_clamped


# ------------------------------------------------------------ operators
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", list(MESHES))
def test_grad_scalar_and_vector(name, precision):
    raw, mo, mg = pair(name, precision=precision)
    for fld, nc, kind in (("s", 1, oracle.BC_FIXED), ("U", 3, oracle.BC_FIXED), ("s", 1, oracle.BC_ZEROGRAD)):
        bo, bg = make_bcs(raw, all_patches(raw, fld, kind, value=(0.3, -0.2, 0.1)), mo, mg)
        x = synth.cell_field(100, mo.N, nc)
        ref = mo.grad(bo, fld, x)
        xg = mg.field("cells", nc, x)
        G = mg.field("cells", 3 * nc)
        dfvm.grad(mg, xg, bg, fld, G)
        got = G.get().reshape(ref.shape)
        scale = grad_scale(mo, mo.interpolate(bo, fld, x), nc)
        assert rel_op_err(got, ref, scale) <= TOL_OP[precision], (fld, kind)


@pytest.mark.parametrize("name", list(MESHES))
def test_grad_from_face_values(name):
    raw, mo, mg = pair(name)
    fv = synth.face_field(300, mo.NF)
    for p in raw.patches:
        if p.kind == synth.PATCH_EMPTY:
            fv[p.start:p.start + p.n] = 0
    ref = mo.grad_faces(fv)
    f = mg.field("faces", 1, fv)
    G = mg.field("cells", 3)
    dfvm.grad_faces(mg, f, G)
    assert rel_op_err(G.get(), ref, grad_scale(mo, fv, 1)) <= 1e-12


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("name", list(MESHES))
def test_div(name, precision):
    raw, mo, mg = pair(name, precision=precision)
    F = synth.face_field(300, mo.NF)
    for p in raw.patches:
        if p.kind == synth.PATCH_EMPTY:
            F[p.start:p.start + p.n] = 0
    ref = mo.div(F)
    f = mg.field("flux", 1, F)
    out = mg.field("cells", 1)
    dfvm.div(mg, f, out)
    scale = np.zeros(mo.N)
    np.add.at(scale, mo.owner, np.abs(F))
    np.add.at(scale, mo.neighbour, np.abs(F[:mo.F]))
    assert rel_op_err(out.get(), ref, scale) <= TOL_OP[precision]


@pytest.mark.parametrize("name", list(MESHES))
def test_interpolate(name):
    raw, mo, mg = pair(name)
    bo, bg = make_bcs(raw, all_patches(raw, "U", oracle.BC_FIXED, value=(1.0, 2.0, 3.0)), mo, mg)
    x = synth.cell_field(100, mo.N, 3)
    ref = mo.interpolate(bo, "U", x)
    out = mg.field("faces", 3)
    dfvm.interpolate(mg, mg.field("cells", 3, x), bg, "U", out)
    assert np.abs(out.get() - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("mode", ["overrelaxed", "minimum", "orthogonal", "none"])
@pytest.mark.parametrize("name", list(MESHES))
def test_laplacian(name, mode, precision):
    raw, mo, mg = pair(name, mode, precision)
    specs = all_patches(raw, "s", oracle.BC_FIXED, value=0.7)
    specs[-1] = (specs[-1][0], "s", oracle.BC_ZEROGRAD, {})
    bo, bg = make_bcs(raw, specs, mo, mg)
    x = synth.cell_field(100, mo.N)
    gam = 1.0 + 0.5 * synth.cell_field(200, mo.N)
    for gamma in (None, gam):
        y, ya = mo.laplacian(bo, "s", x, gamma=gamma)
        out = mg.field("cells", 1)
        dfvm.laplacian(mg, bg, "s", mg.field("cells", 1, x), out,
                       gamma=None if gamma is None else mg.field("cells", 1, gamma))
        assert rel_op_err(out.get(), y, ya) <= TOL_OP[precision]


def test_laplacian_given_gradient_exact_identity():
    # caller-given exact gradient: interior cells of a linear field give 0 on any mesh
    raw, mo, mg = pair("box_tet5_jitter")
    bo, bg = make_bcs(raw, all_patches(raw, "s", oracle.BC_ZEROGRAD), mo, mg)
    a = np.array([0.5, 1.5, -0.7])
    x = mo.xc @ a
    G = np.tile(a, (mo.N, 1))
    y, ya = mo.laplacian(bo, "s", x, grad=G)
    out = mg.field("cells", 1)
    dfvm.laplacian(mg, bg, "s", mg.field("cells", 1, x), out, grad=mg.field("cells", 3, G))
    assert rel_op_err(out.get(), y, ya) <= 1e-12


def test_operators_deterministic():
    raw, mo, mg = pair("pipe_tet")
    bo, bg = make_bcs(raw, all_patches(raw, "s", oracle.BC_FIXED, value=0.1), mo, mg)
    x = mg.field("cells", 1, synth.cell_field(100, mo.N))
    outs = []
    for _ in range(2):
        o = mg.field("cells", 1)
        dfvm.laplacian(mg, bg, "s", x, o)
        outs.append(o.get())
    assert np.array_equal(outs[0], outs[1])


def test_missing_bc_reported():
    raw, mo, mg = pair("cavity")
    bg = dfvm.BCs(mg)
    with pytest.raises(dfvm.DfvmError) as e:
        dfvm.grad(mg, mg.field("cells", 1), bg, "s", mg.field("cells", 3))
    assert e.value.status == "MISSING_BC"


def test_mesh_errors_reported_in_original_numbering():
    raw = synth.fixture_two_boxes(1.0)
    raw.face_points = raw.face_points.copy()
    raw.face_points[raw.face_offsets[3]] = len(raw.points)
    with pytest.raises(dfvm.DfvmError) as e:
        dfvm.Mesh(raw)
    assert e.value.status == "MESH_CONSISTENCY" and e.value.index == 3
