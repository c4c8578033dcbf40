"""OpenFOAM ASCII polyMesh reader (PAPER.md P:431-432
"reads OpenFOAM polyMesh files directly", Table 1): host-only tests.

* golden fixture tests/golden/polymesh_two_hex (hand-written: two unit cubes,
  comments, a face split over two lines, extra patch entries): parsed arrays
  equal the literal ones; the oracle's geometry of the parsed mesh gives the
  closed forms (V = 1 per cell, S = (1, 0, 0) on the shared face);
* round trip: synth.write_polymesh of the generators' meshes read back
  bit-exactly (integers and the 17-digit points);
* errors: binary format, cyclic patch, missing files, truncated list.
"""
import os
import shutil

import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "polymesh_two_hex")


def test_golden_two_hex():
    m = dfvm.read_polymesh(GOLDEN)
    assert m.n_cells == 2 and m.n_faces == 11 and m.n_internal == 1
    assert m.points.shape == (12, 3)
    assert np.array_equal(m.points[8], [2.0, 0.0, 1.0]) and np.array_equal(m.points[10], [1.0, 1.0, 1.0])
    assert np.array_equal(m.face_offsets, np.arange(0, 45, 4))
    assert m.face_points[:4].tolist() == [1, 4, 10, 7]
    assert m.face_points[24:28].tolist() == [4, 10, 11, 5]       # the face written over two lines
    assert m.owner.tolist() == [0, 0, 1, 0, 1, 0, 1, 0, 1, 0, 1] and m.neighbour.tolist() == [1]
    assert [(p.name, p.kind, p.start, p.n) for p in m.patches] == [
        ("inlet", synth.PATCH_GENERIC, 1, 1), ("outlet", synth.PATCH_GENERIC, 2, 1),
        ("walls", synth.PATCH_WALL, 3, 4), ("frontAndBack", synth.PATCH_EMPTY, 7, 4)]
    # the case dir, constant/polyMesh and the polyMesh dir itself all work
    m2 = dfvm.read_polymesh(os.path.join(GOLDEN, "constant", "polyMesh"))
    assert np.array_equal(m2.face_points, m.face_points)
    # closed forms through the oracle's geometry (test infrastructure)
    mo = oracle.Mesh(m)
    assert np.allclose(mo.V, [1.0, 1.0], rtol=0, atol=1e-15)
    assert np.allclose(mo.Sf[0], [1.0, 0.0, 0.0], rtol=0, atol=1e-15)
    assert np.allclose(mo.xc, [[0.5, 0.5, 0.5], [1.5, 0.5, 0.5]], rtol=0, atol=1e-15)


@pytest.mark.parametrize("gen", ["cavity", "pipe_tet", "cylinder_poly", "htree"])
def test_round_trip(gen, tmp_path):
    raw = {"cavity": lambda: synth.cavity(20, scramble=11),
           "pipe_tet": lambda: synth.pipe(4, 2, 6, 0.5, 1.0, tets=True, scramble=21),
           "cylinder_poly": lambda: synth.cylinder_poly(3e3, scramble=13),
           "htree": lambda: synth.htree(target_cells=2e4, scramble=14)}[gen]()
    synth.write_polymesh(raw, str(tmp_path))
    m = dfvm.read_polymesh(str(tmp_path))
    assert np.array_equal(m.points, raw.points)
    for k in ("face_offsets", "face_points", "owner", "neighbour"):
        assert np.array_equal(getattr(m, k), getattr(raw, k)), k
    assert m.n_cells == raw.n_cells
    assert [(p.name, p.kind, p.start, p.n) for p in m.patches] == [(p.name, p.kind, p.start, p.n) for p in raw.patches]
    # renumbering maps of the parsed mesh equal the oracle's maps of the generator's arrays
    R0, R1 = oracle.Renumbering(oracle.Mesh(raw), 1), oracle.Renumbering(oracle.Mesh(m), 1)
    assert np.array_equal(R0.cell_new_of_old, R1.cell_new_of_old)


def _copy(tmp_path):
    d = tmp_path / "case"
    shutil.copytree(GOLDEN, d)
    return d / "constant" / "polyMesh"


def _err(path):
    with pytest.raises(dfvm.DfvmError) as e:
        dfvm.read_polymesh(str(path))
    return str(e.value)


def test_errors(tmp_path):
    assert "INVALID_ARG" in _err(tmp_path / "nowhere")
    d = _copy(tmp_path)
    txt = (d / "points").read_text()
    (d / "points").write_text(txt.replace("format      ascii;", "format      binary;"))
    assert "binary" in _err(d)
    (d / "points").write_text(txt)
    (d / "boundary").write_text((d / "boundary").read_text().replace("type            patch;\n        physicalType",
                                                                     "type            cyclic;\n        physicalType"))
    assert "cyclic" in _err(d)
    d2 = _copy(tmp_path / "b")
    (d2 / "faces").write_text((d2 / "faces").read_text().replace("4(7 8 11 10)\n)", "4(7 8 11"))
    assert "faces" in _err(d2)
    d3 = _copy(tmp_path / "c")
    os.remove(d3 / "owner")
    assert "owner" in _err(d3)
