"""Shared helpers of the GPU parity tests: build the same case on the oracle
and on the CUDA library from one seeded input recipe, and the parity
metrics of SURVEY.md §8(c) "Parity metrics and tolerances"."""
import numpy as np

import oracle
import paper_2603_15920_b200 as dfvm
import synth

TOL_OP = {"f64": 1e-12, "f32": 1e-5}


def rel_op_err(y, yref, scale):
    """||y - yref||_2 / ||scale||_2 with scale the absolute-term sum (§8(c))."""
    return float(np.linalg.norm(np.ravel(y - yref)) / max(np.linalg.norm(np.ravel(scale)), 1e-300))


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def make_bcs(raw, specs, m_or, m_gpu):
    """specs: list of (patch_name, field, kind, kwargs)"""
    bo, bg = oracle.BCs(m_or), dfvm.BCs(m_gpu)
    for name, fld, kind, kw in specs:
        bo.set(name, fld, kind, **kw)
        bg.set(name, fld, kind, **kw)
    return bo, bg


def all_patches(raw, fld, kind, **kw):
    return [(p.name, fld, kind, kw) for p in raw.patches if p.kind != synth.PATCH_EMPTY]


MESHES = {
    "cavity": lambda: synth.cavity(20, scramble=11),
    "box_tet5_jitter": lambda: synth.box(5, 4, 3, 1.0, 0.8, 0.6, split=5, jitter=0.15, scramble=9),
    "kuhn8": lambda: synth.box(8, 8, 8, split=6, scramble=3),
    "pipe_tet": lambda: synth.pipe(6, 3, 20, 0.5, 2.0, tets=True, scramble=12),
    "pipe_hex": lambda: synth.pipe(8, 4, 10, 0.5, 1.0, tets=False, scramble=5),
    "cylinder_poly": lambda: synth.cylinder_poly(6e3, scramble=13),     # C3 family: polygon prisms, F/N ~ 3
    "square_tri": lambda: synth.square_tri(12, jitter=0.2),             # NEXT-1 domain: triangle prisms
    "htree_tet": lambda: synth.htree(target_cells=2e4, scramble=14),    # C4 family: voxel tree, 5-tet
    "sheared_clamp": lambda: synth.sheared_box(6, 5, 3, 25.0),           # > 87 deg faces: A-4 clamp active
}


def grad_scale(m_or, fv, ncomp):
    """per-cell absolute-term sum of the Gauss gradient: sum_f |phi_f||S_f| / V"""
    fv = np.asarray(fv).reshape(m_or.NF, ncomp)
    A = np.linalg.norm(m_or.Sf, axis=1)
    empty = np.zeros(m_or.NF, bool)
    for p in m_or.patches:
        if p.kind == synth.PATCH_EMPTY:
            empty[p.start:p.start + p.n] = True
    t = np.abs(fv) * A[:, None]
    t[empty] = 0
    s = np.zeros((m_or.N, ncomp))
    np.add.at(s, m_or.owner, t)
    np.add.at(s, m_or.neighbour, t[:m_or.F])
    return s / m_or.V[:, None]
