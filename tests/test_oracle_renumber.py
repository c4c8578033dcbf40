"""Oracle pins for O-9 (RCM, face re-sort, CSR, partition, halo lists):
the hand-traced graphs of SURVEY.md §8(c) and structural invariants."""
import numpy as np
import pytest

import oracle
import synth
from synth import _from_cells, _HEX_FACES, _hex_pts, PATCH_WALL


def _boxes_mesh(boxes):
    """cell id i = axis-aligned box boxes[i]; shared vertices merged."""
    pts = []
    for b in boxes:
        pts += _hex_pts(*b)
    P = np.array(pts, np.float64)
    uniq, inv = np.unique(np.round(P, 12), axis=0, return_inverse=True)
    inv = inv.ravel()
    cells = [[[int(inv[8 * c + v]) for v in f] for f in _HEX_FACES] for c in range(len(boxes))]
    return _from_cells(uniq, cells, lambda P_, r: ("walls", 0, PATCH_WALL))


def _renumber(boxes, P=1):
    m = oracle.Mesh(_boxes_mesh(boxes))
    return m, m.renumber(P)


def test_rcm_path(golden):
    g = golden("rcm_hand_traces.json")["path_0_2_1_3"]
    pos = {cid: k for k, cid in enumerate(g["chain_order"])}
    boxes = [(pos[c], pos[c] + 1, 0, 1, 0, 1) for c in range(4)]
    _, R = _renumber(boxes)
    assert R.cell_new_of_old.tolist() == g["new_id"]


def test_rcm_grid_2x3(golden):
    g = golden("rcm_hand_traces.json")["grid_2x3"]
    boxes = [None] * 6
    for col, cid in enumerate(g["top_row"]):
        boxes[cid] = (col, col + 1, 1, 2, 0, 1)
    for col, cid in enumerate(g["bottom_row"]):
        boxes[cid] = (col, col + 1, 0, 1, 0, 1)
    _, R = _renumber(boxes)
    assert R.cell_new_of_old.tolist() == g["new_id"]


def test_rcm_two_components(golden):
    g = golden("rcm_hand_traces.json")["two_components"]
    boxes = [None] * 5
    for ci, chain in enumerate(g["chains"]):
        for k, cid in enumerate(chain):
            boxes[cid] = (k, k + 1, 0, 1, 3 * ci, 3 * ci + 1)
    _, R = _renumber(boxes)
    assert R.cell_new_of_old.tolist() == g["new_id"]


def _check_structure(m, R):
    N, F = m.N, m.F
    new = R.cell_new_of_old
    assert sorted(new.tolist()) == list(range(N))
    fno = R.face_new_of_old
    assert sorted(fno.tolist()) == list(range(m.NF))
    # internal faces: (a, b) sorted, a < b; flips exactly where new(owner) > new(nb)
    a = new[m.owner[:F]]; b = new[m.neighbour]
    flip = a > b
    assert (R.flip_of_old.astype(bool) == flip).all()
    lo = np.minimum(a, b); hi = np.maximum(a, b)
    order = np.empty(F, np.int64); order[fno[:F]] = np.arange(F)
    keys = np.stack([lo[order], hi[order]], 1)
    assert (np.diff(keys[:, 0]) >= 0).all()
    same = np.diff(keys[:, 0]) == 0
    assert (np.diff(keys[:, 1])[same] > 0).all() or (np.diff(keys[:, 1])[same] >= 0).all()
    # boundary faces stay in their patch and are sorted by new owner
    for p in m.patches:
        idx = np.arange(p.start, p.start + p.n)
        assert sorted(fno[idx].tolist()) == idx.tolist()
    # CSR: each internal face appears twice with opposite signs; rows ascending
    rp, inc, nb = R.row_ptr, R.inc_face, R.inc_nb
    assert rp[-1] == 2 * F
    fidx = inc & 0x7FFFFFFF
    for c in range(N):
        row = fidx[rp[c]:rp[c + 1]]
        assert (np.diff(row) > 0).all()
    cnt = np.bincount(fidx, minlength=F)
    assert (cnt == 2).all()
    # neighbours consistent with face endpoints
    rows = np.repeat(np.arange(N), np.diff(rp))
    own_new = np.empty(F, np.int64); own_new[fno[:F]] = lo
    nb_new = np.empty(F, np.int64); nb_new[fno[:F]] = hi
    s_neg = inc < 0
    assert (rows[~s_neg] == own_new[fidx[~s_neg]]).all() and (nb[~s_neg] == nb_new[fidx[~s_neg]]).all()
    assert (rows[s_neg] == nb_new[fidx[s_neg]]).all() and (nb[s_neg] == own_new[fidx[s_neg]]).all()


@pytest.mark.parametrize("P", [1, 2, 4])
def test_renumber_structure_and_partition(P):
    raw = synth.box(16, 3, 3, 8.0, 1.0, 1.0, split=5, scramble=12)
    m = oracle.Mesh(raw)
    R = m.renumber(P)
    _check_structure(m, R)
    assert R.bw_after < R.bw_before
    N = m.N
    sizes = np.bincount(R.part, minlength=P)
    assert sizes.sum() == N and (sizes == [((p + 1) * N) // P - (p * N) // P for p in range(P)]).all()
    rp, nb = R.row_ptr, R.inc_nb
    for p, d in enumerate(R.parts):
        lo, hi = (p * N) // P, ((p + 1) * N) // P
        need = set()
        for c in range(lo, hi):
            for k in range(rp[c], rp[c + 1]):
                if not (lo <= nb[k] < hi):
                    need.add(int(nb[k]))
        assert sorted(need) == sorted(d["ghost"].tolist())
        # ordered by (peer, new id); peers are neighbours in the chain
        key = list(zip(d["ghost_peer"].tolist(), d["ghost"].tolist()))
        assert key == sorted(key)
        assert set(d["ghost_peer"].tolist()) <= {p - 1, p + 1}
        # the send list to q equals q's ghost slice from p, same order
        for q in set(d["send_peer"].tolist()):
            mine = d["send"][d["send_peer"] == q].tolist()
            theirs = R.parts[q]["ghost"][R.parts[q]["ghost_peer"] == p].tolist()
            assert mine == theirs


def test_renumber_identity_option():
    m = oracle.Mesh(synth.box(3, 3, 3, scramble=4))
    R = m.renumber(1, rcm=False)
    assert (R.cell_new_of_old == np.arange(m.N)).all()
    _check_structure(m, R)
