"""Multi-rank host logic on CPU: world_size-2 gloo
processes each build their part of the mesh with the library's host
pipeline (host-only meshes, no GPU) and check
  * the part's ghost / send lists equal the oracle's O-9 partition lists,
  * what rank p sends to q is exactly q's ghost slice for p, in order
    (exchanged over gloo), so NCCL receives land directly in the slice,
  * a halo exchange over gloo of a seeded field followed by a per-rank
    oracle-free gather gives every rank the right ghost values.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth


def _mesh():
    return synth.box(12, 3, 3, 6.0, 1.0, 1.0, split=5, scramble=12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        raw = _mesh()
        m = dfvm.Mesh(raw, n_parts=world, rank=rank, device=-1)
        h = m.export_halo()
        maps = m.export_maps()
        # (1) lists == oracle O-9
        R = oracle.Mesh(raw).renumber(world)
        ok1 = all(np.array_equal(h[k], R.parts[rank][k]) for k in ("ghost", "ghost_peer", "send", "send_peer"))
        # (2) send(p -> q) == ghost(q from p)
        allh = [None] * world
        dist.all_gather_object(allh, {k: v.tolist() for k, v in h.items()})
        ok2 = True
        for qq in range(world):
            if qq == rank:
                continue
            mine = [g for g, pp in zip(h["send"], h["send_peer"]) if pp == qq]
            theirs = [g for g, pp in zip(allh[qq]["ghost"], allh[qq]["ghost_peer"]) if pp == rank]
            ok2 &= mine == theirs
        # (3) halo exchange of a seeded field over gloo (new-id indexed values)
        import torch
        new_of_old = maps["cell_new_of_old"]
        x_old = synth.cell_field(7, raw.n_cells)
        x_new = np.empty_like(x_old)
        x_new[new_of_old] = x_old
        N = raw.n_cells
        lo, hi = rank * N // world, (rank + 1) * N // world
        owned = x_new[lo:hi]
        send_vals = {}
        for qq in set(h["send_peer"].tolist()):
            ids = h["send"][h["send_peer"] == qq]
            send_vals[qq] = owned[ids - lo]
        got = [None] * world
        dist.all_gather_object(got, {int(k): v.tolist() for k, v in send_vals.items()})
        ghosts = np.concatenate([np.array(got[qq][rank]) for qq in sorted(set(h["ghost_peer"].tolist()))]) \
            if len(h["ghost"]) else np.zeros(0)
        ok3 = np.array_equal(ghosts, x_new[h["ghost"]])
        q.put((rank, bool(ok1), bool(ok2), bool(ok3), len(h["ghost"])))
        dist.destroy_process_group()
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, False, False, False, repr(e)))


@pytest.mark.parametrize("world", [2])
def test_partition_halo_gloo(world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for r in res:
        assert r[1] and r[2] and r[3], r


@pytest.mark.parametrize("P", [2, 3, 4])
def test_host_only_parts_cover_and_match_oracle(P):
    raw = _mesh()
    R = oracle.Mesh(raw).renumber(P)
    owned = 0
    for r in range(P):
        m = dfvm.Mesh(raw, n_parts=P, rank=r, device=-1)
        h = m.export_halo()
        for k in ("ghost", "ghost_peer", "send", "send_peer"):
            assert np.array_equal(h[k], R.parts[r][k]), (r, k)
        owned += m.info["n_owned"]
        assert m.info["n_peers"] <= 2            # 1-D chain of RCM blocks
    assert owned == raw.n_cells
