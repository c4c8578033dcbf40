"""Seeded synthetic inputs (meshes and fields) shared by the oracle tests,
the CUDA parity tests, ``smoke()`` and ``bench.py``.

INPUT TOOLING ONLY: nothing here computes any part of the finite-volume
method (no areas, volumes, weights, operators).  Meshes come from
``libsynth.so`` (synth/meshgen.cpp) in OpenFOAM polyMesh convention
(SPEC.md:23-27); fields come from the
counter-based generator ``urand(seed, id)`` of SURVEY.md §8(d2), so a value
depends only on (seed, original id) and is identical for oracle and GPU
regardless of renumbering.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

PATCH_GENERIC, PATCH_WALL, PATCH_EMPTY = 0, 1, 2


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(path)
        vp, i64, i32, f64, u64 = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_uint64
        L.synth_box.restype = vp
        L.synth_box.argtypes = [i32, i32, i32, f64, f64, f64, i32, i32, f64, u64, u64]
        L.synth_pipe.restype = vp
        L.synth_pipe.argtypes = [i32, i32, i32, f64, f64, i32, u64]
        L.synth_voxel_tree.restype = vp
        L.synth_voxel_tree.argtypes = [i32, i32, i32, f64, f64, f64, f64, vp, vp, i32, vp, i32, f64, i32, u64]
        L.synth_extrude_polygons.restype = vp
        L.synth_extrude_polygons.argtypes = [vp, i64, vp, vp, i64, f64, vp, vp, i32, vp, i32, i32, u64]
        L.synth_error.restype = C.c_char_p
        L.synth_error.argtypes = [vp]
        L.synth_sizes.argtypes = [vp, vp]
        L.synth_copy.argtypes = [vp] * 9
        L.synth_patch_name.restype = C.c_char_p
        L.synth_patch_name.argtypes = [vp, i32]
        L.synth_free.argtypes = [vp]
        _LIB = L
    return _LIB


@dataclass
class Patch:
    name: str
    kind: int      # PATCH_GENERIC / PATCH_WALL / PATCH_EMPTY
    start: int
    n: int


@dataclass
class RawMesh:
    """OpenFOAM-style raw mesh: internal faces first with
    owner < neighbour, face rings oriented out of the owner, patches tiling
    the boundary faces in order."""
    points: np.ndarray          # [n_p, 3] f64
    face_offsets: np.ndarray    # [n_f + 1] i64
    face_points: np.ndarray     # [sum] i32
    owner: np.ndarray           # [n_f] i32
    neighbour: np.ndarray       # [F] i32
    patches: list
    n_cells: int
    meta: dict = field(default_factory=dict)

    @property
    def n_faces(self):
        return len(self.owner)

    @property
    def n_internal(self):
        return len(self.neighbour)

    def patch(self, name):
        for i, p in enumerate(self.patches):
            if p.name == name:
                return i
        raise KeyError(name)


def _take(h) -> RawMesh:
    L = _lib()
    if not h:
        raise RuntimeError("generator returned NULL")
    err = L.synth_error(h)
    if err:
        L.synth_free(h)
        raise ValueError(err.decode())
    s = np.zeros(6, np.int64)
    L.synth_sizes(h, s.ctypes.data)
    n_p, n_f, F, n_fp, n_pat, N = (int(x) for x in s)
    pts = np.empty((n_p, 3), np.float64)
    fo = np.empty(n_f + 1, np.int64)
    fp = np.empty(n_fp, np.int32)
    own = np.empty(n_f, np.int32)
    nb = np.empty(F, np.int32)
    ps = np.empty(n_pat, np.int64)
    pn = np.empty(n_pat, np.int64)
    pk = np.empty(n_pat, np.int32)
    L.synth_copy(h, pts.ctypes.data, fo.ctypes.data, fp.ctypes.data, own.ctypes.data,
                 nb.ctypes.data, ps.ctypes.data, pn.ctypes.data, pk.ctypes.data)
    patches = [Patch(L.synth_patch_name(h, i).decode(), int(pk[i]), int(ps[i]), int(pn[i]))
               for i in range(n_pat)]
    L.synth_free(h)
    return RawMesh(pts, fo, fp, own, nb, patches, N)


# ----------------------------------------------------------------- meshes
def box(nx, ny, nz, lx=1.0, ly=1.0, lz=1.0, split=0, patch_mode=0, jitter=0.0,
        jitter_seed=1, scramble=0) -> RawMesh:
    """Structured box [0,lx]x[0,ly]x[0,lz]; split 0 = hex, 5 = alternating
    5-tet (global vertex parity), 6 = Kuhn 6-tet.  patch_mode: 0 six sides,
    1 cavity, 2 single patch, 3 channel slab.  jitter moves interior vertices
    by up to jitter*h per axis (order-independent splitmix64)."""
    m = _take(_lib().synth_box(nx, ny, nz, lx, ly, lz, split, patch_mode, jitter,
                               jitter_seed, scramble))
    m.meta = dict(kind="box", nx=nx, ny=ny, nz=nz, lx=lx, ly=ly, lz=lz, split=split)
    return m


def sheared_box(nx=6, ny=5, nz=3, alpha=25.0, scramble=6) -> RawMesh:
    """Hex box [0,1]^3 mapped by (x, y, z) -> (x, y + alpha x, z): every cell a
    congruent parallelepiped, x- and y-faces at arctan(alpha) to their centroid
    links (alpha = 25: 87.7 deg, beyond the 87.1 deg at which the over-relaxed
    coefficient is clamped, A-4).  Data only: a point transform."""
    m = box(nx, ny, nz, 1.0, 1.0, 1.0, split=0, scramble=scramble)
    m.points = np.array(m.points, np.float64, copy=True)
    m.points[:, 1] += alpha * m.points[:, 0]
    m.meta = dict(m.meta, kind="sheared_box", alpha=alpha)
    return m


def cavity(n=20, scramble=11) -> RawMesh:
    """C1: OpenFOAM cavity tutorial mesh, 0.1 x 0.1 x 0.01 m, n x n x 1 hex
    (reading A-31): movingWall (top), fixedWalls, and
    empty frontAndBack."""
    return box(n, n, 1, 0.1, 0.1, 0.01, split=0, patch_mode=1, scramble=scramble)


def pipe(n=16, m_r=8, n_z=52, R=0.5, L=2.6, tets=True, scramble=12) -> RawMesh:
    """C2/C5: O-grid circular pipe along z; patches inlet
    (z=0), outlet (z=L), wall.  Cells: n_z (n^2 + 4 n m_r) hexes, x5 if tets."""
    m = _take(_lib().synth_pipe(n, m_r, n_z, R, L, 1 if tets else 0, scramble))
    m.meta = dict(kind="pipe", n=n, m_r=m_r, n_z=n_z, R=R, L=L, tets=tets,
                  inlet_center=(0.0, 0.0, 0.0), inlet_radius=R)
    return m


def pipe_c2(scramble=12):
    """configs[1]: ~200k-tet Poiseuille pipe (N = 199 680)."""
    return pipe(16, 8, 52, 0.5, 2.6, True, scramble)


def pipe_c5(n_z=814, scramble=15):
    """configs[4]: 50 012 160-tet pipe (n=64, m_r=32, n_z=814, L=10)."""
    return pipe(64, 32, n_z, 0.5, 10.0 * n_z / 814.0, True, scramble)


def htree(depth=3, r0=1.0, l0=8.0, h=None, target_cells=1.0e7, tets=True, scramble=14):
    """C4: voxelised H-tree vascular geometry: root tube
    radius r0, length l0 along +x; each generation l <- l/sqrt(2),
    r <- r/2^(1/3) (Murray), alternating x/y, branching both ways; depth
    generations -> 2^depth terminal outlets.  Flat-ended cylinders per
    segment plus spheres at joints; voxel -> 5 tets by global parity."""
    segs, rads = [], []
    ports = []  # (cx, cy, cz, ax, ay, az, radius)
    x0 = np.array([0.0, 0.0, 0.0])
    ports.append((*x0, -1.0, 0.0, 0.0, r0))
    x1 = x0 + np.array([l0, 0.0, 0.0])
    segs.append((*x0, *x1)); rads.append(-r0)
    frontier = [(x1, np.array([1.0, 0.0, 0.0]), l0, r0)]
    for g in range(depth):
        nxt = []
        for (p, d, l, r) in frontier:
            l2, r2 = l / math.sqrt(2.0), r / 2.0 ** (1.0 / 3.0)
            perp = np.array([-d[1], d[0], 0.0])
            segs.append((*p, *p)); rads.append(r)          # joint sphere
            for sgn in (1.0, -1.0):
                e = p + sgn * perp * l2
                segs.append((*p, *e)); rads.append(-r2)
                nxt.append((e, sgn * perp, l2, r2))
        frontier = nxt
    for (p, d, l, r) in frontier:
        ports.append((*p, *d, r))
    seg = np.array(segs, np.float64)
    rad = np.array(rads, np.float64)
    lo = np.minimum(seg[:, :3], seg[:, 3:]).min(0) - np.abs(rad).max() - 1e-9
    hi = np.maximum(seg[:, :3], seg[:, 3:]).max(0) + np.abs(rad).max() + 1e-9
    vol = float(np.sum(np.pi * rad ** 2 * np.linalg.norm(seg[:, 3:] - seg[:, :3], axis=1)))
    if h is None:
        nvox = target_cells / (5.0 if tets else 1.0)
        h = (vol / nvox) ** (1.0 / 3.0)
    n = np.ceil((hi - lo) / h).astype(int)
    # shift the voxel lattice so that port planes coincide with voxel faces:
    # ports sit at x0 (inlet) and terminal ends; choose origin at the inlet.
    org = np.floor((lo - x0) / h) * h + x0
    n = np.ceil((hi - org) / h).astype(int)
    P = np.array(ports, np.float64)
    m = _take(_lib().synth_voxel_tree(int(n[0]), int(n[1]), int(n[2]), float(org[0]), float(org[1]),
                                      float(org[2]), float(h), seg.ctypes.data, rad.ctypes.data,
                                      len(rad), P.ctypes.data, len(P), float(0.75 * h),
                                      1 if tets else 0, scramble))
    m.meta = dict(kind="htree", h=h, ports=P, depth=depth)
    return m


def extrude_polygons(pts2, polys, dz, patch_names, patch_kinds, rules, empty_patch, scramble=0):
    """Assemble a one-layer extruded polygon slab (C3 building block).
    polys: list of CCW vertex-id lists, or a pair (offsets[n+1], ids)."""
    pts2 = np.ascontiguousarray(pts2, np.float64)
    if isinstance(polys, tuple):
        off = np.ascontiguousarray(polys[0], np.int64)
        ids = np.ascontiguousarray(polys[1], np.int32)
        polys = range(len(off) - 1)
    else:
        off = np.zeros(len(polys) + 1, np.int64)
        off[1:] = np.cumsum([len(p) for p in polys])
        ids = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in polys]), np.int32)
    names = (C.c_char_p * len(patch_names))(*[s.encode() for s in patch_names])
    kinds = np.asarray(patch_kinds, np.int32)
    R = np.ascontiguousarray(rules, np.float64)
    m = _take(_lib().synth_extrude_polygons(pts2.ctypes.data, len(pts2), off.ctypes.data,
                                            ids.ctypes.data, len(polys), dz, C.cast(names, C.c_void_p),
                                            kinds.ctypes.data, len(patch_names), R.ctypes.data,
                                            len(R), empty_patch, scramble))
    m.meta = dict(kind="extruded", dz=dz)
    return m


# ------------------------------------------------------------ hand fixtures
def _from_cells(points, cell_faces, patch_of_boundary):
    """Tiny hand fixtures: cell_faces[c] = list of
    outward rings.  Internal faces are found by vertex-set matching."""
    points = np.asarray(points, np.float64)
    inst = {}
    for c, faces in enumerate(cell_faces):
        for r in faces:
            inst.setdefault(frozenset(r), []).append((c, list(r)))
    internal, boundary = [], []
    for key, lst in inst.items():
        if len(lst) == 2:
            (c0, r0), (c1, r1) = sorted(lst)
            internal.append((c0, c1, r0))
        else:
            boundary.append((lst[0][0], lst[0][1]))
    internal.sort()
    names = sorted(set(patch_of_boundary(points, r) for _, r in boundary), key=lambda s: s[1])
    rings, own, nb = [], [], []
    for o, n_, r in internal:
        rings.append(r); own.append(o); nb.append(n_)
    patches = []
    for name, order, kind in names:
        start = len(rings)
        for o, r in sorted(boundary):
            if patch_of_boundary(points, r)[0] == name:
                rings.append(r); own.append(o)
        patches.append(Patch(name, kind, start, len(rings) - start))
    fo = np.zeros(len(rings) + 1, np.int64)
    fo[1:] = np.cumsum([len(r) for r in rings])
    return RawMesh(points, fo, np.array([v for r in rings for v in r], np.int32),
                   np.array(own, np.int32), np.array(nb, np.int32), patches, len(cell_faces))


_HEX_FACES = [[0, 3, 2, 1], [4, 5, 6, 7], [0, 1, 5, 4], [3, 7, 6, 2], [0, 4, 7, 3], [1, 2, 6, 5]]


def _hex_pts(x0, x1, y0, y1, z0, z1):
    return [(x0, y0, z0), (x1, y0, z0), (x1, y1, z0), (x0, y1, z0),
            (x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1)]


def fixture_unit_cube():
    """Single unit-cube hexahedron: N=1, F=0, B=6."""
    return _from_cells(_hex_pts(0, 1, 0, 1, 0, 1), [_HEX_FACES],
                       lambda P, r: ("walls", 0, PATCH_WALL))


def fixture_two_boxes(ly2=1.0):
    """Two boxes sharing the unit face x=1: [0,1]^3 and [1,1+ly2]x[0,1]^2
    (ly2=1: SPEC.md:49 two cubes; ly2=3: the 1x1x1 + 1x1x3 pair of
    SURVEY.md §4 whose weight is w = 0.75)."""
    pts = _hex_pts(0, 1, 0, 1, 0, 1) + _hex_pts(1, 1 + ly2, 0, 1, 0, 1)
    # merge the shared vertices (x=1 plane)
    P = np.array(pts)
    uniq, inv = np.unique(np.round(P, 12), axis=0, return_inverse=True)
    inv = inv.ravel()
    c0 = [[int(inv[v]) for v in f] for f in _HEX_FACES]
    c1 = [[int(inv[v + 8]) for v in f] for f in _HEX_FACES]
    return _from_cells(uniq, [c0, c1], lambda P, r: ("walls", 0, PATCH_WALL))


def fixture_unit_tet():
    """Reference tetrahedron (0,0,0),(1,0,0),(0,1,0),(0,0,1): V = 1/6."""
    pts = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    faces = [[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]]
    return _from_cells(pts, [faces], lambda P, r: ("walls", 0, PATCH_WALL))


# ------------------------------------------------------------------ fields
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(x):
    x = x + _GOLD
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def urand(seed, ids):
    """u(seed, id) in [-1, 1) with 53 bits: splitmix64(seed ^ id*golden)
    (SURVEY.md §8(d2)); identical to the generator's C++ jitter stream."""
    ids = np.asarray(ids, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _splitmix64(np.uint64(seed) ^ (ids * _GOLD))
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0


def cell_field(seed, n_cells, n_comp=1):
    """Operator-benchmark input x_c = u(seed + k, original cell id) for
    component k; shape [N] or [N, n_comp]."""
    ids = np.arange(n_cells, dtype=np.uint64)
    if n_comp == 1:
        return urand(seed, ids)
    return np.stack([urand(seed + k, ids) for k in range(n_comp)], axis=1)


def face_field(seed, n_faces):
    return urand(seed, np.arange(n_faces, dtype=np.uint64))


def square_tri(n=20, jitter=0.25, seed=7, scramble=5, y_step=0.5):
    """Unit square [0,1]^2 triangulated (Delaunay of an (n+1)^2 lattice with
    interior vertices jittered by jitter*h, order-independent splitmix64) and
    extruded one layer (dz = 1/n, empty front/back) — the paper's step
    advection domain (§3.1.2, unstructured triangular mesh).
    Patches: inlet_lower (x=0, y<y_step, and y=0), inlet_upper (x=0,
    y>=y_step), outlet (x=1 and y=1), frontAndBack (empty)."""
    from scipy.spatial import Delaunay
    h = 1.0 / n
    ij = np.array([(i, j) for j in range(n + 1) for i in range(n + 1)], np.float64)
    pts = ij * h
    vid = np.arange(len(pts), dtype=np.uint64)
    interior = (ij[:, 0] > 0) & (ij[:, 0] < n) & (ij[:, 1] > 0) & (ij[:, 1] < n)
    pts[interior, 0] += jitter * h * urand(seed, 2 * vid[interior])
    pts[interior, 1] += jitter * h * urand(seed, 2 * vid[interior] + np.uint64(1))
    tri = Delaunay(pts).simplices
    polys = []
    for t in tri:
        a, b, c = pts[t[0]], pts[t[1]], pts[t[2]]
        cross = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
        polys.append([int(t[0]), int(t[1]), int(t[2])] if cross > 0 else [int(t[0]), int(t[2]), int(t[1])])
    e = 1e-9
    rules = [(-1.0, e, -1.0, y_step - e, 0), (-1.0, e, -1.0, 2.0, 1), (-1.0, 2.0, -1.0, e, 0),
             (1 - e, 2.0, -1.0, 2.0, 2), (-1.0, 2.0, 1 - e, 2.0, 2)]
    m = extrude_polygons(pts, polys, h, ["inlet_lower", "inlet_upper", "outlet", "frontAndBack"],
                         [PATCH_GENERIC, PATCH_GENERIC, PATCH_GENERIC, PATCH_EMPTY], rules, 3, scramble)
    m.meta = dict(kind="square_tri", n=n, dz=h, y_step=y_step)
    return m


def cylinder_poly(target_cells=1.0e6, seed=3, scramble=13, jitter=0.25, dz=0.01):
    """C3: flow past a cylinder, 2-D channel
    [-1, 3] x [-1, 1] around a cylinder of diameter 0.2 at the origin.
    Points: staggered polar rings r in [0.1, 0.6) (geometric, near-square
    spacing, jittered except the cylinder ring's radius) and a jittered
    lattice outside; Delaunay; triangles inside the cylinder dropped; the
    POLYGON DUAL (one cell per primal vertex, dual vertices at triangle
    circumcentres, or at the centroid where the circumcentre is not well
    inside its triangle; boundary cells closed through the boundary-edge
    midpoints and the vertex itself) extruded one layer (dz, empty
    front/back).  N = number of primal vertices; F/N ~ 3.
    Patches: inlet (x=-1), outlet (x=3), sides (y=+-1), cylinder (wall),
    frontAndBack (empty)."""
    from scipy.spatial import Delaunay
    x0, x1, y0, y1, rc, rr = -1.0, 3.0, -1.0, 1.0, 0.1, 0.6
    h = np.sqrt(((x1 - x0) * (y1 - y0) - np.pi * rr * rr + 2 * np.pi * rr * rr * np.log(rr / rc)) / target_cells)
    nth = int(round(2 * np.pi * rr / h))
    q = 1.0 + 2 * np.pi / nth
    nring = int(np.floor(np.log(rr / rc) / np.log(q))) + 1
    k, j = np.meshgrid(np.arange(nring), np.arange(nth), indexing="ij")
    k, j = k.ravel(), j.ravel()
    rid = np.arange(len(k), dtype=np.uint64)
    dth = 2 * np.pi / nth
    th = (j + 0.5 * (k % 2)) * dth + 0.1 * dth * urand(seed, 3 * rid)
    r = rc * q ** k * np.where(k > 0, 1.0 + 0.1 * (q - 1.0) * urand(seed, 3 * rid + np.uint64(1)), 1.0)
    ring = np.stack([r * np.cos(th), r * np.sin(th)], 1)
    nx, ny = int(round((x1 - x0) / h)), int(round((y1 - y0) / h))
    I, J = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), indexing="ij")
    I, J = I.ravel(), J.ravel()
    lat = np.stack([x0 + I * (x1 - x0) / nx, y0 + J * (y1 - y0) / ny], 1)
    inner = (I > 0) & (I < nx) & (J > 0) & (J < ny)
    lid = np.arange(len(I), dtype=np.uint64) + np.uint64(1 << 40)
    lat[inner, 0] += jitter * h * urand(seed, 2 * lid[inner])
    lat[inner, 1] += jitter * h * urand(seed, 2 * lid[inner] + np.uint64(1))
    lat = lat[np.hypot(lat[:, 0], lat[:, 1]) > rr + 0.5 * h]
    pts = np.concatenate([ring, lat])
    nv = len(pts)
    tri = Delaunay(pts).simplices.astype(np.int64)
    A, B, Cc = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    cross = (B[:, 0] - A[:, 0]) * (Cc[:, 1] - A[:, 1]) - (B[:, 1] - A[:, 1]) * (Cc[:, 0] - A[:, 0])
    flip = cross < 0
    tri[flip, 1], tri[flip, 2] = tri[flip, 2].copy(), tri[flip, 1].copy()
    A, B, Cc = pts[tri[:, 0]], pts[tri[:, 1]], pts[tri[:, 2]]
    cen = (A + B + Cc) / 3.0
    keep = np.hypot(cen[:, 0], cen[:, 1]) > rc
    tri, A, B, Cc, cen = tri[keep], A[keep], B[keep], Cc[keep], cen[keep]
    nt = len(tri)
    # circumcentre and its barycentric coordinates
    bx, by, cx, cy = B[:, 0] - A[:, 0], B[:, 1] - A[:, 1], Cc[:, 0] - A[:, 0], Cc[:, 1] - A[:, 1]
    d = 2.0 * (bx * cy - by * cx)
    ux = (cy * (bx * bx + by * by) - by * (cx * cx + cy * cy)) / d
    uy = (bx * (cx * cx + cy * cy) - cx * (bx * bx + by * by)) / d
    l1 = (ux * cy - uy * cx) / (bx * cy - by * cx)
    l2 = (bx * uy - by * ux) / (bx * cy - by * cx)
    inside = (l1 > 0.02) & (l2 > 0.02) & (1.0 - l1 - l2 > 0.02)
    dual_t = np.where(inside[:, None], A + np.stack([ux, uy], 1), cen)
    # boundary edges (edges of one kept triangle), oriented as in the CCW triangle
    e = np.concatenate([tri[:, [0, 1]], tri[:, [1, 2]], tri[:, [2, 0]]])
    key = np.minimum(e[:, 0], e[:, 1]) * nv + np.maximum(e[:, 0], e[:, 1])
    uk, cnt = np.unique(key, return_counts=True)
    be = e[np.isin(key, uk[cnt == 1])]
    nb = len(be)
    mid = 0.5 * (pts[be[:, 0]] + pts[be[:, 1]])
    bv = np.unique(be.ravel())
    isb = np.zeros(nv, bool); isb[bv] = True
    vpid = np.full(nv, -1, np.int64); vpid[bv] = nt + nb + np.arange(len(bv))
    dual = np.concatenate([dual_t, mid, pts[bv]])
    # items around each primal vertex: (vertex, angle, dual point, is-midpoint)
    iv = np.concatenate([tri.T.ravel(), be[:, 0], be[:, 1]])
    ip = np.concatenate([np.tile(np.arange(nt), 3), nt + np.arange(nb), nt + np.arange(nb)])
    im = np.concatenate([np.zeros(3 * nt, bool), np.ones(2 * nb, bool)])
    vec = dual[ip] - pts[iv]
    ang = np.arctan2(vec[:, 1], vec[:, 0])
    o = np.lexsort((ang, iv))
    iv, ip, im = iv[o], ip[o], im[o]
    cntv = np.bincount(iv, minlength=nv)
    in_off = np.zeros(nv + 1, np.int64); in_off[1:] = np.cumsum(cntv)
    out_len = cntv + isb
    out_off = np.zeros(nv + 1, np.int64); out_off[1:] = np.cumsum(out_len)
    ids = np.empty(out_off[-1], np.int64)
    pos = np.arange(len(iv)) - in_off[iv]
    inter = ~isb[iv]
    ids[out_off[iv[inter]] + pos[inter]] = ip[inter]
    for v in bv:
        a, b = in_off[v], in_off[v + 1]
        seg_p, seg_m = ip[a:b], im[a:b]
        n = b - a
        gaps = [i for i in range(n) if seg_m[i] and seg_m[(i + 1) % n]]
        if len(gaps) != 1:
            raise ValueError(f"cylinder_poly: boundary vertex {v} has {len(gaps)} exterior gaps")
        i = gaps[0]
        rot = np.concatenate([seg_p[i + 1:], seg_p[:i + 1]])
        ids[out_off[v]:out_off[v + 1]] = np.concatenate([rot, [vpid[v]]])
    eps = 1e-9
    rules = [(-0.2, 0.2, -0.2, 0.2, 3), (x0 - 1, x0 + eps, y0 - 1, y1 + 1, 0), (x1 - eps, x1 + 1, y0 - 1, y1 + 1, 1),
             (x0 - 1, x1 + 1, y0 - 1, y0 + eps, 2), (x0 - 1, x1 + 1, y1 - eps, y1 + 1, 2)]
    m = extrude_polygons(dual, (out_off, ids), dz, ["inlet", "outlet", "sides", "cylinder", "frontAndBack"],
                         [PATCH_GENERIC, PATCH_GENERIC, PATCH_GENERIC, PATCH_WALL, PATCH_EMPTY], rules, 4, scramble)
    m.meta = dict(kind="cylinder_poly", h=h, dz=dz, n_theta=nth, n_ring=nring)
    return m


# ----------------------------------------------------------------- polyMesh I/O
def write_polymesh(raw: RawMesh, case_dir, note=""):
    """Write `raw` as an OpenFOAM ASCII polyMesh under case_dir/constant/polyMesh
    (input tooling for the NEXT-4 reader tests: a plain text dump of the
    arrays, points with 17 significant digits so they round-trip exactly)."""
    d = os.path.join(case_dir, "constant", "polyMesh")
    os.makedirs(d, exist_ok=True)

    def header(f, cls, obj):
        f.write("/*--------------------------------*- C++ -*----------------------------------*\\\n"
                "  synthetic mesh (synth.write_polymesh)\n"
                "\\*---------------------------------------------------------------------------*/\n")
        f.write(f"FoamFile\n{{\n    version     2.0;\n    format      ascii;\n    class       {cls};\n")
        if note:
            f.write(f'    note        "{note}";\n')
        f.write(f'    location    "constant/polyMesh";\n    object      {obj};\n}}\n'
                "// * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * * //\n\n")

    with open(os.path.join(d, "points"), "w") as f:
        header(f, "vectorField", "points")
        f.write(f"{len(raw.points)}\n(\n")
        f.write("".join(f"({x!r} {y!r} {z!r})\n" for x, y, z in np.asarray(raw.points, np.float64).tolist()))
        f.write(")\n")
    with open(os.path.join(d, "faces"), "w") as f:
        header(f, "faceList", "faces")
        fo, fp = raw.face_offsets, raw.face_points
        f.write(f"{raw.n_faces}\n(\n")
        f.write("".join(f"{fo[i + 1] - fo[i]}({' '.join(map(str, fp[fo[i]:fo[i + 1]].tolist()))})\n"
                        for i in range(raw.n_faces)))
        f.write(")\n")
    for name, arr in (("owner", raw.owner), ("neighbour", raw.neighbour)):
        with open(os.path.join(d, name), "w") as f:
            header(f, "labelList", name)
            f.write(f"{len(arr)}\n(\n" + "".join(f"{v}\n" for v in np.asarray(arr).tolist()) + ")\n")
    kinds = {PATCH_GENERIC: "patch", PATCH_WALL: "wall", PATCH_EMPTY: "empty"}
    with open(os.path.join(d, "boundary"), "w") as f:
        header(f, "polyBoundaryMesh", "boundary")
        f.write(f"{len(raw.patches)}\n(\n")
        for p in raw.patches:
            f.write(f"    {p.name}\n    {{\n        type            {kinds[p.kind]};\n"
                    f"        inGroups        List<word> 1({kinds[p.kind]});\n"
                    f"        nFaces          {p.n};\n        startFace       {p.start};\n    }}\n")
        f.write(")\n")
    return d
