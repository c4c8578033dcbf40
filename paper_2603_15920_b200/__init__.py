"""paper_2603_15920_b200 — B200-native hot path of DiFVM (arXiv 2603.15920).

Thin ctypes binding of ``libdfvm.so`` (C ABI in ``include/dfvm.h``): argument
marshalling only — every step of the finite-volume operators and of the PISO
step runs in the library's sm_100a kernels.  There is no CPU fallback: when
the library or a CUDA device is missing, calls raise ``DfvmError``.

Names follow the paper's notation (§2.3-§2.6): ``grad`` (Gauss-Green,
eq:gauss_green), ``div`` (aggregation, eq:aggregate), ``laplacian``
(eq:nonortho_flux), ``Solver.step`` (PISO), ``windkessel_*``
(eq:windkessel_discrete).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdfvm.so")
_LIB = None

STATUS = ["OK", "INVALID_ARG", "MESH_CONSISTENCY", "DEGENERATE_FACE", "INVERTED_CELL", "NONCONVEX_PAIR",
          "EXTREME_NONORTH", "MISSING_BC", "NOT_CONVERGED", "BREAKDOWN", "NONFINITE", "CONTINUITY",
          "INVALID_WK_PARAMS", "CUDA", "NCCL", "OOM"]
NONORTH = {"none": 0, "minimum": 1, "orthogonal": 2, "overrelaxed": 3}
PRECISION = {"f64": 0, "f32": 1}
LOC = {"cells": 0, "faces": 1, "flux": 2}
BC_FIXED, BC_ZEROGRAD, BC_PARABOLIC, BC_WINDKESSEL = 0, 1, 2, 3

# exported symbols declared by include/dfvm.h (checked by the CPU test suite)
SYMBOLS = [
    "dfvm_last_error_message", "dfvm_last_error_index", "dfvm_version", "dfvm_comm_unique_id", "dfvm_comm_create",
    "dfvm_comm_destroy", "dfvm_mesh_create", "dfvm_mesh_info_get", "dfvm_mesh_export_maps", "dfvm_mesh_export_halo",
    "dfvm_mesh_export_geometry", "dfvm_mesh_destroy", "dfvm_field_bytes", "dfvm_field_alloc", "dfvm_field_wrap",
    "dfvm_field_data", "dfvm_field_import", "dfvm_field_export", "dfvm_field_destroy", "dfvm_bcs_create",
    "dfvm_bcs_set", "dfvm_bcs_destroy", "dfvm_fvc_interpolate", "dfvm_fvc_grad", "dfvm_fvc_grad_faces",
    "dfvm_fvc_div", "dfvm_fvm_laplacian_apply", "dfvm_solver_create", "dfvm_pressure_solve",
    "dfvm_momentum_assemble", "dfvm_momentum_apply", "dfvm_piso_step", "dfvm_windkessel_set",
    "dfvm_windkessel_state", "dfvm_windkessel_update", "dfvm_solver_destroy", "dfvm_kernel_launches",
    "dfvm_solver_set_timing", "dfvm_solver_get_timing", "dfvm_comm_create_local", "dfvm_solver_amg_levels",
    "dfvm_transport_step", "dfvm_momentum_apply_transpose", "dfvm_pressure_solve_adjoint", "dfvm_pressure_vjp",
    "dfvm_bcs_set_waveform", "dfvm_bcs_set_time", "dfvm_polymesh_read", "dfvm_polymesh_sizes",
    "dfvm_polymesh_arrays", "dfvm_polymesh_destroy", "dfvm_set_allocator", "dfvm_live_device_bytes",
    "dfvm_solver_profile", "dfvm_solver_profile_get",
]


class DfvmError(RuntimeError):
    def __init__(self, code, msg, index=-1):
        name = STATUS[code] if 0 <= code < len(STATUS) else str(code)
        super().__init__(f"DFVM_E_{name}: {msg} (index {index})")
        self.code, self.status, self.index = code, name, index


class PatchDesc(C.Structure):
    _fields_ = [("name", C.c_char_p), ("kind", C.c_int32), ("start_face", C.c_int64), ("n_faces", C.c_int64)]


class MeshOpts(C.Structure):
    _fields_ = [("renumber_rcm", C.c_int32), ("nonorth", C.c_int32), ("n_parts", C.c_int32), ("rank", C.c_int32),
                ("device", C.c_int32), ("precision", C.c_int32)]


class MeshInfo(C.Structure):
    _fields_ = [("n_cells", C.c_int64), ("n_internal_faces", C.c_int64), ("n_boundary_faces", C.c_int64),
                ("n_empty_faces", C.c_int64), ("n_owned", C.c_int64), ("n_ghost", C.c_int64),
                ("n_local_internal_faces", C.c_int64), ("n_local_boundary_faces", C.c_int64),
                ("n_peers", C.c_int32), ("precision", C.c_int32), ("bandwidth_before", C.c_int64),
                ("bandwidth_after", C.c_int64), ("n_clamped", C.c_int64), ("device_bytes", C.c_int64),
                ("sell_max_row", C.c_int32), ("sell_slices", C.c_int32), ("host_seconds", C.c_double)]


class BcDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value", C.c_double * 3), ("u_max", C.c_double), ("center", C.c_double * 3),
                ("radius", C.c_double)]


class PisoOpts(C.Structure):
    _fields_ = [("nu", C.c_double), ("dt", C.c_double), ("rho", C.c_double), ("n_corr", C.c_int32),
                ("n_nonorth", C.c_int32), ("convection", C.c_int32), ("p_ref_cell", C.c_int64),
                ("p_ref_value", C.c_double), ("p_tol", C.c_double), ("p_rel_tol", C.c_double),
                ("p_rel_tol_final", C.c_double), ("p_maxit", C.c_int32), ("U_tol", C.c_double),
                ("U_rel_tol", C.c_double), ("U_maxit", C.c_int32), ("p_precond", C.c_int32),
                ("time_scheme", C.c_int32), ("ddt_corr", C.c_int32), ("cont_tol", C.c_double)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("level", C.c_int32), ("launches", C.c_int64), ("ms", C.c_double),
                ("alg_bytes", C.c_double)]


class SolveReport(C.Structure):
    _fields_ = [("it", C.c_int32), ("res0", C.c_double), ("res", C.c_double), ("converged", C.c_int32)]


class StepReport(C.Structure):
    _fields_ = [("U", SolveReport * 3), ("p", SolveReport * 16), ("n_p", C.c_int32), ("cont_err_max", C.c_double),
                ("cont_err_sum", C.c_double), ("n_outlets", C.c_int32), ("Q", C.c_double * 64),
                ("p_o", C.c_double * 64), ("nonfinite", C.c_int32), ("gpu_launches", C.c_int32)]


# dfvm_alloc_fn / dfvm_free_fn (include/dfvm.h, §8(b) b3)
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
_ALLOCATOR = None   # keeps the ctypes callbacks alive while installed


def lib():
    """Load libdfvm.so (fails loudly if it was not built)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise DfvmError(13, f"{LIB_PATH} is missing: build it with `make` / __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        for name in SYMBOLS:
            getattr(L, name).restype = C.c_int
        L.dfvm_last_error_message.restype = C.c_char_p
        L.dfvm_last_error_index.restype = i64
        L.dfvm_version.restype = C.c_char_p
        L.dfvm_kernel_launches.restype = i64
        L.dfvm_mesh_create.argtypes = [vp, i64, vp, vp, i64, vp, vp, i64, vp, i32, C.POINTER(MeshOpts), vp, vp,
                                       C.POINTER(vp)]
        L.dfvm_mesh_info_get.argtypes = [vp, C.POINTER(MeshInfo)]
        L.dfvm_mesh_export_maps.argtypes = [vp] * 8
        L.dfvm_mesh_export_halo.argtypes = [vp] * 7
        L.dfvm_mesh_export_geometry.argtypes = [vp] * 9
        L.dfvm_mesh_destroy.argtypes = [vp]
        L.dfvm_field_bytes.argtypes = [vp, i32, i32, C.POINTER(C.c_size_t)]
        L.dfvm_field_alloc.argtypes = [vp, i32, i32, C.POINTER(vp)]
        L.dfvm_field_wrap.argtypes = [vp, vp, i32, i32, C.POINTER(vp)]
        L.dfvm_field_data.argtypes = [vp, C.POINTER(vp)]
        L.dfvm_field_import.argtypes = [vp, vp, i32, vp]
        L.dfvm_field_export.argtypes = [vp, vp, i32, vp]
        L.dfvm_field_destroy.argtypes = [vp]
        L.dfvm_bcs_create.argtypes = [vp, C.POINTER(vp)]
        L.dfvm_bcs_set.argtypes = [vp, i32, C.c_char, C.POINTER(BcDesc)]
        L.dfvm_bcs_destroy.argtypes = [vp]
        L.dfvm_polymesh_read.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.dfvm_polymesh_sizes.argtypes = [vp] + [C.POINTER(i64)] * 4 + [C.POINTER(i32), C.POINTER(i64)]
        L.dfvm_polymesh_arrays.argtypes = [vp] + [C.POINTER(vp)] * 6
        L.dfvm_polymesh_destroy.argtypes = [vp]
        L.dfvm_bcs_set_waveform.argtypes = [vp, i32, C.c_char, f64, i32, vp, vp]
        L.dfvm_bcs_set_time.argtypes = [vp, f64, vp]
        L.dfvm_fvc_interpolate.argtypes = [vp, vp, vp, C.c_char, vp, vp]
        L.dfvm_fvc_grad.argtypes = [vp, vp, vp, C.c_char, vp, vp]
        L.dfvm_fvc_grad_faces.argtypes = [vp, vp, vp, vp]
        L.dfvm_fvc_div.argtypes = [vp, vp, vp, vp]
        L.dfvm_fvm_laplacian_apply.argtypes = [vp, vp, vp, C.c_char, vp, vp, vp, vp]
        L.dfvm_solver_create.argtypes = [vp, vp, C.POINTER(PisoOpts), C.POINTER(vp)]
        L.dfvm_solver_destroy.argtypes = [vp]
        L.dfvm_pressure_solve.argtypes = [vp, vp, vp, vp, f64, f64, i32, C.POINTER(SolveReport), vp]
        L.dfvm_momentum_assemble.argtypes = [vp, vp, vp, vp, vp, vp]
        L.dfvm_momentum_apply.argtypes = [vp, vp, vp, vp]
        L.dfvm_momentum_apply_transpose.argtypes = [vp, vp, vp, vp]
        L.dfvm_pressure_solve_adjoint.argtypes = [vp, vp, vp, vp, f64, f64, i32, C.POINTER(SolveReport), vp]
        L.dfvm_pressure_vjp.argtypes = [vp, vp, vp, vp, vp]
        L.dfvm_piso_step.argtypes = [vp, vp, vp, vp, C.POINTER(StepReport), vp]
        L.dfvm_windkessel_set.argtypes = [vp, i32, f64, f64, f64, f64, i32]
        L.dfvm_windkessel_state.argtypes = [vp, i32, C.POINTER(f64)]
        L.dfvm_windkessel_update.argtypes = [f64, f64, f64, f64, f64, f64, i32, C.POINTER(f64), C.POINTER(f64)]
        L.dfvm_solver_set_timing.argtypes = [vp, i32]
        L.dfvm_solver_get_timing.argtypes = [vp, vp, vp]
        L.dfvm_solver_amg_levels.argtypes = [vp, vp, vp, vp]
        L.dfvm_solver_profile.argtypes = [vp, i32]
        L.dfvm_solver_profile_get.argtypes = [vp, vp, i32, C.POINTER(i32)]
        L.dfvm_transport_step.argtypes = [vp, vp, vp, f64, C.POINTER(SolveReport), vp]
        L.dfvm_comm_unique_id.argtypes = [vp]
        L.dfvm_comm_create.argtypes = [C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]
        L.dfvm_comm_destroy.argtypes = [vp]
        L.dfvm_comm_create_local.argtypes = [C.c_int, vp, vp]
        L.dfvm_set_allocator.argtypes = [ALLOC_FN, FREE_FN, vp]
        L.dfvm_live_device_bytes.restype = i64
        _LIB = L
    return _LIB


def _check(st, allow=()):
    if st != 0 and st not in allow:
        L = lib()
        raise DfvmError(st, L.dfvm_last_error_message().decode(), L.dfvm_last_error_index())
    return st


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def current_stream():
    """The caller's CUDA stream (torch's current stream when torch is in use)."""
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except ImportError:
        pass
    return None


def kernel_launches():
    return int(lib().dfvm_kernel_launches())


def live_device_bytes():
    """Bytes held by library-owned device allocations (dfvm_live_device_bytes)."""
    return int(lib().dfvm_live_device_bytes())


def set_allocator(alloc=None, free=None):
    """dfvm_set_allocator: alloc(nbytes, stream) -> device pointer, free(ptr,
    nbytes, stream); both None restores the default (cudaMallocAsync).  Only
    while no library allocation is live."""
    global _ALLOCATOR
    if (alloc is None) != (free is None):
        raise ValueError("set_allocator needs both callbacks or neither")
    if alloc is None:
        _check(lib().dfvm_set_allocator(C.cast(None, ALLOC_FN), C.cast(None, FREE_FN), None))
        _ALLOCATOR = None
        return
    fa = ALLOC_FN(lambda n, s, ctx: alloc(n, s or 0) or None)
    ff = FREE_FN(lambda p, n, s, ctx: free(p, n, s or 0))
    _check(lib().dfvm_set_allocator(fa, ff, None))
    _ALLOCATOR = (fa, ff)


def use_torch_allocator():
    """Route every library device allocation through PyTorch's caching
    allocator (north star: "PyTorch only for device memory")."""
    import torch

    def alloc(n, stream):
        return torch.cuda.caching_allocator_alloc(int(n), stream=int(stream))

    def free(p, n, stream):
        torch.cuda.caching_allocator_delete(int(p))

    set_allocator(alloc, free)


class Comm:
    """NCCL communicator (one process per GPU); the 128-byte id is broadcast
    with torch.distributed by the caller (see bench.py)."""

    def __init__(self, n_ranks, rank, uid: bytes, device):
        L = lib()
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        _check(L.dfvm_comm_create(n_ranks, rank, C.cast(buf, C.c_void_p), device, C.byref(h)))
        self.h = h.value

    @staticmethod
    def local_group(n_ranks, devices=None):
        """n in-process communicators (ranks = host threads), see dfvm.h."""
        L = lib()
        hs = (C.c_void_p * n_ranks)()
        dv = None if devices is None else (C.c_int * n_ranks)(*devices)
        _check(L.dfvm_comm_create_local(n_ranks, C.cast(dv, C.c_void_p) if dv is not None else None,
                                        C.cast(hs, C.c_void_p)))
        out = []
        for h in hs:
            c = Comm.__new__(Comm)
            c.h = h
            out.append(c)
        return out

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _check(lib().dfvm_comm_unique_id(C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().dfvm_comm_destroy(self.h)
            except (TypeError, AttributeError):   # interpreter shutdown: module globals already cleared
                pass
            self.h = None


class Patch:
    def __init__(self, name, kind, start, n):
        self.name, self.kind, self.start, self.n = name, kind, start, n

    def __repr__(self):
        return f"Patch({self.name!r}, kind={self.kind}, start={self.start}, n={self.n})"


class PolyMesh:
    """Arrays of an OpenFOAM ASCII polyMesh read by dfvm_polymesh_read (NEXT-4;
    P:431-432), in the layout Mesh() / dfvm_mesh_create take (copied out of
    the reader object)."""

    def __init__(self, path):
        L = lib()
        h = C.c_void_p()
        _check(L.dfvm_polymesh_read(os.fspath(path).encode(), C.byref(h)))
        try:
            n = [C.c_int64() for _ in range(4)]
            npat, nc = C.c_int32(), C.c_int64()
            _check(L.dfvm_polymesh_sizes(h, *[C.byref(x) for x in n], C.byref(npat), C.byref(nc)))
            n_p, n_f, n_fp, F = (x.value for x in n)
            ptr = [C.c_void_p() for _ in range(6)]
            _check(L.dfvm_polymesh_arrays(h, *[C.byref(x) for x in ptr]))

            def arr(p, count, ct, dt):
                if count == 0:
                    return np.zeros(0, dt)
                return np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (count,)).astype(dt, copy=True)

            self.points = arr(ptr[0].value, 3 * n_p, C.c_double, np.float64).reshape(n_p, 3)
            self.face_offsets = arr(ptr[1].value, n_f + 1, C.c_int64, np.int64)
            self.face_points = arr(ptr[2].value, n_fp, C.c_int32, np.int32)
            self.owner = arr(ptr[3].value, n_f, C.c_int32, np.int32)
            self.neighbour = arr(ptr[4].value, F, C.c_int32, np.int32)
            pd = C.cast(ptr[5].value, C.POINTER(PatchDesc))
            self.patches = [Patch(pd[i].name.decode(), pd[i].kind, pd[i].start_face, pd[i].n_faces)
                            for i in range(npat.value)]
            self.n_cells = nc.value
            self.meta = dict(kind="polyMesh", path=os.fspath(path))
        finally:
            L.dfvm_polymesh_destroy(h)

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


def read_polymesh(path):
    """OpenFOAM ASCII polyMesh (case dir, constant/polyMesh or the polyMesh dir) -> PolyMesh."""
    return PolyMesh(path)


class Mesh:
    """dfvm_mesh_create from an OpenFOAM-style raw mesh (points, face rings,
    owner, neighbour, patches)."""

    def __init__(self, raw, nonorth="overrelaxed", precision="f64", rcm=True, n_parts=1, rank=0, device=0,
                 comm=None, stream=None):
        L = lib()
        self.raw = raw
        self._names = [p.name.encode() for p in raw.patches]
        pd = (PatchDesc * max(len(raw.patches), 1))()
        for i, p in enumerate(raw.patches):
            pd[i] = PatchDesc(self._names[i], p.kind, p.start, p.n)
        opts = MeshOpts(1 if rcm else 0, NONORTH[nonorth], n_parts, rank, device, PRECISION[precision])
        pts = np.ascontiguousarray(raw.points, np.float64)
        fo = np.ascontiguousarray(raw.face_offsets, np.int64)
        fp = np.ascontiguousarray(raw.face_points, np.int32)
        own = np.ascontiguousarray(raw.owner, np.int32)
        nb = np.ascontiguousarray(raw.neighbour, np.int32)
        h = C.c_void_p()
        _check(L.dfvm_mesh_create(_ptr(pts), len(pts), _ptr(fo), _ptr(fp), len(own), _ptr(own), _ptr(nb), len(nb),
                                  C.cast(pd, C.c_void_p), len(raw.patches), C.byref(opts),
                                  comm.h if comm is not None else None, stream, C.byref(h)))
        self.h = h.value
        self.precision = precision
        self.dtype = np.float64 if precision == "f64" else np.float32
        inf = MeshInfo()
        _check(L.dfvm_mesh_info_get(self.h, C.byref(inf)))
        self.info = {k: getattr(inf, k) for k, _ in MeshInfo._fields_}
        self.N = self.info["n_cells"]
        self.F = self.info["n_internal_faces"]
        self.NF = len(own)
        self.comm = comm

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().dfvm_mesh_destroy(self.h)
            except (TypeError, AttributeError):   # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def export_maps(self):
        F, N = self.F, self.N
        out = dict(cell_new_of_old=np.empty(N, np.int32), face_new_of_old=np.empty(self.NF, np.int32),
                   face_flip=np.empty(F, np.int8), cell_part=np.empty(N, np.int32), row_ptr=np.empty(N + 1, np.int32),
                   inc_face=np.empty(2 * F, np.int32), inc_nb=np.empty(2 * F, np.int32))
        _check(lib().dfvm_mesh_export_maps(self.h, *[_ptr(out[k]) for k in ("cell_new_of_old", "face_new_of_old",
                                                                            "face_flip", "cell_part", "row_ptr",
                                                                            "inc_face", "inc_nb")]))
        return out

    def export_halo(self):
        L = lib()
        ng, ns = C.c_int64(), C.c_int64()
        _check(L.dfvm_mesh_export_halo(self.h, C.byref(ng), None, None, C.byref(ns), None, None))
        g = np.empty(ng.value, np.int32); gp = np.empty(ng.value, np.int32)
        s = np.empty(ns.value, np.int32); sp = np.empty(ns.value, np.int32)
        _check(L.dfvm_mesh_export_halo(self.h, C.byref(ng), _ptr(g), _ptr(gp), C.byref(ns), _ptr(s), _ptr(sp)))
        return dict(ghost=g, ghost_peer=gp, send=s, send_peer=sp)

    def export_geometry(self):
        N, F, NF = self.N, self.F, self.NF
        out = dict(Sf=np.empty((NF, 3)), xf=np.empty((NF, 3)), xc=np.empty((N, 3)), V=np.empty(N), w=np.empty(F),
                   delta=np.empty(F), k=np.empty((F, 3)), delta_b=np.empty(NF - F))
        _check(lib().dfvm_mesh_export_geometry(self.h, *[_ptr(out[k]) for k in ("Sf", "xf", "xc", "V", "w", "delta",
                                                                                "k", "delta_b")]))
        return out

    def field(self, loc="cells", n_comp=1, values=None, stream=None):
        f = Field(self, loc, n_comp)
        if values is not None:
            f.set(values, stream)
        return f


class Field:
    """Library-owned device field (north-star `field_alloc`), or a wrapper
    around caller-owned device memory (e.g. a torch tensor: ``wrap=``)."""

    def __init__(self, mesh, loc="cells", n_comp=1, wrap=None):
        L = lib()
        self.mesh, self.loc, self.n_comp = mesh, loc, n_comp
        h = C.c_void_p()
        if wrap is None:
            _check(L.dfvm_field_alloc(mesh.h, LOC[loc], n_comp, C.byref(h)))
        else:
            self._keep = wrap
            _check(L.dfvm_field_wrap(mesh.h, C.c_void_p(wrap.data_ptr()), LOC[loc], n_comp, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().dfvm_field_destroy(self.h)
            except (TypeError, AttributeError):   # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    @property
    def global_count(self):
        return self.mesh.N if self.loc == "cells" else self.mesh.NF

    def nbytes(self):
        b = C.c_size_t()
        _check(lib().dfvm_field_bytes(self.mesh.h, LOC[self.loc], self.n_comp, C.byref(b)))
        return b.value

    def data_ptr(self):
        p = C.c_void_p()
        _check(lib().dfvm_field_data(self.h, C.byref(p)))
        return p.value

    def set(self, values, stream=None):
        """Import fp64 values [global count(, n_comp)] in ORIGINAL order (host numpy)."""
        a = np.ascontiguousarray(values, np.float64).reshape(self.global_count, self.n_comp)
        _check(lib().dfvm_field_import(self.h, _ptr(a), 1, stream))
        return self

    def get(self, stream=None, out=None):
        """Export to fp64 numpy in ORIGINAL order (synchronises the stream);
        `out` may be a preallocated (e.g. pinned) C-contiguous fp64 array."""
        a = np.zeros((self.global_count, self.n_comp), np.float64) if out is None else out
        assert a.dtype == np.float64 and a.flags.c_contiguous and a.size == self.global_count * self.n_comp
        _check(lib().dfvm_field_export(self.h, _ptr(a), 1, stream))
        if out is not None:
            return out
        return a[:, 0] if self.n_comp == 1 else a

    def import_device(self, dev_ptr, stream=None):
        _check(lib().dfvm_field_import(self.h, C.c_void_p(dev_ptr), 0, stream))

    def export_device(self, dev_ptr, stream=None):
        _check(lib().dfvm_field_export(self.h, C.c_void_p(dev_ptr), 0, stream))


class BCs:
    """Per (patch, field) boundary conditions, field in 'U', 'p', 's'."""

    def __init__(self, mesh):
        self.mesh = mesh
        h = C.c_void_p()
        _check(lib().dfvm_bcs_create(mesh.h, C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().dfvm_bcs_destroy(self.h)
            except (TypeError, AttributeError):   # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def set(self, patch, fld, kind, value=(0.0, 0.0, 0.0), u_max=0.0, center=(0.0, 0.0, 0.0), radius=1.0):
        if isinstance(patch, str):
            patch = self.mesh.raw.patch(patch)
        v = np.zeros(3); v[:len(np.atleast_1d(value))] = np.atleast_1d(value)
        d = BcDesc(kind, (C.c_double * 3)(*v), u_max, (C.c_double * 3)(*center), radius)
        _check(lib().dfvm_bcs_set(self.h, patch, fld.encode(), C.byref(d)))
        return self

    def set_waveform(self, patch, fld, period, a, b=None):
        """Time-varying multiplier g(t) = a0 + sum_k a_k cos(2 pi k t/T) + b_k sin(2 pi k t/T)
        of a fixed-value / parabolic patch value (dfvm_bcs_set_waveform; A-41)."""
        a = np.ascontiguousarray(a, np.float64)
        bb = np.zeros(len(a)) if b is None else np.ascontiguousarray(b, np.float64)
        assert len(bb) == len(a)
        _check(lib().dfvm_bcs_set_waveform(self.h, patch, fld.encode(), period, len(a) - 1,
                                           a.ctypes.data, bb.ctypes.data))
        return self

    def set_time(self, t, stream=None):
        _check(lib().dfvm_bcs_set_time(self.h, t, stream))
        return self


# ------------------------------------------------------------------ operators
def interpolate(mesh, x, bcs, fld, out, stream=None):
    _check(lib().dfvm_fvc_interpolate(mesh.h, x.h, bcs.h, fld.encode(), out.h, stream))
    return out


def grad(mesh, x, bcs, fld, out, stream=None):
    _check(lib().dfvm_fvc_grad(mesh.h, x.h, bcs.h, fld.encode(), out.h, stream))
    return out


def grad_faces(mesh, fv, out, stream=None):
    _check(lib().dfvm_fvc_grad_faces(mesh.h, fv.h, out.h, stream))
    return out


def div(mesh, flux, out, stream=None):
    _check(lib().dfvm_fvc_div(mesh.h, flux.h, out.h, stream))
    return out


def laplacian(mesh, bcs, fld, x, out, gamma=None, grad=None, stream=None):
    _check(lib().dfvm_fvm_laplacian_apply(mesh.h, gamma.h if gamma is not None else None, bcs.h, fld.encode(), x.h,
                                          grad.h if grad is not None else None, out.h, stream))
    return out


def windkessel_update(pc, Q, dt, Rp, Cc, Rd, scheme=0):
    a, b = C.c_double(), C.c_double()
    _check(lib().dfvm_windkessel_update(pc, Q, dt, Rp, Cc, Rd, scheme, C.byref(a), C.byref(b)))
    return a.value, b.value


def _rep(r):
    return dict(it=r.it, res0=r.res0, res=r.res, converged=bool(r.converged))


class Solver:
    """PISO solver (dfvm_solver_create / dfvm_piso_step)."""

    def __init__(self, mesh, bcs, nu, dt, rho=1.0, n_corr=2, n_nonorth=0, convection="upwind", p_ref_cell=0,
                 p_ref_value=0.0, p_tol=1e-14, p_rel_tol=0.0, p_rel_tol_final=0.0, p_maxit=50000, U_tol=1e-14,
                 U_rel_tol=0.0, U_maxit=50000, p_precond="jacobi", theta=1.0, ddt_corr=False, cont_tol=0.0):
        self.mesh, self.bcs = mesh, bcs
        # time scheme (Table 1): theta 1 backward Euler, 0.5 Crank-Nicolson, 0 forward Euler
        schemes = {1.0: 0, 0.5: 1, 0.0: 2}
        if float(theta) not in schemes:
            raise ValueError(f"theta must be 1, 0.5 or 0 (backward Euler, Crank-Nicolson, forward Euler), got {theta}")
        o = PisoOpts(nu, dt, rho, n_corr, n_nonorth, {"upwind": 0, "central": 1, "sou": 2, "quick": 3}[convection],
                     p_ref_cell,
                     p_ref_value, p_tol, p_rel_tol, p_rel_tol_final, p_maxit, U_tol, U_rel_tol, U_maxit,
                     {"jacobi": 0, "amg": 1, "amg32": 2}[p_precond], schemes[float(theta)], 1 if ddt_corr else 0,
                     cont_tol)
        h = C.c_void_p()
        _check(lib().dfvm_solver_create(mesh.h, bcs.h, C.byref(o), C.byref(h)))
        self.h = h.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().dfvm_solver_destroy(self.h)
            except (TypeError, AttributeError):   # interpreter shutdown: module globals already cleared
                pass
            self.h = None

    def windkessel_set(self, patch, Rp, Cc, Rd, pc0=0.0, scheme=0):
        if isinstance(patch, str):
            patch = self.mesh.raw.patch(patch)
        _check(lib().dfvm_windkessel_set(self.h, patch, Rp, Cc, Rd, pc0, scheme))

    def windkessel_state(self, patch):
        if isinstance(patch, str):
            patch = self.mesh.raw.patch(patch)
        v = C.c_double()
        _check(lib().dfvm_windkessel_state(self.h, patch, C.byref(v)))
        return v.value

    def step(self, U, p, phi, stream=None, allow_not_converged=True):
        r = StepReport()
        st = _check(lib().dfvm_piso_step(self.h, U.h, p.h, phi.h, C.byref(r), stream),
                    allow=(8,) if allow_not_converged else ())
        n_out = r.n_outlets
        return dict(status=STATUS[st], U=[_rep(r.U[k]) for k in range(3)],
                    p=[_rep(r.p[i]) for i in range(min(r.n_p, 16))], cont_err_max=r.cont_err_max,
                    cont_err_sum=r.cont_err_sum, n_outlets=n_out, Q=np.array(r.Q[:n_out]),
                    p_o=np.array(r.p_o[:n_out]), nonfinite=bool(r.nonfinite), gpu_launches=r.gpu_launches)

    def pressure_solve(self, rAU, rhs, p, tol=1e-14, rel_tol=0.0, maxit=50000, stream=None):
        r = SolveReport()
        st = _check(lib().dfvm_pressure_solve(self.h, rAU.h, rhs.h, p.h, tol, rel_tol, maxit, C.byref(r), stream),
                    allow=(8,))
        d = _rep(r)
        d["status"] = STATUS[st]
        return d

    def pressure_solve_adjoint(self, rAU, g, lam, tol=1e-14, rel_tol=0.0, maxit=50000, stream=None):
        """NEXT-3: A_p(rAU)^T lambda = g with the forward PCG (eq:implicit_diff P:366-370)."""
        r = SolveReport()
        st = _check(lib().dfvm_pressure_solve_adjoint(self.h, rAU.h, g.h, lam.h, tol, rel_tol, maxit, C.byref(r),
                                                      stream), allow=(8,))
        d = _rep(r)
        d["status"] = STATUS[st]
        return d

    def pressure_vjp(self, p, lam, grad, stream=None):
        """NEXT-3: grad = dL/drAU through the converged pressure solve, from p and lambda."""
        _check(lib().dfvm_pressure_vjp(self.h, p.h, lam.h, grad.h, stream))

    def momentum_apply_transpose(self, x, y, stream=None):
        """NEXT-3: y = M^T x with the last assembled momentum matrix."""
        _check(lib().dfvm_momentum_apply_transpose(self.h, x.h, y.h, stream))

    def transport_step(self, x, phi, gamma, stream=None):
        """One implicit passive-scalar transport step (field 's' BCs); x updated in place."""
        r = SolveReport()
        st = _check(lib().dfvm_transport_step(self.h, x.h, phi.h, gamma, C.byref(r), stream), allow=(8,))
        d = _rep(r)
        d["status"] = STATUS[st]
        return d

    def momentum_assemble(self, U, phi, diag, b, stream=None):
        _check(lib().dfvm_momentum_assemble(self.h, U.h, phi.h, diag.h, b.h, stream))

    def momentum_apply(self, x, y, stream=None):
        _check(lib().dfvm_momentum_apply(self.h, x.h, y.h, stream))

    def set_timing(self, on=True):
        _check(lib().dfvm_solver_set_timing(self.h, 1 if on else 0))

    def timing(self):
        ms = np.zeros(4); n = np.zeros(4, np.int64)
        _check(lib().dfvm_solver_get_timing(self.h, _ptr(ms), _ptr(n)))
        return dict(spmv_ms=float(ms[0]), spmv_n=int(n[0]), cg_iter_ms=float(ms[1]), cg_iter_n=int(n[1]),
                    amg_pre_ms=float(ms[2]), amg_pre_n=int(n[2]), amg_post_ms=float(ms[3]), amg_post_n=int(n[3]))

    def amg_levels(self, nnz=False):
        n = C.c_int32()
        sz = np.zeros(32, np.int64)
        nz = np.zeros(32, np.int64)
        _check(lib().dfvm_solver_amg_levels(self.h, C.byref(n), _ptr(sz), _ptr(nz)))
        if nnz:
            return sz[:n.value].tolist(), nz[:n.value].tolist()
        return sz[:n.value].tolist()

    def profile(self, on=True):
        """dfvm_solver_profile: per-kernel event timing of the following calls (clears the table)."""
        _check(lib().dfvm_solver_profile(self.h, 1 if on else 0))

    def profile_table(self):
        """rows {name, level, launches, ms, alg_bytes} of dfvm_solver_profile_get"""
        n = C.c_int32()
        _check(lib().dfvm_solver_profile_get(self.h, None, 0, C.byref(n)))
        buf = (KernelStat * max(n.value, 1))()
        _check(lib().dfvm_solver_profile_get(self.h, C.cast(buf, C.c_void_p), n.value, C.byref(n)))
        return [dict(name=b.name.decode(), level=b.level, launches=b.launches, ms=b.ms, alg_bytes=b.alg_bytes)
                for b in buf[:n.value]]
