"""ctypes binding of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg may import this module.
The oracle is a plain single-threaded fp64 C++ transcription of the paper's
discretisation and PISO step (§2.3-§2.6) in the readings of
SURVEY.md §8(c); it shares no code with the CUDA library and works in the
caller's original numbering.

Parity status of each function is listed in DESIGN.md ("Oracle pins").
Parity unpinned: the Windkessel coupling inside PISO (reading A-19), the
ddtCorr-free Rhie-Chow flux (A-9) on non-orthogonal tets and the optional
ddtCorr term (A-42) -- checked only against invariants.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS = ["OK", "INVALID_ARG", "MESH_CONSISTENCY", "DEGENERATE_FACE", "INVERTED_CELL",
          "NONCONVEX_PAIR", "EXTREME_NONORTH", "MISSING_BC", "NOT_CONVERGED", "BREAKDOWN",
          "NONFINITE", "CONTINUITY", "INVALID_WK_PARAMS"]

NONORTH = {"none": 0, "minimum": 1, "orthogonal": 2, "overrelaxed": 3}
BC_FIXED, BC_ZEROGRAD, BC_PARABOLIC, BC_WINDKESSEL = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, code, msg, index):
        super().__init__(f"{STATUS[code] if 0 <= code < len(STATUS) else code}: {msg} (index {index})")
        self.code, self.status, self.index = code, STATUS[code] if 0 <= code < len(STATUS) else str(code), index


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make` (or __graft_entry__.build())")
        L = C.CDLL(path)
        vp, i64, i32, f64, ch = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_char
        L.orc_last_error_message.restype = C.c_char_p
        L.orc_last_error_index.restype = i64
        L.orc_mesh_create.argtypes = [vp, i64, vp, vp, i64, vp, vp, i64, vp, vp, vp, i32, i32, C.POINTER(vp)]
        L.orc_mesh_destroy.argtypes = [vp]
        L.orc_mesh_sizes.argtypes = [vp, vp]
        L.orc_mesh_geometry.argtypes = [vp] * 5
        L.orc_mesh_coeffs.argtypes = [vp] * 5
        L.orc_bcs_create.restype = vp
        L.orc_bcs_create.argtypes = [vp]
        L.orc_bcs_destroy.argtypes = [vp]
        L.orc_bcs_set.argtypes = [vp, i32, ch, i32, vp, f64, vp, f64]
        L.orc_bcs_set_wk_value.argtypes = [vp, i32, f64]
        L.orc_bcs_set_waveform.argtypes = [vp, i32, ch, f64, i32, vp, vp]
        L.orc_bcs_set_time.argtypes = [vp, f64]
        L.orc_interpolate.argtypes = [vp, vp, ch, i32, vp, vp]
        L.orc_grad.argtypes = [vp, vp, ch, i32, vp, vp]
        L.orc_grad_faces.argtypes = [vp, i32, vp, vp]
        L.orc_div.argtypes = [vp, vp, vp]
        L.orc_laplacian.argtypes = [vp, vp, ch, vp, vp, vp, vp, vp]
        L.orc_windkessel_update.argtypes = [f64, f64, f64, f64, f64, f64, i32, vp, vp]
        L.orc_ldu_solve.argtypes = [vp, vp, vp, vp, vp, vp, i32, f64, f64, i32, vp]
        L.orc_ldu_apply.argtypes = [vp] * 6
        L.orc_solver_create.restype = vp
        L.orc_solver_create.argtypes = [vp, vp, vp, vp]
        L.orc_solver_destroy.argtypes = [vp]
        L.orc_windkessel_set.argtypes = [vp, i32, f64, f64, f64, f64, i32]
        L.orc_windkessel_pc.restype = f64
        L.orc_windkessel_pc.argtypes = [vp, i32]
        L.orc_piso_step.argtypes = [vp, vp, vp, vp, vp]
        L.orc_momentum_assemble.argtypes = [vp] * 7
        L.orc_pressure_solve.argtypes = [vp, vp, vp, vp, f64, f64, i32, i32, vp]
        L.orc_ldu_apply_transpose.argtypes = [vp] * 6
        L.orc_pressure_adjoint.argtypes = [vp, vp, vp, vp, f64, i32, i32, vp]
        L.orc_pressure_vjp.argtypes = [vp, vp, vp, vp, vp]
        L.orc_transport_step.argtypes = [vp, vp, vp, f64, vp]
        L.orc_poisson_steady.restype = i32
        L.orc_poisson_steady.argtypes = [vp, vp, vp, vp, f64, i32, i32, f64]
        L.orc_renumber_create.restype = vp
        L.orc_renumber_create.argtypes = [vp, i32, i32]
        L.orc_renumber_destroy.argtypes = [vp]
        L.orc_renumber_sizes.argtypes = [vp, vp]
        L.orc_renumber_maps.argtypes = [vp] * 10
        L.orc_renumber_part_sizes.argtypes = [vp, i32, vp]
        L.orc_renumber_part.argtypes = [vp, i32, vp, vp, vp, vp]
        L.orc_laplacian_parts.argtypes = [vp, vp, i32, vp, vp, vp, vp]
        L.orc_pressure_rhs.argtypes = [vp] * 5
        L.orc_flux_correct.argtypes = [vp] * 5
        L.orc_phi_hbya.argtypes = [vp] * 6
        _LIB = L
    return _LIB


def _check(st):
    if st != 0:
        L = lib()
        raise OracleError(st, L.orc_last_error_message().decode(), L.orc_last_error_index())


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


class Mesh:
    """O-0 validation + O-1 geometry + O-2 connectivity + O-3 coefficients."""

    def __init__(self, raw, nonorth="overrelaxed"):
        L = lib()
        self.raw = raw
        pk = np.array([p.kind for p in raw.patches], np.int32)
        ps = np.array([p.start for p in raw.patches], np.int64)
        pn = np.array([p.n for p in raw.patches], np.int64)
        pts = np.ascontiguousarray(raw.points, np.float64)
        fo = np.ascontiguousarray(raw.face_offsets, np.int64)
        fp = np.ascontiguousarray(raw.face_points, np.int32)
        own = np.ascontiguousarray(raw.owner, np.int32)
        nb = np.ascontiguousarray(raw.neighbour, np.int32)
        h = C.c_void_p()
        _check(L.orc_mesh_create(_p(pts), len(pts), _p(fo), _p(fp), len(own), _p(own), _p(nb), len(nb),
                                 _p(pk), _p(ps), _p(pn), len(pk), NONORTH[nonorth], C.byref(h)))
        self.h = h.value
        s = np.zeros(5, np.int64)
        L.orc_mesh_sizes(self.h, _p(s))
        self.N, self.F, self.NF, self.n_clamped, self.n_bad_pyramids = (int(x) for x in s)
        self.Sf = np.empty((self.NF, 3)); self.xf = np.empty((self.NF, 3))
        self.xc = np.empty((self.N, 3)); self.V = np.empty(self.N)
        L.orc_mesh_geometry(self.h, _p(self.Sf), _p(self.xf), _p(self.xc), _p(self.V))
        self.w = np.empty(self.F); self.delta = np.empty(self.F); self.k = np.empty((self.F, 3))
        self.delta_b = np.empty(self.NF - self.F)
        L.orc_mesh_coeffs(self.h, _p(self.w), _p(self.delta), _p(self.k), _p(self.delta_b))
        self.owner, self.neighbour = own, nb
        self.patches = raw.patches

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_mesh_destroy(self.h)
            self.h = None

    # ---- operators (O-4)
    def interpolate(self, bcs, fld, x):
        x = _f64(x)
        nc = 1 if x.ndim == 1 else x.shape[1]
        out = np.empty((self.NF, nc)) if nc > 1 else np.empty(self.NF)
        _check(lib().orc_interpolate(self.h, bcs.h, fld.encode(), nc, _p(x), _p(out)))
        return out

    def grad(self, bcs, fld, x):
        x = _f64(x)
        nc = 1 if x.ndim == 1 else x.shape[1]
        out = np.empty((self.N, 3)) if nc == 1 else np.empty((self.N, nc, 3))
        _check(lib().orc_grad(self.h, bcs.h, fld.encode(), nc, _p(x), _p(out)))
        return out

    def grad_faces(self, fv):
        fv = _f64(fv)
        nc = 1 if fv.ndim == 1 else fv.shape[1]
        out = np.empty((self.N, 3)) if nc == 1 else np.empty((self.N, nc, 3))
        _check(lib().orc_grad_faces(self.h, nc, _p(fv), _p(out)))
        return out

    def div(self, flux):
        flux = _f64(flux)
        out = np.empty(self.N)
        _check(lib().orc_div(self.h, _p(flux), _p(out)))
        return out

    def laplacian(self, bcs, fld, x, gamma=None, grad=None):
        x = _f64(x)
        g = None if gamma is None else _f64(gamma)
        G = None if grad is None else _f64(grad)
        y = np.empty(self.N); ya = np.empty(self.N)
        _check(lib().orc_laplacian(self.h, bcs.h, fld.encode(), _p(g), _p(x), _p(G), _p(y), _p(ya)))
        return y, ya

    # ---- generic LDU solves on this mesh's addressing
    def ldu_solve(self, diag, lower, upper, b, x0=None, mode="cg", tol=1e-14, rel_tol=0.0, maxit=50000):
        x = np.zeros(self.N) if x0 is None else _f64(x0).copy()
        rep = np.zeros(4)
        keep = [_f64(a) for a in (diag, lower, upper, b)]   # keep buffers alive across the call
        st = lib().orc_ldu_solve(self.h, *[_p(a) for a in keep], _p(x),
                                 {"cg": 0, "bicgstab": 1, "lu": 2}[mode], tol, rel_tol, maxit, _p(rep))
        return x, dict(it=int(rep[0]), res0=rep[1], res=rep[2], converged=bool(rep[3]), status=STATUS[st])

    def ldu_apply(self, diag, lower, upper, x):
        y = np.empty(self.N)
        keep = [_f64(a) for a in (diag, lower, upper, x)]
        lib().orc_ldu_apply(self.h, *[_p(a) for a in keep], _p(y))
        return y

    def ldu_apply_transpose(self, diag, lower, upper, x):
        """y = A^T x (NEXT-3; written as a face scatter, independent of ldu_apply)."""
        y = np.empty(self.N)
        keep = [_f64(a) for a in (diag, lower, upper, x)]
        lib().orc_ldu_apply_transpose(self.h, *[_p(a) for a in keep], _p(y))
        return y

    def poisson_steady(self, bcs, src, phi0=None, picard_tol=1e-12, max_picard=200, direct=False, cg_tol=1e-15):
        phi = np.zeros(self.N) if phi0 is None else _f64(phi0).copy()
        src = _f64(src)
        it = lib().orc_poisson_steady(self.h, bcs.h, _p(src), _p(phi), picard_tol, max_picard,
                                      1 if direct else 0, cg_tol)
        return phi, it

    def renumber(self, n_parts=1, rcm=True):
        return Renumbering(self, n_parts, rcm)


class BCs:
    """Per (patch, field) boundary conditions; field in 'U', 'p', 's'."""

    def __init__(self, mesh):
        self.mesh = mesh
        self.h = lib().orc_bcs_create(mesh.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_bcs_destroy(self.h)
            self.h = None

    def set(self, patch, fld, kind, value=(0.0, 0.0, 0.0), u_max=0.0, center=(0.0, 0.0, 0.0), radius=1.0):
        if isinstance(patch, str):
            patch = self.mesh.raw.patch(patch)
        v = np.zeros(3); v[:len(np.atleast_1d(value))] = np.atleast_1d(value)
        c = np.asarray(center, np.float64)
        _check(lib().orc_bcs_set(self.h, patch, fld.encode(), kind, _p(v), u_max, _p(c), radius))
        return self

    def set_wk_value(self, patch, v):
        lib().orc_bcs_set_wk_value(self.h, patch, v)

    def set_waveform(self, patch, fld, period, a, b=None):
        """Time-varying multiplier g(t) = a0 + sum_k a_k cos(2 pi k t/T) + b_k sin(2 pi k t/T)
        of the patch's fixed-value / parabolic value (reading A-41)."""
        a = np.ascontiguousarray(a, np.float64)
        nh = len(a) - 1
        bb = np.zeros(nh + 1) if b is None else np.ascontiguousarray(b, np.float64)
        assert len(bb) == nh + 1
        _check(lib().orc_bcs_set_waveform(self.h, patch, fld.encode(), period, nh, _p(a), _p(bb)))

    def set_time(self, t):
        lib().orc_bcs_set_time(self.h, t)


def windkessel_update(pc, Q, dt, Rp, Cc, Rd, scheme=0):
    """O-8 (eq:windkessel_discrete P:420-425; scheme 0 exact, 1 FE, 2 BE)."""
    a, b = C.c_double(), C.c_double()
    _check(lib().orc_windkessel_update(pc, Q, dt, Rp, Cc, Rd, scheme, C.byref(a), C.byref(b)))
    return a.value, b.value


class Solver:
    """O-5/O-6 PISO step (icoFoam order) in the caller's numbering."""

    def __init__(self, mesh, bcs, nu, dt, rho=1.0, n_corr=2, n_nonorth=0, convection="upwind",
                 p_ref_cell=0, p_ref_value=0.0, direct=False, p_tol=1e-14, p_rel_tol=0.0,
                 p_rel_tol_final=0.0, p_maxit=50000, U_tol=1e-14, U_rel_tol=0.0, U_maxit=50000, p_precond=None,
                 theta=1.0, ddt_corr=False):
        # p_precond is accepted for recipe compatibility and ignored: the oracle
        # always uses Jacobi CG (or dense LU); the converged pressure does not
        # depend on the preconditioner (A-14)
        self.mesh, self.bcs = mesh, bcs
        # theta: time scheme of the momentum / transport predictor (Table 1 P:388,
        # reading A-40): 1 backward Euler, 0.5 Crank-Nicolson, 0 forward Euler
        d = np.array([nu, dt, rho, p_ref_value, p_tol, p_rel_tol, p_rel_tol_final, U_tol, U_rel_tol, theta],
                     np.float64)
        i = np.array([n_corr, n_nonorth, {"upwind": 0, "central": 1, "sou": 2, "quick": 3}[convection], p_ref_cell,
                      1 if direct else 0, p_maxit, U_maxit, 1 if ddt_corr else 0], np.int64)
        self.h = lib().orc_solver_create(mesh.h, bcs.h, _p(d), _p(i))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_solver_destroy(self.h)
            self.h = None

    def windkessel_set(self, patch, Rp, Cc, Rd, pc0=0.0, scheme=0):
        if isinstance(patch, str):
            patch = self.mesh.raw.patch(patch)
        _check(lib().orc_windkessel_set(self.h, patch, Rp, Cc, Rd, pc0, scheme))

    def windkessel_pc(self, patch):
        return lib().orc_windkessel_pc(self.h, patch)

    def step(self, U, p, phi):
        """Advance (U[N,3], p[N], phi[NF]) in place by one PISO step; returns the report."""
        rep = np.zeros(209)
        st = lib().orc_piso_step(self.h, _p(U), _p(p), _p(phi), _p(rep))
        if st not in (0,):
            _check(st)
        return parse_report(rep)

    def momentum_assemble(self, U, phi):
        m = self.mesh
        diag = np.empty(m.N); lo = np.empty(m.F); up = np.empty(m.F); b = np.empty((m.N, 3))
        U, phi = _f64(U), _f64(phi)
        _check(lib().orc_momentum_assemble(self.h, _p(U), _p(phi), _p(diag), _p(lo), _p(up), _p(b)))
        return diag, lo, up, b

    def transport_step(self, x, phi, gamma):
        """One implicit step of passive-scalar transport (field 's' BCs), x updated in place."""
        rep = np.zeros(4)
        phi = _f64(phi)
        st = lib().orc_transport_step(self.h, _p(x), _p(phi), gamma, _p(rep))
        return dict(it=int(rep[0]), res0=rep[1], res=rep[2], converged=bool(rep[3]), status=STATUS[st])

    def pressure_solve(self, rAU, rhs, p0=None, tol=1e-14, rel_tol=0.0, maxit=50000, direct=False):
        p = np.zeros(self.mesh.N) if p0 is None else _f64(p0).copy()
        rep = np.zeros(4)
        rAU, rhs = _f64(rAU), _f64(rhs)
        st = lib().orc_pressure_solve(self.h, _p(rAU), _p(rhs), _p(p), tol, rel_tol, maxit,
                                      2 if direct else 0, _p(rep))
        return p, dict(it=int(rep[0]), res0=rep[1], res=rep[2], converged=bool(rep[3]), status=STATUS[st])


    def pressure_adjoint(self, rAU, g, tol=1e-14, maxit=50000, direct=False):
        """lambda with A_p(rAU)^T lambda = g (eq:implicit_diff P:366-370)."""
        lam = np.zeros(self.mesh.N)
        rep = np.zeros(4)
        rAU, g = _f64(rAU), _f64(g)
        st = lib().orc_pressure_adjoint(self.h, _p(rAU), _p(g), _p(lam), tol, maxit, 2 if direct else 0, _p(rep))
        return lam, dict(it=int(rep[0]), res0=rep[1], res=rep[2], converged=bool(rep[3]), status=STATUS[st])

    def pressure_rhs(self, rAU, phiHbyA, p):
        """O-6 step 3.5 right-hand side (A-9 reading): -D(phiHbyA) + sum_b c_b p_b
        + sum_f s rAU_f k_f . (grad p)_f with the Gauss gradient of p."""
        out = np.empty(self.mesh.N)
        rAU, phiHbyA, p = _f64(rAU), _f64(phiHbyA), _f64(p)
        _check(lib().orc_pressure_rhs(self.h, _p(rAU), _p(phiHbyA), _p(p), _p(out)))
        return out

    def phi_hbya(self, HbyA, rAU, Un, phin):
        """O-6 step 3.3 (+ 3.3' ddtCorr when the solver has ddt_corr, A-42): phiHbyA on every face."""
        out = np.empty(self.mesh.NF)
        HbyA, rAU, Un, phin = _f64(HbyA), _f64(rAU), _f64(Un), _f64(phin)
        _check(lib().orc_phi_hbya(self.h, _p(HbyA), _p(rAU), _p(Un), _p(phin), _p(out)))
        return out

    def flux_correct(self, rAU, phiHbyA, p):
        """Rhie-Chow corrected flux (A-9): phiHbyA - c_f (p_N - p_O) - rAU_f k_f . (grad p)_f."""
        out = np.empty(self.mesh.NF)
        rAU, phiHbyA, p = _f64(rAU), _f64(phiHbyA), _f64(p)
        _check(lib().orc_flux_correct(self.h, _p(rAU), _p(phiHbyA), _p(p), _p(out)))
        return out

    def pressure_vjp(self, rAU, p, lam):
        """dL/drAU through the converged solve A(rAU) p = rhs, given lambda = A^-T dL/dp."""
        out = np.empty(self.mesh.N)
        rAU, p, lam = _f64(rAU), _f64(p), _f64(lam)
        _check(lib().orc_pressure_vjp(self.h, _p(rAU), _p(p), _p(lam), _p(out)))
        return out


def parse_report(rep):
    U = [dict(it=int(rep[4 * k]), res0=rep[4 * k + 1], res=rep[4 * k + 2], converged=bool(rep[4 * k + 3]))
         for k in range(3)]
    n_p = int(rep[12])
    p = [dict(it=int(rep[13 + 4 * i]), res0=rep[14 + 4 * i], res=rep[15 + 4 * i], converged=bool(rep[16 + 4 * i]))
         for i in range(min(n_p, 16))]
    n_out = int(rep[79])
    return dict(U=U, p=p, cont_err_max=rep[77], cont_err_sum=rep[78], n_outlets=n_out,
                Q=rep[80:80 + n_out].copy(), p_o=rep[144:144 + n_out].copy(), nonfinite=bool(rep[208]))


class Renumbering:
    """O-9 integer maps."""

    def __init__(self, mesh, n_parts, rcm=True):
        L = lib()
        self.h = L.orc_renumber_create(mesh.h, n_parts, 1 if rcm else 0)
        s = np.zeros(7, np.int64)
        L.orc_renumber_sizes(self.h, _p(s))
        N, F, NF, I, nB, self.bw_before, self.bw_after = (int(x) for x in s)
        self.cell_new_of_old = np.empty(N, np.int32)
        self.face_new_of_old = np.empty(NF, np.int32)
        self.flip_of_old = np.empty(F, np.int8)
        self.row_ptr = np.empty(N + 1, np.int32)
        self.inc_face = np.empty(I, np.int32)
        self.inc_nb = np.empty(I, np.int32)
        self.brow_ptr = np.empty(N + 1, np.int32)
        self.b_face = np.empty(nB, np.int32)
        self.part = np.empty(N, np.int32)
        L.orc_renumber_maps(self.h, *[_p(a) for a in (self.cell_new_of_old, self.face_new_of_old, self.flip_of_old,
                                                      self.row_ptr, self.inc_face, self.inc_nb, self.brow_ptr,
                                                      self.b_face, self.part)])
        self.parts = []
        for p in range(n_parts):
            ps = np.zeros(2, np.int64)
            L.orc_renumber_part_sizes(self.h, p, _p(ps))
            g = np.empty(ps[0], np.int32); gp = np.empty(ps[0], np.int32)
            sd = np.empty(ps[1], np.int32); sp = np.empty(ps[1], np.int32)
            L.orc_renumber_part(self.h, p, _p(g), _p(gp), _p(sd), _p(sp))
            self.parts.append(dict(ghost=g, ghost_peer=gp, send=sd, send_peer=sp))

    def laplacian_parts(self, mesh, bcs, fld, x, gamma=None):
        """O-10: the Laplacian applied part by part from owned + ghost data only
        (ghosts filled from the owners' send lists); original numbering."""
        y = np.empty(mesh.N)
        x = _f64(x)
        g = None if gamma is None else _f64(gamma)
        _check(lib().orc_laplacian_parts(mesh.h, bcs.h, {"U": 0, "p": 1, "s": 2}[fld], self.h, _p(g), _p(x), _p(y)))
        return y

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_renumber_destroy(self.h)
            self.h = None
