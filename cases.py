"""Workload recipes of BASELINE.json's configs: mesh
generator call, boundary conditions, physical constants, solver settings and
the seeded initial condition.  Data only (no method arithmetic): the same
recipe drives the CUDA library (bench.py, smoke) and the CPU oracle
(tests, cpu_baseline), through their own `BCs.set` / `Solver` calls.
"""
from __future__ import annotations

import numpy as np

import synth

FIXED, ZEROGRAD, PARABOLIC = 0, 1, 2

# throughput-mode Krylov settings (reading A-13: p abs 1e-6 relative to ||b||,
# relTol 0.05 on non-final correctors, 0 on the final one; U 1e-5)
THROUGHPUT = dict(p_tol=1e-6, p_rel_tol=0.05, p_rel_tol_final=0.0, p_maxit=20000, U_tol=1e-5, U_rel_tol=0.0,
                  U_maxit=1000)


class Case:
    def __init__(self, name, raw, bcs, solver, ic, description):
        self.name, self.raw, self.bcs, self.solver, self.ic, self.description = name, raw, bcs, solver, ic, description

    def apply_bcs(self, B):
        for patch, fld, kind, kw in self.bcs:
            B.set(patch, fld, kind, **kw)
        return B

    def initial_state(self, xc, xf, Sf):
        """(U [N,3], p [N], phi [n_faces]) in original numbering, from the
        geometry the caller's own mesh reports."""
        return self.ic(xc, xf, Sf)


def _pipe_bcs(u_max, R):
    return [("inlet", "U", PARABOLIC, dict(u_max=u_max, center=(0.0, 0.0, 0.0), radius=R)),
            ("wall", "U", FIXED, dict(value=(0.0, 0.0, 0.0))), ("outlet", "U", ZEROGRAD, {}),
            ("inlet", "p", ZEROGRAD, {}), ("wall", "p", ZEROGRAD, {}), ("outlet", "p", FIXED, dict(value=0.0))]


def _poiseuille_ic(seed, u_max, R):
    """Poiseuille profile + 1% noise (§8(d2)); phi = u(x_f) . S_f of the
    noise-free profile."""
    def ic(xc, xf, Sf):
        N = len(xc)
        U = np.zeros((N, 3))
        U[:, 2] = u_max * (1.0 - (xc[:, 0] ** 2 + xc[:, 1] ** 2) / (R * R))
        U += 0.01 * u_max * synth.cell_field(seed, N, 3)
        phi = u_max * (1.0 - (xf[:, 0] ** 2 + xf[:, 1] ** 2) / (R * R)) * Sf[:, 2]
        return U, np.zeros(N), phi
    return ic


def c1(scramble=11):
    raw = synth.cavity(20, scramble=scramble)
    bcs = [("movingWall", "U", FIXED, dict(value=(1.0, 0.0, 0.0))), ("fixedWalls", "U", FIXED, dict(value=(0, 0, 0))),
           ("movingWall", "p", ZEROGRAD, {}), ("fixedWalls", "p", ZEROGRAD, {})]
    solver = dict(nu=0.01, dt=0.005, n_corr=2, n_nonorth=0, convection="central", p_ref_cell=0, **THROUGHPUT)
    ic = lambda xc, xf, Sf: (np.zeros((len(xc), 3)), np.zeros(len(xc)), np.zeros(len(Sf)))
    return Case("c1_cavity_20x20x1_hex", raw, bcs, solver, ic, "OpenFOAM cavity 20x20x1 hex, Re=10 (A-31)")


def c2(scramble=12):
    raw = synth.pipe_c2(scramble=scramble)
    # dt = 0.002, not SURVEY's 0.01: on this n=16 O-grid (max non-orthogonality
    # 54 deg, h ~ 0.028) PISO with n_corr = 2 diverges at nu dt / h^2 ~ 1.3
    # (oracle, reading A-34); at 0.002 (nu dt / h^2 ~ 0.26, Co ~ 0.14) it is stable.
    solver = dict(nu=0.1, dt=0.002, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0, **THROUGHPUT)
    return Case("c2_pipe_tet_199680", raw, _pipe_bcs(2.0, 0.5), solver, _poiseuille_ic(21, 2.0, 0.5),
                "O-grid pipe R=0.5 L=2.6, alternating 5-tet, N=199680, Re_D=10")


def c2_small(n_z=8, scramble=12):
    """The C2 recipe (same O-grid cross-section, physics and solver settings)
    on a short pipe (n_z layers of L = 0.05 n_z): a test-sized case."""
    raw = synth.pipe(16, 8, n_z, 0.5, 0.05 * n_z, True, scramble)
    solver = dict(nu=0.1, dt=0.002, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0, **THROUGHPUT)
    return Case(f"c2_small_pipe_tet_{raw.n_cells}", raw, _pipe_bcs(2.0, 0.5), solver, _poiseuille_ic(21, 2.0, 0.5),
                f"C2 cross-section, n_z={n_z}, N={raw.n_cells}")


def c5(n_z=814, scramble=15):
    raw = synth.pipe_c5(n_z=n_z, scramble=scramble)
    solver = dict(nu=0.01, dt=0.001, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0, **THROUGHPUT)
    return Case(f"c5_pipe_tet_{raw.n_cells}", raw, _pipe_bcs(2.0, 0.5), solver, _poiseuille_ic(51, 2.0, 0.5),
                f"O-grid pipe n=64 m_r=32 n_z={n_z}, alternating 5-tet, N={raw.n_cells}, Re_D=100")


def c4(target_cells=1.0e7, scramble=14):
    """configs[3]: voxelised H-tree (Murray radii, 8 terminal outlets) ->
    alternating 5-tet, CGS units (rho 1.06, mu 0.04 -> nu 0.0377 cm^2/s),
    parabolic inlet of mean 10 cm/s, 8 Windkessel RCR outlets alternating the
    Table 2 ground-truth parameters."""
    raw = synth.htree(depth=3, r0=1.0, l0=8.0, target_cells=target_cells, scramble=scramble)
    bcs = [("inlet", "U", PARABOLIC, dict(u_max=20.0, center=(0.0, 0.0, 0.0), radius=1.0)),
           ("wall", "U", FIXED, dict(value=(0.0, 0.0, 0.0))), ("inlet", "p", ZEROGRAD, {}), ("wall", "p", ZEROGRAD, {})]
    outlets = [p.name for p in raw.patches if p.name.startswith("outlet")]
    for o in outlets:
        bcs.append((o, "U", ZEROGRAD, {}))
    gt = [(100.0, 1.1111e-3, 900.0), (160.0, 6.9444e-4, 1440.0)]
    wk = [(o, gt[i % 2]) for i, o in enumerate(outlets)]
    solver = dict(nu=0.04 / 1.06, dt=1e-3, rho=1.06, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0,
                  **THROUGHPUT)
    ic = lambda xc, xf, Sf: (np.zeros((len(xc), 3)), np.zeros(len(xc)), np.zeros(len(Sf)))
    case = Case(f"c4_htree_tet_{raw.n_cells}", raw, bcs, solver, ic,
                f"voxelised H-tree, alternating 5-tet, N={raw.n_cells}, 8 RCR outlets (Table 2 values)")
    case.windkessel = wk     # list of (patch, (Rp, C, Rd)); pc0 = 0, exact integrator
    return case


def c3(target_cells=1.0e6, scramble=13):
    """configs[2]: flow past a cylinder (D = 0.2, Re = 200 with U = 1,
    nu = 1e-3), 2-D polygon dual of a Delaunay triangulation extruded
    one layer; free stream U = (1,0,0) on inlet and sides,
    outlet p = 0, no-slip cylinder; dt = 1e-3, n_corr 2, n_nonorth 1,
    upwind (A-28); U0 = (1,0,0) + 1% noise (seed 31), p0 = 0."""
    raw = synth.cylinder_poly(target_cells=target_cells, scramble=scramble)
    one = dict(value=(1.0, 0.0, 0.0))
    bcs = [("inlet", "U", FIXED, one), ("sides", "U", FIXED, one), ("cylinder", "U", FIXED, dict(value=(0.0, 0.0, 0.0))),
           ("outlet", "U", ZEROGRAD, {}), ("inlet", "p", ZEROGRAD, {}), ("sides", "p", ZEROGRAD, {}),
           ("cylinder", "p", ZEROGRAD, {}), ("outlet", "p", FIXED, dict(value=0.0))]
    solver = dict(nu=1e-3, dt=1e-3, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0, **THROUGHPUT)

    def ic(xc, xf, Sf):
        N = len(xc)
        U = np.zeros((N, 3))
        U[:, 0] = 1.0
        U[:, :2] += 0.01 * synth.cell_field(31, N, 2)
        # free-stream flux, zero on the cylinder wall (face centroids at r <= 0.1)
        phi = Sf[:, 0] * (np.hypot(xf[:, 0], xf[:, 1]) > 0.1 + 1e-9)
        return U, np.zeros(N), phi
    return Case(f"c3_cylinder_poly_{raw.n_cells}", raw, bcs, solver, ic,
                f"cylinder D=0.2 in [-1,3]x[-1,1], polygon dual, 1 layer, N={raw.n_cells}, Re=200")


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}
