"""GPU parity of the solver rows: momentum LDU,
3-component BiCGStab predictor, pressure solve, full PISO steps (cavity C1,
tet pipe with non-orthogonal correction, Windkessel outlets) against the CPU
oracle; converged fields within 1e-8 relative L2 (fp64)."""
import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import make_bcs, rel_l2, rel_op_err

pytestmark = pytest.mark.gpu

TIGHT = dict(p_tol=1e-14, U_tol=1e-14, p_maxit=20000, U_maxit=2000)


def cavity_case(precision="f64", scramble=11, conv="central"):
    raw = synth.cavity(20, scramble=scramble)
    mo = oracle.Mesh(raw)
    mg = dfvm.Mesh(raw, precision=precision)
    specs = [("movingWall", "U", oracle.BC_FIXED, dict(value=(1, 0, 0))),
             ("fixedWalls", "U", oracle.BC_FIXED, dict(value=(0, 0, 0))),
             ("movingWall", "p", oracle.BC_ZEROGRAD, {}), ("fixedWalls", "p", oracle.BC_ZEROGRAD, {})]
    bo, bg = make_bcs(raw, specs, mo, mg)
    kw = dict(nu=0.01, dt=0.005, n_corr=2, n_nonorth=0, convection=conv, p_ref_cell=0)
    return raw, mo, mg, bo, bg, kw


def pipe_case(outlet="fixed", n=4, m_r=2, n_z=6, precision="f64"):
    raw = synth.pipe(n, m_r, n_z, 0.5, 1.0, tets=True, scramble=21)
    mo = oracle.Mesh(raw)
    mg = dfvm.Mesh(raw, precision=precision)
    specs = [("inlet", "U", oracle.BC_PARABOLIC, dict(u_max=2.0, center=(0, 0, 0), radius=0.5)),
             ("wall", "U", oracle.BC_FIXED, dict(value=(0, 0, 0))), ("outlet", "U", oracle.BC_ZEROGRAD, {}),
             ("inlet", "p", oracle.BC_ZEROGRAD, {}), ("wall", "p", oracle.BC_ZEROGRAD, {})]
    if outlet == "fixed":
        specs.append(("outlet", "p", oracle.BC_FIXED, dict(value=0.0)))
    bo, bg = make_bcs(raw, specs, mo, mg)
    kw = dict(nu=0.1, dt=0.01, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=0)
    return raw, mo, mg, bo, bg, kw


def initial_state(mo, seed=21, U0=None):
    U = np.zeros((mo.N, 3)) if U0 is None else U0.copy()
    U += 0.01 * synth.cell_field(seed, mo.N, 3)
    return U, np.zeros(mo.N), np.zeros(mo.NF)


def run_both(raw, mo, mg, bo, bg, kw, steps, U0=None, wk=None, direct=True):
    So = oracle.Solver(mo, bo, direct=direct, **kw, **TIGHT)
    Sg = dfvm.Solver(mg, bg, **kw, **TIGHT)
    if wk:
        for patch, args in wk.items():
            So.windkessel_set(patch, *args)
            Sg.windkessel_set(patch, *args)
    U, p, phi = initial_state(mo, U0=U0)
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
    reps = []
    for _ in range(steps):
        ro = So.step(U, p, phi)
        rg = Sg.step(Ug, pg, phig)
        reps.append((ro, rg))
    return (U, p, phi), (Ug.get(), pg.get(), phig.get()), reps, So, Sg


@pytest.mark.parametrize("conv", ["upwind", "central", "sou", "quick"])
def test_momentum_assembly_and_apply(conv):
    raw, mo, mg, bo, bg, kw = pipe_case()
    kw = dict(kw, convection=conv)
    So = oracle.Solver(mo, bo, **kw)
    Sg = dfvm.Solver(mg, bg, **kw)
    U = synth.cell_field(40, mo.N, 3)
    phi = synth.face_field(41, mo.NF)
    diag, lo, up, b = So.momentum_assemble(U, phi)
    Ug, phig = mg.field("cells", 3, U), mg.field("flux", 1, phi)
    dg, bgf = mg.field("cells", 1), mg.field("cells", 3)
    Sg.momentum_assemble(Ug, phig, dg, bgf)
    assert rel_l2(dg.get(), diag) <= 1e-13
    assert rel_l2(bgf.get(), b) <= 1e-12
    x = synth.cell_field(50, mo.N, 3)
    y = mg.field("cells", 3)
    Sg.momentum_apply(mg.field("cells", 3, x), y)
    ref = np.stack([mo.ldu_apply(diag, lo, up, x[:, k]) for k in range(3)], 1)
    scale = np.stack([mo.ldu_apply(np.abs(diag), np.abs(lo), np.abs(up), np.abs(x[:, k])) for k in range(3)], 1)
    assert rel_op_err(y.get(), ref, scale) <= 1e-12


@pytest.mark.parametrize("precond", ["jacobi", "amg", "amg32"])
@pytest.mark.parametrize("case", ["cavity", "pipe", "pipe_big"])
def test_pressure_solve(case, precond):
    if case == "pipe_big":
        raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)     # 3 AMG levels
    else:
        raw, mo, mg, bo, bg, kw = cavity_case() if case == "cavity" else pipe_case()
    So = oracle.Solver(mo, bo, **kw)
    Sg = dfvm.Solver(mg, bg, p_precond=precond, **kw)
    rAU = 0.01 * (1.5 + 0.5 * synth.cell_field(60, mo.N))
    rhs = 1e-3 * synth.cell_field(61, mo.N)
    p0 = synth.cell_field(62, mo.N)
    po, ro = So.pressure_solve(rAU, rhs, p0=p0, tol=1e-14)
    pg = mg.field("cells", 1, p0)
    rg = Sg.pressure_solve(mg.field("cells", 1, rAU), mg.field("cells", 1, rhs), pg, tol=1e-14)
    assert ro["converged"] and rg["converged"]
    assert rel_l2(pg.get(), po) <= 1e-8, (rg, ro)
    if precond == "jacobi":
        assert abs(rg["it"] - ro["it"]) <= max(5, 0.1 * ro["it"])
    else:
        assert rg["it"] < ro["it"], (rg, ro)          # the preconditioner must pay off


def test_pressure_solve_zero_rhs():
    # b = 0 -> x = 0 with 0 iterations
    raw, mo, mg, bo, bg, kw = pipe_case()
    Sg = dfvm.Solver(mg, bg, **kw)
    pg = mg.field("cells", 1, synth.cell_field(62, mo.N))
    r = Sg.pressure_solve(mg.field("cells", 1, np.full(mo.N, 0.01)), mg.field("cells", 1), pg)
    assert r["it"] == 0 and np.all(pg.get() == 0)


@pytest.mark.parametrize("conv", ["central", "upwind"])
def test_cavity_steps(conv):
    raw, mo, mg, bo, bg, kw = cavity_case(conv=conv)
    (U, p, phi), (Ug, pg, phig), reps, _, _ = run_both(raw, mo, mg, bo, bg, kw, 10)
    assert rel_l2(Ug, U) <= 1e-8 and rel_l2(pg, p) <= 1e-8 and rel_l2(phig, phi) <= 1e-8
    for ro, rg in reps:
        assert rg["cont_err_max"] <= 1e-13 and not rg["nonfinite"]
        assert all(r["converged"] or r["res"] <= 1e-12 * max(r["res0"], 1e-300) for r in rg["p"]), rg["p"]


def test_cavity_regression_values_on_gpu(golden):
    # the oracle pin values reproduced through the CUDA path (A-31 case, unscrambled)
    g = golden("cavity_c1.json")
    raw, mo, mg, bo, bg, kw = cavity_case(scramble=0)
    Sg = dfvm.Solver(mg, bg, **kw, **TIGHT)
    Ug, pg, phig = mg.field("cells", 3), mg.field("cells", 1), mg.field("flux", 1)
    Sg.step(Ug, pg, phig)
    assert abs(np.abs(Ug.get()).max() - g["step1"]["max_abs_U_component"]) <= 1e-9
    p = pg.get()
    assert abs(p.min() - g["step1"]["p_min"]) <= 1e-8 and abs(p.max() - g["step1"]["p_max"]) <= 1e-8


@pytest.mark.parametrize("precond,conv", [("jacobi", "upwind"), ("amg", "upwind"), ("amg", "sou"),
                                          ("jacobi", "quick"), ("amg32", "upwind")])
def test_pipe_nonorth_steps(precond, conv):
    raw, mo, mg, bo, bg, kw = pipe_case()
    kw = dict(kw, p_precond=precond, convection=conv)
    xc = mo.xc
    U0 = np.zeros((mo.N, 3))
    U0[:, 2] = 2.0 * (1 - 4 * (xc[:, 0] ** 2 + xc[:, 1] ** 2))
    (U, p, phi), (Ug, pg, phig), reps, _, _ = run_both(raw, mo, mg, bo, bg, kw, 3, U0=U0)
    assert rel_l2(Ug, U) <= 1e-8 and rel_l2(pg, p) <= 1e-8 and rel_l2(phig, phi) <= 1e-8


def test_windkessel_outlet_steps(golden):
    gt = golden("windkessel.json")["table2_gt"][0]
    raw, mo, mg, bo, bg, kw = pipe_case(outlet="wk")
    xc = mo.xc
    U0 = np.zeros((mo.N, 3))
    U0[:, 2] = 2.0 * (1 - 4 * (xc[:, 0] ** 2 + xc[:, 1] ** 2))
    wk = {"outlet": (gt["Rp"] * 1e-3, gt["C"] * 1e3, gt["Rd"] * 1e-3, 0.0, 0)}
    (U, p, phi), (Ug, pg, phig), reps, So, Sg = run_both(raw, mo, mg, bo, bg, kw, 3, U0=U0, wk=wk)
    assert rel_l2(Ug, U) <= 1e-8 and rel_l2(pg, p) <= 1e-8
    for ro, rg in reps:
        assert np.allclose(rg["Q"], ro["Q"], rtol=1e-8) and np.allclose(rg["p_o"], ro["p_o"], rtol=1e-8)
    assert abs(Sg.windkessel_state("outlet") - So.windkessel_pc(raw.patch("outlet"))) <= 1e-8 * abs(
        So.windkessel_pc(raw.patch("outlet")))


def test_uniform_flow_fixed_point_gpu():
    raw = synth.pipe(4, 2, 6, 0.5, 1.0, tets=True, scramble=3)
    mg = dfvm.Mesh(raw)
    U0 = np.array([0.0, 0.0, 1.0])
    bg = dfvm.BCs(mg)
    bg.set("inlet", "U", dfvm.BC_FIXED, U0); bg.set("wall", "U", dfvm.BC_FIXED, U0)
    bg.set("outlet", "U", dfvm.BC_ZEROGRAD)
    bg.set("inlet", "p", dfvm.BC_ZEROGRAD); bg.set("wall", "p", dfvm.BC_ZEROGRAD)
    bg.set("outlet", "p", dfvm.BC_FIXED, 0.0)
    S = dfvm.Solver(mg, bg, nu=0.1, dt=0.01, n_corr=2, n_nonorth=1, **TIGHT)
    mo = oracle.Mesh(raw)
    Ug = mg.field("cells", 3, np.tile(U0, (mo.N, 1)))
    pg = mg.field("cells", 1)
    phig = mg.field("flux", 1, mo.Sf @ U0)
    for _ in range(3):
        r = S.step(Ug, pg, phig)
    assert np.abs(Ug.get() - U0).max() <= 1e-12 and np.abs(pg.get()).max() <= 1e-12
    assert r["cont_err_max"] <= 1e-13


def test_piso_deterministic():
    raw, mo, mg, bo, bg, kw = pipe_case()
    outs = []
    for _ in range(2):
        S = dfvm.Solver(mg, bg, **kw, **TIGHT)
        U, p, phi = initial_state(mo)
        Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
        for _ in range(2):
            S.step(Ug, pg, phig)
        outs.append((Ug.get(), pg.get(), phig.get()))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_f32_piso_close_to_f64():
    raw, mo, mg, bo, bg, kw = cavity_case(precision="f32")
    Sg = dfvm.Solver(mg, bg, **kw, p_tol=1e-6, U_tol=1e-6)
    Ug, pg, phig = mg.field("cells", 3), mg.field("cells", 1), mg.field("flux", 1)
    for _ in range(5):
        r = Sg.step(Ug, pg, phig)
    So = oracle.Solver(mo, bo, direct=True, **kw)
    U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
    for _ in range(5):
        So.step(U, p, phi)
    assert rel_l2(Ug.get(), U) <= 1e-4 and rel_l2(pg.get(), p) <= 1e-3


@pytest.mark.parametrize("precond", ["jacobi", "amg"])
def test_htree_windkessel_outlets(precond):
    # C4 recipe at small size: voxelised H-tree, 8 RCR outlets (Table 2 values)
    import cases
    case = cases.c4(target_cells=6e4)
    mo = oracle.Mesh(case.raw)
    mg = dfvm.Mesh(case.raw)
    kw = dict(case.solver, **TIGHT)
    # parity needs converged solves: the recipe's loose non-final corrector
    # tolerance (rel 0.05) would compare two different partial iterates
    kw.update(p_tol=1e-13, U_tol=1e-13, p_rel_tol=0.0, p_rel_tol_final=0.0, U_rel_tol=0.0)
    So = oracle.Solver(mo, case.apply_bcs(oracle.BCs(mo)), **kw)
    Sg = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), p_precond=precond, **kw)
    for patch, (Rp, Cc, Rd) in case.windkessel:
        So.windkessel_set(patch, Rp, Cc, Rd, 0.0, 0)
        Sg.windkessel_set(patch, Rp, Cc, Rd, 0.0, 0)
    U, p, phi = case.initial_state(mo.xc, mo.xf, mo.Sf)
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
    for _ in range(3):
        ro = So.step(U, p, phi)
        rg = Sg.step(Ug, pg, phig)
        assert np.allclose(rg["Q"], ro["Q"], rtol=1e-8, atol=1e-12) and np.allclose(rg["p_o"], ro["p_o"], rtol=1e-8)
    assert rel_l2(Ug.get(), U) <= 1e-8 and rel_l2(pg.get(), p) <= 1e-8
    # mass balance of the final fluxes: outlets carry what the inlet brings
    # (walls carry none), to the continuity tolerance
    phig_h = phig.get()
    raw = case.raw
    inflow = sum(phig_h[pt.start:pt.start + pt.n].sum() for pt in raw.patches if pt.name == "inlet")
    outflow = sum(phig_h[pt.start:pt.start + pt.n].sum() for pt in raw.patches if pt.name.startswith("outlet"))
    assert abs(inflow + outflow) <= 1e-9 * abs(inflow)


@pytest.mark.parametrize("conv", ["upwind", "central", "sou", "quick"])
def test_scalar_transport_step_advection(conv):
    # NEXT-1 workload (§3.1.2): step profile, u = (2, 1, 0), Gamma = 1e-3
    raw = synth.square_tri(16, jitter=0.2)
    mo = oracle.Mesh(raw)
    mg = dfvm.Mesh(raw)
    specs = [("inlet_lower", "s", oracle.BC_FIXED, dict(value=1.0)), ("inlet_upper", "s", oracle.BC_FIXED, dict(value=0.0)),
             ("outlet", "s", oracle.BC_ZEROGRAD, {})]
    for pn in ("inlet_lower", "inlet_upper", "outlet"):
        specs += [(pn, "U", oracle.BC_ZEROGRAD, {}), (pn, "p", oracle.BC_ZEROGRAD, {})]
    bo, bg = make_bcs(raw, specs, mo, mg)
    kw = dict(nu=0.0, dt=0.02, convection=conv, U_tol=1e-13, U_maxit=2000)
    So = oracle.Solver(mo, bo, **kw)
    Sg = dfvm.Solver(mg, bg, **kw)
    phi = mo.Sf @ np.array([2.0, 1.0, 0.0])
    for p in raw.patches:
        if p.kind == synth.PATCH_EMPTY:
            phi[p.start:p.start + p.n] = 0.0
    x = np.zeros(mo.N)
    xg = mg.field("cells", 1, x)
    fg = mg.field("flux", 1, phi)
    for _ in range(20):
        So.transport_step(x, phi, 1e-3)
        r = Sg.transport_step(xg, fg, 1e-3)
        assert r["converged"]
    assert rel_l2(xg.get(), x) <= 1e-10


def test_c3_cylinder_poly_piso():
    # C3 recipe at small size (polygon-dual prisms, empty front/back, F/N ~ 3):
    # 3 PISO steps, converged solves, fields within the §8(c) bound
    import cases
    case = cases.c3(target_cells=2e4)
    mo, mg = oracle.Mesh(case.raw), dfvm.Mesh(case.raw)
    kw = dict(case.solver, **TIGHT)
    kw.update(p_tol=1e-13, U_tol=1e-13, p_rel_tol=0.0, p_rel_tol_final=0.0, U_rel_tol=0.0)
    So = oracle.Solver(mo, case.apply_bcs(oracle.BCs(mo)), **kw)
    Sg = dfvm.Solver(mg, case.apply_bcs(dfvm.BCs(mg)), **kw)
    U, p, phi = case.initial_state(mo.xc, mo.xf, mo.Sf)
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
    for _ in range(3):
        So.step(U, p, phi)
        rg = Sg.step(Ug, pg, phig)
        assert rg["cont_err_max"] <= 1e-10
    assert rel_l2(Ug.get(), U) <= 1e-8 and rel_l2(pg.get(), p) <= 1e-8
    assert rel_l2(phig.get(), phi) <= 1e-8
    assert np.abs(Ug.get()[:, 2]).max() <= 1e-12      # A-24: 2-D slab keeps U_z ~ 0


@pytest.mark.parametrize("direct", ["0", "512"])
def test_amg_coarsest_direct_or_sweeps(direct, monkeypatch):
    # coarsest AMG level solved by a dense inverse (default) or by l1-Jacobi
    # sweeps: the converged pressure is the same discrete solution (A-14')
    monkeypatch.setenv("DFVM_AMG_DIRECT", direct)
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    So = oracle.Solver(mo, bo, **kw)
    Sg = dfvm.Solver(mg, bg, p_precond="amg", **kw)
    rAU = 0.01 * (1.5 + 0.5 * synth.cell_field(60, mo.N))
    rhs = 1e-3 * synth.cell_field(61, mo.N)
    po, ro = So.pressure_solve(rAU, rhs, p0=np.zeros(mo.N), tol=1e-14)
    pg = mg.field("cells", 1)
    rg = Sg.pressure_solve(mg.field("cells", 1, rAU), mg.field("cells", 1, rhs), pg, tol=1e-14)
    assert rg["converged"] and len(Sg.amg_levels()) >= 2
    assert rel_l2(pg.get(), po) <= 1e-8


@pytest.mark.parametrize("precond", ["amg", "amg32"])
def test_graph_replay_bitwise(precond):
    # on a non-default stream the AMG-PCG chunks are captured once and replayed
    # as CUDA graphs; the fields must be bitwise those of the direct enqueue
    import ctypes
    import torch
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    U0, p0, phi0 = initial_state(mo)
    out = []
    s = torch.cuda.Stream()
    for sp in (None, ctypes.c_void_p(s.cuda_stream)):
        Sg = dfvm.Solver(mg, bg, p_precond=precond, **kw, **TIGHT)
        Ug, pg, phig = mg.field("cells", 3, U0), mg.field("cells", 1, p0), mg.field("flux", 1, phi0)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(3)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
    assert out[0][3] == out[1][3]
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_live_timing_does_not_change_the_step(graphs, monkeypatch):
    # live kernel timing (bench.py's roofline) records events inside captured
    # graphs or directly on the stream; the fields, iteration counts and the
    # status must be those of an untimed step, and the timers must count
    import ctypes
    import torch
    monkeypatch.setenv("DFVM_GRAPHS", graphs)
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    U0, p0, phi0 = initial_state(mo)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for timing in (False, True):
        Sg = dfvm.Solver(mg, bg, p_precond="amg32", **kw, **TIGHT)
        Sg.set_timing(timing)
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(2)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
        if timing:
            tim = Sg.timing()
            assert tim["spmv_n"] > 0 and tim["spmv_ms"] > 0 and tim["amg_pre_n"] > 0
    assert out[0][3] == out[1][3] and min(out[0][3]) > 0
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)


def test_profile_mode_does_not_change_the_step():
    # dfvm_solver_profile brackets every launch with events (and captures each
    # AMG-PCG chunk afresh): fields and iteration counts bitwise those of an
    # unprofiled step; the table books bytes per kernel and AMG level
    import ctypes
    import torch
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    U0, p0, phi0 = initial_state(mo)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for prof in (False, True):
        Sg = dfvm.Solver(mg, bg, p_precond="amg32", **kw, **TIGHT)
        Sg.profile(prof)
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(2)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
        if prof:
            rows = {(r["name"], r["level"]): r for r in Sg.profile_table()}
            assert rows[("k_cg_spmv", -1)]["launches"] == sum(out[-1][3])
            assert rows[("k_amg_resid", 0)]["alg_bytes"] > 0 and rows[("k_bi_t", -1)]["ms"] > 0
            assert any(k[0].startswith("k_amg_") and k[1] >= 1 for k in rows)   # coarse levels booked per level
    assert out[0][3] == out[1][3]
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)


def test_c1_cavity_100_steps_trajectory():
    # SURVEY §8(c) "Multi-step trajectories: C1 100 steps <= 1e-8" (Re = 10 is
    # strongly damped): the whole t = 0.5 trajectory of the A-31 cavity, oracle
    # and CUDA path at parity tolerance, compared every 10 steps, plus the
    # printed regression values of the survey's independent prototype at t = 0.5
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cavity_c1.json")))
    raw, mo, mg, bo, bg, kw = cavity_case(scramble=0)
    So = oracle.Solver(mo, bo, **kw, **TIGHT)
    Sg = dfvm.Solver(mg, bg, **kw, **TIGHT)
    U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
    Ug, pg, phig = mg.field("cells", 3), mg.field("cells", 1), mg.field("flux", 1)
    for n in range(1, 101):
        So.step(U, p, phi)
        r = Sg.step(Ug, pg, phig)
        assert r["cont_err_max"] <= 1e-13
        if n % 10 == 0:
            assert rel_l2(Ug.get(), U) <= 1e-8 and rel_l2(pg.get(), p) <= 1e-8 and rel_l2(phig.get(), phi) <= 1e-8, n
    Uh, ph = Ug.get(), pg.get()
    t05 = g["step100"]
    assert abs(np.abs(Uh[:, 0]).max() - t05["max_abs_Ux"]) <= 1e-9
    assert abs(np.abs(Uh[:, 1]).max() - t05["max_abs_Uy"]) <= 1e-9
    assert abs(ph.min() - t05["p_min"]) <= 5e-9 and abs(ph.max() - t05["p_max"]) <= 5e-9
    assert abs(np.abs(Uh).sum() - t05["sum_abs_U"]) <= 1e-7


@pytest.mark.parametrize("precond", ["amg", "amg32"])
@pytest.mark.parametrize("size", ["pipe_big", "c5_nz6"])
def test_amg_kernel_variants_bitwise(precond, size, monkeypatch):
    # the fused / unfused coarse kernels (DFVM_AMG_FUSED_FROM) and the
    # CSR-stream / SELL forms of the one-thread-per-row levels (DFVM_AMG_CSR)
    # change the memory traffic only: same rows, same per-row arithmetic in
    # the same order, hence bitwise equal fields and identical iteration counts
    import ctypes
    import torch
    import cases
    if size == "pipe_big":
        raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
        U0, p0, phi0 = initial_state(mo)
        mk = lambda: dfvm.Solver(mg, bg, p_precond=precond, **kw, **TIGHT)
    else:
        case = cases.c5(n_z=6)
        mg = dfvm.Mesh(case.raw)
        geo = mg.export_geometry()
        U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
        bg = case.apply_bcs(dfvm.BCs(mg))
        mk = lambda: dfvm.Solver(mg, bg, **dict(case.solver, p_precond=precond))
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for env in ({"DFVM_AMG_FUSED_FROM": "1"}, {"DFVM_AMG_FUSED_FROM": "3"}, {"DFVM_AMG_FUSED_FROM": "9"},
                {"DFVM_AMG_FUSED_FROM": "3", "DFVM_AMG_CSR": "0"}, {"DFVM_AMG_CSR": "0", "DFVM_AMG_PF": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        Sg = mk()
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(2)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
        assert len(Sg.amg_levels()) >= 3
    for o in out[1:]:
        assert o[3] == out[0][3]
        for a, b in zip(out[0][:3], o[:3]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("perm", ["1", "2"])
def test_amg_sigma_storage_same_hierarchy(perm, monkeypatch):
    # SELL-32-sigma storage of the coarse levels (DFVM_AMG_PERM=1: slot -> row
    # indirection; 2: rows renumbered by slot on the device) keeps the host
    # aggregation, hence the hierarchy and each row's sum order: same level
    # sizes, same iteration counts, fields equal to the natural order up to
    # the round-off of the fp32 coarsest dense inverse (taken in slot order),
    # every pressure solve converged to TIGHT tolerances (no relative stop)
    import ctypes
    import torch
    import cases
    case = cases.c5(n_z=6)
    mg = dfvm.Mesh(case.raw)
    geo = mg.export_geometry()
    U0, p0, phi0 = case.initial_state(geo["xc"], geo["xf"], geo["Sf"])
    bg = case.apply_bcs(dfvm.BCs(mg))
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for v in ("0", perm):
        monkeypatch.setenv("DFVM_AMG_PERM", v)
        Sg = dfvm.Solver(mg, bg, **dict(case.solver, p_precond="amg32", p_rel_tol=0.0, **TIGHT))
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(2)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]],
                    Sg.amg_levels()))
    assert out[0][4] == out[1][4] and len(out[0][4]) >= 3
    assert sum(abs(a - b) for a, b in zip(out[0][3], out[1][3])) <= 2
    for a, b in zip(out[0][:3], out[1][:3]):
        assert rel_l2(b, a) <= 1e-10


@pytest.mark.parametrize("mode", ["1", "2"])
def test_programmatic_launch_bitwise(mode, monkeypatch):
    # programmatic dependent launch inside the device-resident Krylov graphs
    # (DFVM_PDL; every kernel waits for its dependencies first): the fields
    # and iteration counts are bitwise those of ordinary graph edges
    import ctypes
    import torch
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    U0, p0, phi0 = initial_state(mo)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for v in ("0", mode):
        monkeypatch.setenv("DFVM_PDL", v)
        for pc in ("amg32", "jacobi"):
            Sg = dfvm.Solver(mg, bg, p_precond=pc, **kw, **TIGHT)
            Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
            reps = [Sg.step(Ug, pg, phig, sp) for _ in range(3)]
            out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
    for a, b in zip(out[:2], out[2:]):
        assert a[3] == b[3]
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("precond", ["amg32", "amg"])
def test_amg_large_coarsest_inverse(precond, monkeypatch):
    # coarsest levels above the one-block limit (512 rows) are inverted by the
    # blocked symmetric sweep (fp32) / the multi-launch Gauss-Jordan (fp64):
    # the converged pressure equals the oracle's, in no more PCG iterations
    # than with the deeper hierarchy and its 512-row-capped dense coarsest
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    So = oracle.Solver(mo, bo, **kw)
    rAU = 0.01 * (1.5 + 0.5 * synth.cell_field(60, mo.N))
    rhs = 1e-3 * synth.cell_field(61, mo.N)
    po, ro = So.pressure_solve(rAU, rhs, p0=np.zeros(mo.N), tol=1e-14)
    its = []
    for coarse in ("256", "2000"):
        monkeypatch.setenv("DFVM_AMG_COARSE", coarse)
        monkeypatch.setenv("DFVM_AMG_DIRECT", "4000")
        Sg = dfvm.Solver(mg, bg, p_precond=precond, **kw)
        pg = mg.field("cells", 1)
        rg = Sg.pressure_solve(mg.field("cells", 1, rAU), mg.field("cells", 1, rhs), pg, tol=1e-14)
        lv = Sg.amg_levels()
        assert rg["converged"] and rel_l2(pg.get(), po) <= 1e-8
        its.append((rg["it"], lv))
    assert its[1][1][-1] > 512, its          # the large-coarsest path ran
    assert its[1][0] <= its[0][0] + 1, its


def test_amg_refresh_overlap_bitwise(monkeypatch):
    # DFVM_AMG_OVERLAP=1 computes rAU, the pressure matrix and the AMG refresh
    # on a side stream during the predictor: same inputs, same kernels, hence
    # bitwise the fields and iteration counts of the in-corrector refresh
    import ctypes
    import torch
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    U0, p0, phi0 = initial_state(mo)
    s = torch.cuda.Stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    out = []
    for v in ("0", "1"):
        monkeypatch.setenv("DFVM_AMG_OVERLAP", v)
        Sg = dfvm.Solver(mg, bg, p_precond="amg32", **kw, **TIGHT)
        Ug, pg, phig = mg.field("cells", 3, U0, sp), mg.field("cells", 1, p0, sp), mg.field("flux", 1, phi0, sp)
        reps = [Sg.step(Ug, pg, phig, sp) for _ in range(4)]
        out.append((Ug.get(sp), pg.get(sp), phig.get(sp), [r["it"] for rep in reps for r in rep["p"]]))
    assert out[0][3] == out[1][3]
    for a, b in zip(out[0][:3], out[1][:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("env", [{"DFVM_AMG_INV16": "1"}, {"DFVM_AMG_INV_EVERY": "2"}])
def test_amg_large_coarsest_variants(env, monkeypatch):
    # bf16 copy of the blocked inverse / a refresh on every other update only:
    # still an SPD coarse solve, the PISO fields converge to the oracle's
    raw, mo, mg, bo, bg, kw = pipe_case(n=8, m_r=4, n_z=40)
    monkeypatch.setenv("DFVM_AMG_COARSE", "2000")
    monkeypatch.setenv("DFVM_AMG_DIRECT", "4000")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    U0, p0, phi0 = initial_state(mo)
    So = oracle.Solver(mo, bo, **kw, **TIGHT)
    Sg = dfvm.Solver(mg, bg, p_precond="amg32", **kw, **TIGHT)
    U, p, phi = U0.copy(), p0.copy(), phi0.copy()
    Ug, pg, phig = mg.field("cells", 3, U0), mg.field("cells", 1, p0), mg.field("flux", 1, phi0)
    for _ in range(3):
        So.step(U, p, phi)
        Sg.step(Ug, pg, phig)
    assert Sg.amg_levels()[-1] > 512
    assert rel_l2(Ug.get(), U) <= 1e-8 and rel_l2(pg.get(), p) <= 1e-8 and rel_l2(phig.get(), phi) <= 1e-8
