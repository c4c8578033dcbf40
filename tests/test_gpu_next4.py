"""GPU parity of NEXT-4: the theta time schemes of Table 1
(reading A-40: backward Euler, Crank-Nicolson, forward Euler) and the
time-varying inflow waveform (reading A-41), against the CPU
oracle (converged fields within 1e-8 relative L2, fp64) and against the
closed forms the oracle is pinned to (tests/test_oracle_next4.py)."""
import math

import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import rel_l2
from test_gpu_piso import TIGHT, cavity_case, pipe_case, run_both
from test_oracle_next4 import _g, _slab

pytestmark = pytest.mark.gpu

THETAS = [1.0, 0.5, 0.0]


@pytest.mark.parametrize("theta", THETAS)
def test_cavity_theta_steps(theta):
    raw, mo, mg, bo, bg, kw = cavity_case()
    kw = dict(kw, theta=theta, dt=0.0005 if theta == 0.0 else kw["dt"])   # FE: nu dt/h^2 = 0.2
    o, g, reps, _, _ = run_both(raw, mo, mg, bo, bg, kw, steps=4)
    for a, b in zip(g, o):
        assert rel_l2(a, b) <= 1e-8
    if theta == 0.0:   # diagonal predictor: one BiCGStab iteration per component
        assert all(r["it"] <= 1 for _, rg in reps for r in rg["U"])


@pytest.mark.parametrize("theta", THETAS)
@pytest.mark.parametrize("precond", ["jacobi", "amg32"])
def test_pipe_theta_nonorth_steps(theta, precond):
    raw, mo, mg, bo, bg, kw = pipe_case()
    kw = dict(kw, theta=theta, p_precond=precond, dt=0.002 if theta == 0.0 else kw["dt"])
    o, g, _, _, _ = run_both(raw, mo, mg, bo, bg, kw, steps=3)
    for a, b in zip(g, o):
        assert rel_l2(a, b) <= 1e-8


@pytest.mark.parametrize("theta", THETAS)
def test_shear_mode_amplification_gpu(theta):
    n, L, nu, dt, k = 32, 1.0, 0.01, 0.02, 3
    raw = _slab(n, L)
    mg = dfvm.Mesh(raw)
    bg = dfvm.BCs(mg)
    for p in raw.patches:
        if p.kind != synth.PATCH_EMPTY:
            bg.set(p.name, "U", oracle.BC_ZEROGRAD)
            bg.set(p.name, "p", oracle.BC_ZEROGRAD)
    S = dfvm.Solver(mg, bg, nu=nu, dt=dt, n_corr=2, theta=theta, **TIGHT)
    xc = oracle.Mesh(raw).xc
    U = np.zeros((len(xc), 3))
    U[:, 2] = np.cos(k * math.pi * xc[:, 0] / L)
    u0 = U[:, 2].copy()
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1), mg.field("flux", 1)
    lam = 4.0 * nu * n * n / L ** 2 * math.sin(k * math.pi / (2 * n)) ** 2
    G = (1.0 - (1.0 - theta) * dt * lam) / (1.0 + theta * dt * lam)
    for s in range(1, 6):
        S.step(Ug, pg, phig)
        assert np.abs(Ug.get()[:, 2] - G ** s * u0).max() <= 1e-12


def test_pulsatile_plug_flow_gpu():
    period, a, bb = 0.08, [1.0, 0.5, -0.2], [0.0, 0.3, 0.1]
    raw = _slab(16, 1.0, 0.1)
    mo, mg = oracle.Mesh(raw), dfvm.Mesh(raw)
    bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
    for p in raw.patches:
        if p.kind == synth.PATCH_EMPTY:
            continue
        if p.name == "xmin":
            specs = [("U", oracle.BC_FIXED, dict(value=(1.0, 0.0, 0.0))), ("p", oracle.BC_ZEROGRAD, {})]
        elif p.name == "xmax":
            specs = [("U", oracle.BC_ZEROGRAD, {}), ("p", oracle.BC_FIXED, dict(value=0.0))]
        else:
            specs = [("U", oracle.BC_ZEROGRAD, {}), ("p", oracle.BC_ZEROGRAD, {})]
        for fld, kind, kwa in specs:
            bo.set(p.name, fld, kind, **kwa)
            bg.set(p.name, fld, kind, **kwa)
    i_in = raw.patch("xmin")
    bo.set_waveform(i_in, "U", period, a, bb)
    bg.set_waveform(i_in, "U", period, a, bb)
    kw = dict(nu=0.01, dt=0.01, n_corr=2, theta=0.5)
    So = oracle.Solver(mo, bo, **kw, **TIGHT)
    Sg = dfvm.Solver(mg, bg, **kw, **TIGHT)
    U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
    xf = np.abs(mo.Sf[:, 0]) > 0.5 * np.abs(mo.Sf).max()
    for s in range(1, 7):
        So.step(U, p, phi)
        Sg.step(Ug, pg, phig)
        ph = phig.get()
        assert np.abs(ph[xf] / mo.Sf[xf, 0] - _g(s * 0.01, period, a, bb)).max() <= 1e-11
        assert rel_l2(ph, phi) <= 1e-10 and rel_l2(Ug.get(), U) <= 1e-10 and rel_l2(pg.get(), p) <= 1e-8


@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_pulsatile_parabolic_pipe(theta):
    # the paper's pulsatile parabolic inflow on the non-orthogonal tet pipe
    raw, mo, mg, bo, bg, kw = pipe_case()
    wave = (0.05, [1.0, 0.4, 0.1], [0.0, -0.3, 0.2])
    bo.set_waveform(raw.patch("inlet"), "U", *wave)
    bg.set_waveform(raw.patch("inlet"), "U", *wave)
    kw = dict(kw, theta=theta)
    o, g, reps, _, _ = run_both(raw, mo, mg, bo, bg, kw, steps=4)
    for a, b in zip(g, o):
        assert rel_l2(a, b) <= 1e-8


def test_waveform_errors():
    raw, mo, mg, bo, bg, kw = pipe_case()
    with pytest.raises(dfvm.DfvmError):
        bg.set_waveform(raw.patch("inlet"), "s", 1.0, [1.0])
    with pytest.raises(dfvm.DfvmError):
        bg.set_waveform(raw.patch("inlet"), "U", 0.0, [1.0])
    bg.set_waveform(raw.patch("outlet"), "U", 1.0, [1.0])          # zeroGradient patch: rejected at the step
    S = dfvm.Solver(mg, bg, **kw)
    Ug, pg, phig = mg.field("cells", 3), mg.field("cells", 1), mg.field("flux", 1)
    with pytest.raises(dfvm.DfvmError):
        S.step(Ug, pg, phig)
    with pytest.raises(ValueError):
        dfvm.Solver(mg, bg, **dict(kw, theta=0.7))


def test_polymesh_case_on_gpu(tmp_path):
    # NEXT-4 reader: a cavity written as an OpenFOAM ASCII case, read back by the
    # library and solved on the GPU, equals the oracle on the generator's arrays
    raw = synth.cavity(20, scramble=11)
    synth.write_polymesh(raw, str(tmp_path))
    pm = dfvm.read_polymesh(str(tmp_path))
    mo, mg = oracle.Mesh(raw), dfvm.Mesh(pm)
    specs = [("movingWall", "U", oracle.BC_FIXED, dict(value=(1, 0, 0))),
             ("fixedWalls", "U", oracle.BC_FIXED, dict(value=(0, 0, 0))),
             ("movingWall", "p", oracle.BC_ZEROGRAD, {}), ("fixedWalls", "p", oracle.BC_ZEROGRAD, {})]
    bo, bg = oracle.BCs(mo), dfvm.BCs(mg)
    for name, fld, kind, kwa in specs:
        bo.set(name, fld, kind, **kwa)
        bg.set(name, fld, kind, **kwa)
    kw = dict(nu=0.01, dt=0.005, n_corr=2, convection="central", theta=0.5)
    o, g, _, _, _ = run_both(raw, mo, mg, bo, bg, kw, steps=3)
    for a, b in zip(g, o):
        assert rel_l2(a, b) <= 1e-8


@pytest.mark.parametrize("theta", [0.5, 0.0])
def test_f32_theta_waveform_close_to_oracle(theta):
    # the fp32 library path of NEXT-4 (theta assembly, k_bc_wave in float)
    raw, mo, mg, bo, bg, kw = cavity_case(precision="f32")
    wave = (0.02, [1.0, 0.3], [0.0, 0.2])
    bo.set_waveform(raw.patch("movingWall"), "U", *wave)
    bg.set_waveform(raw.patch("movingWall"), "U", *wave)
    kw = dict(kw, theta=theta, dt=0.0005 if theta == 0.0 else kw["dt"])
    Sg = dfvm.Solver(mg, bg, **kw, p_tol=1e-6, U_tol=1e-6)
    Ug, pg, phig = mg.field("cells", 3), mg.field("cells", 1), mg.field("flux", 1)
    So = oracle.Solver(mo, bo, direct=True, **kw)
    U, p, phi = np.zeros((mo.N, 3)), np.zeros(mo.N), np.zeros(mo.NF)
    for _ in range(5):
        Sg.step(Ug, pg, phig)
        So.step(U, p, phi)
    assert rel_l2(Ug.get(), U) <= 1e-4 and rel_l2(pg.get(), p) <= 1e-3


@pytest.mark.parametrize("case", ["cavity", "pipe"])
def test_ddtcorr_steps(case):
    # OpenFOAM's Euler ddtCorr Rhie-Chow term (A-42) against the oracle
    if case == "cavity":
        raw, mo, mg, bo, bg, kw = cavity_case()
    else:
        raw, mo, mg, bo, bg, kw = pipe_case()
        kw = dict(kw, p_precond="amg32")
    kw = dict(kw, ddt_corr=True)
    o, g, _, _, _ = run_both(raw, mo, mg, bo, bg, kw, steps=4)
    for a, b in zip(g, o):
        assert rel_l2(a, b) <= 1e-8
