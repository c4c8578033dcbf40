"""The A-19 pins of tests/test_oracle_pins_r2.py run through the CUDA path:
the Windkessel coupling inside the PISO step against closed forms (steady
uniform flow: exact fixed point on the analytic RCR solution; pulsatile plug
flow: the exact-integrator recurrence on the last corrector's Q), and the
same two cases against the oracle step by step."""
import math

import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth

pytestmark = pytest.mark.gpu

WK = dict(Rp=120.0, Cc=2.0e-3, Rd=800.0, pc0=0.4)
TIGHT = dict(U_tol=1e-15, p_tol=1e-15, p_maxit=20000, U_maxit=2000)


def _duct(lib, U0, rho, wave=None, walls="fixed", nyz=3):
    raw = synth.box(6, nyz, nyz, 2.0, 1.0, 1.0, scramble=4)
    m = lib.Mesh(raw)
    b = lib.BCs(m)
    for p in raw.patches:
        if p.name == "xmin":
            b.set(p.name, "U", 0, (U0, 0.0, 0.0)); b.set(p.name, "p", 1)
        elif p.name == "xmax":
            b.set(p.name, "U", 1)
        else:
            if walls == "fixed":
                b.set(p.name, "U", 0, (U0, 0.0, 0.0))
            else:
                b.set(p.name, "U", 1)
            b.set(p.name, "p", 1)
    if wave is not None:
        b.set_waveform(raw.patch("xmin"), "U", *wave)
    S = lib.Solver(m, b, nu=0.05, dt=0.01, rho=rho, n_corr=2, **TIGHT)
    S.windkessel_set(raw.patch("xmax"), WK["Rp"], WK["Cc"], WK["Rd"], WK["pc0"], 0)
    return raw, m, S


def test_uniform_flow_rcr_fixed_point_gpu():
    U0, rho, dt = 0.8, 1.06, 0.01
    raw, mg, Sg = _duct(dfvm, U0, rho)
    mo = oracle.Mesh(raw)
    Ug = mg.field("cells", 3, np.tile([U0, 0.0, 0.0], (mo.N, 1)))
    pg = mg.field("cells", 1)
    phig = mg.field("flux", 1, U0 * mo.Sf[:, 0])
    Q = U0 * 1.0
    for n in range(1, 6):
        r = Sg.step(Ug, pg, phig)
        pc = WK["Rd"] * Q + (WK["pc0"] - WK["Rd"] * Q) * math.exp(-n * dt / (WK["Rd"] * WK["Cc"]))
        po = pc + WK["Rp"] * Q
        assert abs(r["Q"][0] - Q) <= 1e-12 * Q
        assert abs(Sg.windkessel_state("xmax") - pc) <= 1e-12 * abs(pc)
        assert abs(r["p_o"][0] - po) <= 1e-12 * abs(po)
        assert np.abs(pg.get() - po / rho).max() <= 1e-12 * abs(po / rho), n
        assert np.abs(Ug.get() - [U0, 0.0, 0.0]).max() <= 1e-12 * U0


def test_pulsatile_rcr_recurrence_gpu_and_oracle():
    U0, rho, dt = 0.8, 1.06, 0.01
    period, a, bb = 0.08, [1.0, 0.5], [0.0, 0.3]
    g = lambda t: a[0] + a[1] * math.cos(2 * math.pi * t / period) + bb[1] * math.sin(2 * math.pi * t / period)
    raw, mg, Sg = _duct(dfvm, U0, rho, wave=(period, a, bb), walls="zerograd", nyz=1)
    _, mo, So = _duct(oracle, U0, rho, wave=(period, a, bb), walls="zerograd", nyz=1)
    U = np.tile([U0 * g(0.0), 0.0, 0.0], (mo.N, 1))
    p = np.zeros(mo.N)
    phi = U0 * g(0.0) * mo.Sf[:, 0].copy()
    Ug, pg, phig = mg.field("cells", 3, U), mg.field("cells", 1, p), mg.field("flux", 1, phi)
    e = math.exp(-dt / (WK["Rd"] * WK["Cc"]))
    pc = WK["pc0"]
    for n in range(1, 7):
        So.step(U, p, phi)
        r = Sg.step(Ug, pg, phig)
        Ql = g(n * dt) * U0
        pc = pc * e + WK["Rd"] * Ql * (1 - e)
        assert abs(r["Q"][0] - Ql) <= 1e-11, n
        assert abs(Sg.windkessel_state("xmax") - pc) <= 1e-11 * abs(pc), n
        assert abs(r["p_o"][0] - (pc + WK["Rp"] * Ql)) <= 1e-11 * abs(pc + WK["Rp"] * Ql), n
        assert np.linalg.norm(pg.get() - p) <= 1e-10 * np.linalg.norm(p)
        assert np.linalg.norm(Ug.get() - U) <= 1e-10 * np.linalg.norm(U)
