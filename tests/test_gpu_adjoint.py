"""GPU parity for NEXT-3: transposed momentum apply,
adjoint pressure solve and the pressure VJP of the implicit differentiation
(eq:vjp P:352-358, eq:implicit_diff P:366-370), through the C ABI, against
the oracle on the same seeded inputs."""
import numpy as np
import pytest

import oracle
import paper_2603_15920_b200 as dfvm
import synth
from gpu_common import make_bcs, rel_l2, rel_op_err

pytestmark = pytest.mark.gpu


def _pipe(outlet_fixed=True):
    raw = synth.pipe(6, 3, 16, 0.5, 1.5, tets=True, scramble=21)
    mo, mg = oracle.Mesh(raw), dfvm.Mesh(raw)
    specs = [("inlet", "U", oracle.BC_PARABOLIC, dict(u_max=2.0, center=(0, 0, 0), radius=0.5)),
             ("wall", "U", oracle.BC_FIXED, dict(value=(0, 0, 0))), ("outlet", "U", oracle.BC_ZEROGRAD, {}),
             ("inlet", "p", oracle.BC_ZEROGRAD, {}), ("wall", "p", oracle.BC_ZEROGRAD, {}),
             ("outlet", "p", oracle.BC_FIXED if outlet_fixed else oracle.BC_ZEROGRAD,
              dict(value=0.3) if outlet_fixed else {})]
    bo, bg = make_bcs(raw, specs, mo, mg)
    kw = dict(nu=0.1, dt=0.01, n_corr=2, n_nonorth=1, convection="upwind", p_ref_cell=7)
    return raw, mo, mg, bo, bg, kw


@pytest.mark.parametrize("conv", ["upwind", "central", "sou"])
def test_momentum_transpose_apply(conv):
    raw, mo, mg, bo, bg, kw = _pipe()
    kw = dict(kw, convection=conv)
    So, Sg = oracle.Solver(mo, bo, **kw), dfvm.Solver(mg, bg, **kw)
    U, phi = synth.cell_field(40, mo.N, 3), synth.face_field(41, mo.NF)
    diag, lo, up, _ = So.momentum_assemble(U, phi)
    Sg.momentum_assemble(mg.field("cells", 3, U), mg.field("flux", 1, phi), mg.field("cells", 1), mg.field("cells", 3))
    x = synth.cell_field(50, mo.N, 3)
    y = mg.field("cells", 3)
    Sg.momentum_apply_transpose(mg.field("cells", 3, x), y)
    ref = np.stack([mo.ldu_apply_transpose(diag, lo, up, x[:, k]) for k in range(3)], 1)
    scale = np.stack([mo.ldu_apply(np.abs(diag), np.abs(up), np.abs(lo), np.abs(x[:, k])) for k in range(3)], 1)
    assert rel_op_err(y.get(), ref, scale) <= 1e-12
    # adjointness on the GPU alone: <M a, b> = <a, M^T b>
    a, b = synth.cell_field(51, mo.N, 3), synth.cell_field(52, mo.N, 3)
    Ma, Mtb = mg.field("cells", 3), mg.field("cells", 3)
    Sg.momentum_apply(mg.field("cells", 3, a), Ma)
    Sg.momentum_apply_transpose(mg.field("cells", 3, b), Mtb)
    lhs, rhs = np.sum(Ma.get() * b), np.sum(a * Mtb.get())
    assert abs(lhs - rhs) <= 1e-12 * np.sum(np.abs(Ma.get() * b))


@pytest.mark.parametrize("fixed", [True, False])
@pytest.mark.parametrize("precond", ["jacobi", "amg"])
def test_adjoint_solve_and_vjp(fixed, precond):
    raw, mo, mg, bo, bg, kw = _pipe(outlet_fixed=fixed)
    So, Sg = oracle.Solver(mo, bo, **kw), dfvm.Solver(mg, bg, p_precond=precond, **kw)
    rAU = 0.01 * (1.5 + 0.5 * synth.cell_field(60, mo.N))
    rhs = 1e-3 * synth.cell_field(61, mo.N)
    g = synth.cell_field(63, mo.N)
    lam_o, ro = So.pressure_adjoint(rAU, g, tol=1e-14)
    lam_g = mg.field("cells", 1)
    rg = Sg.pressure_solve_adjoint(mg.field("cells", 1, rAU), mg.field("cells", 1, g), lam_g, tol=1e-14)
    assert ro["converged"] and rg["converged"]
    assert rel_l2(lam_g.get(), lam_o) <= 1e-8
    # VJP on identical inputs (the oracle's p and lambda): an operator, 1e-12
    p_o, _ = So.pressure_solve(rAU, rhs, tol=1e-14)
    grad_o = So.pressure_vjp(rAU, p_o, lam_o)
    grad_g = mg.field("cells", 1)
    Sg.pressure_vjp(mg.field("cells", 1, p_o), mg.field("cells", 1, lam_o), grad_g)
    assert rel_l2(grad_g.get(), grad_o) <= 1e-12
