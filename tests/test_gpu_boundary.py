"""GPU checks of the §8(b) boundary contract beyond the compute calls:

* b3 ownership: dfvm_set_allocator routes every library device buffer
  through the caller's allocator (torch's caching allocator here), with
  results bitwise equal to the default allocator;
* b5 errors: DFVM_E_CONTINUITY ("divergence check failure ->
  ContinuityViolation") above the caller's threshold, never below it.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2603_15920_b200 as dfvm
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import gc, sys
import numpy as np, torch
sys.path.insert(0, %r)
import paper_2603_15920_b200 as dfvm, cases

def run():
    case = cases.c2_small()
    m = dfvm.Mesh(case.raw)
    g = m.export_geometry()
    U0, p0, phi0 = case.initial_state(g["xc"], g["xf"], g["Sf"])
    B = case.apply_bcs(dfvm.BCs(m))
    kw = dict(case.solver); kw["p_precond"] = "amg32"
    S = dfvm.Solver(m, B, **kw)
    s = torch.cuda.Stream()
    sp = s.cuda_stream
    import ctypes
    sp = ctypes.c_void_p(sp)
    U, p, phi = m.field("cells", 3, U0, sp), m.field("cells", 1, p0, sp), m.field("flux", 1, phi0, sp)
    for _ in range(2):
        S.step(U, p, phi, sp)
    live = dfvm.live_device_bytes()
    out = (U.get(sp), p.get(sp), phi.get(sp))
    del S, U, p, phi, B, m
    gc.collect()
    return out, live

torch.cuda.init()
ref, live_default = run()
assert dfvm.live_device_bytes() == 0, dfvm.live_device_bytes()
dfvm.use_torch_allocator()
torch.cuda.synchronize()
a0 = torch.cuda.memory_allocated()
peak0 = torch.cuda.max_memory_allocated()
got, live_torch = run()
assert live_torch == live_default > 0, (live_torch, live_default)
assert torch.cuda.max_memory_allocated() - a0 >= live_torch, (torch.cuda.max_memory_allocated(), a0, live_torch)
assert dfvm.live_device_bytes() == 0
torch.cuda.synchronize()
assert torch.cuda.memory_allocated() == a0, (torch.cuda.memory_allocated(), a0)
for a, b in zip(ref, got):
    assert np.array_equal(a, b)
dfvm.set_allocator()
print("ALLOC_OK", live_torch)
""" % ROOT


def test_torch_caching_allocator_owns_library_memory():
    r = subprocess.run([sys.executable, "-c", _SCRIPT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALLOC_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_set_allocator_refused_while_allocations_live():
    raw = synth.cavity(6)
    m = dfvm.Mesh(raw)
    assert dfvm.live_device_bytes() > 0
    with pytest.raises(dfvm.DfvmError) as ei:
        dfvm.set_allocator(lambda n, s: 0, lambda p, n, s: None)
    assert ei.value.status == "INVALID_ARG"
    del m


def test_continuity_status():
    import cases
    case = cases.c2_small()
    m = dfvm.Mesh(case.raw)
    g = m.export_geometry()
    U0, p0, phi0 = case.initial_state(g["xc"], g["xf"], g["Sf"])
    B = case.apply_bcs(dfvm.BCs(m))
    # converged final corrector: continuity at round-off, far below 1e-6
    ok = dfvm.Solver(m, B, **dict(case.solver, p_tol=1e-12, cont_tol=1e-6))
    U, p, phi = m.field("cells", 3, U0), m.field("cells", 1, p0), m.field("flux", 1, phi0)
    r = ok.step(U, p, phi)
    assert r["status"] == "OK" and r["cont_err_max"] <= 1e-6
    # a threshold below round-off must trip, and the report still names the value
    bad = dfvm.Solver(m, B, **dict(case.solver, p_tol=1e-12, cont_tol=1e-300))
    with pytest.raises(dfvm.DfvmError) as ei:
        bad.step(U, p, phi)
    assert ei.value.status == "CONTINUITY" and "cont_tol" in str(ei.value)
