"""CPU-side checks of the C-ABI boundary (no compute calls without a GPU):
libdfvm.so loads, exports every entry point include/dfvm.h declares, the
pure-host Windkessel update matches the closed form, and compute entry points
fail loudly (DFVM_E_CUDA) when no GPU is present instead of falling back."""
import math
import os
import re

import numpy as np
import pytest

import paper_2603_15920_b200 as dfvm
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dfvm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfvm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_binding_symbols():
    assert set(_declared()) == set(dfvm.SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = dfvm.lib()
    for name in _declared():
        assert hasattr(L, name), name


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dfvm.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_windkessel_update_host_scalar():
    # eq:windkessel_discrete closed form; FE/BE alternatives
    Rp, Cc, Rd, pc, Q, dt = 100.0, 1.1111e-3, 900.0, 0.3, 0.01, 1e-3
    e = math.exp(-dt / (Rd * Cc))
    a, po = dfvm.windkessel_update(pc, Q, dt, Rp, Cc, Rd, 0)
    assert abs(a - (pc * e + Rd * Q * (1 - e))) <= 1e-15 and abs(po - (a + Rp * Q)) <= 1e-15
    a, _ = dfvm.windkessel_update(pc, Q, dt, Rp, Cc, Rd, 1)
    assert abs(a - (pc + dt * (Q - pc / Rd) / Cc)) <= 1e-15
    a, _ = dfvm.windkessel_update(pc, Q, dt, Rp, Cc, Rd, 2)
    assert abs(a - (pc + dt * Q / Cc) / (1 + dt / (Rd * Cc))) <= 1e-15
    with pytest.raises(dfvm.DfvmError) as ei:
        dfvm.windkessel_update(pc, Q, dt, Rp, 0.0, Rd, 0)
    assert ei.value.status == "INVALID_WK_PARAMS"


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(dfvm.DfvmError) as ei:
        dfvm.Mesh(synth.cavity())
    assert ei.value.status == "CUDA"


def test_missing_library_raises(monkeypatch, tmp_path):
    """Without libdfvm.so the binding raises instead of running anything else:
    there is no CPU or oracle fallback on the product path."""
    monkeypatch.setattr(dfvm, "_LIB", None)
    monkeypatch.setattr(dfvm, "LIB_PATH", str(tmp_path / "libdfvm.so"))
    with pytest.raises(dfvm.DfvmError) as ei:
        dfvm.lib()
    assert "missing" in str(ei.value)


def test_product_path_never_imports_oracle():
    """The package and bench's timed arm share no code with oracle/: no module
    of the package imports it, and the library does not link liboracle."""
    pkg = os.path.join(ROOT, "paper_2603_15920_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "liboracle" not in src, f
                assert "oracle/" not in src.replace("oracle/`", ""), f


def test_set_allocator_contract():
    """§8(b) b3: dfvm_set_allocator takes both callbacks or neither, and may
    be changed while no library allocation is live (true here: no GPU, so no
    mesh / field was ever created)."""
    assert dfvm.live_device_bytes() == 0
    calls = []
    dfvm.set_allocator(lambda n, s: calls.append(n) or 0, lambda p, n, s: None)
    dfvm.set_allocator()
    L = dfvm.lib()
    st = L.dfvm_set_allocator(dfvm.ALLOC_FN(lambda n, s, c: None), dfvm.FREE_FN(0), None)
    assert st == 1   # DFVM_E_INVALID_ARG: one callback without the other
    assert calls == []   # installing never allocates


def test_piso_opts_layout_matches_header():
    """the binding's PisoOpts mirrors dfvm_piso_opts field for field (cont_tol last)"""
    src = open(os.path.join(ROOT, "include", "dfvm.h")).read()
    body = src[src.index("/* --------------------------------------------------------------- solver */"):]
    body = body[:body.index("} dfvm_piso_opts;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    names = re.findall(r"(?:double|int32_t|int64_t)\s+([^;]+);", body)
    flat = [n.strip() for grp in names for n in grp.split(",")]
    assert flat == [f for f, _ in dfvm.PisoOpts._fields_]
