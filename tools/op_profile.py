"""Apply each FVM operator a few times on a BASELINE mesh (for ncu captures
of the operator kernels outside the PISO step).
usage: python tools/op_profile.py [c5|c3|c4] [f64|f32] [nz]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import cases  # noqa: E402
import paper_2603_15920_b200 as dfvm  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
nz = int(sys.argv[3]) if len(sys.argv) > 3 else None
case = cases.c5(n_z=nz) if (cfg == "c5" and nz) else cases.CONFIGS[cfg]()
raw = case.raw
m = dfvm.Mesh(raw, precision=prec)
B = dfvm.BCs(m)
for pt in raw.patches:
    if pt.kind != synth.PATCH_EMPTY:
        B.set(pt.name, "s", 0, value=0.5)
        B.set(pt.name, "U", 0, value=(0.3, -0.2, 0.1))
        B.set(pt.name, "p", 0, value=0.0)
n = raw.n_cells
x = m.field("cells", 1, synth.cell_field(100, n))
X3 = m.field("cells", 3, synth.cell_field(100, n, 3))
G, G9, y = m.field("cells", 3), m.field("cells", 9), m.field("cells", 1)
xf = m.field("faces", 1)
fl = m.field("flux", 1, synth.face_field(300, raw.n_faces))
for _ in range(3):
    dfvm.interpolate(m, x, B, "s", xf)
    dfvm.grad(m, x, B, "s", G)
    dfvm.grad(m, X3, B, "U", G9)
    dfvm.div(m, fl, y)
    dfvm.laplacian(m, B, "p", x, y, grad=G)
print("ok", float(np.abs(y.get()).max()))
