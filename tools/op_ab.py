"""A/B of the FVM operator kernels on one BASELINE mesh: the bench's
operator section under each value of an environment knob read per launch.
usage: python tools/op_ab.py [c5|c3|c4] [f64|f32] [VAR v1 v2 ...]
(default: DFVM_LD3 1 0 1)"""
import json
import os
import sys
import ctypes as C

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import cases  # noqa: E402
import paper_2603_15920_b200 as dfvm  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
var = sys.argv[3] if len(sys.argv) > 3 else "DFVM_LD3"
vals = sys.argv[4:] if len(sys.argv) > 4 else ["1", "0", "1"]


class A:
    precision = prec


case = cases.CONFIGS[cfg]()
mesh = dfvm.Mesh(case.raw, precision=prec)
info = mesh.info
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sp = C.c_void_p(stream.cuda_stream)
hbm, _ = bench.peaks()
res = {}
for i, v in enumerate(vals):
    os.environ[var] = v
    res[f"{i}:{var}={v}"] = bench.operator_bench(dfvm, torch, mesh, case, info, stream, sp, hbm, A, lambda x: x,
                                            lambda: None)
print(json.dumps({"config": cfg, "precision": prec, "n_cells": info["n_cells"], "ops": res}))
