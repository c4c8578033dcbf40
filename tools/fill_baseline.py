"""Print BASELINE.md §4 rows from a directory of bench lines (gpu_final_r2b.sh
output): python tools/fill_baseline.py gpurun_out/TAG"""
import json
import os
import sys

D = sys.argv[1]


def L(f):
    p = os.path.join(D, f)
    try:
        return json.loads(open(p).read().strip().splitlines()[-1])
    except Exception:
        return None


b, f32, ref = L("bench.json"), L("bench_f32.json"), L("bench_ref.json")
c4, c3, c2, c1 = L("bench_c4.json"), L("bench_c3.json"), L("bench_c2.json"), L("bench_c1.json")
peak = b["roofline"]["peak"]


def op(d, k):
    o = (d or {}).get("operators") or {}
    return o.get(k, {})


def g(v, f="%.0f"):
    return (f % v) if v is not None else "—"


rows = []
lb, lf = op(b, "laplacian_p"), op(f32, "laplacian_p")
rows.append(("C5 pipe 50.0M tets (O-grid, alternating 5-tet, L/D = 10)", "`lap_apply` GB/s (ALG 28N + 24F; over-relaxed Laplacian with a given gradient, `operators.laplacian_p`)", "1",
             g(lb.get("GBps")), g(lf.get("GBps")), "%.0f %% / %.0f %%" % (100 * lb["frac"], 100 * lf["frac"]), "—"))
r = b["roofline"]
rows.append(("C5", "PCG SpMV `k_cg_spmv` inside the PISO step (roofline kernel of the bench line; ALG 28N + 24F)", "1",
             g(r["achieved"]), "—", "%.1f %% (ncu DRAM %.2f GB / launch)" % (100 * r["frac"], (r.get("traffic") or 0) / 1e9), "—"))
ops = ["interpolate_s", "grad_s", "grad_U", "div"]
rows.append(("C5", "`fvc_interpolate` / `fvc_grad` scalar / vector / `fvc_div` GB/s", "1",
             " / ".join(g(op(b, k).get("GBps")) for k in ops), " / ".join(g(op(f32, k).get("GBps")) for k in ops),
             " / ".join("%.0f %%" % (100 * op(b, k)["frac"]) for k in ops), "—"))
kb = b["krylov"]
rows.append(("C5", "PISO cell-updates/s (PCG it/solve, BiCGStab it/component); e2e through the C ABI with host buffers", "1",
             "%.3e (%.1f, %.1f); e2e %.3e" % (b["value"], kb["pcg_iterations_per_solve"], kb["bicgstab_iterations_per_component"], b["e2e"]["value"]),
             "%.3e; e2e %.3e" % (f32["value"], f32["e2e"]["value"]) if f32 else "—", "—",
             "%.3e (%s)" % (ref["value"], ref["cpu_baseline"]["sample"].split(",")[0]) if ref else "—"))
for name, d, extra in (("C4 vascular H-tree 9.54M tets, 8 RCR outlets", c4, ""), ("C3 cylinder 1.00M poly (F/N = 3)", c3, ""),
                       ("C2 pipe 199 680 tets", c2, ""), ("C1 cavity 400 hex", c1, "")):
    if not d:
        continue
    kd = d["krylov"]
    lap = op(d, "laplacian_p")
    rows.append((name, "PISO cell-updates/s (ms/step; PCG it/solve); `lap_apply` GB/s", "1",
                 "%.3e (%.2f ms; %.1f); lap %s GB/s" % (d["value"], d["ms_per_step"], kd["pcg_iterations_per_solve"], g(lap.get("GBps"))),
                 "—", "lap %.0f %%" % (100 * lap["frac"]) if lap.get("frac") else "—", "—"))
print("| Config | Metric | P | fp64 | fp32 | %% of %.0f GB/s | Oracle (1 core) |" % peak)
print("|---|---|---|---|---|---|---|")
for rw in rows:
    print("| " + " | ".join(rw) + " |")
