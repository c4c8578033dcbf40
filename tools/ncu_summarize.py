"""Compact summaries of ncu CSV output (run on the GPU box by gpu_ncu_r2.sh).
  launches IN OUT: per (kernel, grid) launch count, total / mean duration, share
  full IN OUT:     per launch, the metrics that explain a bandwidth-bound kernel
"""
import csv
import sys
from collections import defaultdict

mode, src, dst = sys.argv[1:4]
rows = list(csv.reader(open(src, errors="replace")))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
if mode == "launches":
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        if r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        key = (r[col["Kernel Name"]].split("(")[0], r[col["Grid Size"]], r[col["Block Size"]])
        v = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)   # -> usecond
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "grid", "block", "launches", "total_us", "mean_us", "share"])
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            w.writerow([k[0], k[1], k[2], v[0], round(v[1], 1), round(v[1] / v[0], 2), round(v[1] / tot, 4)])
else:
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
            "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
            "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"]
    keep = [h for h in want if h in col]
    with open(dst, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(keep)
        for r in data:
            w.writerow([r[col[h]] for h in keep])
