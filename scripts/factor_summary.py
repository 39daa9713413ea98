"""Summarise an ncu --metrics CSV launch log (coarse factorization capture):
per kernel name -- launches, total time, time-weighted FP64 pipe / DMMA pipe
utilisation, DRAM bytes.  usage: python scripts/factor_summary.py log.csv out.json"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
names = {}
for r in rows[1:]:
    try:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    names[r[ii]] = r[ki]
agg = defaultdict(lambda: defaultdict(float))
for i, m in per.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    a = agg[names[i][:90]]
    a["launches"] += 1
    a["time_ns"] += t
    for k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
              "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active"):
        if k in m:
            a[k + "_x_time"] += m[k] * t
    a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a["time_ns"] for a in agg.values()) or 1
out = {}
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_ns"]):
    t = a["time_ns"] or 1
    out[k] = {"launches": int(a["launches"]), "total_ms": a["time_ns"] / 1e6, "share": a["time_ns"] / tot,
              "fp64_pipe_cycles_pct": a.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active_x_time", 0) / t,
              "fp64_inst_pct": a.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active_x_time", 0) / t,
              "dmma_pipe_pct": a.get("sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active_x_time", 0) / t,
              "dram_GB": a["dram_bytes"] / 1e9}
json.dump({"total_ms": tot / 1e6, "kernels": out}, open(sys.argv[2], "w"), indent=1)
for k, v in list(out.items())[:15]:
    print(f"{v['share']:.3f} {v['total_ms']:8.2f} ms x{v['launches']:5d} fp64cyc {v['fp64_pipe_cycles_pct']:5.1f} dmma {v['dmma_pipe_pct']:5.1f}  {k}")
