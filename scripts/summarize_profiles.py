"""Summarise gpurun_out/prof (scripts/profile_round.sh) into profiles/round1/.
usage: python scripts/summarize_profiles.py [src] [dst]"""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/round1"
os.makedirs(dst, exist_ok=True)
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return None
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (v[i], u[i]) for i, k in enumerate(h)}
    res = {"kernel": d.get("Kernel Name", ("?",))[0]}
    for k in KEYS:
        if k in d:
            val, unit = d[k]
            try:
                val = float(val.replace(",", ""))
            except ValueError:
                pass
            res[k] = [val, unit]
    st = [(k.split("stalled_")[1], float(d[k][0].replace(",", "") or 0)) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    tot = sum(x for _, x in st) or 1
    res["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(st, key=lambda kv: -kv[1])[:8]}
    return res


summary = {}
for q in ("2", "3", "4"):
    for kind in ("fused", "fixup"):
        rep = os.path.join(src, f"{kind}_q{q}.ncu-rep")
        if os.path.exists(rep):
            r = raw(rep)
            if r:
                summary[f"{kind}_q{q}"] = r
json.dump({"command": "ncu --set full --clock-control none --import-source on -k regex:<kernel> "
                      "-s 2 -c 1 python scripts/profile_apply.py <order> <cells> 0 4 "
                      "(Q2 64^3, Q3 43^3, Q4 32^3; fused = fused_jacobian_kernel, fixup = "
                      "fused_fixup_kernel)",
           "kernels": summary}, open(os.path.join(dst, "ncu_full_summary.json"), "w"), indent=1)

lf = os.path.join(src, "launches_bench.csv")
if os.path.exists(lf):
    rows = [r for r in csv.reader(open(lf)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[1:]:
        try:
            d[r[ki]].append(float(r[vi].replace(",", "")) / 1e3)
        except ValueError:
            pass
    tot = sum(sum(v) for v in d.values())
    shares = {k[:100]: {"launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
                        "share": sum(v) / tot}
              for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))}
    json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python "
                          "bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-newton",
               "note": "cold-cache, serialised per-launch times: compare shares, not absolutes; "
                       "includes the e2e host-pipelined chunk launches",
               "kernels": shares}, open(os.path.join(dst, "launch_shares.json"), "w"), indent=1)
    shutil.copy(lf, os.path.join(dst, "launches_bench.csv"))
for f in ("bench_n1.json", "pmg_breakdown.log", "smi.txt"):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))
if "fused_q2" in summary:
    f = summary["fused_q2"]
    rd, wr = f["dram__bytes_read.sum"], f["dram__bytes_write.sum"]
    traffic = rd[0] * SCALE.get(rd[1], 1) + wr[0] * SCALE.get(wr[1], 1)
    json.dump({"kernel": "fused_jacobian_kernel<2,3>", "config": "Q2 64^3",
               "dram_bytes_per_launch": traffic, "algorithmic_bytes": 1065633840.0,
               "source": f"ncu --set full, {dst}/ncu_full_summary.json"},
              open("profiles/ncu_apply_summary.json", "w"), indent=1)
print(json.dumps({k: {"time": v.get("gpu__time_duration.sum"),
                      "dram_pct": v.get("dram__throughput.avg.pct_of_peak_sustained_elapsed"),
                      "fp64_pct": v.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")}
                  for k, v in summary.items()}, indent=1))
