"""Compact JSON summary of .ncu-rep files (run on the GPU box so only small
files come back).  usage: python scripts/ncu_summary.py out.json rep1 [rep2 ...]
Every kernel row of every report: duration, DRAM bytes, FP64 pipe, issue,
occupancy, shared-memory wavefronts / conflicts, L2 hit rate, top stalls."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size",
        "launch__block_size"]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {k: (v[i], u[i]) for i, k in enumerate(h) if i < len(v)}
        r = {"kernel": d.get("Kernel Name", ("?",))[0][:140]}
        for k in KEYS:
            if k in d:
                val, unit = d[k]
                try:
                    val = float(val.replace(",", ""))
                except ValueError:
                    pass
                r[k] = [val, unit]
        st = []
        for k in h:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and k in d:
                try:
                    st.append((k.split("stalled_")[1], float(d[k][0].replace(",", "") or 0)))
                except ValueError:
                    pass
        tot = sum(x for _, x in st) or 1
        r["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(st, key=lambda kv: -kv[1])[:8]}
        res.append(r)
    return res


out = {}
for rep in sys.argv[2:]:
    name = rep.split("/")[-1].replace(".ncu-rep", "")
    out[name] = rows_of(rep)
json.dump(out, open(sys.argv[1], "w"), indent=1)
for k, v in out.items():
    for r in v:
        t = r.get("gpu__time_duration.sum", ["?"])[0]
        print(k, r["kernel"][:60], t, r.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", ["?"])[0])
