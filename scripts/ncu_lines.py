"""Summarise `ncu -i R --page source --csv --print-source cuda,sass` output:
per CUDA source line, share of executed warp instructions and stall samples
(with the top stall reasons).  usage: ncu_lines.py dump.csv [n] [lo-hi]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rng = tuple(map(int, sys.argv[3].split("-"))) if len(sys.argv) > 3 else None
cur = hdr = None
agg = defaultdict(lambda: defaultdict(float))
src = {}
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:  # a source line row: its SASS rows follow
        line = (cur, int(r[0]))
        src[line] = r[1][:80]
        continue
    if line is None or not r[2].startswith("0x"):
        continue
    if True:  # a SASS row, attributed to the preceding source line
        d = agg[line]
        for k, col in enumerate(hdr):
            if k >= 4 and (col.startswith("stall_") and "Not Issued" not in col
                           or col in ("Instructions Executed", "L1 Wavefronts Shared")):
                try:
                    d[col] += float(r[k])
                except ValueError:
                    pass
tot_i = sum(d["Instructions Executed"] for d in agg.values()) or 1
tot_s = sum(sum(v for k, v in d.items() if k.startswith("stall_")) for d in agg.values()) or 1
tot_w = sum(d["L1 Wavefronts Shared"] for d in agg.values()) or 1
print(f"warp inst {tot_i:.0f}  stall samples {tot_s:.0f}  smem wavefronts {tot_w:.0f}")
items = list(agg.items())
if rng:
    items = [it for it in items if rng[0] <= it[0][1] <= rng[1]]
    si = sum(d["Instructions Executed"] for _, d in items)
    ss = sum(sum(v for k, v in d.items() if k.startswith("stall_")) for _, d in items)
    print(f"lines {rng}: {100*si/tot_i:.1f}% inst {100*ss/tot_s:.1f}% stall")
def stalls(d):
    return sum(v for k, v in d.items() if k.startswith("stall_"))
for key, d in sorted(items, key=lambda kv: -stalls(kv[1]))[:n]:
    top = sorted(((v, k[6:]) for k, v in d.items() if k.startswith("stall_")), reverse=True)[:3]
    tops = " ".join(f"{k}:{100*v/max(stalls(d),1):.0f}" for v, k in top if v)
    print(f"{100*d['Instructions Executed']/tot_i:5.1f}%i {100*stalls(d)/tot_s:5.1f}%s "
          f"{100*d['L1 Wavefronts Shared']/tot_w:5.1f}%w {key[0]}:{key[1]:<4} {src[key]:<60} [{tops}]")
