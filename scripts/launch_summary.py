"""Aggregate an ncu --csv --metrics gpu__time_duration.sum launch list by kernel name."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    try:
        d[r[ki][:90]].append(float(r[vi].replace(",", "")))
    except ValueError:
        pass
tot = sum(sum(v) for v in d.values())
print(f"total {tot/1e3:.1f} us over {sum(len(v) for v in d.values())} launches")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{len(v):6d} x {sum(v)/len(v)/1e3:9.2f} us = {sum(v)/1e3:10.1f} us {100*sum(v)/tot:5.1f}%  {k}")
