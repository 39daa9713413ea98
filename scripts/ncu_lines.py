"""Summarise an ncu --page source --csv --print-source cuda,sass dump:
top CUDA source lines by executed instructions and stall samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cur, hdr, out = None, None, []
tot_i = tot_s = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 9: continue
    try:
        ln = int(r[0])
    except ValueError:
        continue  # SASS rows are listed with address columns; skip
    try:
        inst = int(r[hdr.index("Instructions Executed")]) if r[hdr.index("Instructions Executed")] not in ("", "-") else 0
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")]) if r[hdr.index("Warp Stall Sampling (All Samples)")] not in ("", "-") else 0
    except (ValueError, IndexError):
        continue
    tot_i += inst; tot_s += st
    out.append((inst, st, cur, ln, r[1][:90]))
print(f"total inst {tot_i}  stall samples {tot_s}")
for inst, st, f, ln, src in sorted(out, reverse=True)[:n]:
    print(f"{inst/max(tot_i,1)*100:5.1f}% inst {st/max(tot_s,1)*100:5.1f}% stall  {f}:{ln}  {src}")
