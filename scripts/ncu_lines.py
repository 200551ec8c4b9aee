"""Per-source-line stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur_file = "?"
hdr = None
lines = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit() and r[2] == "-":
        si = 4; ii = 7
        try:
            lines.append((cur_file, int(r[0]), r[1], int(r[si] or 0), int(r[ii] or 0),
                          {hdr[k]: r[k] for k in range(len(hdr)) if hdr[k].startswith("stall_") and "Not" not in hdr[k]}))
        except ValueError:
            pass
tot = sum(l[3] for l in lines) or 1
toti = sum(l[4] for l in lines) or 1
print(f"total samples {tot}, warp-instructions {toti}")
for f, ln, src, s, i, st in sorted(lines, key=lambda x: -x[3])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    top = sorted(((k, int(v)) for k, v in st.items() if v.isdigit()), key=lambda x: -x[1])[:2]
    print(f"{f[:14]:14s}:{ln:<4d} {100*s/tot:5.1f}%  inst {100*i/toti:5.1f}%  {top}  {src.strip()[:70]}")
