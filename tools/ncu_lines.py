"""Dev tool: per-CUDA-source-line totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
acc = defaultdict(lambda: [0.0, 0.0, ""])
fpath = ""; hdr = None; line = None; src = ""
for r in rows:
    if r and r[0] == "File Path":
        fpath = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        line = r[0]; src = r[1]
    try:
        ex = float(r[7] or 0); sm = float(r[6] or 0)
    except ValueError:
        continue
    key = (fpath, line)
    acc[key][0] += ex; acc[key][1] += sm; acc[key][2] = src
te = sum(v[0] for v in acc.values()); ts = sum(v[1] for v in acc.values())
print(f"total warp-inst {te:.3e}, samples {ts:.0f}")
for (f, l), (e, s, src) in sorted(acc.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{f}:{l:>5} exec {e / te * 100:5.1f}% samp {s / ts * 100:5.1f}%  {src.strip()[:80]}")
