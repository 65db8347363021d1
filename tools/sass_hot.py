"""Dev tool: summarise an `ncu --page source --csv --print-source sass` export:
stall-reason totals and the hottest instructions (by samples / executed)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, h):
    try:
        return float(r[ix[h]])
    except Exception:
        return 0.0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for h in stalls:
        tot[h] += num(r, h)
S = sum(tot.values())
print("stall samples:", int(S))
for h, v in tot.most_common(12):
    print(f"  {h:28s} {v / S * 100:5.1f}%")
ie = sum(num(r, "Instructions Executed") for r in data)
print("instructions executed (warp):", int(ie))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("\nhottest by samples:")
for r in sorted(data, key=lambda r: -num(r, "# Samples"))[:top]:
    st = sorted(((num(r, h), h[6:]) for h in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {int(num(r, '# Samples')):6d} exec {int(num(r, 'Instructions Executed')):9d}  {r[ix['Source']][:60]:60s} {st}")
