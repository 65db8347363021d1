"""Dev tool: print SASS lines [addr_lo, addr_hi] (hex suffix match) with exec count and samples."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
lo, hi = int(sys.argv[2], 16), int(sys.argv[3], 16)
for r in data:
    a = int(r[ix["Address"]], 16) & 0xffffff
    if lo <= a <= hi:
        print(f"{a:06x} {r[ix['# Samples']]:>6} {r[ix['Instructions Executed']]:>10}  {r[ix['Source']]}")
