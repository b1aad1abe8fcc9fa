"""Stall-reason totals of an ncu SASS source page, per contiguous region of the kernel.
python tools/stall_regions.py page.csv start:end[:name] ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in rows[2:] if len(r) > len(cols)]
for spec in sys.argv[2:]:
    p = spec.split(":")
    a, b = int(p[0]), int(p[1])
    name = p[2] if len(p) > 2 else spec
    tot = {c: sum(int(r[h.index(c)] or 0) for r in data[a:b]) for c in cols}
    s = sum(tot.values())
    top = sorted(tot.items(), key=lambda x: -x[1])[:6]
    print(f"{name:12s} {s:7d} " + " ".join(f"{k[6:]}={v}" for k, v in top))
