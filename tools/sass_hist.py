"""Opcode histogram of an ncu source page (--page source --csv --print-source sass):
warp-level 'Instructions Executed' summed per SASS opcode, optionally per unit of work."""
import csv
import sys
from collections import Counter


def hist(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
    c = Counter()
    for r in rows[2:]:
        if len(r) <= i_ex or not r[i_ex].strip().isdigit():
            continue
        op = r[i_src].split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        c[o.split(".")[0]] += int(r[i_ex])
    return c


if __name__ == "__main__":
    c = hist(sys.argv[1])
    div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    tot = sum(c.values())
    print(f"total {tot / div:.1f}")
    for o, n in c.most_common(40):
        print(f"{o:12s} {n / div:10.1f} {100 * n / tot:5.1f}%")
