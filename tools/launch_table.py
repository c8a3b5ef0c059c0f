"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel name
(template arguments kept) count, total and mean time; optionally the launch sequence."""
import csv
import sys
from collections import OrderedDict


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    return [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr + 1:] if len(r) > vi]


if __name__ == "__main__":
    L = load(sys.argv[1])
    skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    L = L[skip:]
    agg = OrderedDict()
    for k, v in L:
        name = k.split("(")[0][:70]
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + v)
    tot = sum(v for _, v in L)
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{name:72s} n={c:5d} total={t / 1e3:10.1f} us mean={t / c / 1e3:8.1f} us  {100 * t / tot:5.1f}%")
    print(f"total {tot / 1e3:.1f} us over {len(L)} launches")
