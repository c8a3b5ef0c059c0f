"""Instruction mix and stall shares of an ncu `--page source --csv --print-source sass`
export: executed warp-instructions per opcode (and per pair when npairs is given), the
hottest straight-line blocks and their stall samples."""
import csv
import re
import sys
from collections import Counter

path = sys.argv[1]
npairs = float(sys.argv[2]) if len(sys.argv) > 2 else None
r = list(csv.reader(open(path)))
h = r[1]
si, ii, sa = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
rows = []
for row in r[2:]:
    try:
        rows.append((int(row[0], 16), row[si].strip(), int(row[ii] or 0), int(row[sa] or 0)))
    except (ValueError, IndexError):
        pass
ops, stalls = Counter(), Counter()
for a, s, n, st in rows:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", s)
    op = m.group(2) if m else s.split()[0]
    ops[op] += n
    stalls[op] += st
tot = sum(ops.values())
stot = sum(stalls.values())
print(f"total warp-instructions {tot:.4g}" + (f"  per pair {tot * 32 / npairs:.2f} thread-instr" if npairs else ""))
for op, n in ops.most_common(22):
    print(f"  {op:10s} {n / tot * 100:5.1f}%  stalls {stalls[op] / max(1, stot) * 100:5.1f}%" +
          (f"  {n * 32 / npairs:6.2f}/pair" if npairs else ""))
