"""Hot straight-line SASS blocks of an ncu `--page source --csv` export:
consecutive instructions with equal execution counts, ranked by share."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
h = r[1]
si, ii, sa = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
rows = []
for row in r[2:]:
    try:
        rows.append((int(row[0], 16), row[si].strip(), int(row[ii]), int(row[sa])))
    except (ValueError, IndexError):
        pass
base = rows[0][0]
blocks, cur = [], None
for a, s, n, st in rows:
    if cur and n == cur[2]:
        cur[3] += 1
        cur[4] += st
        cur[5] = a
    else:
        cur = [a, s, n, 1, st, a]
        blocks.append(cur)
tot = sum(b[2] * b[3] for b in blocks)
stot = sum(b[4] for b in blocks)
print("total warp-instructions", tot)
for b in sorted(sorted(blocks, key=lambda b: -b[2] * b[3])[:top_n], key=lambda b: b[0]):
    print(f"{(b[0]-base):6x}-{(b[5]-base):6x} n={b[2]:11d} len={b[3]:4d} share={b[2]*b[3]/tot*100:5.1f}% "
          f"stall={b[4]/stot*100:4.1f}% first: {b[1][:60]}")
