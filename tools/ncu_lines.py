"""Per-CUDA-line instruction and stall shares from an ncu
`--page source --csv --print-source cuda,sass` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 50
path = None
hdr = None
out = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) >= 2 and r[0] == "Function Name":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or r[2] != "-":
        continue
    try:
        n = int(r[hdr.index("Instructions Executed")] or 0)
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    if n or s:
        out.append((n, s, path, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
stot = sum(o[1] for o in out) or 1
print("total warp-instructions", tot)
for n, s, f, l, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{n / tot * 100:5.1f}% st{s / stot * 100:5.1f}% {f}:{l} {src}")
