"""Join an ncu SASS source-page CSV (--page source --print-source sass) with
nvdisasm line info of the same kernel: instructions executed and stall
samples per source line.  Usage: sass_lines.py <ncu_sass.csv[.gz]> <obj.o> <kernel-substring>"""
import csv
import collections
import gzip
import os
import re
import subprocess
import sys
import tempfile


def line_map(obj, kern):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    m, cur, inside = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = kern in ln
            continue
        if not inside:
            continue
        f = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
        if f:
            cur = (os.path.basename(f.group(1)), int(f.group(2)))
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a and cur:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    path, obj, kern = sys.argv[1:4]
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    h = rows[1]
    body = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":  # next function (device function listings follow the kernel)
            break
        body.append(r)
    iA, iE, iS = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    addrs = [int(r[iA], 16) for r in body]
    base = min(addrs)
    m = line_map(obj, kern)
    ex, st = collections.Counter(), collections.Counter()
    for r, a in zip(body, addrs):
        key = m.get(a - base, ("?", 0))
        ex[key] += float(r[iE] or 0)
        st[key] += float(r[iS] or 0)
    te, ts = sum(ex.values()), sum(st.values())
    print(f"total warp-instructions {te:.4g}, samples {ts:.4g}")
    for key, v in sorted(ex.items(), key=lambda x: -x[1])[:60]:
        print(f"{key[0]:22s}:{key[1]:<5d} inst {v / te * 100:5.1f}%  stall {st[key] / ts * 100:5.1f}%")


if __name__ == "__main__":
    main()
