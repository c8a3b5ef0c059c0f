"""bench.py's distance step alone: the packed fp32 Gini matrix of the metric data
(image-like, p = 784) at a given n and nu -- for launch lists and kernel profiles.
Prints the median time of 3 steps (CUDA events) after one warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
nus = [float(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2.0]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
X = make_image_like(n, 784)
dX = torch.from_numpy(X).cuda()
out = torch.zeros(len(nus) * G.packed_elems(n), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
G.pairwise_gini_device(dX.data_ptr(), G.F32, n, 784, nus, G.F32, True, out.data_ptr(), 0, 1, st.cuda_stream)
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, 784, nus, G.F32, True, out.data_ptr(), 0, 1, st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"n={n} nus={nus} ms={np.median(ts):.3f} pairs/s={n * (n - 1) / 2 / (np.median(ts) / 1e3):.4g} checksum={float(out.double().sum()):.10g}")
