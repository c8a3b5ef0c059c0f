"""C4's distance step alone (log-normal fp32, p = 128, 1% duplicated rows, 4 nu in one
launch, full fp32 n x n out) at a given n -- for launch lists and kernel profiles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import synth as S  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nus = S.C4_NUS
X, _, _ = S.lognormal_dup(n, 128, 4)
dX = torch.from_numpy(X).cuda()
out = torch.zeros((len(nus), n, n), dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
run = lambda: G.pairwise_gini_device(dX.data_ptr(), G.F32, n, 128, nus, G.F32, False, out.data_ptr(), 0, 1,
                                     st.cuda_stream)
run()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run()
    e1.record(st)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"C4 n={n} ms={np.median(ts):.2f} pairs/s(all 4 nu)={n * (n - 1) / 2 / (np.median(ts) / 1e3):.4g}")
