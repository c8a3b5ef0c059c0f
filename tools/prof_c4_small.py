"""C4-shaped split-kernel workload at a reduced n for ncu captures (p = 128 log-normal, 4 nu, fp32 out)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
g = np.random.default_rng(4)
X = np.exp(g.standard_normal((n, 128))).astype(np.float32)
dX = torch.from_numpy(X).cuda()
nus = [1.5, 2.0, 3.0, 5.0]
out = torch.zeros(len(nus) * n * n, dtype=torch.float32, device="cuda")
for _ in range(2):
    G.pairwise_gini_device(dX.data_ptr(), G.F32, n, 128, nus, G.F32, False, out.data_ptr())
torch.cuda.synchronize()
print("done", float(out[:n * n].double().sum()))
