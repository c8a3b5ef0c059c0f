"""Distance-step time at the metric shape (n=20000, p=784 image-like) for a
few nu values: nu = 2 / 3 take the linear-weight kernel, others the merge
kernel.  Wall time around one device-resident call (not a bench number)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from bench import make_image_like  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

nus = [float(v) for v in sys.argv[1:]] or [2.0, 2.5, 1.5]
X = make_image_like(20000, 784)
dX = torch.from_numpy(X).cuda()
dD = torch.zeros(G.packed_elems(20000), dtype=torch.float32, device="cuda")
G.pairwise_gini_device(dX.data_ptr(), G.F32, 20000, 784, [nus[0]], G.F32, True, dD.data_ptr())  # warm-up
for nu in nus:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    G.pairwise_gini_device(dX.data_ptr(), G.F32, 20000, 784, [nu], G.F32, True, dD.data_ptr())
    torch.cuda.synchronize()
    print(f"nu {nu}: {time.perf_counter() - t0:.4f} s", flush=True)
