"""Euclidean pairwise_matrix on the device: the tcgen05 path (mode 2) vs
the exact fp64 CUDA-core kernel (mode 1), CUDA events on the launching stream, at C4's
shape (n = 20000, p = 128 log-normal fp32, 1% duplicated rows).  Prints one JSON line
with the tensor-pipe and HBM-write rooflines of the tcgen05 kernel."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import synth as S  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
X, _, _ = S.lognormal_dup(n, 128, 4)
p = X.shape[1]
dX = torch.from_numpy(X).cuda()
dD = torch.empty((n, n), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()


def run(mode):
    G._check(G.lib().gmds_pairwise_euclidean_device(ctypes.c_void_p(dX.data_ptr()), G._i32(G.F32), G._i64(n),
                                                    G._i64(p), ctypes.c_void_p(dD.data_ptr()), G._i32(mode),
                                                    ctypes.c_void_p(st.cuda_stream)))


out = {"n": n, "p": p}
for mode, name in ((2, "tc"), (1, "exact")):
    run(mode)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run(mode)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    out[name + "_s"] = float(np.median(ts))
pp = -(-p // 64) * 64
T = -(-n // 128)
flops = T * (T + 1) / 2 * 128 * 128 * 6 * pp * 2  # bf16 MMA work issued (upper tiles, 3-way split)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
out["tc_tflops"] = flops / out["tc_s"] / 1e12
out["tc_tensor_frac_of_bf16_peak"] = out["tc_tflops"] / peaks["bf16_tflops"]
out["tc_hbm_write_gbs"] = 8.0 * n * n / out["tc_s"] / 1e9
out["tc_hbm_frac"] = out["tc_hbm_write_gbs"] / peaks["hbm_gbs"]
out["speedup_vs_exact"] = out["exact_s"] / out["tc_s"]
print(json.dumps(out), flush=True)
