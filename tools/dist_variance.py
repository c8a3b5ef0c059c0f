"""Diagnose run-to-run variance of the metric distance step: K timed steps
with CUDA events and per-phase host traces, while nvidia-smi logs clocks,
power and throttle reasons every 100 ms."""
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_image_like, N, P  # noqa: E402
from paper_2605_25124_b200 import gmds as G  # noqa: E402


def main():
    import torch

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/smi_log.csv"
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                            "clocks_throttle_reasons.active", "--format=csv", "-lms", "100"],
                           stdout=open(out, "w"), stderr=subprocess.DEVNULL)
    X = make_image_like(N, P)
    dX = torch.from_numpy(X).cuda()
    dD = torch.zeros(G.packed_elems(N), dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for k in range(steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(st)
        G.pairwise_gini_device(dX.data_ptr(), G.F32, N, P, [2.0], G.F32, True, dD.data_ptr(), 0, 1, st.cuda_stream)
        e1.record(st)
        e1.synchronize()
        print(f"step {k}: events {e0.elapsed_time(e1):.1f} ms, wall {1e3 * (time.perf_counter() - t0):.1f} ms "
              f"t={time.time():.2f}", flush=True)
    smi.terminate()


if __name__ == "__main__":
    main()
