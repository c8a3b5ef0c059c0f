"""Facade e2e (ginimds::pairwise_matrix(X, gini(2)).matrix() from C++, tools/cpp/facade_e2e.cpp) at the
metric shape, with the download's huge-page hint / populate threads (GMDS_PREFAULT=huge|pop|both)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import make_image_like  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N, P = 20000, 784
X = make_image_like(N, P)
Xcm = np.asfortranarray(X.astype(np.float64))
Lf = ctypes.CDLL(os.path.join(ROOT, "paper_2605_25124_b200", "lib", "libfacade_e2e.so"))
Lf.facade_e2e.restype = ctypes.c_int
cs, secs = ctypes.c_double(0.0), ctypes.c_double(0.0)


def call():
    rc = Lf.facade_e2e(ctypes.c_void_p(Xcm.ctypes.data), ctypes.c_int64(N), ctypes.c_int64(P), ctypes.c_double(2.0),
                       ctypes.byref(secs), ctypes.byref(cs))
    assert rc == 0
    return secs.value


call()
for mode in ("none", "huge", "pop", "both", "none"):
    if mode == "none":
        os.environ.pop("GMDS_PREFAULT", None)
    else:
        os.environ["GMDS_PREFAULT"] = mode
    ts = [call() for _ in range(3)]
    print(f"{mode}: {np.mean(ts) * 1e3:.1f} ms  ({N * (N - 1) / 2 / np.mean(ts) / 1e6:.0f} M pairs/s)  checksum {cs.value:.6g}", flush=True)
