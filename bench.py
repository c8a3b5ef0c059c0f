#!/usr/bin/env python3
"""bench.py -- BASELINE.json's metric on the B200 engine (and the reference arm).

Metric: "Gini distance-matrix pairs/sec; stress iters/sec at n=20k,p=784,q=2
vs roofline".  Workload (BASELINE metric config = SURVEY 8(d) "metric" row):
n = 20000 rows, p = 784 features, fp32, image-like synthetic data (80% exact
zeros per row, the rest uniform over the 256 levels k/255 plus N(0, 0.1^2)
noise, clipped to [0, 1]; seeded numpy PCG64), nu = 2, q = 2.

One step = one full Gini distance matrix (n(n-1)/2 = 199,990,000 pairs, one
sort per pair) written as the packed fp32 triangle the fit consumes, followed
by S Kruskal stress iterations (Armijo gradient descent, seeded N(0, 0.1^2)
init, rel_tol 1e-300) on that matrix.
  value  = distance pairs/s (device-resident X, CUDA events on the launch stream)
  stress = stress iterations/s of the same step (reported beside value)
  e2e    = pairs/s through the drop-in C-ABI pairwise_matrix call
           (gmds_pairwise_gini: pinned host X in, host n x n fp64 D out;
           host<->device copies inside the timed region)

``--impl reference`` times the reference's own CPU implementation (the
UNMODIFIED reference core compiled by oracle/Makefile, all host threads) on a
bounded sample of the same workload.  Multi-GPU (torchrun): the pair tiles are
split across ranks (strong scaling, no collective on the data path); the fit
runs on each rank's share of D's packed blocks (gmds_dmat_gini_sharded) with one
in-stream NCCL all-reduce of [gradient | loss sums] per pass
(gmds_minimize_stress_sharded).  The timed regions are bracketed by a barrier and
the time is the max over ranks.  ``--gpus N`` without torchrun re-launches
itself under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, P, Q, NU = 20000, 784, 2, 2.0
NU_GENERAL = 2.5  # a weight outside the linear case (nu in {2, 3}), reported beside the headline
STRESS_ITERS = 50
SEED = 2605


def make_image_like(n, p, seed=SEED):
    """SURVEY 8(d) C3 generator: 80% exact zeros, 256 levels + N(0, 0.1^2) noise, clipped."""
    g = np.random.default_rng(seed)
    X = g.integers(0, 256, size=(n, p)).astype(np.float64) / 255.0
    X += g.normal(0.0, 0.1, size=(n, p))
    np.clip(X, 0.0, 1.0, out=X)
    X[g.random((n, p)) < 0.8] = 0.0
    return X.astype(np.float32)


def ops_per_pair(p, nnu):
    """p*ceil(log2 p) comparisons + p differences + 2*p*Nnu LUT FMAs."""
    return p * int(np.ceil(np.log2(p))) + p + 2 * p * nnu


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            t = json.load(f)
        g = lambda k: t[k]["dram_read_bytes"] + t[k]["dram_write_bytes"]
        return g("gini_gmd_kernel"), g("stress_tma_kernel_fused")
    except (OSError, KeyError, ValueError):
        return None, None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region, in-process
    through NVML (nvidia-ml-py) every 500 ms -- spawning nvidia-smi at 200 ms was
    measured to slow the distance kernel by ~10% on this box.  Falls back to
    nvidia-smi when NVML is unavailable."""

    def __init__(self, device_index=0, period=0.5):
        self.dev = device_index
        self.period = period
        self.samples = []
        self.max_mhz = None

    def __enter__(self):
        import threading

        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = {"hw_slowdown": getattr(N, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                    "sw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                    "hw_thermal_slowdown": getattr(N, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                    "sw_power_cap": getattr(N, "nvmlClocksThrottleReasonSwPowerCap", 0x4)}

            def run():
                while True:
                    try:
                        mhz = float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.samples.append((mhz, [k for k, b in bits.items() if r & b]))
                    except Exception:
                        pass
                    if self._stop.wait(self.period):
                        return

            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)

    def summary(self):
        sm = [m for m, _ in self.samples]
        reasons = sorted({x for _, rs in self.samples for x in rs})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(sm), "source": "nvml"}


# ---------------------------------------------------------------------------------------------------
# reference arm / cpu baseline


def reference_rate(X, seconds_target=12.0, threads=0):
    """Reference pairs/s on host cores: the UNMODIFIED reference per-pair code
    (gen_gini_distance under its own parallel_for) over a bounded block of rows.
    Falls back to the oracle restatement when oracle/_ref was not built."""
    from oracle import ref_lib

    L = ref_lib.load()
    n = X.shape[0]
    Xd = np.ascontiguousarray(X, dtype=np.float64)
    if L is not None:
        ref_lib.set_max_threads(threads)
        cores = ref_lib.max_threads()
        kind = "reference"
        # calibrate on one row per thread, then size the sample to ~seconds_target
        rows = max(1, cores)
        t0 = time.perf_counter()
        ref_lib.gini_rows(Xd, NU, 0, rows)
        dt = time.perf_counter() - t0
        per_pair = dt / sum(n - 1 - i for i in range(rows))
        want = int(seconds_target / per_pair)
        rows = max(cores, int(np.ceil(want / max(1, n - 1) / cores)) * cores)
        rows = min(rows, n - 1)
        pairs = sum(n - 1 - i for i in range(rows))
        t0 = time.perf_counter()
        ref_lib.gini_rows(Xd, NU, 0, rows)
        dt = time.perf_counter() - t0
        sample = f"rows 0..{rows - 1} of the n={n}, p={X.shape[1]} matrix ({pairs} pairs), reference gen_gini_distance"
        return pairs / dt, cores, kind, sample, dt
    from oracle import gini_oracle as O

    rows = 8
    I, J = [], []
    for i in range(rows):
        I.extend([i] * (n - 1 - i))
        J.extend(range(i + 1, n))
    I, J = np.array(I), np.array(J)
    t0 = time.perf_counter()
    O.gini_pairs(Xd, I, J, NU)
    dt = time.perf_counter() - t0
    return I.size / dt, 1, "port", f"rows 0..{rows - 1} ({I.size} pairs), numpy restatement", dt


def reference_stress_rate(seconds_cap=8.0):
    """Reference serial Kruskal iterate loop (embed.cpp:222-272): per-iteration
    time at n=2500 (on the reference's Euclidean distances of the same data --
    the iterate loop's cost does not depend on the metric that built D, and a
    Gini D at n=2500 would itself take ~40 s on the host), scaled to n=20000 by
    the pair count (each iteration is >= 3 O(n^2) passes); an extrapolation."""
    from oracle import ref_lib

    if ref_lib.load() is None:
        return None
    n_s = 2500
    Xs = make_image_like(n_s, P, seed=SEED + 1).astype(np.float64)
    D = ref_lib.pairwise_matrix(Xs, None)
    t0 = time.perf_counter()
    r = ref_lib.minimize_stress(D, Q, "kruskal", max_iters=3, rel_tol=1e-300)
    dt_with_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref_lib.classical_mds(D, Q)
    dt_init = time.perf_counter() - t0
    per_iter = max(1e-9, (dt_with_init - dt_init) / max(1, r["iterations"]))
    scale = (N * (N - 1)) / (n_s * (n_s - 1))
    return {"iters_per_sec": 1.0 / (per_iter * scale), "sample": f"3 Kruskal iterations at n={n_s} "
            f"({per_iter * 1e3:.1f} ms/iter), x{scale:.0f} pair-count extrapolation to n={N}", "cores": 1}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """The reference's own CPU path, W untimed + K timed steps; each step is the same bounded
    sample of the workload (a block of rows of the n x n matrix through the reference's
    gen_gini_distance under its parallel_for), sized so the whole run ends in a few minutes."""
    if rank != 0:
        return
    from oracle import ref_lib

    X = make_image_like(N, P)
    steps, warm = max(1, args.steps), max(0, args.warmup)
    per_step = min(8.0, max(1.0, 150.0 / (steps + warm)))
    rate0, cores, kind, sample, _ = reference_rate(X, seconds_target=per_step)  # calibration (untimed)
    rows = int(sample.split("rows 0..")[1].split(" ")[0]) + 1 if kind == "reference" else None
    Xd = np.ascontiguousarray(X, dtype=np.float64)
    pairs = sum(N - 1 - i for i in range(rows)) if rows else None
    times = []
    for k in range(warm + steps):
        if rows:
            t0 = time.perf_counter()
            ref_lib.gini_rows(Xd, NU, 0, rows)
            dt = time.perf_counter() - t0
        else:
            r, _, _, _, dt = reference_rate(X, seconds_target=per_step)
        if k >= warm:
            times.append(dt)
    rate = (pairs / float(np.mean(times))) if rows else rate0
    srate = reference_stress_rate()
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "pairs/s", "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": float(np.mean(times)) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "metric: n=20000 p=784 image-like fp32 (widened exactly to f64), nu=2, q=2",
                   "n": N, "p": P, "q": Q, "nu": NU},
        "cpu_baseline": {"value": rate, "unit": "pairs/s", "cores": cores, "cpu_model": cpu_model(), "kind": kind,
                         "sample": sample + f"; {warm} untimed + {steps} timed repetitions of this sample"},
        "e2e": {"value": rate, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_times_s": [round(t, 3) for t in times],
    }
    if srate:
        line["stress_iters_per_sec"] = srate["iters_per_sec"]
        line["stress_sample"] = srate["sample"]
        line["stress_cores"] = srate["cores"]
    print(json.dumps(line), flush=True)


METRIC = "Gini distance-matrix pairs/sec; stress iters/sec at n=20k,p=784,q=2 vs roofline"


# ---------------------------------------------------------------------------------------------------
# B200 arm


def run_engine(args, rank, world, dist):
    import torch

    from paper_2605_25124_b200 import gmds as G

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    G.lib().gmds_set_device(dev)
    stream = torch.cuda.current_stream()
    G.lib().gmds_set_stream(ctypes_void(stream.cuda_stream))

    X = make_image_like(N, P)
    dX = torch.from_numpy(X).cuda()
    npairs = N * (N - 1) // 2
    pe = G.packed_elems(N)
    dD = torch.zeros(pe, dtype=torch.float32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def distance_step():
        G.pairwise_gini_device(dX.data_ptr(), G.F32, N, P, [NU], G.F32, True, dD.data_ptr(), rank, world,
                               stream.cuda_stream)

    # ---- distance: warm-up, then K timed steps (L2 flushed between steps)
    for _ in range(args.warmup):
        distance_step()
    barrier()
    launches0 = G.launch_count()
    times = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            distance_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    barrier()
    dist_launches = G.launch_count() - launches0
    print(f"[bench] distance step times (ms): {[round(t * 1e3, 2) for t in times]}", file=sys.stderr, flush=True)
    t_dist = max_over_ranks(dist, float(np.mean(times)))

    # ---- the same step at a nu outside {2, 3} (general-weight kernel), reported beside `value`
    def general_step():
        G.pairwise_gini_device(dX.data_ptr(), G.F32, N, P, [NU_GENERAL], G.F32, True, dD.data_ptr(), rank, world,
                               stream.cuda_stream)

    general_step()
    gtimes = []
    for _ in range(2):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        general_step()
        e1.record(stream)
        e1.synchronize()
        gtimes.append(e0.elapsed_time(e1) / 1e3)
    t_general = max_over_ranks(dist, float(np.mean(gtimes)))

    # ---- stress: S Kruskal iterations on the packed matrix of this step.  One GPU: the
    # device-controlled fit.  Several ranks: the row-sharded device-controlled fit of libgmds.
    Y0 = np.random.default_rng(SEED).normal(0.0, 0.1, (N, Q))
    # GMDS_BENCH_SHARDED=1 runs the multi-GPU code path at one rank too (a 1-rank NCCL
    # communicator): the glue below is then exercised on a single-GPU box
    if world > 1 or os.environ.get("GMDS_BENCH_SHARDED"):
        # libgmds multi-GPU path: an NCCL communicator (unique id shared over torch.distributed),
        # this rank's share of D's packed blocks, and the device-resident sharded fit with one
        # in-stream all-reduce of [gradient | loss sums] per pass
        uid = [G.comm_unique_id() if rank == 0 else None]
        if dist is not None:
            dist.broadcast_object_list(uid, src=0)
        comm = G.comm_init_nccl(uid[0], world, rank)
        Dm = G.dmat_gini_sharded(comm, dX.data_ptr(), G.F32, N, P, NU, G.F32)

        def fit(iters):
            return G.minimize_stress_sharded(comm, Dm, Y0, "kruskal", max_iters=iters, rel_tol=1e-300)
    else:
        comm = None
        Dm = G.dmat_gini_device(dX.data_ptr(), G.F32, N, P, NU, G.F32)

        def fit(iters):
            return G.minimize_stress(Dm, Q, "kruskal", max_iters=iters, rel_tol=1e-300, Y0=Y0)
    fit(2)  # warm-up
    barrier()
    launches1 = G.launch_count()
    stimes, siters, spasses = [], 0, 0
    with ClockSampler(dev) as clk2:
        for _ in range(max(1, args.steps)):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r = fit(STRESS_ITERS)
            e1.record(stream)
            e1.synchronize()
            stimes.append(e0.elapsed_time(e1) / 1e3)
            siters += r["iterations"]
            spasses += r["passes"]
    stress_launches = G.launch_count() - launches1
    print(f"[bench] stress step times (ms): {[round(t * 1e3, 2) for t in stimes]}", file=sys.stderr, flush=True)
    t_stress = max_over_ranks(dist, float(np.sum(stimes)))
    iters_per_sec = siters / t_stress
    # steady-state rate: iterations 51-100 of the same (deterministic) fit, as the difference
    # of a 100- and the 50-iteration run -- by then every step is above fp32 storage's
    # resolution (no difference passes); reported beside the headline rate
    resolved = None
    if True:
        def timed_fit(iters):
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rr = fit(iters)
            e1.record(stream)
            e1.synchronize()
            return e0.elapsed_time(e1) / 1e3, rr

        t100, r100 = timed_fit(2 * STRESS_ITERS)
        t50, r50 = timed_fit(STRESS_ITERS)
        t100, t50 = max_over_ranks(dist, t100), max_over_ranks(dist, t50)
        if r100["iterations"] == 2 * STRESS_ITERS and t100 > t50:
            resolved = {"iters_per_sec": STRESS_ITERS / (t100 - t50), "ms_per_iter": 1e3 * (t100 - t50) / STRESS_ITERS,
                        "passes_per_iter": (r100["passes"] - r50["passes"]) / STRESS_ITERS,
                        "iterations": "51-100 of the fit (t(100) - t(50))"}
    Dm.free()
    if comm is not None:
        comm.free()

    # ---- e2e: the drop-in pairwise_matrix call, pinned host X -> host fp64 n x n D
    e2e = None
    if world == 1 and not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory().numpy()
        Dh = torch.empty((1, N, N), dtype=torch.float64).pin_memory().numpy()
        etimes = []
        G.lib().gmds_set_stream(ctypes_void(0))

        def e2e_call():
            G.lib().gmds_pairwise_gini(G._vp(Xh), G._i32(G.F32), G._i32(G.ROW_MAJOR), G._i64(N), G._i64(P),
                                       G._p(np.array([NU])), G._i32(1), G._i32(G.F64), G._vp(Dh))

        for _ in range(max(1, min(args.warmup, 2))):  # untimed warm-up (first call maps the output buffers)
            e2e_call()
        for k in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            e2e_call()
            etimes.append(time.perf_counter() - t0)
        e2e = {"value": npairs / float(np.mean(etimes)), "unit": "pairs/s", "h2d_bytes_per_step": int(X.nbytes),
               "d2h_bytes_per_step": int(Dh.nbytes), "ms_per_step": float(np.mean(etimes)) * 1e3,
               "call": "gmds_pairwise_gini (pairwise_matrix drop-in, fp64 n x n out)"}
        del Dh
        # the same call as a C++ caller of the reference API makes it (tools/cpp/facade_e2e.cpp):
        # const Matrix& D = ginimds::pairwise_matrix(X, MetricSpec::gini(2)).matrix(); X an Eigen-layout
        # (column-major) fp64 matrix, D the facade's own (pageable) host Matrix
        try:
            import ctypes

            Lf = ctypes.CDLL(os.path.join(ROOT, "paper_2605_25124_b200", "lib", "libfacade_e2e.so"))
            Xcm = np.asfortranarray(X.astype(np.float64))
            secs, chk = ctypes.c_double(), ctypes.c_double()

            def facade_call():
                rc = Lf.facade_e2e(ctypes.c_void_p(Xcm.ctypes.data), ctypes.c_int64(N), ctypes.c_int64(P),
                                   ctypes.c_double(NU), ctypes.byref(secs), ctypes.byref(chk))
                if rc != 0:
                    raise RuntimeError("facade_e2e failed")
                return secs.value

            facade_call()  # warm-up (pinned staging, pool)
            ftimes = [facade_call() for _ in range(max(1, min(args.steps, 3)))]
            e2e["facade"] = {"value": npairs / float(np.mean(ftimes)), "unit": "pairs/s",
                             "ms_per_step": float(np.mean(ftimes)) * 1e3, "h2d_bytes_per_step": int(Xcm.nbytes),
                             "d2h_bytes_per_step": int(8 * N * N),
                             "call": "ginimds::pairwise_matrix(X, MetricSpec::gini(2)).matrix() (C++ facade, "
                                     "fp64 column-major X, host Matrix D)"}
        except (OSError, RuntimeError) as ex:
            e2e["facade"] = {"unavailable": str(ex)}
        G.lib().gmds_set_stream(ctypes_void(stream.cuda_stream))

    # ---- roofline of the dominant kernel (gini_gmd_kernel: the whole distance step is this kernel
    # plus a 12 KB LUT upload and two 4-byte flag copies).  Peak: the NOMINAL FP32/INT32 lane-op
    # rate (SMs x 128 lanes x max SM clock; MEASURED_PEAKS.json has no ALU figure); the probe's
    # measured rate is reported beside it
    alu = ctypes_double()
    G.lib().gmds_probe_alu(ctypes_ref(alu))
    props = torch.cuda.get_device_properties(dev)
    sm_max = clk.summary().get("sm_max_mhz") or 1965.0
    alu_nominal = props.multi_processor_count * 128 * sm_max * 1e6 * world  # whole job
    ops_pair = ops_per_pair(P, 1)
    my_pairs = npairs  # all ranks together
    achieved = my_pairs * ops_pair / t_dist
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0) * world  # whole job: every rank streams its share of D
    traffic_dist, traffic_stress = load_traffic()
    # stress: unit = one iteration; algorithmic bytes = one read of the packed fp32
    # triangle (n(n-1)/2 x 4 B) per iteration, whatever the passes per iteration
    bytes_iter = npairs * 4
    ms_iter = 1e3 / iters_per_sec
    ach_iter = bytes_iter / (ms_iter * 1e-3) / 1e9
    value = npairs / t_dist
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": (t_dist + t_stress / max(1, args.steps)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy PCG64, SURVEY 8(d) image-like generator)",
        "config": {"workload": "metric: n=20000 p=784 q=2 nu=2 (BASELINE metric config; C3 generator at n=20k)",
                   "n": N, "p": P, "q": Q, "nu": NU, "input_dtype": "f32", "D_storage": "f32 packed triangle",
                   "stress_iters_per_step": STRESS_ITERS, "stress_kind": "kruskal (Armijo GD)",
                   "init": "seeded N(0, 0.1^2) (SURVEY F4)", "l2": "flushed (256 MB write) before every "
                   "distance step; the packed D (800 MB) exceeds L2 for the stress passes",
                   "parallelism": f"dp{world}: distance pair tiles and the fit's packed blocks sharded over {world} GPU(s), one NCCL all-reduce per stress pass"},
        "distance_ms": t_dist * 1e3,
        "distance_general_nu": {"nu": NU_GENERAL, "ms": t_general * 1e3, "pairs_per_s": npairs / t_general,
                                "kernel": "gini_gen2_kernel (midranks counted, one LUT pass)",
                                "alu_frac_of_nominal": npairs * ops_pair / t_general / alu_nominal},
        "stress_iters_per_sec": iters_per_sec,
        "stress_resolved_steps": resolved,
        "stress_ms_per_iter": ms_iter,
        "stress_passes_per_iter": spasses / max(1, siters),
        "gpu_launches": int(dist_launches + stress_launches),
        "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": alu_nominal / 1e12, "unit": "Tops/s",
                     "frac": achieved / alu_nominal, "traffic": traffic_dist, "traffic_unit": "bytes/launch (ncu)",
                     "kernel": "gini_gmd2_kernel (nu = 2: linear-weight path)", "ops_per_pair": ops_pair,
                     "peak_source": f"nominal: {props.multi_processor_count} SMs x 128 lanes x {sm_max:.0f} MHz "
                                    "(MEASURED_PEAKS.json has no ALU figure)",
                     "probe_peak": alu.value / 1e12, "frac_of_probe": achieved / alu.value,
                     "probe_source": "gmds_probe_alu on this GPU (FFMA + IADD3/LOP3 lane-op rate)"},
        "stress_roofline": {"bound": "hbm", "unit": "GB/s", "peak": hbm,
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs" + (" (fallback)" if peaks.get("fallback") else ""),
                            "bytes_per_iter": bytes_iter,
                            "achieved": ach_iter, "frac": ach_iter / hbm,
                            "iterations": f"1-{STRESS_ITERS} of the fit (the bench's stress step)",
                            "traffic": traffic_stress, "kernel": "stress_tma_multi_kernel<2,1> fused body (+ reductions, gd_step)"},
        "clocks": clk.summary(),
        "clocks_stress": clk2.summary(),
    }
    if resolved:
        a2 = bytes_iter / (resolved["ms_per_iter"] * 1e-3) / 1e9
        line["stress_roofline"]["resolved"] = {"achieved": a2, "frac": a2 / hbm,
                                               "iterations": resolved["iterations"]}
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, kind, sample, _ = reference_rate(X, seconds_target=10.0)
        line["cpu_baseline"] = {"value": rate, "unit": "pairs/s", "cores": cores, "cpu_model": cpu_model(),
                                "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)


def ctypes_void(v):
    import ctypes

    return ctypes.c_void_p(v)


def ctypes_double():
    import ctypes

    return ctypes.c_double()


def ctypes_ref(x):
    import ctypes

    return ctypes.byref(x)


def max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:  # self-launch N ranks, one per GPU
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist_mod

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist_mod.init_process_group("nccl")
        dist = dist_mod
    try:
        run_engine(args, rank, world, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
