#!/usr/bin/env python
"""Benchmark of the B200 structured-sketch apply (BASELINE.json metric: sketch input GB/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference] [--config cfg2]

One step = one pass of the hot path over one config-sized batch of synthetic input already
resident in HBM (config 2 by default: the SRTT sketch Y = A*Omega of a 65536 x 8192 float32 A,
2 GiB, larger than the 126 MB L2, so no flush is needed between steps).  Under torchrun every
rank processes its own batch (row blocks of a N*65536-row matrix; no collective on the data path)
and `value` = all ranks' input bytes / the max-over-ranks device time ("scaling": "weak").

`--impl reference` times the reference algorithm on the host (the CPU oracle port in oracle/,
which restates sketchkit's NumPy/SciPy path) on a bounded row sample with every host core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sketch input GB/s (% of HBM peak) for sparse/SRTT/KR Y=AΩ, 1–8 B200"
FALLBACK_HBM_GBS = 6650.0


# ---------------------------------------------------------------------------------------------
# workloads (BASELINE.json configs; synthetic inputs with the configs' shapes and distributions)
# ---------------------------------------------------------------------------------------------
def _cfg2(torch, dev, rank):
    from paper_2508_21189_b200.sketch import SparseRttTM

    n, d, k = 65536, 8192, 512
    make = lambda: SparseRttTM(d, k, 1, "wht", seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    a /= torch.arange(1, d + 1, dtype=torch.float32, device=dev)  # sigma_j = 1/j
    return dict(name="cfg2", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=1, kernel="srtt_wht_tc",
                workload="cfg2 SRTT sketch Y=A*D*H*S: A 65536x8192 f32 (sigma_j=1/j), WHT d=8192, k=512, xi=1",
                op="right")


def _cfg1(torch, dev, rank):
    from paper_2508_21189_b200.sketch import SparseUniformTM

    n, d, k = 16384, 4096, 256
    make = lambda: SparseUniformTM(d, k, 4, seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(2000 + rank)
    a = torch.randn(n, d, dtype=torch.float64, device=dev, generator=g)
    return dict(name="cfg1", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=1, kernel="sparse_right_cols_kernel",
                workload="cfg1 sparse sign Y=A*Omega: A 16384x4096 f64, zeta=4, k=256", op="right")


def _cfg3(torch, dev, rank):
    from paper_2508_21189_b200.sketch import SparseUniformTM

    n, d, k = 131072, 16384, 200
    make = lambda: SparseUniformTM(d, k, 8, seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(3000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    return dict(name="cfg3", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=1, kernel="dense_tc_pair_kernel<1,0,0> (sparse sign as exact bf16 Omega^T)",
                workload="cfg3 RSVD sketch Y=A*Omega: A 131072x16384 f32 (iid input for throughput), zeta=8, k=200",
                op="right")


def _cfg4(torch, dev, rank):
    from paper_2508_21189_b200.sketch import SparseUniformTM

    n, d, k = 4194304, 512, 2048
    make = lambda: SparseUniformTM(n, k, 8, seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(4000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    # rows scaled by 1 + Pareto(1.5) weights (coherent rows, as the config states; inverse CDF)
    a *= (torch.rand(n, 1, device=dev, generator=g).clamp_min(1e-12) ** (-1.0 / 1.5))
    return dict(name="cfg4", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=2, kernel="sparse_adjoint_gather",
                workload="cfg4 SA sketch: S (2048 x 4194304, zeta=8) applied to A 4194304x512 f32", op="adjoint")


def _cfg5(torch, dev, rank):
    from paper_2508_21189_b200.sketch import KhatriRaoTM

    n, d, k = 16384, 65536, 512
    make = lambda: KhatriRaoTM(256, 2, k, "real_rademacher", seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(5000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    return dict(name="cfg5", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=None, kernel="dense_tc_pair_kernel<1,0,1> (sk_kr_right_signs: F resident, +-1 weights as sign bits, Omega never formed)",
                flops=2.0 * n * d * k, flops_executed_x=2,
                workload="cfg5 Khatri-Rao sketch: A 16384x65536 f32, ell=2, d0=256, k=512", op="right")


def _gauss(torch, dev, rank):
    """Gaussian Omega at the config-3 sketch shape: the dense tcgen05 GEMM kept as the tensor-core
    reference (north star); Omega's float64 draws split into bf16 hi + lo, A into hi + lo (BF16x3)."""
    from paper_2508_21189_b200.sketch import GaussianTM

    n, d, k = 131072, 16384, 200
    make = lambda: GaussianTM(d, k, seed=0)  # noqa: E731
    tm = make()
    g = torch.Generator(device=dev).manual_seed(6000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    return dict(name="gauss", tm=tm, make=make, a=a, n=n, d=d, k=k, launches=1,
                kernel="dense_tc_pair_kernel<2> (Gaussian Omega, BF16x3)", flops=2.0 * n * d * k, flops_executed_x=3,
                workload="Gaussian Y=A*Omega at the cfg3 shape: A 131072x16384 f32, k=200", op="right")


def _cfg2dct(torch, dev, rank):
    """Config 2's shape with the reference's DEFAULT real-field transform (DCT, rtt.py:92-93)."""
    from paper_2508_21189_b200.sketch import SparseRttTM

    w = _cfg2(torch, dev, rank)
    make = lambda: SparseRttTM(8192, 512, 1, "dct", seed=0)  # noqa: E731
    w.update(name="cfg2dct", tm=make(), make=make, kernel="dense_tc_pair_kernel<2,0,0> (materialised D C^T S, BF16x3)",
             workload="cfg2 shape with the DCT SRTT (reference default transform): A 65536x8192 f32, k=512, xi=1")
    return w


def _twosided(torch, dev, rank):
    """The generalized-Nystrom sketch stage at DESIGN's shape: Y = A Omega and
    X = A^T Psi from one read of A on the fused kernel."""
    from paper_2508_21189_b200.sketch import SparseRttTM, SparseUniformTM

    n, d, k, p = 1 << 21, 512, 64, 96
    g = torch.Generator(device=dev).manual_seed(7000 + rank)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)
    make = lambda: (SparseRttTM(d, k, 1, "wht", seed=1), SparseUniformTM(n, p, 8, seed=2))  # noqa: E731
    return dict(name="twosided", tm=make(), make=make, a=a, n=n, d=d, k=k, p=p, launches=2,
                kernel="two_sided_kernel", op="twosided",
                workload="two-sided sketch: A 2097152x512 f32, Omega SRTT (k=64), Psi sparse sign (p=96, zeta=8)")


WORKLOADS = {"cfg1": _cfg1, "cfg2": _cfg2, "cfg3": _cfg3, "cfg4": _cfg4, "cfg5": _cfg5, "gauss": _gauss,
             "cfg2dct": _cfg2dct, "twosided": _twosided}


def _apply(w, x):
    if w["op"] == "twosided":
        from paper_2508_21189_b200 import rand_nla

        om, ps = w["tm"]
        return rand_nla.two_sided_sketch(x, om, ps)
    return w["tm"].apply_right(x) if w["op"] == "right" else w["tm"].apply_adjoint(x)


def _bytes(w, dtype_size):
    a_bytes = w["n"] * w["d"] * dtype_size
    if w["op"] == "twosided":
        out_elems = w["n"] * w["k"] + w["p"] * w["d"]
    else:
        out_elems = w["n"] * w["k"] if w["op"] == "right" else w["k"] * w["d"]
    return a_bytes, a_bytes + out_elems * dtype_size


# ---------------------------------------------------------------------------------------------
# clocks sampling during the timed region
# ---------------------------------------------------------------------------------------------
class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML every 5 ms while the timed region runs."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self.error = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        except Exception as exc:  # noqa: BLE001 - reported in the JSON
            self.error = f"{type(exc).__name__}: {exc}"
        return self

    def _run(self):
        nv = self._nvml
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                try:
                    rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                except AttributeError:
                    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                self.samples.append((mhz, rs))
            except Exception as exc:  # noqa: BLE001
                self.error = f"{type(exc).__name__}: {exc}"
                return
            self._stop.wait(0.005)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "error": self.error}
        reasons = sorted({nm for _, rs in self.samples for nm, bit in self.REASONS if rs & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML, 5 ms period"}


# ---------------------------------------------------------------------------------------------
def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def _traffic(name):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(name)
        return None if ent is None else float(ent["bytes_per_launch"])
    except (OSError, ValueError, KeyError, TypeError):
        return None


def _dist(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # one process per GPU; SKETCH_B200_DIST_BACKEND=gloo + fewer GPUs than ranks is a functional
        # dry run only (ranks then share a device: NCCL refuses duplicate GPUs)
        dev_idx = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev_idx)
        backend = os.environ.get("SKETCH_B200_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return world, rank, local


def _backend():
    import torch.distributed as dist

    return dist.get_backend() if dist.is_available() and dist.is_initialized() else "none"


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(world, value, dev):
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def time_device(torch, w, steps, warmup, world, dev):
    """Device-timed steps (CUDA events on the launching stream); returns (total_s, per-step list)."""
    a = w["a"]
    for _ in range(warmup):
        _apply(w, a)
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    start_all = torch.cuda.Event(enable_timing=True)
    end_all = torch.cuda.Event(enable_timing=True)
    start_all.record(stream)
    for i in range(steps):
        ev[i][0].record(stream)
        _apply(w, a)
        ev[i][1].record(stream)
    end_all.record(stream)
    torch.cuda.synchronize()
    _barrier(world)
    torch.cuda.synchronize()
    per = [s.elapsed_time(e) / 1e3 for s, e in ev]
    total = start_all.elapsed_time(end_all) / 1e3
    return total, per


def _downstream(torch, w, dev):
    """The config's downstream pipeline on the same input (warm, wall clock around a synchronized
    call): config 3 rsvd (sketch, orth, Q^T A, SVD), config 4 sketch-and-precondition LSQR and
    sketch-and-solve, the two-sided leg's generalized Nystrom SVD (the paper's headline application)."""
    from paper_2508_21189_b200 import rand_nla

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        return out, (time.perf_counter() - t0) * 1e3

    if w["name"] == "cfg3":
        # the config's A = U diag(i^-2) V^T (Haar U, V: QR of Gaussians with the diag(R) sign fix),
        # truncated to its leading r = 2048 terms (the dropped tail is 6e-6 of ||A||_F), written over
        # the throughput input: the SVD stage's cost depends on the spectrum, so time it on the real one
        a = w["a"]
        n, d, r = a.shape[0], a.shape[1], 2048
        g = torch.Generator(device=dev).manual_seed(3333)

        def haar(rows):
            q, rr = torch.linalg.qr(torch.randn(rows, r, device=dev, dtype=torch.float32, generator=g))
            return q * torch.sign(rr.diagonal())[None, :]

        u, v = haar(n), haar(d)
        sig = torch.arange(1, r + 1, device=dev, dtype=torch.float32) ** -2.0
        with rand_nla._no_tf32():
            torch.matmul(u * sig[None, :], v.T, out=a)
        del u, v
        fac, ms = timed(lambda: rand_nla.rsvd(a, w["k"], w["tm"]))
        res = rand_nla.rsvd_residual(a, fac)
        s2 = sig.double() ** 2
        best = float(torch.sqrt(s2[w["k"]:].sum() / s2.sum()))
        return {"rsvd_ms": ms, "residual_rel_fro": res, "best_rank_k_residual": best,
                "input": "A = U diag(i^-2) V^T, Haar U (131072 x 2048), V (16384 x 2048), seed 3333",
                "what": "rank-200 rsvd of A (sketch, CholeskyQR2, Q^T A on the tensor cores, SVD); ||A - QB||_F / ||A||_F"}
    if w["name"] == "cfg4":
        a = w["a"]
        g = torch.Generator(device=dev).manual_seed(4444)
        x0 = torch.randn(a.shape[1], device=dev, dtype=torch.float64, generator=g)
        b = (rand_nla._matvec_blocks(a, x0, 0) + 1e-3 * torch.randn(a.shape[0], device=dev, dtype=torch.float64,
                                                                      generator=g)).float()
        res, ms = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, w["tm"], atol=1e-6, btol=0.0))
        _, ms_ss = timed(lambda: rand_nla.sketch_and_solve(a, b, w["tm"]))
        return {"lsqr_ms": ms, "iterations": res.itn, "istop": res.istop, "sketch_and_solve_ms": ms_ss,
                "what": "sketch-and-precondition LSQR to the 1e-6 normal-equation test (SA, QR(SA), LSQR on A R^-1); "
                        "sketch-and-solve (SA, Sb, truncated pseudo-inverse)"}
    if w["name"] == "twosided":
        om, ps = w["tm"]
        fac, ms = timed(lambda: rand_nla.gen_nystrom_svd(w["a"], w["k"], w["p"], om, ps))
        return {"gen_nystrom_svd_ms": ms, "rank": int(fac.sigma.numel()),
                "what": "generalized Nystrom in SVD form (two-sided sketch, QR of Y and of X, the core SVDs) on the leg's A"}
    return None


def time_setup(torch, w, steady_s):
    """Operator construction + device encoding/upload, reported apart from the apply:
    a fresh operator's first apply on the step's input minus one steady apply."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    y = _apply(dict(w, tm=w["make"]()), w["a"])
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    del y
    return {"ms": max(0.0, first - steady_s) * 1e3, "first_call_ms": first * 1e3,
            "what": "constructor draws + device encoding and upload of Omega (first apply minus a steady apply)"}


def time_e2e(torch, w, steps, world, dev):
    """Through the public API with pinned HOST buffers: H2D of A, kernel, D2H of Y, every step."""
    a_host = torch.empty(w["a"].shape, dtype=w["a"].dtype, pin_memory=True)
    a_host.copy_(w["a"])
    for _ in range(3):  # warm-up of the host path: device chunk buffers and the two pinned result
        y = _apply(w, a_host)  # blocks the caching host allocator alternates between steps
    torch.cuda.synchronize()
    _barrier(world)
    t0 = time.perf_counter()
    marks = []
    for _ in range(steps):
        y = _apply(w, a_host)  # returns after the D2H of the step's result has completed
        marks.append(time.perf_counter())
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    el = _max_over_ranks(world, el, dev)
    h2d = a_host.numel() * a_host.element_size()
    d2h = y.numel() * y.element_size()
    del a_host
    step_ms = [1e3 * (b - a) for a, b in zip([t0] + marks[:-1], marks)]
    return el, h2d, d2h, step_ms


def cpu_reference_step(w, a_host, procs):
    """The reference algorithm (oracle port) on host rows `a_host`."""
    import oracle as orc

    name = w["name"]
    tm = w["tm"]
    if name in ("cfg2", "cfg2dct"):
        dv, samp = orc.srtt_parts(tm.d, tm.k, tm.xi, tm.seed)
        fn = lambda x: orc.srtt_right(dv, samp, x, tm.transform)  # noqa: E731
    elif name == "twosided":  # the Y = A Omega half on the sample rows (X needs every row of A)
        om = tm[0]
        dv, samp = orc.srtt_parts(om.d, om.k, om.xi, om.seed)
        fn = lambda x: orc.srtt_right(dv, samp, x, "wht")  # noqa: E731
    elif name in ("cfg1", "cfg3"):
        om = orc.sparse_uniform_csr(tm.d, tm.k, tm.zeta, tm.seed)
        fn = lambda x: orc.csr_right(om, x)  # noqa: E731
    elif name == "cfg5":
        f = orc.kr_factors(tm.d0, tm.ell, tm.k, tm.seed, tm.base)
        fn = lambda x: orc.kr_right(f, x)  # noqa: E731
    elif name == "gauss":  # the reference: a dense float64 GEMM with its Omega (gaussian.py:19-30)
        om = orc.gaussian_dense(tm.d, tm.k, tm.seed)
        fn = lambda x: orc.dense_right(om, x)  # noqa: E731
    elif name == "cfg4":  # S A restricted to the sample rows: Omega[:rows]^T A[:rows] (scipy, one core)
        csr = _cfg4_csr(tm)[: a_host.shape[0]]
        t0 = time.perf_counter()
        y = orc.csr_adjoint(csr, a_host)
        return time.perf_counter() - t0, y
    else:
        raise ValueError(name)
    t0 = time.perf_counter()
    y = orc.right_multiprocess(fn, a_host, procs=procs, rows=max(1, a_host.shape[0] // (4 * procs)))
    return time.perf_counter() - t0, y


_CSR_CACHE = {}


def _cfg4_csr(tm):
    import oracle as orc

    key = (tm.d, tm.k, tm.zeta, tm.seed)
    if key not in _CSR_CACHE:
        _CSR_CACHE[key] = orc.sparse_uniform_csr(*key)
    return _CSR_CACHE[key]


def sample_parity(w, procs):
    """(cpu_baseline dict, rel-F error of the GPU result vs the oracle) on the config's row sample."""
    rows = SAMPLE_ROWS[w["name"]]
    a_host = w["a"][:rows].cpu().numpy()
    dt, y_ref = cpu_reference_step(w, a_host, procs)
    if w["op"] == "right":
        y_gpu = _apply(w, w["a"][:rows]).double().cpu().numpy()
    elif w["op"] == "twosided":
        y_gpu = _apply(w, w["a"][:rows])[0].double().cpu().numpy()
    else:  # the row block of S that multiplies the sample rows (device-sliced draws)
        y_gpu = w["tm"].row_block(0, rows).apply_adjoint(w["a"][:rows]).double().cpu().numpy()
    err = float(np.linalg.norm(y_gpu - y_ref) / np.linalg.norm(y_ref))
    cores = procs if w["op"] in ("right", "twosided") else 1
    cpu = {"value": a_host.nbytes / dt / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
           "sample": f"{rows} rows of the {w['name']} input ({a_host.nbytes / 1e6:.0f} MB), oracle/ port of the "
                     f"sketchkit float64 path" + (f", row-parallel over {procs} processes" if cores > 1 else
                                                  ", scipy sparse on one core (as the reference)"),
           "parity_rel_fro_err_vs_gpu": err}
    return cpu, err


SAMPLE_ROWS = {"cfg1": 4096, "cfg2": 2048, "cfg3": 512, "cfg4": 1 << 18, "cfg5": 16, "cfg2dct": 1024,
               "twosided": 8192, "gauss": 2048}


def run_reference(args):
    """--impl reference: the reference's CPU algorithm (oracle port) on all host cores, rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch

    procs = os.cpu_count() or 1
    w = WORKLOADS[args.config](torch, torch.device("cpu") if not torch.cuda.is_available() else torch.device("cuda", 0), 0)
    rows = SAMPLE_ROWS[args.config]
    a_host = w["a"][:rows].cpu().numpy()
    del w["a"]
    a_bytes_row = w["d"] * a_host.itemsize
    times = []
    for i in range(args.warmup + args.steps):
        dt, _ = cpu_reference_step(w, a_host, procs)
        if i >= args.warmup:
            times.append(dt)
    med = statistics.median(times)
    value = rows * a_bytes_row / med / 1e9
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": med * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if a_host.dtype == np.float32 else "f64", "data": "synthetic",
        "config": {"workload": w["workload"], "rows_per_step": rows, "parallelism": f"{procs} host processes"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": procs, "kind": "port",
                         "sample": f"{rows} rows of the {args.config} input per step (oracle/ port of sketchkit, "
                                   f"float64 NumPy/SciPy, row-parallel over {procs} processes)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def measure_sharded_sa(torch, world, rank, dev, steps=5, warmup=3):
    """Config 4 SA over row shards with the NCCL all-reduce of the partials.

    Strong scaling: the 4194304-row A is split into `world` row blocks; rank g holds its block
    and the matching rows of Omega (`SparseRowBlockTM`), runs K2g on them and the 2048 x 512
    float64 partials are summed by one all-reduce (`dist.sharded_adjoint`).  Timed on the device
    (events on the launching stream, barrier on both sides, max over ranks), all-reduce included;
    the all-reduce alone is timed the same way and reported apart.
    """
    from paper_2508_21189_b200 import dist as skd
    from paper_2508_21189_b200.sketch import SparseUniformTM

    n, d, k = 4194304, 512, 2048
    r0, r1 = skd.row_range(n, world, rank)
    tm = SparseUniformTM(n, k, 8, seed=0)
    g = torch.Generator(device=dev).manual_seed(4000 + rank)
    a = torch.randn(r1 - r0, d, dtype=torch.float32, device=dev, generator=g)
    a *= (torch.rand(r1 - r0, 1, device=dev, generator=g).clamp_min(1e-12) ** (-1.0 / 1.5))
    step = lambda: skd.sharded_adjoint(tm, a, r0)  # noqa: E731
    part = step()  # builds the row block's device encoding (setup, untimed)

    def timed(fn):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        _barrier(world)
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        _barrier(world)
        return _max_over_ranks(world, e0.elapsed_time(e1) / 1e3 / steps, dev)

    t_step = timed(step)
    t_ar = timed(lambda: skd.allreduce_sum(part))
    out = {"workload": f"cfg4 SA, A 4194304x512 f32 split into {world} row block(s), all-reduce ({_backend()}) of the "
                       "2048x512 float64 partials", "scaling": "strong",
           "value_gbs": n * d * 4 / t_step / 1e9, "ms_per_step": t_step * 1e3, "allreduce_ms": t_ar * 1e3,
           "rows_per_gpu": r1 - r0, "allreduce_bytes": part.numel() * part.element_size()}
    del a, part
    torch.cuda.empty_cache()
    return out


def measure_strong_cfg2(torch, world, rank, dev, steps=10, warmup=3):
    """Config 2 with the 65536-row A split across the ranks (strong scaling: 65536 / N rows each,
    no collective); device time max over ranks."""
    from paper_2508_21189_b200 import dist as skd
    from paper_2508_21189_b200.sketch import SparseRttTM

    n, d, k = 65536, 8192, 512
    r0, r1 = skd.row_range(n, world, rank)
    tm = SparseRttTM(d, k, 1, "wht", seed=0)
    g = torch.Generator(device=dev).manual_seed(1000)
    a = torch.randn(n, d, dtype=torch.float32, device=dev, generator=g)[r0:r1].contiguous()
    a /= torch.arange(1, d + 1, dtype=torch.float32, device=dev)
    w = dict(tm=tm, a=a, op="right")
    total, _ = time_device(torch, w, steps, warmup, world, dev)
    total = _max_over_ranks(world, total, dev)
    out = {"workload": f"cfg2 SRTT, A 65536x8192 f32 split into {world} row block(s) of ~{r1 - r0} rows",
           "scaling": "strong", "value_gbs": n * d * 4 * steps / total / 1e9, "ms_per_step": total / steps * 1e3,
           "rows_per_gpu": r1 - r0}
    del a
    torch.cuda.empty_cache()
    return out


def measure(torch, w, steps, warmup, world, rank, dev, with_e2e, clocks_idx):
    a = w["a"]
    esize = a.element_size()
    a_bytes, alg_bytes = _bytes(w, esize)
    with ClockSampler(clocks_idx) as cs:
        total, per = time_device(torch, w, steps, warmup, world, dev)
    total = _max_over_ranks(world, total, dev)
    mean_step = statistics.mean(per)
    res = {
        "value": world * a_bytes * steps / total / 1e9,
        "ms_per_step": total / steps * 1e3,
        "kernel_ms": mean_step * 1e3,
        "alg_bytes": alg_bytes,
        "achieved_gbs": alg_bytes / mean_step / 1e9,
        "clocks": cs.summary(),
    }
    res["omega_setup"] = time_setup(torch, w, mean_step)
    if with_e2e:
        e_steps = max(1, min(steps, 5))
        el, h2d, d2h, step_ms = time_e2e(torch, w, e_steps, world, dev)
        res["e2e"] = {"value": world * a_bytes * e_steps / el / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": d2h, "steps": e_steps, "step_ms": [round(x, 2) for x in step_ms],
                      "path": f"tm.{'apply_adjoint' if w['op'] == 'adjoint' else 'apply_right'}(pinned host torch tensor)"
                              " -> host tensor (H2D+kernel+D2H)"}
    return res


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--others", default="cfg1,cfg3,cfg4,cfg5,gauss,cfg2dct,twosided",
                    help="extra configs measured at N=1 ('' = none)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg (quick kernel experiments)")
    ap.add_argument("--no-sharded", action="store_true", help="skip the sharded config-4 SA (NCCL all-reduce) leg")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world, rank, local = _dist(args)
    dev = torch.device("cuda", (local % max(1, torch.cuda.device_count())) if world > 1 else 0)
    peak, peak_src = _peaks()

    w = WORKLOADS[args.config](torch, dev, rank)
    m = measure(torch, w, args.steps, max(3, args.warmup), world, rank, dev, True, dev.index)
    esize = w["a"].element_size()
    launches = w["launches"]

    cpu = None
    procs = os.cpu_count() or 1
    if world == 1 and rank == 0 and not args.no_cpu:
        cpu, _ = sample_parity(w, procs)

    others = {}
    del w["a"]
    torch.cuda.empty_cache()
    if not args.no_sharded:
        try:  # the one path with a collective, at every N (strong scaling)
            others["cfg4_sharded"] = measure_sharded_sa(torch, world, rank, dev)
        except Exception as exc:  # report, never hide
            others["cfg4_sharded"] = {"error": f"{type(exc).__name__}: {exc}"}
        if args.config == "cfg2":
            try:  # the headline workload at fixed total size (strong scaling), next to the weak headline
                others["cfg2_strong"] = measure_strong_cfg2(torch, world, rank, dev)
            except Exception as exc:
                others["cfg2_strong"] = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        bf16_burst, bf16_sust = float(pk["bf16_tflops"]), float(pk["bf16_tflops_sustained"])
    except (OSError, KeyError, ValueError):
        bf16_burst, bf16_sust = None, None
    if world == 1 and args.others:
        for name in [s for s in args.others.split(",") if s and s != args.config]:
            try:
                ow = WORKLOADS[name](torch, dev, rank)
                # sized by time, not count: >= 30 ms of warm-up launches (clocks ramp back up after the
                # previous leg's setup) and >= 30 ms timed, so a 0.1 ms kernel is not timed on 3 launches
                est, _ = time_device(torch, ow, 1, 1, 1, dev)
                o_warm = int(min(300, max(3, math.ceil(0.03 / max(est, 1e-6)))))
                o_steps = int(min(200, max(3, math.ceil(0.03 / max(est, 1e-6)))))
                om = measure(torch, ow, o_steps, o_warm, 1, 0, dev, False, 0)
                oes = ow["a"].element_size()
                downstream = _downstream(torch, ow, dev)
                others[name] = {"workload": ow["workload"], "value_gbs": om["value"], "ms_per_step": om["ms_per_step"],
                                "steps": o_steps, "warmup": o_warm,
                                "dtype": "f32" if oes == 4 else "f64", "kernel": ow["kernel"],
                                "pct_hbm_peak": 100.0 * om["achieved_gbs"] / peak,
                                "roofline_achieved_gbs": om["achieved_gbs"], "alg_bytes": om["alg_bytes"],
                                "traffic": _traffic(name), "omega_setup_ms": om["omega_setup"]["ms"],
                                "clocks": om["clocks"]}
                if name in SAMPLE_ROWS and not args.no_cpu:
                    ocpu, oerr = sample_parity(ow, procs)
                    others[name]["cpu_baseline"] = ocpu
                    others[name]["parity_rel_fro_err"] = oerr
                if downstream:
                    others[name]["downstream"] = downstream
                if ow.get("flops"):
                    tf = ow["flops"] / (om["kernel_ms"] / 1e3) / 1e12
                    ex = tf * ow["flops_executed_x"]
                    others[name]["tensor"] = {
                        "useful_tflops": tf, "executed_tflops": ex,
                        "executed_frac_of_burst_bf16": ex / bf16_burst if bf16_burst else None,
                        "useful_frac_of_burst_bf16": tf / bf16_burst if bf16_burst else None,
                        "executed_frac_of_sustained_bf16": ex / bf16_sust if bf16_sust else None,
                        "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst: a kernel timed alone) and "
                                       "bf16_tflops_sustained"}
                del ow
                torch.cuda.empty_cache()
            except Exception as exc:  # report, never hide
                others[name] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        a_gib = w["n"] * w["d"] * esize / 2**30
        out = {
            "metric": METRIC,
            "value": m["value"],
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": m["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32" if esize == 4 else "f64",
            "data": "synthetic",
            "config": {"workload": w["workload"], "rows_per_gpu": w["n"], "d": w["d"], "k": w["k"],
                       "parallelism": f"row blocks over {world} GPU(s), no data-path collective",
                       "l2": f"input {a_gib:.1f} GiB per step > 126 MB L2: no flush between steps"},
            "pct_hbm_peak": 100.0 * m["achieved_gbs"] / peak,
            "roofline": {"bound": "hbm", "achieved": m["achieved_gbs"], "peak": peak, "unit": "GB/s",
                         "frac": m["achieved_gbs"] / peak, "traffic": _traffic(args.config),
                         "kernel": w["kernel"], "alg_bytes_per_launch": m["alg_bytes"],
                         "kernel_ms_mean": m["kernel_ms"], "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": m["e2e"],
            "gpu_launches": (launches * args.steps) if launches else None,
            "clocks": m["clocks"],
            "omega_setup": m["omega_setup"],
            "others": others,
        }
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
