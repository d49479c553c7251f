"""Full-size downstream pipelines of BASELINE configs 3 and 4 on one GPU (results -> JSON).

config 3: A = U diag(i^-2) V^T (131072 x 16384 float32, U and V Haar via QR of Gaussian matrices
          generated on the GPU), rsvd with SparseUniformTM(16384, 200, zeta=8), report
          ||A - QB||_F / ||A||_F (k = 200) and the rank-100 truncation error.
config 4: A 4194304 x 512 float32 rows scaled by 1 + Pareto(1.5) weights, b = A x0 + 1e-3 N(0,1),
          S = SparseUniformTM(4194304, 2048, zeta=8) as the adjoint sketch, QR(SA) = QR, LSQR on
          A R^-1 to relative normal-equation residual 1e-6.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2508_21189_b200 import rand_nla  # noqa: E402
from paper_2508_21189_b200.sketch import SparseUniformTM  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def config3(dev, n=131072, d=16384, k=200, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    # Haar U (n x d) and V (d x d): QR of Gaussians with the diag(R) sign fix, float32 to bound memory
    u, r = torch.linalg.qr(torch.randn(n, d, device=dev, dtype=torch.float32, generator=g))
    u *= torch.sign(torch.diagonal(r))[None, :]
    del r
    v, r = torch.linalg.qr(torch.randn(d, d, device=dev, dtype=torch.float32, generator=g))
    v *= torch.sign(torch.diagonal(r))[None, :]
    del r
    s = torch.arange(1, d + 1, device=dev, dtype=torch.float32) ** -2.0
    u *= s[None, :]
    a = u @ v.T
    del u
    torch.cuda.empty_cache()
    tm = SparseUniformTM(d, k, 8, seed=0)
    tm.apply_right(a[:256])  # build and cache the device form of Omega outside the timing
    y, t_sketch = timed(lambda: tm.apply_right(a))
    f, t_rsvd = timed(lambda: rand_nla.rsvd(a, k, tm))
    err, t_err = timed(lambda: rand_nla.rsvd_residual(a, f))
    # rank-100 truncation of the same factorization
    f100 = rand_nla.SvdFactorization(f.u[:, :100], f.sigma[:100], f.v[:, :100])
    err100 = rand_nla.rsvd_residual(a, f100)
    sig = s.double()
    opt_k = float(torch.sqrt((sig[k:] ** 2).sum() / (sig ** 2).sum()))
    opt_100 = float(torch.sqrt((sig[100:] ** 2).sum() / (sig ** 2).sum()))
    return {"config": "cfg3", "shape": [n, d], "k": k, "sketch_ms": t_sketch * 1e3, "rsvd_ms": t_rsvd * 1e3,
            "residual_ms": t_err * 1e3, "rel_err_k200": err, "optimal_rank200": opt_k, "rel_err_rank100": err100,
            "optimal_rank100": opt_100, "sketch_input_GBps": n * d * 4 / t_sketch / 1e9}


def config4(dev, n=4194304, d=512, k=2048, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    gen = np.random.default_rng(seed)
    w = torch.from_numpy(1.0 + gen.pareto(1.5, size=n).astype(np.float32)).to(dev)
    a = torch.randn(n, d, device=dev, dtype=torch.float32, generator=g) * w[:, None]
    x0 = torch.randn(d, device=dev, dtype=torch.float64, generator=g)
    b = (a.double() @ x0 + 1e-3 * torch.randn(n, device=dev, dtype=torch.float64, generator=g)).float()
    tm = SparseUniformTM(n, k, 8, seed=0)
    tm.apply_adjoint(a)  # encode / upload Omega once (the encodings depend on the operand width)
    _, t_sketch = timed(lambda: tm.apply_adjoint(a))
    res, t_lsqr = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0))
    # second call: cuSOLVER / kernel first-use costs paid
    _, t_lsqr_warm = timed(lambda: rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0))
    x = res.x
    r = (a.double() @ x - b.double())
    rel_res = float(r.norm() / b.double().norm())
    # ||A||_2 from the Gram matrix (512 x 512) instead of an SVD of the tall matrix
    gram = torch.zeros(d, d, dtype=torch.float64, device=dev)
    for s0 in range(0, n, 1 << 18):
        blk = a[s0:s0 + (1 << 18)].double()
        gram += blk.T @ blk
    anorm = float(torch.linalg.eigvalsh(gram)[-1].sqrt())
    ne = float((a.double().T @ r).norm() / (r.norm() * anorm))
    return {"config": "cfg4", "shape": [n, d], "k": k, "sketch_ms": t_sketch * 1e3, "lsqr_ms": t_lsqr * 1e3, "lsqr_warm_ms": t_lsqr_warm * 1e3,
            "iterations": res.itn, "istop": res.istop, "rel_residual": rel_res,
            "lsqr_normal_eq_test_preconditioned": res.normal_eq_test, "normal_eq_residual_unpreconditioned": ne, "sketch_input_GBps": n * d * 4 / t_sketch / 1e9}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/pipelines.json")
    ap.add_argument("--which", default="cfg3,cfg4")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = []
    for w in args.which.split(","):
        res.append(config3(dev) if w == "cfg3" else config4(dev))
        print(json.dumps(res[-1]), flush=True)
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
