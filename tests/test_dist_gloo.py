"""World-size-2 gloo tests (CPU) of the row-sharded multi-GPU logic: sharding, the all-reduced
adjoint sketch, CholeskyQR2, the distributed rSVD and the distributed LSQR.

The CUDA kernels are not available on CPU, so a test-only NumPy operator (the oracle) stands in
for the per-rank apply; what is under test is the host-side partition and reduction logic.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_2508_21189_b200 import dist as skd


class OracleRowOp:
    """CPU stand-in with the product operator's interface (apply_right/apply_adjoint/row_block)."""

    def __init__(self, csr, r0=0):
        self.csr = csr
        self.d, self.k = csr.shape
        self.r0 = r0

    def row_block(self, r0, r1):
        return OracleRowOp(self.csr[r0:r1], r0)

    def apply_right(self, a):
        return torch.from_numpy(orc.csr_right(self.csr, a.double().numpy()))

    def apply_adjoint(self, b):
        return torch.from_numpy(orc.csr_adjoint(self.csr, b.double().numpy()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as exc:  # surface in the parent
        q.put((rank, exc))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return out


def _problem():
    rng = np.random.default_rng(0)
    n, d, k = 3001, 24, 96
    a = rng.standard_normal((n, d)) * (1.0 + rng.pareto(1.5, size=n))[:, None]
    b = a @ rng.standard_normal(d) + 1e-3 * rng.standard_normal(n)
    return a, b, orc.sparse_uniform_csr(n, k, 8, 7)


def _adjoint_job(rank, world):
    a, _, csr = _problem()
    r0, r1 = skd.row_range(a.shape[0], world, rank)
    sa = skd.sharded_adjoint(OracleRowOp(csr), torch.from_numpy(a[r0:r1]), r0)
    return sa.numpy()


def _lsqr_job(rank, world):
    a, b, csr = _problem()
    r0, r1 = skd.row_range(a.shape[0], world, rank)
    res = skd.sharded_lsqr(torch.from_numpy(a[r0:r1]), torch.from_numpy(b[r0:r1]), OracleRowOp(csr), r0,
                           atol=1e-12, btol=1e-12, _host_scaffold=True)
    return res.x.numpy() if hasattr(res.x, "numpy") else np.asarray(res.x)


def _rsvd_job(rank, world):
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((1200, 40)))
    a = (u * np.arange(1, 41) ** -2.0) @ np.linalg.qr(rng.standard_normal((64, 40)))[0].T
    csr = orc.sparse_uniform_csr(64, 16, 4, 2)
    r0, r1 = skd.row_range(a.shape[0], world, rank)
    f = skd.sharded_rsvd(torch.from_numpy(a[r0:r1]), 16, OracleRowOp(csr))
    err = skd.sharded_residual(torch.from_numpy(a[r0:r1]), f)
    return f.sigma.numpy(), err


def test_row_range_partition():
    for n in (1, 7, 100, 4194304):
        for w in (1, 2, 3, 8):
            ranges = [skd.row_range(n, w, r) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(w - 1))
            sizes = [r1 - r0 for r0, r1 in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_sharded_adjoint_gloo():
    out = _run(_adjoint_job)
    a, _, csr = _problem()
    ref = orc.csr_adjoint(csr, a)
    for r in out:
        assert np.allclose(out[r], ref, rtol=1e-12, atol=1e-10)


def test_sharded_lsqr_gloo():
    import scipy.sparse.linalg as sla

    out = _run(_lsqr_job)
    a, b, _ = _problem()
    ref = sla.lsqr(a, b, atol=1e-14, btol=1e-14, iter_lim=10000)[0]
    for r in out:
        assert np.allclose(out[r], ref, rtol=1e-7, atol=1e-9)
    assert np.array_equal(out[0], out[1])


def test_sharded_rsvd_gloo():
    out = _run(_rsvd_job)
    rng = np.random.default_rng(1)
    u, _ = np.linalg.qr(rng.standard_normal((1200, 40)))
    a = (u * np.arange(1, 41) ** -2.0) @ np.linalg.qr(rng.standard_normal((64, 40)))[0].T
    csr = orc.sparse_uniform_csr(64, 16, 4, 2)
    u_r, s_ref, v_r = orc.rsvd(a, lambda x: orc.csr_right(csr, x), 16)
    err_ref = np.linalg.norm(a - (u_r * s_ref) @ v_r.T) / np.linalg.norm(a)
    for r, (s, err) in out.items():
        assert np.allclose(s, s_ref, rtol=1e-8)
        assert abs(err - err_ref) <= 1e-8
