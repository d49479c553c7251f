"""Parity at BASELINE config size on the production paths (slow GPU tests, one config each).

* config 2 (the headline): all 65536 rows of the SRTT sketch against the CPU oracle.
* config 3 sketch: all 131072 rows against a float64 device product with the oracle's Omega, plus
  oracle rows from three tiles.

* config 4 S A: the full 4194304 x 512 float32 sketch (K2g) against the chunked CPU oracle
  (`csr_adjoint_chunked`, the reference's `matrix.conj().T @ b` by row blocks);
  and the same rows split into 3 uneven row blocks (the multi-GPU shards) whose partials sum to it.
* config 4 LSQR: sketch-and-precondition LSQR at full size against the float64 least-squares
  optimum formed on the host (normal equations in float64, chunked): unpreconditioned SciPy `lsqr`
  on this coherent (Pareto-weighted) A needs thousands of passes over 8 GiB, so the exact optimum
  is the reference; tolerance 1e-4 relative on ||Ax - b|| / ||b||.
* config 3 rsvd: rank-200 rSVD of A = U diag(i^-2) V^T (131072 x 16384 float32) against the
  reference's algorithm (oracle `rsvd`: Y = A Omega, Q = orth(Y), B = Q^T A, SVD) in float64 on the
  host with the same Omega; ||A - QB|| / ||A|| and the rank-100 truncation error within 1e-2
  relative.  The float64 products use a dense copy of Omega with BLAS (the sparse
  `csc_matvecs` path is single-threaded: ~70 s at this size, App. B); same arithmetic up to rounding.
* float64 (the reference's dtype) at the config-2 (WHT and DCT), config-3 and config-5 shapes: row
  samples from several tiles against the oracle at 1e-12.
"""

import numpy as np
import pytest

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import rand_nla
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu

N4, D4, K4 = 4194304, 512, 2048


def _cfg4_input(cuda, seed=41):
    import torch

    g = torch.Generator(device=cuda).manual_seed(seed)
    a = torch.randn(N4, D4, dtype=torch.float32, device=cuda, generator=g)
    a *= torch.rand(N4, 1, device=cuda, generator=g).clamp_min(1e-12) ** (-1.0 / 1.5)  # 1 + Pareto(1.5) weights
    return a


@pytest.fixture(scope="module")
def cfg4(cuda):
    a = _cfg4_input(cuda)
    tm = skb.SparseUniformTM(N4, K4, 8, seed=0)
    csr = orc.sparse_uniform_csr(N4, K4, 8, 0)
    return a, tm, csr


def test_config4_sketch_full_size(cfg4):
    a, tm, csr = cfg4
    sa = tm.apply_adjoint(a).double().cpu().numpy()
    ref = orc.csr_adjoint_chunked(csr, a.cpu().numpy())
    err = np.linalg.norm(sa - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err


def test_config4_uneven_row_blocks_sum(cfg4):
    """Three uneven row blocks (multi-GPU shards) on one GPU: K2g partials of the blocks (device-
    sliced draws, no host triplets) sum to the full sketch and to the oracle."""
    import torch

    a, tm, csr = cfg4
    cuts = [0, 1000003, 2900000, N4]
    total = torch.zeros((K4, D4), dtype=torch.float64, device=a.device)
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        blk = tm.row_block(r0, r1)
        assert blk._coo is None  # sliced from the device draws
        total += blk.apply_adjoint(a[r0:r1]).double()
    ref = orc.csr_adjoint_chunked(csr, a.cpu().numpy())
    err = np.linalg.norm(total.cpu().numpy() - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err
    empty = tm.row_block(N4, N4)
    assert float(empty.apply_adjoint(a[:0]).abs().sum()) == 0.0


def test_config4_lsqr_full_size(cfg4):
    import torch

    a, tm, _ = cfg4
    g = torch.Generator(device=a.device).manual_seed(4444)
    x0 = torch.randn(D4, device=a.device, dtype=torch.float64, generator=g)
    b = (rand_nla._matvec_blocks(a, x0, 0) + 1e-3 * torch.randn(N4, device=a.device, dtype=torch.float64,
                                                                  generator=g)).float()
    res = rand_nla.sketch_precondition_lsqr(a, b, tm, atol=1e-6, btol=0.0)
    x = res.x.double().cpu().numpy()
    # float64 least-squares optimum on the host: G = A^T A, c = A^T b by row chunks, then Cholesky
    ah = a.cpu().numpy()
    bh = b.cpu().numpy().astype(np.float64)
    G = np.zeros((D4, D4))
    c = np.zeros(D4)
    for s in range(0, N4, 1 << 18):
        blk = ah[s:s + (1 << 18)].astype(np.float64)
        G += blk.T @ blk
        c += blk.T @ bh[s:s + (1 << 18)]
    x_ref = np.linalg.solve(G, c)

    def rel_res(xx):
        r2 = 0.0
        for s in range(0, N4, 1 << 18):
            blk = ah[s:s + (1 << 18)].astype(np.float64)
            r2 += float(((blk @ xx - bh[s:s + (1 << 18)]) ** 2).sum())
        return np.sqrt(r2) / np.linalg.norm(bh)

    r_gpu, r_ref = rel_res(x), rel_res(x_ref)
    assert r_ref <= r_gpu * (1 + 1e-12)  # the optimum is the optimum
    assert abs(r_gpu - r_ref) <= 1e-4 * r_ref, (r_gpu, r_ref, res.itn)


def test_config3_rsvd_full_size(cuda):
    import torch

    n, d, k, r = 131072, 16384, 200, 2048
    g = torch.Generator(device=cuda).manual_seed(3333)

    def haar(rows):
        q, rr = torch.linalg.qr(torch.randn(rows, r, device=cuda, dtype=torch.float32, generator=g))
        return q * torch.sign(rr.diagonal())[None, :]

    u, v = haar(n), haar(d)
    sig = torch.arange(1, r + 1, device=cuda, dtype=torch.float32) ** -2.0
    with rand_nla._no_tf32():
        a = (u * sig[None, :]) @ v.T  # A = U diag(i^-2) V^T, leading 2048 terms (tail 6e-6 of ||A||)
    del u, v
    tm = skb.SparseUniformTM(d, k, 8, seed=0)
    fac = rand_nla.rsvd(a, k, tm)
    res_gpu = rand_nla.rsvd_residual(a, fac)
    res100_gpu = rand_nla.rsvd_residual(a, rand_nla.SvdFactorization(fac.u[:, :100], fac.sigma[:100],
                                                                     fac.v[:, :100]))
    # the reference algorithm in float64 on the host (oracle rsvd with the same Omega)
    ah = a.cpu().numpy()
    del a, fac
    torch.cuda.empty_cache()
    om = orc.sparse_uniform_csr(d, k, 8, 0).toarray()
    step = 8192
    y = np.concatenate([ah[s:s + step].astype(np.float64) @ om for s in range(0, n, step)])
    q = orc.orth(y)
    bmat = np.zeros((q.shape[1], d))
    a2 = 0.0
    for s in range(0, n, step):
        blk = ah[s:s + step].astype(np.float64)
        bmat += q[s:s + step].T @ blk
        a2 += float((blk ** 2).sum())
    sv = np.linalg.svd(bmat, compute_uv=False)
    res_ref = np.sqrt(max(a2 - float((sv ** 2).sum()), 0.0) / a2)
    res100_ref = np.sqrt(max(a2 - float((sv[:100] ** 2).sum()), 0.0) / a2)
    assert abs(res_gpu - res_ref) <= 1e-2 * res_ref, (res_gpu, res_ref)
    assert abs(res100_gpu - res100_ref) <= 1e-2 * res100_ref, (res100_gpu, res100_ref)


def test_config2_full_vs_oracle(cuda):
    """The headline: all 65536 rows of the config-2 SRTT sketch (tcgen05 kernel) against the CPU oracle,
    row-parallel on the host cores (the oracle's float64 WHT path, ~5 s on 16 processes)."""
    import os

    import torch

    n, d, k = 65536, 8192, 512
    tm = skb.SparseRttTM(d, k, 1, "wht", seed=0)
    g = torch.Generator(device=cuda).manual_seed(1000)
    a = torch.randn(n, d, dtype=torch.float32, device=cuda, generator=g)
    a /= torch.arange(1, d + 1, dtype=torch.float32, device=cuda)
    y = tm.apply_right(a).double().cpu().numpy()
    dv, samp = orc.srtt_parts(d, k, 1, 0)
    ref = orc.right_multiprocess(lambda x: orc.srtt_right(dv, samp, x, "wht"), a.cpu().numpy(),
                                 procs=os.cpu_count() or 1, rows=1024)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err


def test_config3_sketch_full(cuda):
    """Config 3's sketch Y = A Omega at full size (131072 x 16384 f32, zeta = 8, k = 200) on the CTA-pair
    tensor-core engine: against a float64 device product with the oracle's Omega for every row, and
    the oracle itself on rows from three tiles."""
    import torch

    n, d, k = 131072, 16384, 200
    tm = skb.SparseUniformTM(d, k, 8, seed=0)
    g = torch.Generator(device=cuda).manual_seed(3000)
    a = torch.randn(n, d, dtype=torch.float32, device=cuda, generator=g)
    y = tm.apply_right(a).double()
    csr = orc.sparse_uniform_csr(d, k, 8, 0)
    om = torch.as_tensor(csr.toarray(), device=cuda)
    ref = torch.empty_like(y)
    for r0 in range(0, n, 8192):
        ref[r0:r0 + 8192] = a[r0:r0 + 8192].double() @ om
    err = float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref))
    assert err <= 1e-5, err
    rows = np.r_[0:8, 65536:65544, n - 8:n]
    assert rel_err(y[rows].cpu().numpy(), orc.csr_right(csr, a[rows].cpu().numpy())) <= 1e-5


def test_float64_config_shapes_vs_oracle(cuda):
    """The reference's own dtype at the BASELINE shapes (what a NumPy float64 caller runs): config-2
    SRTT with the WHT (K3) and with the DCT default (K3b), config-3 sparse sign (K1r row slabs) and
    config-5 Khatri-Rao (K5d, the tile synthesised from the factors) — row samples from several tiles
    against the oracle at 1e-12."""
    import torch

    rows = np.r_[0:16, 20000:20008, -16:0]

    def check(tm, n, d, ref_fn, seed):
        g = torch.Generator(device=cuda).manual_seed(seed)
        a = torch.randn(n, d, dtype=torch.float64, device=cuda, generator=g)
        y = tm.apply_right(a)
        idx = rows % n
        got = y[torch.as_tensor(idx, device=cuda)].cpu().numpy()
        ref = ref_fn(a[torch.as_tensor(idx, device=cuda)].cpu().numpy())
        assert rel_err(got, ref) <= 1e-12, type(tm).__name__
        del a, y
        torch.cuda.empty_cache()

    tm = skb.SparseRttTM(8192, 512, 1, "wht", seed=0)
    dv, samp = orc.srtt_parts(8192, 512, 1, 0)
    check(tm, 65536, 8192, lambda x: orc.srtt_right(dv, samp, x, "wht"), 1)
    tm = skb.SparseRttTM(8192, 512, 1, "dct", seed=0)
    check(tm, 32768, 8192, lambda x: orc.srtt_right(dv, samp, x, "dct"), 2)
    tm = skb.SparseUniformTM(16384, 200, 8, seed=0)
    csr = orc.sparse_uniform_csr(16384, 200, 8, 0)
    assert len(tm._ring_on(cuda)[0]) > 1  # row slabs
    check(tm, 65536, 16384, lambda x: orc.csr_right(csr, x), 3)
    tm = skb.KhatriRaoTM(256, 2, 512, "real_rademacher", seed=0)
    fac = orc.kr_factors(256, 2, 512, 0)
    check(tm, 8192, 65536, lambda x: orc.kr_right(fac, x), 4)
