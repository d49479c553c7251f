"""NumPy/SciPy restatement of the reference sketch path (test infrastructure).

Functional style on purpose: each test-matrix family is described by a small
parameter tuple and the oracle returns plain arrays (scipy CSR, dense
float64), so the checker shares no code with the product package.

Reference anchors (relative to /root/reference/pkg/src/sketchkit/):
  RNG streams ............ core/rng.py:27-70
  entry distributions .... sketch/base.py:23-45
  w/o-replacement rows ... sketch/sparse.py:18-43
  SparseStack ............ sketch/sparse.py:118-139
  SparseUniform .......... sketch/sparse.py:187-194
  SparseCol .............. sketch/sparse.py:308-320
  CSR apply paths ........ sketch/sparse.py:63-78
  WHT / DCT .............. sketch/rtt.py:28-60
  SparseRTT .............. sketch/rtt.py:78-154
  Khatri-Rao ............. sketch/khatri_rao.py:46-74, 132-164
  Gaussian ............... sketch/gaussian.py:19-30
"""

from __future__ import annotations

import numpy as np
import scipy.fft
import scipy.sparse as sp

__all__ = [
    "stream",
    "rademacher",
    "distinct_rows",
    "sparse_uniform_csr",
    "sparse_stack_csr",
    "sparse_col_csr",
    "srtt_parts",
    "stack_from_assignments",
    "kr_factors",
    "gaussian_dense",
    "csr_right",
    "csr_adjoint",
    "wht_rows",
    "dct3_rows",
    "srtt_right",
    "kr_right",
    "dense_right",
    "right_chunked",
    "csr_adjoint_chunked",
    "right_multiprocess",
    "orth",
    "rsvd",
    "truncated_pinv_apply",
    "sketch_and_solve",
]


# --------------------------------------------------------------------------
# RNG: (seed, path) -> SeedSequence entropy -> Philox -> Generator
# --------------------------------------------------------------------------
def _entropy_words(label):
    """core/rng.py:27-36 — int -> [v mod 2^64, is_negative]; str -> [LE int, len, 2]."""
    if isinstance(label, (int, np.integer)):
        v = int(label)
        return [v & (2**64 - 1), int(v < 0)]
    if isinstance(label, str):
        b = label.encode("utf-8")
        return [int.from_bytes(b, "little"), len(b), 2]
    raise TypeError(type(label))


def stream(seed: int, *path) -> np.random.Generator:
    """core/rng.py:65-70 (RngStream(seed, path).generator()); base.py:60-61 path = (ClassName, label)."""
    ent = _entropy_words(int(seed))
    for p in path:
        ent += _entropy_words(p)
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(ent)))


def rademacher(g: np.random.Generator, size) -> np.ndarray:
    """sketch/base.py:30-31 — integers(0,2) as float64 * 2 - 1."""
    return g.integers(0, 2, size=size).astype(np.float64) * 2.0 - 1.0


def distinct_rows(g, n_sets: int, take: int, universe: int) -> np.ndarray:
    """sketch/sparse.py:18-43 — rejection on iid draws, permutation when acceptance < 5%."""
    if take > universe:
        raise ValueError("take > universe")
    if take == universe:
        return np.tile(np.arange(universe), (n_sets, 1)) if n_sets else np.empty((0, take), int)
    p_all_distinct = np.prod(1.0 - np.arange(take) / universe)
    if p_all_distinct < 0.05:
        res = np.empty((n_sets, take), dtype=np.int64)
        for s in range(n_sets):
            res[s] = g.permutation(universe)[:take]
        return res
    res = g.integers(0, universe, size=(n_sets, take))
    while True:
        dup = (np.diff(np.sort(res, axis=1), axis=1) == 0).any(axis=1)
        redo = np.flatnonzero(dup)
        if redo.size == 0:
            return res
        res[redo] = g.integers(0, universe, size=(redo.size, take))


# --------------------------------------------------------------------------
# Constructors (real field only — the B200 path has no complex config)
# --------------------------------------------------------------------------
def sparse_uniform_csr(d: int, k: int, zeta: int, seed: int) -> sp.csr_array:
    """sketch/sparse.py:187-194 (SparseUniformTM._build)."""
    g = stream(seed, "SparseUniformTM", "entries")
    cols = distinct_rows(g, d, zeta, k)
    cols.sort(axis=1)
    sg = g.integers(0, 2, size=(d, zeta)) * 2.0 - 1.0
    vals = (sg / np.sqrt(zeta)).astype(np.float64).ravel()
    return sp.csr_array((vals, cols.ravel(), np.arange(d + 1) * zeta), shape=(d, k))


def sparse_stack_csr(d: int, zeta: int, block: int, seed: int) -> sp.csr_array:
    """sketch/sparse.py:128-139 (SparseStackTM._assemble/_build, real Rademacher)."""
    g = stream(seed, "SparseStackTM", "entries")
    buckets = g.integers(0, block, size=(d, zeta))
    sg = rademacher(g, (d, zeta))
    return stack_from_assignments(sg, buckets, block)


def stack_from_assignments(signs, buckets, block: int) -> sp.csr_array:
    """sketch/sparse.py:118-132 — column = bucket + j*b, value sign/sqrt(zeta)."""
    signs = np.asarray(signs, dtype=np.float64)
    buckets = np.asarray(buckets)
    d, zeta = signs.shape
    cols = buckets + np.arange(zeta)[None, :] * block
    vals = (signs / np.sqrt(zeta)).ravel()
    return sp.csr_array((vals, cols.ravel(), np.arange(d + 1) * zeta), shape=(d, block * zeta))


def sparse_col_csr(d: int, k: int, xi: int, seed: int) -> sp.csr_array:
    """sketch/sparse.py:308-320 (SparseColTM._build) — xi distinct rows per column, value
    +-sqrt(d/xi)/sqrt(k); rows may repeat across columns."""
    g = stream(seed, "SparseColTM", "entries")
    rows = distinct_rows(g, k, xi, d)
    sg = g.integers(0, 2, size=(k, xi)) * 2.0 - 1.0
    mag = np.sqrt(d / xi) / np.sqrt(k)
    coo = sp.coo_array(((sg.ravel() * mag), (rows.ravel(), np.repeat(np.arange(k), xi))), shape=(d, k))
    out = sp.csr_array(coo)
    out.sort_indices()
    return out


def srtt_parts(d: int, k: int, xi: int, seed: int, diagonal: str = "real_rademacher"):
    """sketch/rtt.py:114-121 — D from stream (SparseRttTM, diagonal), sampler = SparseColTM(seed)."""
    g = stream(seed, "SparseRttTM", "diagonal")
    if diagonal == "real_rademacher":
        dv = rademacher(g, d)
    elif diagonal == "uniform_symmetric":
        dv = g.uniform(-np.sqrt(3.0), np.sqrt(3.0), size=d)
    else:
        raise ValueError(diagonal)
    return dv.astype(np.float64), sparse_col_csr(d, k, xi, seed)


def kr_factors(d0: int, ell: int, k: int, seed: int, base: str = "real_rademacher") -> np.ndarray:
    """sketch/khatri_rao.py:46-59, 132-139 — ell sequential (d0, k) draws from (KhatriRaoTM, factors)."""
    g = stream(seed, "KhatriRaoTM", "factors")
    blocks = []
    for _ in range(ell):
        if base == "real_rademacher":
            blocks.append(rademacher(g, (d0, k)))
        elif base == "real_gaussian":
            blocks.append(g.standard_normal((d0, k)))
        elif base == "real_spherical":
            x = g.standard_normal((d0, k))
            blocks.append(x * (np.sqrt(d0) / np.linalg.norm(x, axis=0)))
        else:
            raise ValueError(base)
    return np.stack(blocks).astype(np.float64)


def gaussian_dense(d: int, k: int, seed: int) -> np.ndarray:
    """sketch/gaussian.py:19-30 (real) — N(0,1) * k^-1/2 from (GaussianTM, entries)."""
    return stream(seed, "GaussianTM", "entries").standard_normal((d, k)) * (1.0 / np.sqrt(k))


# --------------------------------------------------------------------------
# Apply paths (float64, as the reference computes)
# --------------------------------------------------------------------------
def csr_right(omega: sp.csr_array, a) -> np.ndarray:
    """sketch/sparse.py:63-66 — A @ Omega (scipy csc_matvecs on Omega^T after A's transpose copy)."""
    return np.asarray(np.asarray(a, dtype=np.float64) @ omega)


def csr_adjoint(omega: sp.csr_array, b) -> np.ndarray:
    """sketch/sparse.py:68-78 — Omega^T @ B; a 1-D B is treated as a column and squeezed."""
    b = np.asarray(b, dtype=np.float64)
    one = b.ndim == 1
    out = np.asarray(omega.T @ (b[:, None] if one else b))
    return out[:, 0] if one else out


def wht_rows(x: np.ndarray) -> np.ndarray:
    """sketch/rtt.py:28-44 along axis 1 — unnormalised butterflies on adjacent blocks, then /sqrt(d)."""
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    if d <= 0 or d & (d - 1):
        raise ValueError("WHT requires a power-of-two length")
    y = np.ascontiguousarray(x.T)  # (d, n): butterflies run over the leading axis as in the reference
    h = 1
    while h < d:
        v = y.reshape(d // (2 * h), 2, h, n)
        y = np.stack([v[:, 0] + v[:, 1], v[:, 0] - v[:, 1]], axis=1).reshape(d, n)
        h *= 2
    return (y / np.sqrt(d)).T


def dct3_rows(x: np.ndarray) -> np.ndarray:
    """sketch/rtt.py:136-137 — right-multiplying by the DCT-II applies DCT-III (ortho) to each row."""
    return scipy.fft.dct(np.asarray(x, dtype=np.float64), type=3, norm="ortho", axis=1)


def srtt_right(dvals, sampler: sp.csr_array, a, transform: str) -> np.ndarray:
    """sketch/rtt.py:129-140 — (A * D) -> row transform -> @ S."""
    ad = np.asarray(a, dtype=np.float64) * dvals[None, :]
    adf = dct3_rows(ad) if transform == "dct" else wht_rows(ad)
    return np.asarray(adf @ sampler)


def kr_right(factors: np.ndarray, a) -> np.ndarray:
    """sketch/khatri_rao.py:62-74, 158-164 — mode-by-mode einsum on A^T, factor 0 on the slow index."""
    ell, d0, k = factors.shape
    bt = np.asarray(a, dtype=np.float64).T
    m = bt.shape[1]
    t = np.einsum("dk,dr->kr", factors[0], bt.reshape(d0, -1))
    for i in range(1, ell):
        t = np.einsum("dk,kdr->kr", factors[i], t.reshape(k, d0, -1))
    return t.reshape(k, m).T / np.sqrt(k)


def dense_right(omega: np.ndarray, a) -> np.ndarray:
    """sketch/base.py:75-79 — A @ materialize()."""
    return np.asarray(a, dtype=np.float64) @ omega


def right_chunked(fn, a, rows: int = 4096, threads: int = 1) -> np.ndarray:
    """Row-chunked right apply (rows are independent) with an optional thread pool."""
    a = np.asarray(a)
    n = a.shape[0]
    starts = list(range(0, n, rows))
    parts = [None] * len(starts)

    def run(j):
        s = starts[j]
        parts[j] = fn(a[s:s + rows])

    if threads <= 1:
        for j in range(len(starts)):
            run(j)
    else:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(run, range(len(starts))))
    return np.concatenate(parts, axis=0) if parts else np.zeros((0, 0))


def csr_adjoint_chunked(omega: sp.csr_array, b, rows: int = 1 << 18) -> np.ndarray:
    """Row-block partial sums of Omega^T B using omega[r0:r1]."""
    b = np.asarray(b)
    out = None
    for s in range(0, b.shape[0], rows):
        part = csr_adjoint(omega[s:s + rows], b[s:s + rows])
        out = part if out is None else out + part
    return out


# --------------------------------------------------------------------------
# Multi-process row-parallel driver for the CPU baseline (all host cores)
# --------------------------------------------------------------------------
_POOL_STATE = {}


def _pool_run(bounds):
    fn, a = _POOL_STATE["fn"], _POOL_STATE["a"]
    s, e = bounds
    return s, fn(a[s:e])


def right_multiprocess(fn, a, procs: int, rows: int = 256) -> np.ndarray:
    """Row-parallel apply over `procs` forked worker processes (rows are independent).

    The input is shared copy-on-write through fork; only the (small) outputs travel back.  Used by
    bench.py's cpu_baseline / reference arm so the reference algorithm gets every host core.
    """
    import multiprocessing as mp

    a = np.asarray(a)
    n = a.shape[0]
    bounds = [(s, min(n, s + rows)) for s in range(0, n, rows)]
    if procs <= 1 or len(bounds) <= 1:
        return fn(a)
    _POOL_STATE["fn"], _POOL_STATE["a"] = fn, a
    try:
        with mp.get_context("fork").Pool(procs) as pool:
            parts = dict(pool.map(_pool_run, bounds))
    finally:
        _POOL_STATE.clear()
    return np.concatenate([parts[s] for s, _ in bounds], axis=0)


# --------------------------------------------------------------------------
# Downstream drivers (float64, as the reference)
# --------------------------------------------------------------------------
RANK_TOL = 5.0 * float(np.finfo(np.float64).eps)  # core/factor.py:27-28


def orth(m, rel_tol: float = RANK_TOL) -> np.ndarray:
    """core/factor.py:63-82 — Householder QR, SVD basis when R reveals rank deficiency."""
    m = np.asarray(m)
    if m.shape[1] == 0:
        return m.copy()
    q, r = np.linalg.qr(m, mode="reduced")
    dg = np.abs(np.diag(r))
    top = dg.max(initial=0.0)
    if top == 0.0:
        return q[:, :0]
    if dg.min() > rel_tol * top:
        return q
    u, s, _ = np.linalg.svd(m, full_matrices=False)
    return u[:, : int(np.count_nonzero(s > rel_tol * s[0]))]


def rsvd(a, omega_apply, k: int):
    """rand_nla.py:84-109 — Y = A Omega, Q = orth(Y), B = Q^* A, SVD(B) -> (Q U_B, sigma, V)."""
    a = np.asarray(a, dtype=np.float64)
    q = orth(omega_apply(a))
    if q.shape[1] == 0:
        return np.zeros((a.shape[0], 0)), np.zeros(0), np.zeros((a.shape[1], 0))
    u, s, vh = np.linalg.svd(q.conj().T @ a, full_matrices=False)
    return q @ u, s, vh.conj().T


def truncated_pinv_apply(m, b, rel_tol: float = RANK_TOL):
    """core/factor.py:112-136."""
    b = np.asarray(b)
    one = b.ndim == 1
    b = b[:, None] if one else b
    u, s, vh = np.linalg.svd(m, full_matrices=False)
    rank = 0 if s.size == 0 or s[0] == 0.0 else int(np.count_nonzero(s > rel_tol * s[0]))
    out = np.zeros((m.shape[1], b.shape[1])) if rank == 0 else vh[:rank].conj().T @ ((u[:, :rank].conj().T @ b) / s[:rank, None])
    return out[:, 0] if one else out


def sketch_and_solve(a, b, adjoint_apply):
    """rand_nla.py:278-297 — (Psi^* A)^+ (Psi^* B)."""
    return truncated_pinv_apply(adjoint_apply(np.asarray(a, dtype=np.float64)),
                                adjoint_apply(np.asarray(b, dtype=np.float64)))
