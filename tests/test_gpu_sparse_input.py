"""SciPy-sparse operands for the sparse-sign families (K1s): the reference's SuiteSparse path
(src/sketch/sparse.py:63-78: `a @ self.matrix`, `self.matrix.conj().T @ b`, never densified)."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as orc
from _cases import rel_err
from paper_2508_21189_b200 import sketch as skb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,k,zeta,density", [(2000, 3000, 64, 4, 0.01), (500, 40000, 200, 8, 0.001),
                                                 (7, 100, 30, 3, 0.3), (300, 64, 9000, 2, 0.05)])
def test_sparse_a_right(n, d, k, zeta, density, cuda):
    a = sp.random(n, d, density=density, format="csr", random_state=n + d, dtype=np.float64)
    tm = skb.SparseUniformTM(d, k, zeta, seed=4)
    y = tm.apply_right(a)
    assert isinstance(y, np.ndarray) and y.dtype == np.float64 and y.shape == (n, k)
    ref = (a @ orc.sparse_uniform_csr(d, k, zeta, 4)).toarray()  # the reference's own expression
    assert rel_err(y, ref) <= 1e-12


def test_sparse_b_adjoint(cuda):
    b = sp.random(5000, 70, density=0.02, format="csc", random_state=1)
    tm = skb.SparseStackTM(5000, 4, 32, seed=2)
    out = tm.apply_adjoint(b)
    ref = (orc.sparse_stack_csr(5000, 4, 32, 2).T @ b).toarray()
    assert out.shape == (128, 70) and rel_err(out, ref) <= 1e-12


def test_sparse_empty_rows_and_iid(cuda):
    a = sp.csr_array((np.array([1.5, -2.0]), np.array([3, 999]), np.array([0, 0, 1, 1, 2, 2])), shape=(5, 1000))
    tm = skb.SparseIIDTM(1000, 50, 3.0, seed=6)
    ref = a @ tm.materialize()
    assert rel_err(tm.apply_right(a), ref) <= 1e-12
    assert np.all(tm.apply_right(sp.csr_array((3, 1000))) == 0)
