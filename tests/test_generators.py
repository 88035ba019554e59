"""Host generators (harness inputs): the reference's own generators reproduced exactly, and the
properties of the configs the reference has no generator for (27-point stencil, scramble, R-MAT)."""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise


def _same(A, r):
    np.testing.assert_array_equal(A.row_ptr, r[0])
    np.testing.assert_array_equal(A.col_idx, r[1])
    assert_bitwise(A.values, r[2])


def test_reference_generators_reproduced(ref):
    _same(mpkg.poisson1d(9), ref.gen(1, 9))
    _same(mpkg.poisson2d(13, 7), ref.gen(2, 13, 7))
    _same(mpkg.poisson3d(6, 5, 4), ref.gen(3, 6, 5, 4))
    _same(mpkg.random_csr(500, 6, 3), ref.gen(4, 500, 6, 0, 3))
    _same(mpkg.random_spd(700, 5, 777), ref.gen(5, 700, 5, 0, 777))
    np.testing.assert_array_equal(mpkg.random_vector(4096, 42), ref.random_vector(4096, 42))


def test_golden_random_vector(golden):
    assert_bitwise(mpkg.random_vector(1000, 42), golden["rv.x"])


def test_generator_errors():
    with pytest.raises(ValueError):
        mpkg.poisson1d(0)
    with pytest.raises(ValueError):
        mpkg.random_csr(10, 0, 1)
    with pytest.raises(ValueError):
        mpkg.random_csr(10, 11, 1)


def _dense(A):
    D = np.zeros((A.n_rows, A.n_cols))
    for r in range(A.n_rows):
        s, e = A.row_ptr[r], A.row_ptr[r + 1]
        D[r, A.col_idx[s:e]] = A.values[s:e]
    return D


def _check_csr(A):
    rp = A.row_ptr.astype(np.int64)
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0)
    for r in range(A.n_rows):
        c = A.col_idx[rp[r]:rp[r + 1]]
        assert np.all(np.diff(c.astype(np.int64)) > 0)


def test_stencil27():
    A = mpkg.stencil27(5, 4, 3)
    _check_csr(A)
    D = _dense(A)
    assert np.all(np.diag(D) == 26.0)
    assert A.nnz == (3 * 5 - 2) * (3 * 4 - 2) * (3 * 3 - 2)
    assert np.array_equal(D, D.T)
    assert set(np.unique(D[D != 0])) == {26.0, -1.0}
    full = mpkg.stencil27(160, 160, 160)  # config C2/C4 size check (fast, direct CSR)
    assert full.nnz == 478 ** 3 and full.n_rows == 4096000


def test_stencil27_random_sym():
    A = mpkg.stencil27_random_sym(6, 5, 4, 7)
    _check_csr(A)
    D = _dense(A)
    assert np.array_equal(D, D.T)  # exactly symmetric
    off = D[(D != 0) & ~np.eye(A.n_rows, dtype=bool)]
    assert np.all(off <= -0.9) and np.all(off >= -1.1)
    assert np.all(np.diag(D) == 26.0)
    B = mpkg.stencil27_random_sym(6, 5, 4, 7)
    assert_bitwise(A.values, B.values)


def test_scramble_semantics(oracle):
    A = mpkg.stencil27_random_sym(5, 5, 5, 3)
    B, perm = mpkg.scramble(A, 11, return_perm=True)
    assert sorted(perm.tolist()) == list(range(A.n_rows))
    prp, pci, pv = oracle.permute(A.row_ptr, A.col_idx, A.values, perm)
    np.testing.assert_array_equal(B.row_ptr, prp)
    np.testing.assert_array_equal(B.col_idx, pci)
    assert_bitwise(B.values, pv)


def test_rmat_properties():
    A = mpkg.rmat(10, 16, 5)
    assert A.n_rows == 1024
    _check_csr(A)
    D = _dense(A)
    assert np.array_equal(D, D.T)
    off = D - np.diag(np.diag(D))
    assert np.all(off <= 0)
    nz = off[off != 0]
    assert np.all(nz <= -0.1) and np.all(nz >= -1.0)
    np.testing.assert_allclose(np.diag(D), 1.0 + np.abs(off).sum(axis=1), rtol=1e-14)
    B = mpkg.rmat(10, 16, 5)
    assert_bitwise(A.values, B.values)
    # power law: a handful of hub rows, many isolated vertices
    deg = np.diff(A.row_ptr.astype(np.int64)) - 1
    assert deg.max() > 20 * max(1, np.median(deg))
