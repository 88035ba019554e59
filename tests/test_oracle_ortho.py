"""Pins the oracle's block-orthogonalisation restatement (oracle.c orc_block_dots / update /
icgs / tsqr; reference ortho.hpp) before it checks the GPU.  ortho.hpp needs Eigen, which is not
in this container, so the pins are the reference's own known-answer tests (test_ortho.cpp),
restated here with the same inputs, tolerances and expectations, plus an independent
LAPACK (numpy) QR for the tsqr factors."""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise


def random_block(rows, cols, seed):
    """test_ortho.cpp:32-38: mt19937_64(seed), U[-1,1), column-major (returned as (cols, rows))."""
    return mpkg.random_vector(rows * cols, seed).reshape(cols, rows)


def ortho_defect(q):
    return np.abs(q @ q.T - np.eye(q.shape[0])).max()


def fact_defect(v_in, q, r):
    return np.abs(q.T @ r - v_in.T).max()


def test_tsqr_random_block_bounds(oracle):  # test_ortho.cpp:119-133
    v_in = random_block(1000, 4, 17)
    q, r = oracle.tsqr(v_in)
    vmax = np.abs(v_in).max()
    assert ortho_defect(q) <= 1e-13
    assert fact_defect(v_in, q, r) <= 1e-13 * vmax
    assert np.all(np.diag(r) >= 0) and np.all(np.tril(r, -1) == 0)
    # LAPACK's Householder QR with the same sign normalisation (unique factorisation)
    qn, rn = np.linalg.qr(v_in.T)
    s = np.sign(np.diag(rn))
    np.testing.assert_allclose(r, s[:, None] * rn, atol=1e-13 * vmax)
    np.testing.assert_allclose(q, (qn * s).T, atol=1e-13)


def test_tsqr_orthonormal_input_gives_identity_r(oracle):  # test_ortho.cpp:135-146
    q, _ = oracle.tsqr(random_block(600, 5, 3))
    _, r = oracle.tsqr(q)
    np.testing.assert_allclose(r, np.eye(5), atol=1e-13)


def test_tsqr_duplicate_columns_flag_rank_deficiency(oracle):  # test_ortho.cpp:148-159
    v = random_block(500, 3, 5).copy()
    v[1] = v[0]
    vmax = np.abs(v).max()
    _, r = oracle.tsqr(v)
    assert mpkg.tsqr_rank_deficient(r, 1e-14 * vmax * np.sqrt(500.0))
    assert not mpkg.tsqr_rank_deficient(np.array([[2.0, 0.0], [0.0, 1.0]]), 1e-14)


def test_tsqr_rejects_wide_blocks(oracle):  # test_ortho.cpp:192-196
    with pytest.raises(ValueError):
        oracle.tsqr(np.ones((3, 2)))


def test_icgs_exactly_orthogonal_input_is_untouched(oracle):  # test_ortho.cpp:198-211
    rows, qcols, vcols = 64, 4, 2
    q = np.zeros((qcols, rows))
    q[np.arange(qcols), np.arange(qcols)] = 1.0
    v = random_block(rows, vcols, 7).copy()
    v[:, :qcols] = 0.0
    out, coeff = oracle.icgs(q, v, 2)
    assert np.all(coeff == 0.0)
    assert_bitwise(out, v)


def test_icgs_duplicate_of_basis_column_projects_to_zero(oracle):  # test_ortho.cpp:213-224
    q, _ = oracle.tsqr(random_block(1000, 5, 11))
    out, coeff = oracle.icgs(q, q[:1], 1)
    assert np.abs(out).max() <= 1e-13
    assert abs(coeff[0, 0] - 1.0) <= 1e-12
    assert np.abs(coeff[1:, 0]).max() <= 1e-12


def test_icgs_cross_products_after_sweeps(oracle):  # test_ortho.cpp:226-244
    q, _ = oracle.tsqr(random_block(1000, 8, 13))
    v_in = random_block(1000, 4, 19)
    v1, _ = oracle.icgs(q, v_in, 1)
    assert np.abs(q @ v1.T).max() <= 1e-10
    v2, _ = oracle.icgs(q, v_in, 2)
    assert np.abs(q @ v2.T).max() <= 1e-12


def test_icgs_coefficients_reconstruct_the_projection(oracle):  # test_ortho.cpp:246-264
    rows, qcols, vcols = 128, 3, 2
    q = np.zeros((qcols, rows))
    q[np.arange(qcols), np.arange(qcols)] = 1.0
    c0 = np.array([0.5, -2.0, 1.25, 3.0, 0.0, -0.75]).reshape(vcols, qcols)  # column-major
    w = random_block(rows, vcols, 23).copy()
    w[:, :qcols] = 0.0
    v = w.copy()
    v[:, :qcols] = c0
    out, coeff = oracle.icgs(q, v, 2)
    assert np.abs(coeff - c0.T).max() <= 1e-15
    assert np.abs(out - w).max() <= 1e-15


def test_icgs_rejects_non_positive_sweeps_and_empty_basis(oracle):  # test_ortho.cpp:284-297
    with pytest.raises(ValueError):
        oracle.icgs(np.zeros((1, 8)), np.ones((1, 8)), 0)
    v = random_block(32, 2, 43)
    out, coeff = oracle.icgs(None, v, 1)
    assert coeff.size == 0
    assert_bitwise(out, v)


def test_block_dots_update_are_the_serial_loops(oracle):
    """ortho.hpp:46-92 literally: serial ascending sums, ascending-k updates (mul then sub)."""
    rng = np.random.default_rng(1)
    q, v = rng.standard_normal((3, 257)), rng.standard_normal((2, 257))
    c = oracle.block_dots(q, v)
    for k in range(3):
        for j in range(2):
            acc = 0.0
            for i in range(257):
                acc += float(q[k, i]) * float(v[j, i])
            assert c[k, j] == acc
    out = oracle.block_update(q, c, v)
    want = v.copy()
    for j in range(2):
        for k in range(3):
            want[j] = want[j] - c[k, j] * q[k]
    assert_bitwise(out, want)
