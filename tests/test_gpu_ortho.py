"""GPU block orthogonalisation (reference ortho.hpp) against the oracle.

Bitwise mode: block_dots is the reference's serial sum per entry, block_update the ascending-k
update, so dots / update / icgs are bit-identical to the oracle.  Fast mode: block_dots runs on
the fp64 tensor cores with a fixed-order reduction; it is checked entry-wise against the serial
sum with the tolerance |dC_kj| <= 1e-13 |q_k| |v_j| (forward error bound of a dot product, with
room), and icgs / tsqr against the reference's own acceptance tolerances (test_ortho.cpp).
tsqr: (Q, R) with a non-negative R diagonal is unique for a full-rank block; R and Q are
compared with the oracle within 1e-10 vmax (the reference's panel-tree tolerance,
test_ortho.cpp:176), orthogonality within 1e-13 and Q R = V within 1e-13 vmax."""
import contextlib

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def random_block(rows, cols, seed):
    return mpkg.random_vector(rows * cols, seed).reshape(cols, rows)


@contextlib.contextmanager
def mode(ctx, m):
    ctx.set_mode(m)
    try:
        yield
    finally:
        ctx.set_mode(ctx.MODE_BITWISE)


MODES = ["bitwise", "fast"]


def _mode(ctx, name):
    return mode(ctx, ctx.MODE_FAST if name == "fast" else ctx.MODE_BITWISE)


SHAPES = [(1, 1, 1), (31, 3, 2), (33, 7, 1), (1000, 25, 8), (4099, 50, 11), (100_003, 9, 4)]


@pytest.mark.parametrize("rows,qcols,vcols", SHAPES)
def test_block_dots(ctx, oracle, rows, qcols, vcols):
    rng = np.random.default_rng(rows + qcols)
    q, v = rng.uniform(-1, 1, (qcols, rows)), rng.uniform(-1, 1, (vcols, rows))
    want = oracle.block_dots(q, v)
    with _mode(ctx, "bitwise"):
        assert_bitwise(ctx.block_dots(q, v), want, "bitwise dots")
    with _mode(ctx, "fast"):
        got = ctx.block_dots(q, v)
        got2 = ctx.block_dots(q, v)
    assert_bitwise(got, got2, "fast dots are deterministic")
    bound = 1e-13 * np.outer(np.linalg.norm(q, axis=1), np.linalg.norm(v, axis=1))
    assert np.all(np.abs(got - want) <= bound)


@pytest.mark.parametrize("rows,qcols,vcols", SHAPES)
@pytest.mark.parametrize("m", MODES)
def test_block_update_bitwise(ctx, oracle, rows, qcols, vcols, m):
    rng = np.random.default_rng(7 * rows + vcols)
    q, v = rng.uniform(-1, 1, (qcols, rows)), rng.uniform(-1, 1, (vcols, rows))
    c = rng.uniform(-2, 2, (qcols, vcols))
    with _mode(ctx, m):
        assert_bitwise(ctx.block_update(q, c, v), oracle.block_update(q, c, v), "update")


@pytest.mark.parametrize("rows,qcols,vcols", SHAPES[1:])
@pytest.mark.parametrize("sweeps", [1, 2, 3])
def test_icgs_bitwise_mode_matches_oracle(ctx, oracle, rows, qcols, vcols, sweeps):
    q, _ = oracle.tsqr(random_block(rows, qcols, 31 + qcols)) if rows >= qcols else (None, None)
    v = random_block(rows, vcols, 37)
    want_v, want_c = oracle.icgs(q, v, sweeps)
    with _mode(ctx, "bitwise"):
        got_v, got_c = ctx.icgs_block_orthogonalize(q, v, sweeps)
    assert_bitwise(got_v, want_v, "v")
    assert_bitwise(got_c, want_c, "coeff")


@pytest.mark.parametrize("m", MODES)
def test_icgs_reference_known_answers(ctx, oracle, m):
    with _mode(ctx, m):
        # test_ortho.cpp:198-211 exactly orthogonal input is untouched
        rows = 64
        q = np.zeros((4, rows))
        q[np.arange(4), np.arange(4)] = 1.0
        v = random_block(rows, 2, 7).copy()
        v[:, :4] = 0.0
        out, coeff = ctx.icgs_block_orthogonalize(q, v, 2)
        assert np.all(coeff == 0.0)
        assert_bitwise(out, v)
        # test_ortho.cpp:213-224 a duplicate of a basis column projects to zero
        qb, _ = ctx.tsqr(random_block(1000, 5, 11))
        out, coeff = ctx.icgs_block_orthogonalize(qb, qb[:1], 1)
        assert np.abs(out).max() <= 1e-13
        assert abs(coeff[0, 0] - 1.0) <= 1e-12 and np.abs(coeff[1:, 0]).max() <= 1e-12
        # test_ortho.cpp:226-244 cross products after one / two sweeps
        qb, _ = ctx.tsqr(random_block(1000, 8, 13))
        v_in = random_block(1000, 4, 19)
        v1, _ = ctx.icgs_block_orthogonalize(qb, v_in, 1)
        assert np.abs(qb @ v1.T).max() <= 1e-10
        v2, _ = ctx.icgs_block_orthogonalize(qb, v_in, 2)
        assert np.abs(qb @ v2.T).max() <= 1e-12
        # test_ortho.cpp:246-264 coefficients reconstruct a known projection
        q = np.zeros((3, 128))
        q[np.arange(3), np.arange(3)] = 1.0
        c0 = np.array([0.5, -2.0, 1.25, 3.0, 0.0, -0.75]).reshape(2, 3)
        w = random_block(128, 2, 23).copy()
        w[:, :3] = 0.0
        v = w.copy()
        v[:, :3] = c0
        out, coeff = ctx.icgs_block_orthogonalize(q, v, 2)
        assert np.abs(coeff - c0.T).max() <= 1e-15 and np.abs(out - w).max() <= 1e-15
        # test_ortho.cpp:284-297 bad sweeps, empty basis
        with pytest.raises(ValueError, match="sweeps must be >= 1"):
            ctx.icgs_block_orthogonalize(np.zeros((1, 8)), np.ones((1, 8)), 0)
        v = random_block(32, 2, 43)
        out, coeff = ctx.icgs_block_orthogonalize(None, v, 1)
        assert coeff.size == 0
        assert_bitwise(out, v)


@pytest.mark.parametrize("sweeps", [2, 3])
@pytest.mark.parametrize("rows,qcols,vcols", [(1000, 25, 8), (100_003, 9, 4), (20_001, 64, 12),
                                              (5000, 70, 3), (33, 1, 1)])
def test_icgs_fast_mode_tolerance(ctx, oracle, rows, qcols, vcols, sweeps):
    """Fast mode: tensor-core dots, and every update but the last fused with the next sweep's
    dots (k_update_dots; qcols <= 64).  Within tolerance of the oracle's serial ICGS."""
    q, _ = oracle.tsqr(random_block(rows, qcols, 5))
    v = random_block(rows, vcols, 6)
    want_v, want_c = oracle.icgs(q, v, sweeps)
    with _mode(ctx, "fast"):
        got_v, got_c = ctx.icgs_block_orthogonalize(q, v, sweeps)
    vmax = np.abs(v).max()
    assert np.abs(got_c - want_c).max() <= 1e-12 * np.sqrt(rows) * vmax
    assert np.abs(got_v - want_v).max() <= 1e-12 * vmax
    assert np.abs(q @ got_v.T).max() <= 1e-12


TSQR = [(1, 1), (5, 5), (600, 5), (1000, 4), (8192, 6), (10_000, 5), (200_000, 8), (70_001, 3),
        (20_000, 16), (5000, 64), (128, 64)]


@pytest.mark.parametrize("rows,cols", TSQR)
def test_tsqr_matches_oracle(ctx, oracle, rows, cols):
    v_in = random_block(rows, cols, rows + cols)
    q_o, r_o = oracle.tsqr(v_in)
    q, r = ctx.tsqr(v_in)
    vmax = np.abs(v_in).max()
    assert np.all(np.diag(r) >= 0) and np.all(np.tril(r, -1) == 0)
    assert np.abs(q @ q.T - np.eye(cols)).max() <= 1e-13
    assert np.abs(q.T @ r - v_in.T).max() <= 1e-13 * vmax
    assert np.abs(r - r_o).max() <= 1e-10 * vmax
    assert np.abs(q - q_o).max() <= 1e-10
    q2, r2 = ctx.tsqr(v_in)
    assert_bitwise(q2, q, "tsqr is deterministic")
    assert_bitwise(r2, r)


def test_tsqr_ill_conditioned_newton_like_block(ctx, oracle):
    """s-step blocks are graded and nearly dependent (cond ~1e9): the narrow (c <= 8) register /
    compact-WY path must keep Q orthonormal to roundoff like Householder does (a Gram-based QR
    would lose ~cond * eps of orthogonality)."""
    rows, cols = 120_000, 8
    base = random_block(rows, 1, 77)[0]
    noise = random_block(rows, cols, 78)
    v_in = np.stack([(base + 10.0 ** (-j - 1) * noise[j]) * 10.0 ** (-j) for j in range(cols)])
    q, r = ctx.tsqr(v_in)
    assert np.abs(q @ q.T - np.eye(cols)).max() <= 1e-13
    assert np.abs(q.T @ r - v_in.T).max() <= 1e-13 * np.abs(v_in).max()
    q_o, r_o = oracle.tsqr(v_in)
    assert np.abs(r - r_o).max() <= 1e-10 * np.abs(v_in).max()


def test_tsqr_reference_known_answers(ctx):
    # test_ortho.cpp:135-146 orthonormal input gives R = I
    q, _ = ctx.tsqr(random_block(600, 5, 3))
    _, r = ctx.tsqr(q)
    np.testing.assert_allclose(r, np.eye(5), atol=1e-13)
    # test_ortho.cpp:148-159 duplicate columns flag rank deficiency
    v = random_block(500, 3, 5).copy()
    v[1] = v[0]
    _, r = ctx.tsqr(v)
    assert mpkg.tsqr_rank_deficient(r, 1e-14 * np.abs(v).max() * np.sqrt(500.0))
    # zero block: R = 0, no NaN
    q, r = ctx.tsqr(np.zeros((2, 300)))
    assert np.all(r == 0.0) and np.all(np.isfinite(q))
    # test_ortho.cpp:192-196 wide blocks rejected; the GPU's column cap
    with pytest.raises(ValueError, match="at least as many rows"):
        ctx.tsqr(np.ones((3, 2)))
    with pytest.raises(ValueError, match="at most 64 columns"):
        ctx.tsqr(np.ones((65, 100)))
    q, r = ctx.tsqr(np.zeros((0, 10)))
    assert q.shape == (0, 10) and r.shape == (0, 0)


def test_device_pointer_variants_and_full_size_block(ctx):
    """C4-sized Newton block (n = 192^3, s = 8) against a 25-column basis through the _dev entry
    points; properties checked on the device."""
    import torch
    dev = torch.device("cuda", 0)
    n, qc, s = 192 ** 3, 25, 8
    g = torch.Generator(device=dev).manual_seed(5)
    Q = torch.rand((qc, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    R = torch.empty((qc, qc), dtype=torch.float64, device=dev)
    ctx.tsqr_dev(Q.data_ptr(), n, qc, R.data_ptr())
    ctx.synchronize()
    assert (Q @ Q.T - torch.eye(qc, device=dev, dtype=torch.float64)).abs().max().item() <= 1e-12
    V = torch.rand((s, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    V0 = V.clone()
    coeff = torch.empty((s, qc), dtype=torch.float64, device=dev)
    for m in MODES:
        V.copy_(V0)
        with _mode(ctx, m):
            ctx.icgs_block_orthogonalize_dev(Q.data_ptr(), n, qc, V.data_ptr(), s, 2, coeff.data_ptr())
            ctx.synchronize()
        assert (Q @ V.T).abs().max().item() <= 1e-12 * V0.abs().max().item() * 10
        # V0 = Q C + V  (coefficients column-major qc x s == row-major (s, qc))
        rec = coeff @ Q + V
        assert (rec - V0).abs().max().item() <= 1e-12
    Vin = V.clone()
    Rv = torch.empty((s, s), dtype=torch.float64, device=dev)
    ctx.tsqr_dev(V.data_ptr(), n, s, Rv.data_ptr())
    ctx.synchronize()
    Rm = Rv.T  # column-major
    assert (V @ V.T - torch.eye(s, device=dev, dtype=torch.float64)).abs().max().item() <= 1e-13
    assert (Rm.T @ V - Vin).abs().max().item() <= 1e-13 * Vin.abs().max().item()
    assert bool((torch.diag(Rm) >= 0).all())


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("rows,qcols,vcols,sweeps", [(200_003, 25, 8, 2), (50_000, 9, 5, 3), (70_000, 64, 8, 2),
                                                     (1000, 3, 2, 1), (300, 4, 8, 2), (90_000, 70, 4, 2)])
def test_ortho_block_equals_icgs_then_tsqr(ctx, oracle, mode, rows, qcols, vcols, sweeps):
    """mpkg_ortho_block (ICGS's last update fused into TSQR's first factor kernel) returns exactly
    what icgs_block_orthogonalize followed by tsqr returns, in both modes."""
    q, _ = oracle.tsqr(random_block(rows, qcols, 41))
    v = random_block(rows, vcols, 42)
    with _mode(ctx, mode):
        v1, c1 = ctx.icgs_block_orthogonalize(q, v, sweeps)
        q1, r1 = ctx.tsqr(v1)
        q2, c2, r2 = ctx.ortho_block(q, v, sweeps)
    assert_bitwise(c2, c1, "coefficients")
    assert_bitwise(q2, q1, "Q")
    assert_bitwise(r2, r1, "R")
