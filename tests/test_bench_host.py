"""Host-side pieces of bench.py that run without a GPU: the flop conventions, the seeded stand-in
roots, and the CPU baselines the reference arm reports for the Eigen-dependent configs (the
oracle's C restatement of the same computation)."""
import numpy as np
import pytest

import bench
import paper_2309_02228_b200 as mpkg


def test_chain_flops_conventions():
    c = bench.CONFIGS
    assert bench.chain_flops(c["c4jac"], 100, 10) == 2.0 * 100 * 8 * 2
    assert bench.chain_flops(c["c4gs2"], 100, 10) == 8 * (1 * (200.0 + 100.0) + 200.0)
    assert bench.chain_flops(c["c4prod"], 100, 10) == 2.0 * 100 * 39
    with pytest.raises(ValueError):
        bench.chain_flops(c["c2"], 100, 10)


def test_leja_chebyshev_roots():
    r = bench.leja_chebyshev_roots(8, 0.5, 52.0)
    assert len(r) == 8 and len(set(r)) == 8
    assert abs(r[0]) == max(abs(v) for v in r)  # Leja order starts at the largest modulus
    assert all(0.5 <= v <= 52.0 for v in r)


@pytest.mark.parametrize("cfg", ["c4jac", "c4gs2", "c4prod"])
def test_port_chain_baseline_small(oracle, cfg):
    A = mpkg.poisson3d(8, 8, 8)
    lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
    P = oracle.permute(A.row_ptr, A.col_idx, A.values, pm)
    x = mpkg.random_vector(A.n_rows, 5)
    cb = bench.port_chain_baseline(bench.CONFIGS[cfg], P, x, 1)
    assert cb["kind"] == "port" and cb["cores"] == 1 and cb["value"] > 0 and cb["ms"] > 0


def test_port_ortho_baseline_small():
    cb = bench.port_ortho_baseline(bench.CONFIGS["c4ortho"], 5000, 7, 1)
    assert cb["kind"] == "port" and cb["value"] > 0


def test_newton_shifts_are_chebyshev_points():
    th = bench.newton_shifts(8)
    want = [26 + 26 * np.cos(np.pi * (2 * k - 1) / 16) for k in range(1, 9)]
    np.testing.assert_allclose(th, want, rtol=0, atol=0)
