"""Pins the CPU oracle (oracle/oracle.c) before it is trusted as the checker:
(1) against the golden fixtures generated from the reference itself (tests/golden/), and
(2) against the reference compiled in place (oracle/_ref) on fresh inputs, bit for bit, and
(3) against the literal known answers of the reference's own tests / SPEC examples."""
import numpy as np
import pytest

from conftest import assert_bitwise

LEV_CASES = ["tridiag5", "grid3x3", "poisson2d_20x17", "poisson3d_7x8x9", "random_spd_200_5_77",
             "random_csr_300_5_11", "diag6", "two_paths"] + [f"random_csr_120_4_{s}" for s in range(1, 6)]


@pytest.mark.parametrize("name", LEV_CASES)
def test_levels_and_permute_match_golden(oracle, golden, name):
    g = lambda k: golden[f"lev.{name}.{k}"]
    lv, pm, ip, lp = oracle.build_levels(g("rp"), g("ci"))
    for got, key in ((lv, "levels"), (pm, "perm"), (ip, "inv_perm"), (lp, "level_ptr")):
        np.testing.assert_array_equal(got, g(key), err_msg=key)
    prp, pci, pv = oracle.permute(g("rp"), g("ci"), g("v"), pm)
    np.testing.assert_array_equal(prp, g("prp"))
    np.testing.assert_array_equal(pci, g("pci"))
    assert_bitwise(pv, g("pv"), "values")
    assert oracle.validate_levels(prp, pci, lv, ip)


def test_known_answer_levels(oracle, golden):
    # test_levels.cpp:15-24 tridiagonal: 5 levels of one row, identity perm
    lv, pm, ip, lp = oracle.build_levels(golden["lev.tridiag5.rp"], golden["lev.tridiag5.ci"])
    assert list(np.diff(lp)) == [1] * 5 and list(pm) == list(range(5))
    # test_levels.cpp:26-33 3x3 grid -> [1,2,3,2,1]
    lp = oracle.build_levels(golden["lev.grid3x3.rp"], golden["lev.grid3x3.ci"])[3]
    assert list(np.diff(lp)) == [1, 2, 3, 2, 1]
    # test_levels.cpp:35-46 diagonal -> one level
    lp = oracle.build_levels(golden["lev.diag6.rp"], golden["lev.diag6.ci"])[3]
    assert list(lp) == [0, 6]
    # test_levels.cpp:58-72 two disjoint paths -> [2,2,1]
    lp = oracle.build_levels(golden["lev.two_paths.rp"], golden["lev.two_paths.ci"])[3]
    assert list(np.diff(lp)) == [2, 2, 1]


def test_validate_levels_detects_violation(oracle):
    # test_levels.cpp:95-107
    rp = np.array([0, 2, 3, 4, 5]); ci = np.array([0, 3, 1, 2, 3])
    ident = np.arange(4)
    assert not oracle.validate_levels(rp, ci, ident, ident)


def test_greedy_group_known_answers(oracle, golden):
    # test_levels.cpp:109-122
    assert oracle.greedy_group([1000] * 10, 2500) == [0, 2, 4, 6, 8, 10] == list(golden["greedy.a"])
    assert oracle.greedy_group([1000, 5000, 1000, 1000], 2500) == [0, 1, 2, 4] == list(golden["greedy.b"])
    assert oracle.greedy_group([10, 10, 10], 0) == [0, 1, 2, 3] == list(golden["greedy.c"])


def test_group_levels_matches_golden(oracle, golden):
    g = lambda k: golden[f"plan.poisson2d_64.{k}"]
    gr, glp, gfp, tgt = oracle.group_levels(g("level_ptr"), g("prp"), 100 * 1024, 4)
    np.testing.assert_array_equal(gr, g("group_rows"))
    np.testing.assert_array_equal(glp, g("group_level_ptr"))
    np.testing.assert_array_equal(gfp, g("group_footprint"))
    assert tgt == int(g("target")) == 100 * 1024 // 5
    with pytest.raises(ValueError):
        oracle.group_levels(g("level_ptr"), g("prp"), 1024, 0)


def test_wavefront_known_answer(oracle):
    # test_mpk.cpp:47-58 / SPEC.md:232
    assert oracle.wavefront_schedule(3, 2) == [(0, 1), (1, 1), (0, 2), (2, 1), (1, 2), (2, 2)]
    for ng in range(1, 11):
        for pm in range(1, 9):
            order = oracle.wavefront_schedule(ng, pm)
            assert len(order) == ng * pm and len(set(order)) == ng * pm
            done = set()
            for g, q in order:  # test_mpk.cpp:72-102 dependency audit
                if q > 1:
                    for nb in (g - 1, g, g + 1):
                        if 0 <= nb < ng:
                            assert (nb, q - 1) in done
                done.add((g, q))


def test_mpk_matches_golden(oracle, golden):
    g = lambda k: golden[f"mpk.poisson2d_12x9_p5.{k}"]
    assert_bitwise(oracle.baseline_mpk(g("rp"), g("ci"), g("v"), g("x"), 5), g("block"))
    for name in ("poisson2d_48x37", "poisson3d_9x10x11", "random_csr_2000_5_3"):
        for p in (1, 3, 6):
            h = lambda k: golden[f"mpk.{name}_p{p}.{k}"]
            prp, pci, pv = oracle.permute(h("rp"), h("ci"), h("v"), h("perm"))
            blk = oracle.mpk(prp, pci, pv, h("group_rows"), p, h("x"), p)
            assert_bitwise(blk, h("block"), f"{name} p={p} blocked")
            assert_bitwise(oracle.baseline_mpk(prp, pci, pv, h("x"), p), h("block"), "baseline")


def test_shifted_matches_golden(oracle, golden):
    g = lambda k: golden[f"shift.random_csr_150.{k}"]
    assert_bitwise(oracle.baseline_mpk_shifted(g("rp"), g("ci"), g("v"), g("x"), g("shifts")),
                   g("block"))
    h = lambda k: golden[f"shift.poisson2d_30.{k}"]
    prp, pci, pv = oracle.permute(h("rp"), h("ci"), h("v"), h("perm"))
    blk = oracle.mpk_shifted(prp, pci, pv, h("group_rows"), 5, h("x"), h("shifts"))
    assert_bitwise(blk, h("block"))
    assert_bitwise(oracle.baseline_mpk_shifted(prp, pci, pv, h("x"), h("shifts")), h("block"))


def test_shift_chain_rules(oracle):
    # test_mpk.cpp:208-222
    assert not oracle.check_shift_chain([1.0, 2.0 + 1.0j])
    assert not oracle.check_shift_chain([2.0 + 1.0j, 0.5, 2.0 - 1.0j])
    assert not oracle.check_shift_chain([2.0 - 1.0j, 2.0 + 1.0j, 0.0])
    assert oracle.check_shift_chain([0.4, 1.2 + 0.7j, 1.2 - 0.7j, -0.3])


def test_spec_examples(oracle):
    # SPEC.md:242 [[2,1],[0,3]], x=(1,1), p=2 -> (3,3), (9,9)
    blk = oracle.baseline_mpk([0, 2, 3], [0, 1, 1], [2.0, 1.0, 3.0], [1.0, 1.0], 2)
    assert blk[1].tolist() == [3.0, 3.0] and blk[2].tolist() == [9.0, 9.0]
    # SPEC.md:262 diag(1,3), lambda=2 -> (-1,1)
    blk = oracle.baseline_mpk_shifted([0, 1, 2], [0, 1], [1.0, 3.0], [1.0, 1.0], [2.0])
    assert blk[1].tolist() == [-1.0, 1.0]
    # SPEC.md:241 A=I -> y_p = x
    blk = oracle.baseline_mpk([0, 1, 2, 3], [0, 1, 2], [1.0] * 3, [1.0, 2.0, 3.0], 4)
    assert all(blk[p].tolist() == [1.0, 2.0, 3.0] for p in range(5))


def test_tune_select(oracle):
    # test_mpk.cpp:224-234
    assert oracle.tune_select([1.0, 1.8, 2.1, 2.0], 1, 4) == 3
    assert oracle.tune_select([1.0, 2.1, 1.5, 2.1], 1, 4) == 2


def test_dense_power_oracle(oracle, golden):
    """test_mpk.cpp:125-139: baseline vs a dense restatement, |d| <= 1e-13 max|ref|."""
    g = lambda k: golden[f"mpk.poisson2d_12x9_p5.{k}"]
    rp, ci, v, x = g("rp"), g("ci"), g("v"), g("x")
    n = len(rp) - 1
    D = np.zeros((n, n))
    for r in range(n):
        D[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    blk = oracle.baseline_mpk(rp, ci, v, x, 5)
    y = x.copy()
    for p in range(1, 6):
        y = D @ y
        assert np.max(np.abs(blk[p] - y)) <= 1e-13 * np.max(np.abs(y))


def test_oracle_vs_reference_fresh(oracle, ref):
    """Fresh (non-fixture) inputs: the restatement equals the reference bit for bit."""
    for args in [(5, 5000, 7, 0, 9), (4, 3000, 6, 0, 17), (3, 11, 9, 7)]:
        rp, ci, v = ref.gen(*args)
        a = oracle.build_levels(rp, ci)
        b = ref.build_levels(rp, ci, v)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)
        po = oracle.permute(rp, ci, v, a[1])
        pr = ref.permute(rp, ci, v, a[1])
        for x, y in zip(po, pr):
            np.testing.assert_array_equal(x, y)
        x = ref.random_vector(len(rp) - 1, 42)
        for p in (2, 5):
            gr = oracle.group_levels(a[3], po[0], 256 * 1024, p)
            np.testing.assert_array_equal(gr[0], ref.group_levels(*pr, a[3], 256 * 1024, p)[0])
            assert_bitwise(oracle.mpk(*po, gr[0], p, x, p), ref.mpk(*pr, gr[0], p, x, p, threads=4))


# ---- Jacobi chains (jacobi.hpp) -------------------------------------------
JAC_CASES = [f"{m}_s{s}" for m in ("random_spd_400_5_9", "poisson2d_17x13") for s in (1, 2, 4)]


@pytest.mark.parametrize("name", JAC_CASES)
def test_jacobi_matches_golden(oracle, golden, name):
    g = lambda k: golden[f"jac.{name}.{k}"]
    sw = int(name.rsplit("_s", 1)[1])
    pos, inv = oracle.diag_info(g("prp"), g("pci"), g("pv"))
    np.testing.assert_array_equal(pos, g("pos"))
    assert_bitwise(inv, g("inv"))
    assert_bitwise(oracle.jacobi_apply(g("prp"), g("pci"), g("pv"), sw, g("x")), g("apply"))
    y = oracle.jacobi_op(g("prp"), g("pci"), g("pv"), sw, g("x"))
    assert_bitwise(y, g("op"))
    assert_bitwise(y, g("op_blocked"))  # jacobi.hpp:196: the blocked twin is bitwise equal


def test_jacobi_setup_errors(oracle):
    # jacobi.hpp:48-64: non-square -> invalid_argument; missing / zero diagonal -> runtime_error
    with pytest.raises(ValueError):
        oracle.diag_info([0, 1], [0], [1.0], n_cols=2)
    with pytest.raises(RuntimeError):
        oracle.diag_info([0, 1, 2], [1, 0], [1.0, 1.0])  # no diagonal at all
    with pytest.raises(RuntimeError):
        oracle.diag_info([0, 1, 2], [0, 1], [2.0, 0.0])  # zero diagonal


def test_sstep_jacobi_chain_composition(oracle, golden):
    """The s-step Jacobi chain (sstep.hpp:122-157, which needs Eigen and cannot be compiled here)
    is pinned by composition: zero shifts give jacobi_op applied s times (pinned above against
    the compiled jacobi.hpp), and the shift terms follow mpk.hpp's shifted rows."""
    g = lambda k: golden[f"jac.random_spd_400_5_9_s2.{k}"]
    rp, ci, v, x = g("prp"), g("pci"), g("pv"), g("x")
    for sw in (1, 2, 3):
        blk = oracle.sstep_jacobi_block(rp, ci, v, sw, x, [0.0] * 4)
        y = x.copy()
        for p in range(1, 5):
            y = oracle.jacobi_op(rp, ci, v, sw, y)
            assert_bitwise(blk[p], y, f"sweeps={sw} p={p}")
        sh = [0.5, 1.5 + 0.5j, 1.5 - 0.5j, 2.0]
        blk = oracle.sstep_jacobi_block(rp, ci, v, sw, x, sh)
        w = [x]
        for p, s in enumerate(sh, 1):
            t = oracle.jacobi_op(rp, ci, v, sw, w[p - 1])
            b2 = s.imag ** 2 if s.imag < 0 else 0.0
            nxt = t - s.real * w[p - 1]
            if b2 != 0.0:
                nxt = nxt + b2 * w[p - 2]
            w.append(nxt)
            assert_bitwise(blk[p], nxt, f"shifted sweeps={sw} p={p}")
    with pytest.raises(ValueError):
        oracle.sstep_jacobi_block(rp, ci, v, 1, x, [1.0 - 1.0j, 1.0 + 1.0j])


def test_jacobi_oracle_vs_reference_fresh(oracle, ref):
    for args in [(5, 3000, 6, 0, 4), (3, 8, 9, 10), (4, 700, 5, 0, 8)]:
        rp, ci, v = ref.gen(*args)
        x = ref.random_vector(len(rp) - 1, 42)
        for sw in (1, 3):
            assert_bitwise(oracle.jacobi_apply(rp, ci, v, sw, x), ref.jacobi_apply(rp, ci, v, sw, x))
            assert_bitwise(oracle.jacobi_op(rp, ci, v, sw, x), ref.jacobi_op(rp, ci, v, sw, x))


# ---- GS2 chains (gs2.hpp) -------------------------------------------------------------------------
GS2_CASES = ["g0_k1_f1", "g2_k2_f1", "g3_k2_f0"]


@pytest.mark.parametrize("name", GS2_CASES)
def test_gs2_matches_golden(oracle, golden, name):
    g = lambda k: golden[f"gs2.{name}.{k}"]
    gamma, K, fw = (int(t[1:]) for t in name.split("_"))
    for mode in ("smooth", "apply", "smooth_residual", "op"):
        z, out = oracle.gs2(g("prp"), g("pci"), g("pv"), gamma, K, bool(fw), mode, g("x"), g("z0"))
        if mode != "op":
            assert_bitwise(z, g(f"{mode}_z"), mode)
        if out is not None:
            assert_bitwise(out, g(f"{mode}_out"), mode)


def test_sstep_gs2_chain_composition(oracle, golden):
    """sstep.hpp:160-198 (Eigen-dependent header) pinned by composition: zero shifts give gs2_op
    applied s times; shift terms as mpk.hpp's shifted rows."""
    g = lambda k: golden[f"gs2.g2_k2_f1.{k}"]
    rp, ci, v, x = g("prp"), g("pci"), g("pv"), g("x")
    for gamma, K, fw in ((0, 1, True), (2, 2, True), (1, 3, False)):
        sh = [0.5, 1.5 + 0.5j, 1.5 - 0.5j, 2.0]
        blk = oracle.sstep_gs2_block(rp, ci, v, gamma, K, fw, x, sh)
        w = [x]
        for p, s in enumerate(sh, 1):
            _, t = oracle.gs2(rp, ci, v, gamma, K, fw, "op", w[p - 1])
            nxt = t - s.real * w[p - 1]
            if s.imag < 0:
                nxt = nxt + (s.imag ** 2) * w[p - 2]
            w.append(nxt)
            assert_bitwise(blk[p], nxt, f"gamma={gamma} K={K} p={p}")


def test_from_coo_oracle_vs_reference(oracle, ref):
    """csr.hpp:72-110: stable sort, input-order duplicate sums from 0.0 (-0.0 alone -> +0.0)."""
    rng = np.random.default_rng(8)
    for _ in range(20):
        nr, nc = int(rng.integers(1, 80)), int(rng.integers(1, 80))
        m = int(rng.integers(0, 600))
        r = rng.integers(0, nr, m).astype(np.uint32)
        c = rng.integers(0, nc, m).astype(np.uint32)
        v = rng.choice([-0.0, 1.0, -1.0, 2.5, 1e-300], m) * rng.uniform(0.5, 2, m)
        a = oracle.from_coo(nr, nc, r, c, v)
        b = ref.from_coo(nr, nc, r, c, v)
        np.testing.assert_array_equal(a[0], b[2])
        np.testing.assert_array_equal(a[1], b[3])
        assert_bitwise(a[2], b[4])
    with pytest.raises(ValueError):
        oracle.from_coo(2, 2, [0, 2], [0, 0], [1.0, 1.0])


# ---- product-form polynomial (poly.hpp:146-281; the header needs Eigen, absent here) -------------
def _dense(rp, ci, v, n):
    D = np.zeros((n, n))
    for r in range(n):
        for k in range(rp[r], rp[r + 1]):
            D[r, ci[k]] += v[k]
    return D


def test_poly_known_answers(oracle):
    # test_poly.cpp:150-167 ScaledIdentityDegreeOne: root 2 on diag(2,2): z = v / 2 exactly
    z = oracle.poly_apply([0, 1, 2], [0, 1], [2.0, 2.0], [2.0], [4.0, 6.0])
    assert z.tolist() == [2.0, 3.0]
    with pytest.raises(ValueError):  # poly.hpp:85-87: pair members must be adjacent conjugates
        oracle.poly_apply([0, 1, 2], [0, 1], [2.0, 2.0], [1.0 + 1.0j, 2.0], [1.0, 1.0])


@pytest.mark.parametrize("case", ["diag", "complex_pair"])
def test_poly_exact_on_known_spectrum(oracle, case):
    """Roots = the exact spectrum: the GMRES polynomial inverts A, i.e. A z = v (test_poly.cpp:
    187-215 restated with the roots given instead of computed by the Eigen-based setup), and more
    generally A z = v - prod_i (I - A / theta_i) v for any roots."""
    if case == "diag":
        eigs = [1.0, 2.5, 3.0, 4.2, 5.0, 6.7]
        n = 12
        d = [eigs[i % 6] for i in range(n)]
        rp, ci, v = list(range(n + 1)), list(range(n)), d
        roots = [6.7, 1.0, 5.0, 2.5, 4.2, 3.0]
    else:  # eigenvalues 1 +- 2i and 3 (test_poly.cpp:202-215)
        rp, ci, v = [0, 2, 4, 5], [0, 1, 0, 1, 2], [1.0, -2.0, 2.0, 1.0, 3.0]
        n = 3
        roots = [3.0, 1.0 + 2.0j, 1.0 - 2.0j]
    A = _dense(rp, ci, v, n)
    x = np.linspace(-1.0, 1.3, n)
    z = oracle.poly_apply(rp, ci, v, roots, x)
    assert np.max(np.abs(A @ z - x)) <= 1e-10 * np.max(np.abs(x))
    # the residual-polynomial identity with arbitrary (non-spectral) roots
    roots2 = [0.7, 2.0 + 0.5j, 2.0 - 0.5j, 4.0]
    z2 = oracle.poly_apply(rp, ci, v, roots2, x)
    R = x.astype(complex)
    for th in roots2:
        R = R - (A @ R) / th
    assert np.max(np.abs(A @ z2 - (x - R.real))) <= 1e-12 * max(1.0, np.max(np.abs(x)))


def test_poly_inner_preconditioned_identity(oracle):
    """Inner Jacobi / GS2: the same identity for the combined operator A M^{-1} (M^{-1} from the
    pinned jacobi_apply / gs2 stages)."""
    A_ = __import__("paper_2309_02228_b200").random_spd(60, 4, 17)
    rp, ci, v = A_.row_ptr, A_.col_idx, A_.values
    n = A_.n_rows
    A = _dense(rp, ci, v, n)
    x = np.cos(0.3 * np.arange(n))
    roots = [0.9, 1.6 + 0.4j, 1.6 - 0.4j, 0.5, 1.2]
    for inner, kw in (("jacobi", dict(sweeps=1)), ("jacobi", dict(sweeps=3)),
                      ("gs2", dict(gamma=0)), ("gs2", dict(gamma=2, forward=False))):
        z = oracle.poly_apply(rp, ci, v, roots, x, inner=inner, **kw)

        def minv(y):
            if inner == "jacobi":
                return oracle.jacobi_apply(rp, ci, v, kw["sweeps"], y)
            return oracle.gs2(rp, ci, v, kw["gamma"], 1, kw.get("forward", True), "apply", y)[0]

        R = x.astype(complex)
        for th in roots:
            op = (A @ minv(R.real)) + 1j * (A @ minv(R.imag))
            R = R - op / th
        lhs = A @ minv(z)
        assert np.max(np.abs(lhs - (x - R.real))) <= 1e-11 * max(1.0, np.max(np.abs(x))), inner
