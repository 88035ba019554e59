"""GPU parity: every output of the sm_100a path against the pinned CPU oracle, bit for bit.

Restates the reference's hot-path tests (proj/tests/test_levels.cpp, test_mpk.cpp,
acceptance.cpp C1-C3) against the mpkg C ABI.  Levels/perm/inv_perm/level_ptr/A_perm must be
bit-identical; basis vectors are bitwise equal in MPKG_MODE_BITWISE (the north star's 1e-12
inf-norm tolerance is the looser bar, asserted too where stated)."""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu


def corpus():
    """The acceptance C1/C2 corpus (acceptance.cpp:118-160) plus irregular / scrambled cases."""
    return {
        "poisson1d_1000": mpkg.poisson1d(1000),
        "poisson2d_256": mpkg.poisson2d(256, 256),
        "poisson3d_32": mpkg.poisson3d(32, 32, 32),
        "random_spd_50k": mpkg.random_spd(50000, 5, 777),
        "random_spd_4000": mpkg.random_spd(4000, 6, 123),
        "random_csr_2000": mpkg.random_csr(2000, 5, 3),  # nonsymmetric pattern
        "stencil27_scrambled_20": mpkg.scramble(mpkg.stencil27_random_sym(20, 20, 20, 1), 2),
        "rmat_12": mpkg.rmat(12, 8, 3),
    }


@pytest.fixture(scope="module")
def cases(oracle):
    out = {}
    for name, A in corpus().items():
        lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
        prp, pci, pv = oracle.permute(A.row_ptr, A.col_idx, A.values, pm)
        out[name] = dict(A=A, levels=lv, perm=pm, inv_perm=ip, level_ptr=lp,
                         P=mpkg.HostCsr.from_arrays(prp, pci, pv))
    return out


# ---- level engine -----------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tridiag5", "grid3x3", "poisson2d_20x17", "poisson3d_7x8x9",
                                  "random_spd_200_5_77", "random_csr_300_5_11", "diag6",
                                  "two_paths"] + [f"random_csr_120_4_{s}" for s in range(1, 6)])
def test_levels_golden(ctx, golden, name):
    g = lambda k: golden[f"lev.{name}.{k}"]
    A = ctx.csr(mpkg.HostCsr.from_arrays(g("rp"), g("ci"), g("v")))
    ls = ctx.build_levels(A)
    for key in ("levels", "perm", "inv_perm", "level_ptr"):
        np.testing.assert_array_equal(getattr(ls, key), g(key), err_msg=key)
    P = ctx.permute(A, ls).download()
    np.testing.assert_array_equal(P.row_ptr, g("prp"))
    np.testing.assert_array_equal(P.col_idx, g("pci"))
    assert_bitwise(P.values, g("pv"))
    assert ctx.validate_levels(ctx.csr(P), ls)


def test_levels_corpus_bit_exact(ctx, cases):
    for name, c in cases.items():
        A = ctx.csr(c["A"])
        ls = ctx.build_levels(A)
        for key in ("levels", "perm", "inv_perm", "level_ptr"):
            np.testing.assert_array_equal(getattr(ls, key), c[key], err_msg=f"{name} {key}")
        P = ctx.permute(A, ls).download()
        np.testing.assert_array_equal(P.row_ptr, c["P"].row_ptr, err_msg=name)
        np.testing.assert_array_equal(P.col_idx, c["P"].col_idx, err_msg=name)
        assert_bitwise(P.values, c["P"].values, name)
        # host-perm permute path (csr.hpp:159 signature) agrees too
        P2 = ctx.permute(A, c["perm"]).download()
        np.testing.assert_array_equal(P2.col_idx, c["P"].col_idx)
        assert ctx.validate_levels(ctx.csr(c["P"]), ls)


def test_validate_levels_detects_violation(ctx):
    # test_levels.cpp:95-107
    A = ctx.csr(mpkg.HostCsr.from_arrays([0, 2, 3, 4, 5], [0, 3, 1, 2, 3], [1.0] * 5))
    ident = np.arange(4)
    fake = ctx.levels_from_host(ident, ident, ident, [0, 1, 2, 3, 4])
    assert not ctx.validate_levels(A, fake)


def test_permute_rejects_non_permutation(ctx):
    A = ctx.csr(mpkg.poisson1d(5))
    with pytest.raises(ValueError):
        ctx.permute(A, [0, 1, 2, 2, 4])
    with pytest.raises(ValueError):
        ctx.permute(A, [0, 1, 2, 3, 7])
    with pytest.raises(ValueError):
        ctx.build_levels(ctx.csr(mpkg.HostCsr.from_arrays([0, 1], [1], [1.0], n_cols=2)))


def test_permute_vector_roundtrip(ctx, oracle):
    rng = np.random.default_rng(0)
    perm = rng.permutation(1000).astype(np.uint32)
    v = rng.standard_normal(1000)
    pv = ctx.permute_vector(v, perm)
    assert_bitwise(pv[perm], v)
    assert_bitwise(ctx.unpermute_vector(pv, perm), v)


def test_group_levels_golden(ctx, golden, oracle):
    g = lambda k: golden[f"plan.poisson2d_64.{k}"]
    A = ctx.csr(mpkg.poisson2d(64, 64))
    ls = ctx.build_levels(A)
    Ap = ctx.permute(A, ls)
    plan = ctx.group_levels(ls, Ap, 100 * 1024, 4)
    np.testing.assert_array_equal(plan.group_rows, g("group_rows"))
    np.testing.assert_array_equal(plan.group_level_ptr, g("group_level_ptr"))
    np.testing.assert_array_equal(plan.group_footprint, g("group_footprint"))
    assert plan.target_bytes == 100 * 1024 // 5
    # test_levels.cpp:124-147 plan invariants
    for gi in range(plan.n_groups()):
        assert plan.group_footprint[gi] == ctx.row_range_footprint(
            Ap, int(plan.group_rows[gi]), int(plan.group_rows[gi + 1]), 4)
        if plan.group_footprint[gi] > plan.target_bytes:
            assert plan.group_level_ptr[gi + 1] - plan.group_level_ptr[gi] == 1
    with pytest.raises(ValueError):
        ctx.group_levels(ls, Ap, 1024, 0)  # test_levels.cpp:149-155
    with pytest.raises(ValueError):
        ctx.group_levels(ls, ctx.csr(mpkg.poisson1d(11)), 1024, 2)


def test_group_levels_corpus(ctx, cases, oracle):
    for name, c in cases.items():
        ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
        Ap = ctx.csr(c["P"])
        for cache, p in ((1 << 20, 3), (64 << 10, 8), (1 << 30, 1)):
            plan = ctx.group_levels(ls, Ap, cache, p)
            gr, glp, gfp, tgt = oracle.group_levels(c["level_ptr"], c["P"].row_ptr, cache, p)
            np.testing.assert_array_equal(plan.group_rows, gr, err_msg=name)
            np.testing.assert_array_equal(plan.group_footprint, gfp, err_msg=name)


# ---- power kernels ----------------------------------------------------------------------------
def test_spmv_and_baseline_golden(ctx, golden):
    g = lambda k: golden[f"mpk.poisson2d_12x9_p5.{k}"]
    A = ctx.csr(mpkg.HostCsr.from_arrays(g("rp"), g("ci"), g("v")))
    blk = ctx.baseline_mpk(A, g("x"), 5)
    assert_bitwise(blk.as_matrix(), g("block"))
    assert_bitwise(ctx.spmv(A, g("x")), g("block")[1])


@pytest.mark.parametrize("name", ["poisson2d_48x37", "poisson3d_9x10x11", "random_csr_2000_5_3"])
@pytest.mark.parametrize("p", [1, 3, 6])
def test_fused_mpk_golden(ctx, golden, name, p):
    h = lambda k: golden[f"mpk.{name}_p{p}.{k}"]
    A = ctx.csr(mpkg.HostCsr.from_arrays(h("rp"), h("ci"), h("v")))
    ls = ctx.build_levels(A)
    np.testing.assert_array_equal(ls.perm, h("perm"))
    Ap = ctx.permute(A, ls)
    plan = ctx.group_levels(ls, Ap, 64 * 1024, p)
    np.testing.assert_array_equal(plan.group_rows, h("group_rows"))
    assert_bitwise(ctx.mpk(plan, Ap, h("x"), p).as_matrix(), h("block"), "fused")
    assert_bitwise(ctx.baseline_mpk(Ap, h("x"), p).as_matrix(), h("block"), "baseline")


def test_fused_mpk_corpus_all_p(ctx, cases, oracle):
    """acceptance.cpp C1: blocked == baseline bitwise, corpus x p 1..8 (here both GPU paths also
    equal the oracle)."""
    for name, c in cases.items():
        P = c["P"]
        Ap = ctx.csr(P)
        ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
        x = mpkg.random_vector(P.n_rows, 42)
        ref8 = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 8)
        for p in range(1, 9):
            plan = ctx.group_levels(ls, Ap, 1 << 20, p)
            assert_bitwise(ctx.mpk(plan, Ap, x, p).as_matrix(), ref8[: p + 1], f"{name} p={p}")
        assert_bitwise(ctx.baseline_mpk(Ap, x, 8).as_matrix(), ref8, f"{name} baseline")


DEFAULT_KNOBS = {"order": -1, "slack": -1, "schedule": 0, "kernel": 0, "tile_rows": 128,
                 "producers": 0, "cgroups": 0, "stages": 0, "pass": 0, "l2_budget": 0, "ctas_per_sm": 0,
                 "wave_dict": 1, "wave_affine": 2}

SCHEDULES = {
    "sweeps": {"schedule": 2},
    "wave": {"schedule": 3},
    "wave-plain": {"schedule": 3, "wave_dict": 0},
    "wave-noaffine": {"schedule": 3, "wave_affine": 0},
    "wave-affine-only": {"schedule": 3, "wave_affine": 1},
    "wave-1cta": {"schedule": 3, "ctas_per_sm": 1},
    "wave-pass1": {"schedule": 3, "pass": 1},
    "wave-pass2-slack1": {"schedule": 3, "pass": 2, "slack": 1},
    "wave-pass6-tiny-budget": {"schedule": 3, "pass": 6, "slack": 0, "l2_budget": 4096},
    "fused-lean": {"schedule": 1},
    "fused-lean-slack0": {"schedule": 1, "slack": 0},
    "fused-lean-slack1": {"schedule": 1, "slack": 1},
    "fused-lean-slack7": {"schedule": 1, "slack": 7},
    "fused-lean-tile64": {"schedule": 1, "tile_rows": 64},
    "fused-staged": {"schedule": 1, "kernel": 1},
    "fused-warptile": {"schedule": 1, "kernel": 2},
    "fused-async": {"schedule": 1, "kernel": 4},
    "fused-async-tile32": {"schedule": 1, "kernel": 4, "tile_rows": 32, "producers": 2, "cgroups": 4},
    "fused-async-tile64": {"schedule": 1, "kernel": 4, "tile_rows": 64, "producers": 8},
}


def set_knobs(ctx, knobs):
    for k, v in {**DEFAULT_KNOBS, **knobs}.items():
        ctx.set_param(k, v)


@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("sched", list(SCHEDULES))
def test_orders_and_schedules(ctx, cases, oracle, order, sched):
    """Every private row order (A_perm / Cuthill-McKee / longest-first inside levels), schedule
    (one launch per power, or the fused tile-DAG kernel with any ticket slack) and fused-kernel
    variant gives the same bits: they change only which rows run where and when."""
    try:
        set_knobs(ctx, {"order": order, **SCHEDULES[sched]})
        for name in ("stencil27_scrambled_20", "random_csr_2000", "rmat_12", "poisson2d_256"):
            c = cases[name]
            P = c["P"]
            Ap = ctx.csr(P)
            ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
            x = mpkg.random_vector(P.n_rows, 9)
            plan = ctx.group_levels(ls, Ap, 1 << 20, 6)
            ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 6)
            assert_bitwise(ctx.mpk(plan, Ap, x, 6).as_matrix(), ref, f"{name} {sched} order={order}")
            info = plan.exec_info()
            assert_bitwise(ctx.mpk(plan, Ap, x, 6).as_matrix(), ref, f"{name} {sched} order={order} again")
            assert info["order"] == order
            want = ("sweeps" if sched == "sweeps" else
                    ("sweeps" if info["long_rows"] else "wave") if sched.startswith("wave") else "fused")
            assert info["schedule"] == want
            sh = [0.5, 1.0 + 2.0j, 1.0 - 2.0j, -1.0, 3.0, 0.25]
            ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
            assert_bitwise(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref, f"{name} shifted")
            coef = np.linspace(-1, 1, 7)
            zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
            assert_bitwise(ctx.mpk_poly(plan, Ap, x, coef), zr, f"{name} poly")
    finally:
        set_knobs(ctx, {})


def _arrow_matrix(n=6000, hubs=(0, 17, 2500), seed=5):
    """Tridiagonal band plus a few dense hub rows/columns (rows far longer than the SELL long-row
    cap), symmetric pattern."""
    rng = np.random.default_rng(seed)
    rows = {i: {i: 4.0} for i in range(n)}
    for i in range(n - 1):
        rows[i][i + 1] = rows[i + 1][i] = -1.0
    for h in hubs:
        for j in rng.choice(n, size=n // 2, replace=False):
            if j != h:
                v = -float(rng.uniform(0.1, 1.0))
                rows[h][int(j)] = v
                rows[int(j)][h] = v
    rp, ci, vv = [0], [], []
    for i in range(n):
        for j in sorted(rows[i]):
            ci.append(j)
            vv.append(rows[i][j])
        rp.append(len(ci))
    return mpkg.HostCsr.from_arrays(rp, ci, vv)


@pytest.mark.parametrize("schedule", [0, 1, 2])
@pytest.mark.parametrize("order", [-1, 0, 1, 2])
def test_long_rows_and_length_order(ctx, oracle, order, schedule):
    """Hub rows (>1024 entries) are added in stored order by a CTA each: beside the sweeps on a
    side stream (auto / schedule=2, k_long_rows_bitwise) or inside the fused kernel (schedule=1).
    Every order and schedule gives the reference's bits, on the host- and device-pointer paths."""
    import torch
    try:
        set_knobs(ctx, {"order": order, "schedule": schedule})
        for A in (_arrow_matrix(), mpkg.rmat(15, 16, 7)):
            lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
            P = mpkg.HostCsr.from_arrays(*oracle.permute(A.row_ptr, A.col_idx, A.values, pm))
            assert np.diff(P.row_ptr.astype(np.int64)).max() > 1024
            Ap = ctx.csr(P)
            ls = ctx.levels_from_host(lv, pm, ip, lp)
            x = mpkg.random_vector(P.n_rows, 3)
            plan = ctx.group_levels(ls, Ap, 8 << 20, 4)
            ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 4)
            assert_bitwise(ctx.mpk(plan, Ap, x, 4).as_matrix(), ref, f"order={order}")
            info = plan.exec_info()
            if order != 0:  # the private-order SELL leaves hub rows out: CTA-cooperative path
                assert info["long_rows"] > 0
            want = "fused" if schedule == 1 else "sweeps"
            assert info["schedule"] == want
            n = P.n_rows
            d_x = torch.from_numpy(x).cuda()
            d_b = torch.full((5 * n,), float("nan"), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()  # torch's stream is not ordered with the context's stream
            for _ in range(2):  # capture, then replay
                ctx.mpk_dev(plan, Ap, d_x.data_ptr(), 4, d_b.data_ptr(), n, 5)
                ctx.synchronize()
                assert_bitwise(d_b.view(5, n).cpu().numpy(), ref, f"device path order={order}")
            sh = [1.0, 2.0 + 0.5j, 2.0 - 0.5j, 0.5]
            ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
            assert_bitwise(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref, "shifted")
            coef = [0.5, -1.0, 0.25, 2.0, -0.125]
            zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
            assert_bitwise(ctx.mpk_poly(plan, Ap, x, coef), zr, "poly")
    finally:
        set_knobs(ctx, {})


def _rel_inf_err(got, ref):
    """max|got - ref| / max|ref| per basis vector (the north star's 1e-12 bar)."""
    got, ref = np.atleast_2d(got), np.atleast_2d(ref)
    return [float(np.abs(g - r).max() / max(np.abs(r).max(), 1e-300)) for g, r in zip(got, ref)]


@pytest.mark.parametrize("schedule", [0, 1])
def test_fast_mode_long_rows_within_tolerance(ctx, oracle, schedule):
    """MPKG_MODE_FAST reduces hub rows in parallel (sweep schedule) -- or, with the fused
    schedule forced, keeps the stored-order path: every basis vector within 1e-12 of the oracle
    in the inf-norm relative sense, run-to-run deterministic, and the baseline still bitwise."""
    try:
        set_knobs(ctx, {"schedule": schedule})
        ctx.set_mode(ctx.MODE_FAST)
        for A in (_arrow_matrix(), mpkg.rmat(15, 16, 7)):
            lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
            P = mpkg.HostCsr.from_arrays(*oracle.permute(A.row_ptr, A.col_idx, A.values, pm))
            Ap = ctx.csr(P)
            ls = ctx.levels_from_host(lv, pm, ip, lp)
            x = mpkg.random_vector(P.n_rows, 3)
            plan = ctx.group_levels(ls, Ap, 8 << 20, 4)
            ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 4)
            got = ctx.mpk(plan, Ap, x, 4).as_matrix()
            errs = _rel_inf_err(got, ref)
            assert max(errs) <= 1e-12, errs
            assert_bitwise(ctx.mpk(plan, Ap, x, 4).as_matrix(), got, "deterministic")
            info = plan.exec_info()
            assert info["schedule"] == ("fused" if schedule == 1 else "sweeps")
            if schedule == 1:
                assert_bitwise(got, ref, "fused keeps stored order")
            sh = [1.0, 2.0 + 0.5j, 2.0 - 0.5j, 0.5]
            ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
            assert max(_rel_inf_err(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref)) <= 1e-12
            coef = [0.5, -1.0, 0.25, 2.0, -0.125]
            zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
            assert max(_rel_inf_err(ctx.mpk_poly(plan, Ap, x, coef), zr)) <= 1e-12
            assert_bitwise(ctx.baseline_mpk(Ap, x, 4).as_matrix(),
                           oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 4), "baseline")
    finally:
        ctx.set_mode(ctx.MODE_BITWISE)
        set_knobs(ctx, {})


@pytest.mark.parametrize("order", [-1, 0])
def test_fast_mode_coop_rows_graph_and_host_paths(ctx, oracle, order):
    """Fast-mode sweeps send rows longer than 128 entries to k_coop_rows on a side stream (hub rows
    split into 2048-entry items, partials added in order by k_coop_finish).  The device-pointer
    call (CUDA-graph replay) and the host-pointer call (eager, streamed copies) agree bit for bit,
    repeat bit for bit, and stay within 1e-12 of the oracle; A_perm order (order=0) too."""
    import torch
    try:
        set_knobs(ctx, {"order": order})
        ctx.set_mode(ctx.MODE_FAST)
        for A in (_arrow_matrix(), mpkg.rmat(14, 16, 11)):
            lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
            P = mpkg.HostCsr.from_arrays(*oracle.permute(A.row_ptr, A.col_idx, A.values, pm))
            Ap = ctx.csr(P)
            ls = ctx.levels_from_host(lv, pm, ip, lp)
            n, p = P.n_rows, 5
            x = mpkg.random_vector(n, 9)
            plan = ctx.group_levels(ls, Ap, 8 << 20, p)
            ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, p)
            host = ctx.mpk(plan, Ap, x, p).as_matrix().copy()
            assert max(_rel_inf_err(host, ref)) <= 1e-12
            d_x = torch.from_numpy(x).cuda()
            d_b = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
            for _ in range(2):  # capture, then replay
                d_b.fill_(float("nan"))
                torch.cuda.synchronize()  # torch's stream is not ordered with the context's stream
                ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_b.data_ptr(), n, p + 1)
                ctx.synchronize()
                assert_bitwise(d_b.view(p + 1, n).cpu().numpy(), host, "graph == host path")
            sh = [1.0, 2.0 + 0.5j, 2.0 - 0.5j, 0.5, 3.0]
            ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
            assert max(_rel_inf_err(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref)) <= 1e-12
            assert plan.exec_info()["schedule"] == "sweeps"
    finally:
        ctx.set_mode(ctx.MODE_BITWISE)
        set_knobs(ctx, {})


@pytest.mark.parametrize("name", ["poisson3d_32", "stencil27_scrambled_20", "random_csr_2000",
                                  "random_spd_50k"])
def test_resident_single_launch_matches_oracle(ctx, cases, oracle, name):
    """L2-resident matrices run all p powers in one cooperative launch (grid barrier between
    powers) on the device-pointer path: plain, shifted (with a conjugate pair) and polynomial
    results bit-identical to the oracle and to the per-power graph path (resident=0)."""
    import torch
    c = cases[name]
    P = c["P"]
    Ap = ctx.csr(P)
    ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
    n, p = P.n_rows, 6
    x = mpkg.random_vector(n, 21)
    d_x = torch.from_numpy(x).cuda()
    sh = [1.5, 2.0 + 0.5j, 2.0 - 0.5j, 0.25, -1.0, 3.0]
    coef = [0.5, -1.0, 0.25, 2.0, -0.125, 1.0, 0.75]
    refs = {"plain": oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, p),
            "shifted": oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)}
    zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
    try:
        for resident in (1, 0, 1):
            ctx.set_param("resident", resident)
            plan = ctx.group_levels(ls, Ap, 8 << 20, p)
            for kind in ("plain", "shifted", "poly"):
                d_b = torch.full(((p + 1) * n,), float("nan"), dtype=torch.float64, device="cuda")
                d_z = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
                torch.cuda.synchronize()  # torch's stream is not ordered with the context's stream
                if kind == "plain":
                    ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_b.data_ptr(), n, p + 1)
                elif kind == "shifted":
                    ctx.mpk_shifted_dev(plan, Ap, d_x.data_ptr(), sh, d_b.data_ptr(), n, p + 1)
                else:
                    ctx.mpk_poly_dev(plan, Ap, d_x.data_ptr(), coef, d_z.data_ptr(), d_b.data_ptr(), n, p + 1)
                ctx.synchronize()
                if kind == "poly":
                    assert_bitwise(d_z.cpu().numpy(), zr, f"{name} poly resident={resident}")
                    assert_bitwise(d_b.view(p + 1, n).cpu().numpy(), refs["plain"], "poly block")
                else:
                    assert_bitwise(d_b.view(p + 1, n).cpu().numpy(), refs[kind], f"{name} {kind} resident={resident}")
            assert plan.exec_info()["schedule"] == "sweeps"
    finally:
        ctx.set_param("resident", 0)
        set_knobs(ctx, {})


@pytest.mark.parametrize("name", ["poisson3d_32", "stencil27_scrambled_20"])
def test_long_chains_run_in_segments(ctx, cases, oracle, name):
    """p above the executor's 32 powers per call runs segment by segment (each from the previous
    segment's last slice): plain and shifted bases of 45 powers, with a conjugate pair straddling
    the segment boundary, are bit-identical to the oracle on the host- and device-pointer paths."""
    import torch
    c = cases[name]
    P = c["P"]
    Ap = ctx.csr(P)
    ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
    n, p = P.n_rows, 45
    x = mpkg.random_vector(n, 13)
    plan = ctx.group_levels(ls, Ap, 8 << 20, p)
    # values grow like 12^45 (finite in fp64); the bits must match the oracle's arithmetic
    ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, p)
    assert_bitwise(ctx.mpk(plan, Ap, x, p).as_matrix(), ref, "plain host path")
    d_x = torch.from_numpy(x).cuda()
    d_b = torch.full(((p + 1) * n,), float("nan"), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_b.data_ptr(), n, p + 1)
    ctx.synchronize()
    assert_bitwise(d_b.view(p + 1, n).cpu().numpy(), ref, "plain device path")
    sh = [4.0 + 0.1 * k for k in range(31)] + [3.0 + 0.5j, 3.0 - 0.5j] + [2.0 + 0.05 * k for k in range(12)]
    assert len(sh) == p and sh[31].imag > 0  # the pair occupies powers 32 and 33
    ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
    assert_bitwise(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref, "shifted, pair across the boundary")


def test_fused_repeatable_and_plan_reuse(ctx, cases):
    c = cases["stencil27_scrambled_20"]
    Ap = ctx.csr(c["P"])
    ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
    plan = ctx.group_levels(ls, Ap, 1 << 20, 8)
    x = mpkg.random_vector(Ap.n_rows, 7)
    first = ctx.mpk(plan, Ap, x, 8).as_matrix().copy()
    for p in (8, 5, 8, 2):  # p below the plan budget reuses the plan (execute.hpp:74-83)
        assert_bitwise(ctx.mpk(plan, Ap, x, p).as_matrix(), first[: p + 1])
    info = plan.exec_info()
    assert info["tiles"] == (Ap.n_rows + 127) // 128


def test_shifted_golden(ctx, golden):
    g = lambda k: golden[f"shift.random_csr_150.{k}"]
    A = ctx.csr(mpkg.HostCsr.from_arrays(g("rp"), g("ci"), g("v")))
    assert_bitwise(ctx.baseline_mpk_shifted(A, g("x"), g("shifts")).as_matrix(), g("block"))
    h = lambda k: golden[f"shift.poisson2d_30.{k}"]
    A = ctx.csr(mpkg.HostCsr.from_arrays(h("rp"), h("ci"), h("v")))
    ls = ctx.build_levels(A)
    Ap = ctx.permute(A, ls)
    plan = ctx.group_levels(ls, Ap, 16 * 1024, 5)
    assert_bitwise(ctx.mpk_shifted(plan, Ap, h("x"), h("shifts")).as_matrix(), h("block"))


def test_newton_basis_config4_shape(ctx, oracle):
    """C4's Newton basis (real Chebyshev shifts on [0,52]) on a reduced 27-point grid."""
    A = mpkg.stencil27(24, 24, 24)
    lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
    P = mpkg.HostCsr.from_arrays(*oracle.permute(A.row_ptr, A.col_idx, A.values, pm))
    Ap = ctx.csr(P)
    ls = ctx.levels_from_host(lv, pm, ip, lp)
    theta = [26 + 26 * np.cos(np.pi * (2 * k - 1) / 16) for k in range(1, 9)]
    x = mpkg.random_vector(P.n_rows, 5)
    plan = ctx.group_levels(ls, Ap, 32 << 20, 8)
    ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, theta)
    assert_bitwise(ctx.mpk_shifted(plan, Ap, x, theta).as_matrix(), ref)
    assert_bitwise(ctx.baseline_mpk_shifted(Ap, x, theta).as_matrix(), ref)


def test_poly_coefficient_form(ctx, cases, oracle):
    rng = np.random.default_rng(11)
    for name in ("poisson3d_32", "stencil27_scrambled_20", "random_spd_4000"):
        c = cases[name]
        P = c["P"]
        Ap = ctx.csr(P)
        ls = ctx.levels_from_host(c["levels"], c["perm"], c["inv_perm"], c["level_ptr"])
        coef = rng.uniform(-1, 1, 9)
        x = mpkg.random_vector(P.n_rows, 3)
        plan = ctx.group_levels(ls, Ap, 1 << 20, 8)
        z_ref, blk_ref = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
        z, blk = ctx.mpk_poly(plan, Ap, x, coef, return_block=True)
        assert_bitwise(z, z_ref, name)
        assert_bitwise(blk.as_matrix(), blk_ref, name)
        assert_bitwise(ctx.mpk_poly(plan, Ap, x, coef), z_ref, name + " no block")


def test_spec_examples(ctx):
    A = ctx.csr(mpkg.HostCsr.from_arrays([0, 2, 3], [0, 1, 1], [2.0, 1.0, 3.0]))
    blk = ctx.baseline_mpk(A, [1.0, 1.0], 2)
    assert blk.slice(1).tolist() == [3.0, 3.0] and blk.slice(2).tolist() == [9.0, 9.0]
    D = ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2], [0, 1], [1.0, 3.0]))
    assert ctx.baseline_mpk_shifted(D, [1.0, 1.0], [2.0]).slice(1).tolist() == [-1.0, 1.0]
    I = ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2, 3], [0, 1, 2], [1.0] * 3))
    ls = ctx.build_levels(I)
    Ip = ctx.permute(I, ls)
    plan = ctx.group_levels(ls, Ip, 1 << 20, 4)
    blk = ctx.mpk(plan, Ip, [1.0, 2.0, 3.0], 4)
    assert all(blk.slice(p).tolist() == [1.0, 2.0, 3.0] for p in range(5))


def test_argument_errors(ctx):
    # test_mpk.cpp:247-259
    A = ctx.csr(mpkg.poisson1d(10))
    ls = ctx.build_levels(A)
    P = ctx.permute(A, ls)
    plan = ctx.group_levels(ls, P, 1024, 2)
    x = np.ones(10)
    with pytest.raises(ValueError):
        ctx.mpk(plan, P, x, 2, mpkg.VectorBlock(10, 2))  # needs 3 slices
    with pytest.raises(ValueError):
        ctx.mpk(plan, P, x, 3, mpkg.VectorBlock(10, 4))  # p_m > plan
    with pytest.raises(ValueError):
        ctx.baseline_mpk(A, np.ones(9), 2)
    with pytest.raises(ValueError):
        ctx.baseline_mpk_shifted(A, x, [1.0, 2.0 + 1.0j])
    with pytest.raises(ValueError):
        ctx.mpk_shifted(plan, P, x, [2.0 - 1.0j, 2.0 + 1.0j])
    with pytest.raises(ValueError):
        ctx.mpk(plan, ctx.csr(mpkg.poisson1d(11)), np.ones(11), 2)


def test_empty_and_edge_matrices(ctx):
    # empty rows, a single row, a matrix with no entries at all
    E = mpkg.HostCsr.from_arrays([0, 0, 1, 1], [1], [2.0])
    A = ctx.csr(E)
    ls = ctx.build_levels(A)
    assert ls.n_levels() == 1  # no off-diagonal edge: every row roots its own component
    blk = ctx.baseline_mpk(A, [1.0, 3.0, 5.0], 2)
    assert blk.slice(1).tolist() == [0.0, 6.0, 0.0]
    Z = ctx.csr(mpkg.HostCsr.from_arrays([0, 0, 0], [], []))
    lz = ctx.build_levels(Z)
    assert list(lz.level_ptr) == [0, 2]
    Zp = ctx.permute(Z, lz)
    plan = ctx.group_levels(lz, Zp, 1 << 20, 3)
    assert ctx.mpk(plan, Zp, [4.0, -1.0], 3).as_matrix()[1:].tolist() == [[0.0, 0.0]] * 3


def test_special_values_propagate(ctx, oracle):
    """0*Inf = NaN must appear exactly where the reference's row loop produces it."""
    A = mpkg.poisson2d(40, 40)
    x = mpkg.random_vector(A.n_rows, 1)
    x[17] = np.inf
    x[1000] = np.nan
    ref = oracle.baseline_mpk(A.row_ptr, A.col_idx, A.values, x, 3)
    assert_bitwise(ctx.baseline_mpk(ctx.csr(A), x, 3).as_matrix(), ref)


def test_tune_p_measured(ctx):
    # test_mpk.cpp:236-245
    A = ctx.csr(mpkg.poisson2d(48, 48))
    ls = ctx.build_levels(A)
    Ap = ctx.permute(A, ls)
    res = ctx.tune_p(ls, Ap, 256 * 1024, 1, 3)
    assert 1 <= res.p_opt <= 3 and len(res.table) == 3
    assert all(g > 0 for _, g in res.table)
    with pytest.raises(ValueError):
        ctx.tune_p(ls, Ap, 256 * 1024, 0, 3)


def test_config1_full_size_bitwise(ctx, oracle):
    """BASELINE config C1 (64^3 7-point, p=4) at full size, end to end on the GPU, against the
    oracle: levels/perm bit-exact, all 4 basis vectors bit-exact."""
    A = mpkg.poisson3d(64, 64, 64)
    assert A.n_rows == 262144 and A.nnz == 1810432
    lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
    assert len(lp) - 1 == 190
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    np.testing.assert_array_equal(ls.perm, pm)
    np.testing.assert_array_equal(ls.level_ptr, lp)
    Ap = ctx.permute(dA, ls)
    P = Ap.download()
    prp, pci, pv = oracle.permute(A.row_ptr, A.col_idx, A.values, pm)
    np.testing.assert_array_equal(P.col_idx, pci)
    x = mpkg.random_vector(A.n_rows, 42)
    plan = ctx.group_levels(ls, Ap, 100 << 20, 4)
    ref = oracle.baseline_mpk(prp, pci, pv, x, 4)
    assert_bitwise(ctx.mpk(plan, Ap, x, 4).as_matrix(), ref)


@pytest.mark.parametrize("knobs", [{}, {"pass": 2, "slack": 1}, {"pass": 8}, {"order": 1}, {"wave_affine": 0},
                                   {"wave_affine": 1}, {"pass": 3, "ctas_per_sm": 1}])
def test_wave_affine_records(ctx, oracle, knobs):
    """Affine chunk records (32 full rows whose entry k is column base_k + lane with one value:
    the interior of a level-ordered stencil) hold the same entries in the same stored order as the
    general records: bitwise equal powers, Newton basis and polynomial, with most chunks of a
    72^3 7-point Laplacian stored that way; Inf / NaN / the sentinel pattern in x flow through."""
    A = mpkg.poisson3d(72, 72, 72)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    P = Ap.download()
    x = mpkg.random_vector(A.n_rows, 11)
    try:
        set_knobs(ctx, {"schedule": 3, **knobs})
        plan = ctx.group_levels(ls, Ap, 1 << 20, 8)
        got = ctx.mpk(plan, Ap, x, 8).as_matrix()
        info = plan.exec_info()
        assert info["schedule"] == "wave" and info["wave_format"] == 1
        if knobs.get("wave_affine", 2) and not knobs.get("order", 0):
            assert info["wave_affine_chunks"] > 0.25 * info["wave_chunks"], info
        elif not knobs.get("wave_affine", 2):
            assert info["wave_affine_chunks"] == 0
        if knobs.get("wave_affine", 2) == 2 and not knobs.get("order", 0):
            # the chunks where the grid's diagonals break are banded: almost nothing stays general
            assert info["wave_banded_chunks"] > 0.25 * info["wave_chunks"], info
            assert info["wave_affine_chunks"] + info["wave_banded_chunks"] > 0.9 * info["wave_chunks"], info
        elif knobs.get("wave_affine", 2) < 2:
            assert info["wave_banded_chunks"] == 0
        ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 8)
        assert_bitwise(got, ref, f"affine {knobs}")
        sh = [0.5, 1.0 + 2.0j, 1.0 - 2.0j, -1.0, 3.0, 0.25]
        ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
        assert_bitwise(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref, "affine shifted")
        coef = np.linspace(-1, 1, 9)
        zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
        assert_bitwise(ctx.mpk_poly(plan, Ap, x, coef), zr, "affine poly")
        xs = x.copy()
        xs[1234] = np.inf
        xs[200000] = np.nan
        xs[300000:300001].view(np.uint64)[0] = np.uint64(0x7FF4DEAD5EED0001)
        got = ctx.mpk(plan, Ap, xs, 5).as_matrix()
        ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, xs, 5)
        assert np.array_equal(np.isnan(got), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert_bitwise(got[ok], ref[ok], "affine special values")
    finally:
        set_knobs(ctx, {})


def test_auto_schedule_picks_the_wave_above_l2(ctx, oracle):
    """Auto schedule: a short-row matrix larger than the L2 (128^3 7-point Laplacian, 175 MB) runs
    on the wave, powers / Newton basis / polynomial (plain powers + k_poly_combine) all bitwise; a
    64^3 one (22 MB, L2-resident) stays on the sweeps."""
    set_knobs(ctx, {})
    for n, want in ((128, "wave"), (64, "sweeps")):
        A = mpkg.poisson3d(n, n, n)
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        P = Ap.download()
        x = mpkg.random_vector(A.n_rows, 21)
        plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], 4)
        got = ctx.mpk(plan, Ap, x, 4).as_matrix()
        assert plan.exec_info()["schedule"] == want, plan.exec_info()
        ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 4)
        assert_bitwise(got, ref, f"auto {n}^3")
        coef = np.linspace(-1, 1, 5)
        zr, _ = oracle.poly(P.row_ptr, P.col_idx, P.values, x, coef)
        assert_bitwise(ctx.mpk_poly(plan, Ap, x, coef), zr, f"auto poly {n}^3")
        assert plan.exec_info()["schedule"] == want
        sh = [0.5, 1.0 + 2.0j, 1.0 - 2.0j, -1.0]
        ref = oracle.baseline_mpk_shifted(P.row_ptr, P.col_idx, P.values, x, sh)
        assert_bitwise(ctx.mpk_shifted(plan, Ap, x, sh).as_matrix(), ref, f"auto shifted {n}^3")


@pytest.mark.parametrize("dict_fmt", [1, 0])
def test_wave_special_values_and_sentinel_pattern(ctx, oracle, dict_fmt):
    """The wave schedule synchronises by value (a signalling-NaN sentinel in the slices a pass
    writes): caller data in x may hold any bit pattern, including Inf, NaN and the sentinel itself,
    and must flow through exactly as in the reference's row loop.  NaN payloads are compared as
    NaN (CPU and GPU quiet a signalling NaN differently); every other value bitwise."""
    A = mpkg.poisson3d(24, 24, 24)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    P = Ap.download()
    x = mpkg.random_vector(A.n_rows, 5)
    x[17] = np.inf
    x[2000] = -np.inf
    x[4000] = np.nan
    x[9000:9001].view(np.uint64)[0] = np.uint64(0x7FF4DEAD5EED0001)  # kWaveEmpty, as caller data
    try:
        set_knobs(ctx, {"schedule": 3, "pass": 3})
        ctx.set_param("wave_dict", dict_fmt)
        plan = ctx.group_levels(ls, Ap, 1 << 20, 6)
        got = ctx.mpk(plan, Ap, x, 6).as_matrix()
        assert plan.exec_info()["schedule"] == "wave"
    finally:
        set_knobs(ctx, {})
        ctx.set_param("wave_dict", 1)
    ref = oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, 6)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert_bitwise(got[ok], ref[ok], "non-NaN values")
    assert np.isnan(got[1:]).sum() > 100  # the NaNs really spread through the powers
