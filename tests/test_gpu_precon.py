"""GPU parity of the Jacobi-preconditioned chains: jacobi_setup /
jacobi_apply / jacobi_op / jacobi_op_blocked (reference jacobi.hpp) and the s-step Jacobi basis
(sstep.hpp:122-157), bit for bit against the golden fixtures generated from the compiled
reference and against the pinned oracle."""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

JAC_CASES = [f"{m}_s{s}" for m in ("random_spd_400_5_9", "poisson2d_17x13") for s in (1, 2, 4)]


@pytest.mark.parametrize("name", JAC_CASES)
def test_jacobi_golden(ctx, golden, name):
    g = lambda k: golden[f"jac.{name}.{k}"]
    sw = int(name.rsplit("_s", 1)[1])
    A = ctx.csr(mpkg.HostCsr.from_arrays(g("prp"), g("pci"), g("pv")))
    J = ctx.jacobi_setup(A, sw)
    pos, inv = J.diag()
    np.testing.assert_array_equal(pos, g("pos"))
    assert_bitwise(inv, g("inv"), "inv")
    assert_bitwise(ctx.jacobi_apply(J, A, g("x")), g("apply"), "apply")
    assert_bitwise(ctx.jacobi_op(J, A, g("x")), g("op"), "op")
    n = A.n_rows
    gr = g("group_rows")
    plan = mpkg.ExecutionPlan.from_groups(n, gr, p_m=1, sub_powers=J.stages())
    assert_bitwise(ctx.jacobi_op_blocked(J, plan, A, g("x")), g("op_blocked"), "op_blocked")


def _cases(oracle):
    mats = {"random_spd_50k": mpkg.random_spd(50000, 5, 777), "poisson3d_32": mpkg.poisson3d(32, 32, 32),
            "stencil27_scrambled": mpkg.scramble(mpkg.stencil27_random_sym(18, 17, 16, 3), 4)}
    out = {}
    for name, A in mats.items():
        lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
        P = mpkg.HostCsr.from_arrays(*oracle.permute(A.row_ptr, A.col_idx, A.values, pm))
        out[name] = (P, lv, pm, ip, lp)
    return out


def test_jacobi_corpus_vs_oracle(ctx, oracle):
    for name, (P, lv, pm, ip, lp) in _cases(oracle).items():
        Ap = ctx.csr(P)
        x = mpkg.random_vector(P.n_rows, 42)
        for sw in (1, 2, 3, 5):
            J = ctx.jacobi_setup(Ap, sw)
            assert_bitwise(ctx.jacobi_apply(J, Ap, x), oracle.jacobi_apply(P.row_ptr, P.col_idx, P.values, sw, x),
                           f"{name} apply sweeps={sw}")
            assert_bitwise(ctx.jacobi_op(J, Ap, x), oracle.jacobi_op(P.row_ptr, P.col_idx, P.values, sw, x),
                           f"{name} op sweeps={sw}")


@pytest.mark.parametrize("sweeps", [1, 2, 3])
def test_sstep_jacobi_basis(ctx, oracle, sweeps):
    shifts = [0.5, 2.0 + 0.75j, 2.0 - 0.75j, 1.0, 3.0 + 1.0j, 3.0 - 1.0j, 0.25, 1.5]
    for name, (P, lv, pm, ip, lp) in _cases(oracle).items():
        Ap = ctx.csr(P)
        ls = ctx.levels_from_host(lv, pm, ip, lp)
        J = ctx.jacobi_setup(Ap, sweeps)
        x = mpkg.random_vector(P.n_rows, 5)
        ref = oracle.sstep_jacobi_block(P.row_ptr, P.col_idx, P.values, sweeps, x, shifts)
        # sequential form (plan = NULL) and the cache-blocked form (plan with the chain's stages)
        assert_bitwise(ctx.sstep_jacobi(J, None, Ap, x, shifts).as_matrix(), ref, f"{name} seq")
        plan = ctx.group_levels(ls, Ap, 1 << 20, len(shifts)).with_sub_powers(J.stages(), lp)
        assert_bitwise(ctx.sstep_jacobi(J, plan, Ap, x, shifts).as_matrix(), ref, f"{name} plan")


def test_jacobi_errors(ctx):
    # jacobi.hpp:48-64 / 73: invalid_argument vs runtime_error, first failing row reported
    A = ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2, 3], [1, 0, 2], [1.0, 1.0, 1.0]))  # row 0 no diag
    with pytest.raises(mpkg.MpkgError, match="missing diagonal entry at row 0"):
        ctx.jacobi_setup(A, 1)
    Z = ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2, 3], [0, 1, 2], [1.0, 0.0, 1.0]))
    with pytest.raises(mpkg.MpkgError, match="zero diagonal entry at row 1"):
        ctx.jacobi_setup(Z, 1)
    G = ctx.csr(mpkg.poisson2d(6, 5))
    with pytest.raises(ValueError):
        ctx.jacobi_setup(G, 0)
    J = ctx.jacobi_setup(G, 2)
    ls = ctx.build_levels(G)
    Gp = ctx.permute(G, ls)
    J = ctx.jacobi_setup(Gp, 2)
    plan = ctx.group_levels(ls, Gp, 1 << 16, 4)  # sub_powers 1 != 3 stages
    with pytest.raises(ValueError, match="sub_powers"):
        ctx.jacobi_op_blocked(J, plan, Gp, np.ones(30))
    with pytest.raises(ValueError, match="sub_powers"):
        ctx.sstep_jacobi(J, plan, Gp, np.ones(30), [1.0, 2.0])
    ok = plan.with_sub_powers(3)
    with pytest.raises(ValueError, match="p_m"):  # execute.hpp:81-83 power budget
        ctx.sstep_jacobi(J, ok, Gp, np.ones(30), [1.0] * 5)
    with pytest.raises(ValueError):  # conjugate pair straddling the end (mpk.hpp:111-127)
        ctx.sstep_jacobi(J, None, Gp, np.ones(30), [1.0, 1.0 + 2.0j])


# ---- GS2 (gs2.hpp) ----------------------------------------------------------------------------
GS2_CASES = ["g0_k1_f1", "g2_k2_f1", "g3_k2_f0"]


@pytest.mark.parametrize("name", GS2_CASES)
def test_gs2_golden(ctx, golden, name):
    g = lambda k: golden[f"gs2.{name}.{k}"]
    gamma, K, fw = (int(t[1:]) for t in name.split("_"))
    A = ctx.csr(mpkg.HostCsr.from_arrays(g("prp"), g("pci"), g("pv")))
    G = ctx.gs2_setup(A, gamma, K, bool(fw))
    plan = mpkg.ExecutionPlan.from_groups(A.n_rows, g("group_rows"), p_m=K, sub_powers=G.stages())
    for pl in (None, plan):  # sequential form and the blocked twin
        assert_bitwise(ctx.gs2_smooth(G, A, g("x"), g("z0"), pl), g("smooth_z"), "smooth")
        assert_bitwise(ctx.gs2_apply(G, A, g("x"), pl), g("apply_z"), "apply")
        z, r = ctx.gs2_smooth_residual(G, A, g("x"), g("z0"), pl)
        assert_bitwise(z, g("smooth_residual_z"), "smooth_residual z")
        assert_bitwise(r, g("smooth_residual_out"), "smooth_residual r")
        assert_bitwise(ctx.gs2_op(G, A, g("x"), pl), g("op_out"), "op")


@pytest.mark.parametrize("gamma,K,fw", [(0, 1, True), (1, 2, True), (2, 3, False)])
def test_gs2_corpus_and_sstep_vs_oracle(ctx, oracle, gamma, K, fw):
    shifts = [0.5, 2.0 + 0.75j, 2.0 - 0.75j, 1.0]
    for name, (P, lv, pm, ip, lp) in _cases(oracle).items():
        Ap = ctx.csr(P)
        ls = ctx.levels_from_host(lv, pm, ip, lp)
        G = ctx.gs2_setup(Ap, gamma, K, fw)
        x = mpkg.random_vector(P.n_rows, 42)
        z0 = mpkg.random_vector(P.n_rows, 43)
        rp, ci, vv = P.row_ptr, P.col_idx, P.values
        z, _ = oracle.gs2(rp, ci, vv, gamma, K, fw, "smooth", x, z0)
        assert_bitwise(ctx.gs2_smooth(G, Ap, x, z0), z, f"{name} smooth")
        _, y = oracle.gs2(rp, ci, vv, gamma, K, fw, "op", x)
        assert_bitwise(ctx.gs2_op(G, Ap, x), y, f"{name} op")
        ref = oracle.sstep_gs2_block(rp, ci, vv, gamma, K, fw, x, shifts)
        assert_bitwise(ctx.sstep_gs2(G, None, Ap, x, shifts).as_matrix(), ref, f"{name} sstep")
        plan = ctx.group_levels(ls, Ap, 1 << 20, len(shifts) * K).with_sub_powers(G.stages(), lp)
        assert_bitwise(ctx.sstep_gs2(G, plan, Ap, x, shifts).as_matrix(), ref, f"{name} sstep plan")


def test_gs2_errors(ctx):
    A = ctx.csr(mpkg.poisson2d(6, 5))
    with pytest.raises(ValueError, match="gamma"):
        ctx.gs2_setup(A, -1)
    with pytest.raises(ValueError, match="sweeps"):
        ctx.gs2_setup(A, 1, 0)
    M = ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2, 3], [1, 0, 2], [1.0, 1.0, 1.0]))
    with pytest.raises(mpkg.MpkgError, match="gs2_setup: missing diagonal entry at row 0"):
        ctx.gs2_setup(M, 1)
    G = ctx.gs2_setup(A, 2, 2)
    bad = mpkg.ExecutionPlan.from_groups(30, [0, 30], p_m=2, sub_powers=3)
    with pytest.raises(ValueError, match="sub_powers"):
        ctx.gs2_apply(G, A, np.ones(30), bad)
    small = mpkg.ExecutionPlan.from_groups(30, [0, 30], p_m=1, sub_powers=4)
    with pytest.raises(ValueError, match="p_m"):
        ctx.gs2_apply(G, A, np.ones(30), small)
    with pytest.raises(ValueError, match="p_m"):  # s * sweeps > budget
        ctx.sstep_gs2(G, mpkg.ExecutionPlan.from_groups(30, [0, 30], p_m=3, sub_powers=4), A,
                      np.ones(30), [1.0, 2.0])


# ---- product-form polynomial (poly.hpp:146-281) -------------------------------------------------
ROOTS = {
    "real": [4.0, 0.7, 2.5, 1.3],
    "pairs": [3.5, 1.0 + 0.6j, 1.0 - 0.6j, 2.2, 0.9 + 0.2j, 0.9 - 0.2j],      # ends on a pair
    "mixed": [2.0 + 1.0j, 2.0 - 1.0j, 0.8, 3.1, 1.7 + 0.3j, 1.7 - 0.3j, 1.1],  # trailing real root
}


@pytest.mark.parametrize("inner", ["none", "jacobi1", "jacobi3", "gs2_0", "gs2_2b"])
def test_poly_apply_vs_oracle(ctx, oracle, inner):
    for name, (P, lv, pm, ip, lp) in _cases(oracle).items():
        Ap = ctx.csr(P)
        x = mpkg.random_vector(P.n_rows, 17)
        kw, prec = {}, None
        if inner.startswith("jacobi"):
            kw = dict(inner="jacobi", sweeps=int(inner[-1]))
            prec = ctx.jacobi_setup(Ap, kw["sweeps"])
        elif inner.startswith("gs2"):
            kw = dict(inner="gs2", gamma=int(inner[4]), forward=not inner.endswith("b"))
            prec = ctx.gs2_setup(Ap, kw["gamma"], 1, kw["forward"])
        stages = 1 if prec is None else prec.stages()
        ls = ctx.levels_from_host(lv, pm, ip, lp)
        for rname, roots in ROOTS.items():
            ref = oracle.poly_apply(P.row_ptr, P.col_idx, P.values, roots, x, **kw)
            assert_bitwise(ctx.poly_apply(Ap, roots, x, prec), ref, f"{name} {inner} {rname}")
            plan = ctx.group_levels(ls, Ap, 1 << 20, 3).with_sub_powers(stages, lp)  # root slicing
            assert_bitwise(ctx.poly_apply(Ap, roots, x, prec, plan), ref, f"{name} {inner} {rname} plan")


def test_poly_apply_errors(ctx):
    A = ctx.csr(mpkg.poisson2d(6, 5))
    with pytest.raises(ValueError, match="conjugate pair"):
        ctx.poly_apply(A, [1.0 + 1.0j, 2.0], np.ones(30))
    with pytest.raises(ValueError, match="not set up"):
        ctx.poly_apply(A, [], np.ones(30))
    G = ctx.gs2_setup(A, 1, 2)
    with pytest.raises(ValueError, match="single sweep"):
        ctx.poly_apply(A, [1.0], np.ones(30), G)
    plan = mpkg.ExecutionPlan.from_groups(30, [0, 30], p_m=2, sub_powers=3)
    with pytest.raises(ValueError, match="sub_powers"):
        ctx.poly_apply(A, [1.0, 2.0], np.ones(30), None, plan)
    z = ctx.poly_apply(ctx.csr(mpkg.HostCsr.from_arrays([0, 1, 2], [0, 1], [2.0, 2.0])), [2.0], [4.0, 6.0])
    assert z.tolist() == [2.0, 3.0]  # test_poly.cpp:160-166
