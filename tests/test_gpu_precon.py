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
