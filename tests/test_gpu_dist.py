"""The NCCL shard layer (mpkg_dist_*, csrc/dist.cu) on the GPU box's single B200: a one-rank NCCL
communicator runs the whole C++ path -- host broadcast, halo plan with its preallocated local x,
block and row scatter from the root, exchange + local MPK -- and must reproduce the single-GPU MPK
bit for bit.  (NCCL does not allow two ranks on one GPU; the multi-rank plan and exchange are
covered on CPU by tests/test_dist_abi.py and on the device with gloo by test_gpu_sharded.py.)"""
import numpy as np
import pytest
import torch

import paper_2309_02228_b200 as mpkg
from paper_2309_02228_b200 import multi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,p", [("stencil", 4), ("poisson", 8)])
def test_nccl_one_rank_dist_mpk_bitwise(kind, p):
    A = (mpkg.scramble(mpkg.stencil27_random_sym(20, 18, 16, 3), 4) if kind == "stencil"
         else mpkg.poisson3d(40, 36, 32))
    ctx = mpkg.Context(0)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    n = A.n_rows
    lp = np.asarray(ls.level_ptr, np.uint32)
    x = ctx.permute_vector(mpkg.random_vector(n, 17), ls.perm)
    d_x = torch.from_numpy(x).cuda()
    ref = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
    ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), p, ref.data_ptr(), n, p + 1)

    D = multi.NcclDist(ctx, 1, 0, multi.NcclDist.unique_id())
    meta = D.bcast_host(np.array([len(lp) - 1], np.uint32))
    assert int(meta[0]) == len(lp) - 1
    rp = Ap.download().row_ptr.astype(np.int64)
    bounds = multi.dist_partition(lp, rp[lp.astype(np.int64)], 1)
    D.set_plan(lp, bounds, p)
    info = D.info()
    assert info["own"] == (0, n) and info["local"] == (0, n)
    assert info["send_bytes"] == info["recv_bytes"] == 0
    A_loc = D.scatter_blocks(0, Ap)
    assert (A_loc.n_rows, A_loc.nnz) == (n, Ap.nnz)
    x_own = torch.empty(n, dtype=torch.float64, device="cuda")
    D.scatter_rows(0, d_x.data_ptr(), x_own.data_ptr())
    ctx.synchronize()
    assert torch.equal(x_own, d_x)
    ident = np.arange(n, dtype=np.uint32)
    lls = ctx.levels_from_host(np.zeros(n, np.uint32), ident, ident, lp)
    plan = ctx.group_levels(lls, A_loc, ctx.device_info()["l2_bytes"], p)
    blk = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
    for _ in range(2):  # the preallocated exchange buffer is reused across steps
        D.mpk(plan, A_loc, x_own.data_ptr(), p, blk.data_ptr(), n, p + 1)
        ctx.synchronize()
        assert torch.equal(blk.view(torch.int64), ref.view(torch.int64))
    D.close()
    ctx.close()
