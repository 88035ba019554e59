"""The device-resident multi-GPU path (multi.ShardedMPK: level-range shards with p ghost levels,
one halo exchange of x, local MPK on the GPU) run as world-size 2 and 3 on ONE GPU: the ranks
share cuda:0 and exchange through gloo (host staging).  Ranks never wait on each other inside a
kernel -- the only synchronisation is the host-side exchange before each local MPK -- so
sharing the device is a faithful test of the partition / halo / local-matrix logic that NCCL
drives across GPUs.  Own rows must equal the oracle bit for bit."""
import os
import socket

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    if kind == "stencil":
        return mpkg.scramble(mpkg.stencil27_random_sym(22, 20, 18, 4), 5)
    return mpkg.random_spd(20000, 5, 9)


def _worker(rank, world, port, kind, p, order, q):
    import torch
    import torch.distributed as dist

    from paper_2309_02228_b200 import multi
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = mpkg.Context(0)
        ctx.set_param("order", order)
        A = _problem(kind)
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        lens = np.diff(A.row_ptr.astype(np.int64))[ls.inv_perm.astype(np.int64)]
        prefix = np.concatenate([[0], np.cumsum(lens)])
        shard = multi.ShardedMPK(ctx, Ap, ls.level_ptr, prefix, p, rank, world)
        x = ctx.permute_vector(mpkg.random_vector(A.n_rows, 42), ls.perm)
        o0, o1 = shard.halo_plan.own_rows
        dev = torch.device("cuda", 0)
        x_own = torch.from_numpy(np.ascontiguousarray(x[o0:o1])).to(dev)
        blk = torch.empty((p + 1) * max(shard.n_local, 1), dtype=torch.float64, device=dev)
        shard.step(x_own, blk, dist)
        ctx.synchronize()
        a0, a1 = shard.own
        own = blk.view(p + 1, -1)[:, a0:a1].cpu().numpy() if shard.n_local else np.zeros((p + 1, 0))
        q.put((rank, o0, o1, own))
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,p,order", [(2, "stencil", 4, -1), (3, "stencil", 8, 1),
                                                (2, "random", 6, 0)])
def test_sharded_mpk_own_rows_bitwise(oracle, world, kind, p, order):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, p, order, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    A = _problem(kind)
    n = A.n_rows
    lv, pm, ip, lp = oracle.build_levels(A.row_ptr, A.col_idx)
    rp, ci, v = oracle.permute(A.row_ptr, A.col_idx, A.values, pm)
    x = np.empty(n)
    x[pm] = mpkg.random_vector(n, 42)  # csr.hpp:191 permute_vector: out[perm[i]] = in[i]
    ref = oracle.baseline_mpk(rp, ci, v, x, p)
    got = np.zeros_like(ref)
    covered = 0
    for _, o0, o1, own in res:
        got[:, o0:o1] = own
        covered += o1 - o0
    assert covered == n
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
