"""N>1 path of the level-partitioned MPK (paper_2309_02228_b200/multi.py) on CPU: partition and
halo-plan invariants, and world_size-2/3 gloo runs whose assembled own rows must equal the
single-rank result bit for bit.  The local compute is injected: the CPU oracle here (tests may
use it as the checker), the sm_100a path in production."""
import os
import socket

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from paper_2309_02228_b200 import multi


def _problem(kind="stencil", seed=3):
    from oracle.oracle import Oracle
    O = Oracle()
    A = (mpkg.scramble(mpkg.stencil27_random_sym(9, 8, 7, seed), seed + 1) if kind == "stencil"
         else mpkg.random_spd(3000, 5, seed))
    lv, pm, ip, lp = O.build_levels(A.row_ptr, A.col_idx)
    P = O.permute(A.row_ptr, A.col_idx, A.values, pm)
    return P, lp


def _oracle_local(rp, ci, v, lp, x, p):
    from oracle.oracle import Oracle
    return Oracle().baseline_mpk(rp, ci, v, x, p)


def test_partition_balances_and_covers():
    (rp, ci, v), lp = _problem()
    for world in (1, 2, 3, 5):
        parts = multi.partition_levels(lp, rp, world)
        assert parts[0][0] == 0 and parts[-1][1] == len(lp) - 1
        assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
        nnz = [int(rp[lp[b]] - rp[lp[a]]) for a, b in parts]
        assert sum(nnz) == rp[-1]
        level_nnz = np.diff(np.asarray(rp, dtype=np.int64)[np.asarray(lp, dtype=np.int64)])
        assert max(nnz) <= rp[-1] / world + level_nnz.max()  # balanced to one level's nnz


def test_halo_plan_pieces_cover_local_rows():
    (rp, ci, v), lp = _problem()
    parts = multi.partition_levels(lp, rp, 3)
    for p in (1, 3, 6):
        for r in range(3):
            h = multi.halo_plan(lp, parts, r, p)
            g0, g1 = h.local_rows
            cov = sorted((a, b) for _, a, b in h.pieces)
            assert cov[0][0] == g0 and cov[-1][1] == g1
            assert all(cov[i][1] == cov[i + 1][0] for i in range(len(cov) - 1))
            assert g0 <= h.own_rows[0] <= h.own_rows[1] <= g1


def test_local_matrix_keeps_entry_order():
    (rp, ci, v), lp = _problem()
    lrp, lci, lv = multi.local_matrix(rp, ci, v, int(lp[2]), int(lp[9]))
    for r in range(len(lrp) - 1):
        cols = lci[lrp[r]:lrp[r + 1]]
        assert np.all(np.diff(cols.astype(np.int64)) > 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, p, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        (rp, ci, v), lp = _problem(kind)
        n = len(rp) - 1
        x = mpkg.random_vector(n, 42)
        d = multi.DistributedMPK(rp, ci, v, lp, p, rank, world, local_mpk=_oracle_local)
        o0, o1 = d.plan.own_rows
        own = d.run(x[o0:o1], dist)
        q.put((rank, o0, o1, own))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,p", [(2, "stencil", 4), (2, "random", 6), (3, "stencil", 8)])
def test_gloo_distributed_mpk_bitwise(world, kind, p):
    import torch.multiprocessing as tmp
    from oracle.oracle import Oracle
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    (rp, ci, v), lp = _problem(kind)
    n = len(rp) - 1
    ref = Oracle().baseline_mpk(rp, ci, v, mpkg.random_vector(n, 42), p)
    got = np.zeros_like(ref)
    covered = 0
    for _, o0, o1, own in res:
        got[:, o0:o1] = own
        covered += o1 - o0
    assert covered == n
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
