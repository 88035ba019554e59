"""The C-ABI shard layer (csrc/dist.cu, include/mpkg.h mpkg_dist_*) on CPU: its partition and halo
plan agree with multi.py's for many level structures, and world-2/3 gloo exchanges move exactly the
bytes the plan lists and assemble the right local x.  (The NCCL entry points need GPUs:
tests/test_gpu_dist.py.)"""
import os
import socket

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from paper_2309_02228_b200 import multi


def _levels(rng, nl):
    sizes = rng.integers(0, 40, size=nl)
    sizes[rng.integers(0, nl)] += 1
    lp = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint32)
    nnz_row = rng.integers(1, 9, size=int(lp[-1]))
    rp = np.concatenate([[0], np.cumsum(nnz_row)]).astype(np.int64)
    return lp, rp


def test_partition_matches_multi():
    rng = np.random.default_rng(7)
    for _ in range(200):
        lp, rp = _levels(rng, int(rng.integers(1, 60)))
        for world in (1, 2, 3, 4, 5, 8):
            py = multi.partition_levels(lp, rp, world)
            b = multi.dist_partition(lp, rp[lp.astype(np.int64)], world)
            assert [(int(b[r]), int(b[r + 1])) for r in range(world)] == py


def test_halo_matches_multi():
    rng = np.random.default_rng(11)
    for _ in range(150):
        lp, rp = _levels(rng, int(rng.integers(1, 50)))
        world = int(rng.integers(1, 6))
        p = int(rng.integers(0, 9))
        parts = multi.partition_levels(lp, rp, world)
        bounds = [parts[0][0]] + [b for _, b in parts]
        plans = [multi.halo_plan(lp, parts, r, p) for r in range(world)]
        for r in range(world):
            h = multi.dist_halo(lp, bounds, world, r, p)
            assert h["own"] == plans[r].own_rows and h["local"] == plans[r].local_rows
            for s in range(world):
                if s == r:
                    assert h["recv"][s] == (0, 0) and h["send"][s] == (0, 0)
                    continue
                rec = [(a, b) for o, a, b in plans[r].pieces if o == s]
                assert h["recv"][s] == (rec[0] if rec else (0, 0))
                snd = [(a, b) for o, a, b in plans[s].pieces if o == r]
                assert h["send"][s] == (snd[0] if snd else (0, 0))


def test_halo_rejects_bad_bounds():
    lp = np.array([0, 3, 5, 9], np.uint32)
    with pytest.raises(ValueError, match="monotone"):
        multi.dist_halo(lp, [0, 2, 1, 3], 3, 0, 1)
    with pytest.raises(ValueError, match="rank"):
        multi.dist_halo(lp, [0, 3], 1, 1, 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        lp, rp = _levels(rng, 30)
        n = int(lp[-1])
        x = np.arange(n, dtype=np.float64) * 1.5 - 7.0
        parts = multi.partition_levels(lp, rp, world)
        bounds = [0] + [b for _, b in parts]
        plans = [multi.halo_plan(lp, parts, r, p) for r in range(world)]
        o0, o1 = plans[rank].own_rows
        stats = {}
        xl = multi.exchange_halo(torch.from_numpy(x[o0:o1].copy()), plans, rank, dist, stats=stats).numpy()
        h = multi.dist_halo(lp, bounds, world, rank, p)
        g0, g1 = h["local"]
        q.put((rank, stats.get("send_bytes", 0), stats.get("recv_bytes", 0),
               8 * sum(b - a for a, b in h["send"]), 8 * sum(b - a for a, b in h["recv"]),
               bool(np.array_equal(xl, x[g0:g1]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,p", [(2, 3), (3, 5)])
def test_gloo_exchange_moves_exactly_the_plan(world, p):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, sent, recvd, plan_send, plan_recv, ok in res:
        assert ok, rank
        assert (sent, recvd) == (plan_send, plan_recv), rank
    assert sum(r[1] for r in res) == sum(r[2] for r in res) > 0
