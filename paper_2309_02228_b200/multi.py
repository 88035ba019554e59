"""Multi-GPU MPK: contiguous BFS-level ranges per rank with p-deep ghost levels.

The level adjacency property (levels.hpp:17-24) confines row i's columns to levels
level(i)-1 .. level(i)+1.  Rank r owns the levels [L_r, L_{r+1}) (balanced by nnz) and also
holds p ghost levels on each side, i.e. the rows of levels [L_r - p, L_{r+1} + p).  Power k is
valid on own rows plus ghost depth p-k (redundant-compute, communication-avoiding MPK), so the
only exchange is ONE halo of x before the sweep; no collective runs inside the p powers.  The
local matrix is A_perm restricted to the local rows with columns outside the local range
dropped: rows that lose a column are exactly the outermost ghost rows, whose (wrong) values can
reach at most ghost depth p-k at power k and never an own row.  Own rows are therefore computed
by the same formula from the same inputs as on one GPU: bit-identical results for any N.

The host logic (partition, halo plan, local matrix, exchange, assembly) is independent of the
device; `DistributedMPK` runs the local MPK through a callable (default: the sm_100a path of
this package).  Communication uses torch.distributed point-to-point (NCCL on GPUs, gloo in the
CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


def partition_levels(level_ptr: Sequence[int], row_ptr: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous level ranges [L_r, L_{r+1}) balancing nnz (row count breaks ties)."""
    lp = np.asarray(level_ptr, dtype=np.int64)
    rp = np.asarray(row_ptr, dtype=np.int64)
    nl = len(lp) - 1
    if world < 1:
        raise ValueError("partition_levels: world must be >= 1")
    cum = rp[lp]  # nnz before each level boundary
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        L = int(np.searchsorted(cum, target, side="left"))
        L = max(L, bounds[-1])
        bounds.append(min(L, nl))
    bounds.append(nl)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


@dataclass
class HaloPlan:
    rank: int
    levels: Tuple[int, int]      # own level range
    own_rows: Tuple[int, int]    # own rows [o0, o1) of A_perm
    local_rows: Tuple[int, int]  # rows held locally [g0, g1) (own + p ghost levels each side)
    pieces: List[Tuple[int, int, int]]  # (owner rank, row0, row1) covering local_rows

    @property
    def n_local(self) -> int:
        return self.local_rows[1] - self.local_rows[0]


def halo_plan(level_ptr: Sequence[int], parts: Sequence[Tuple[int, int]], rank: int, p: int) -> HaloPlan:
    lp = list(int(v) for v in level_ptr)
    nl = len(lp) - 1
    L0, L1 = parts[rank]
    o0, o1 = lp[L0], lp[L1]
    g0, g1 = lp[max(0, L0 - p)], lp[min(nl, L1 + p)]
    if o0 == o1:  # empty rank: holds nothing
        g0 = g1 = o0
    pieces = []
    for s, (a, b) in enumerate(parts):
        r0, r1 = max(lp[a], g0), min(lp[b], g1)
        if r0 < r1:
            pieces.append((s, r0, r1))
    return HaloPlan(rank, (L0, L1), (o0, o1), (g0, g1), pieces)


def local_matrix(row_ptr, col_idx, values, g0: int, g1: int):
    """Rows [g0, g1) of A_perm, columns outside [g0, g1) dropped, indices shifted by -g0 (the
    stored order of the kept entries is unchanged)."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    ci = np.asarray(col_idx, dtype=np.int64)
    v = np.asarray(values)
    b, e = rp[g0], rp[g1]
    cols = ci[b:e]
    keep = (cols >= g0) & (cols < g1)
    rows = np.repeat(np.arange(g1 - g0), np.diff(rp[g0:g1 + 1]))
    counts = np.bincount(rows[keep], minlength=g1 - g0)
    lrp = np.zeros(g1 - g0 + 1, dtype=np.uint32)
    np.cumsum(counts, out=lrp[1:])
    return lrp, (cols[keep] - g0).astype(np.uint32), np.ascontiguousarray(v[b:e][keep])


def local_level_ptr(level_ptr, L0: int, L1: int, p: int):
    lp = np.asarray(level_ptr, dtype=np.int64)
    nl = len(lp) - 1
    a, b = max(0, L0 - p), min(nl, L1 + p)
    return (lp[a:b + 1] - lp[a]).astype(np.uint32)


def exchange_halo(x_own, plans: Sequence[HaloPlan], rank: int, dist, group=None, stats=None):
    """The one collective of the level-partitioned MPK: builds this rank's local x (rows
    [g0, g1)) from the owners' pieces with grouped point-to-point transfers.  `x_own` is a torch
    tensor holding rows [o0, o1); the result lives on the same device (NCCL over NVLink between
    GPUs, gloo in the CPU tests).  Every rank calls this with its own x_own."""
    import torch
    if x_own.is_cuda and dist.get_backend(group) == "gloo":  # gloo moves host tensors only
        return exchange_halo(x_own.cpu(), plans, rank, dist, group, stats).to(x_own.device)
    me = plans[rank]
    g0, g1 = me.local_rows
    o0 = me.own_rows[0]
    out = torch.empty(g1 - g0, dtype=x_own.dtype, device=x_own.device)
    ops = []
    for other in plans:  # my own rows to every rank whose local range overlaps them
        if other.rank == rank:
            continue
        for s, r0, r1 in other.pieces:
            if s == rank:
                ops.append(dist.P2POp(dist.isend, x_own[r0 - o0:r1 - o0].contiguous(), other.rank, group))
                if stats is not None:
                    stats["send_bytes"] = stats.get("send_bytes", 0) + 8 * (r1 - r0)
    for s, r0, r1 in me.pieces:
        if s == rank:
            out[r0 - g0:r1 - g0] = x_own[r0 - o0:r1 - o0]
        else:
            ops.append(dist.P2POp(dist.irecv, out[r0 - g0:r1 - g0], s, group))
            if stats is not None:
                stats["recv_bytes"] = stats.get("recv_bytes", 0) + 8 * (r1 - r0)
    if ops:
        for rq in dist.batch_isend_irecv(ops):
            rq.wait()
    return out


def exchange_x(x_own: np.ndarray, plans: Sequence[HaloPlan], rank: int, dist, group=None) -> np.ndarray:
    """Host-array form of exchange_halo."""
    import torch
    return exchange_halo(torch.from_numpy(np.ascontiguousarray(x_own, dtype=np.float64)), plans, rank,
                         dist, group).numpy()


LocalMPK = Callable[[np.ndarray, np.ndarray, np.ndarray, np.ndarray, np.ndarray, int], np.ndarray]


def gpu_local_mpk(ctx=None, cache_bytes: Optional[int] = None) -> LocalMPK:
    """The default local compute: this package's fused sm_100a MPK on the rank's GPU."""
    from . import api

    def run(rp, ci, v, lp, x, p):
        c = ctx or api.Context(0)
        A = c.csr(api.HostCsr.from_arrays(rp, ci, v))
        n = len(rp) - 1
        ident = np.arange(n, dtype=np.uint32)
        ls = c.levels_from_host(np.zeros(n, np.uint32), ident, ident, lp)
        plan = c.group_levels(ls, A, cache_bytes or c.device_info()["l2_bytes"], p)
        return c.mpk(plan, A, x, p).as_matrix()

    return run


class DistributedMPK:
    """One rank's share of a level-partitioned MPK over A_perm (global arrays on every rank for
    simplicity of setup; only the local slice is kept)."""

    def __init__(self, row_ptr, col_idx, values, level_ptr, p: int, rank: int, world: int,
                 local_mpk: Optional[LocalMPK] = None):
        self.p, self.rank, self.world = p, rank, world
        self.parts = partition_levels(level_ptr, row_ptr, world)
        self.plans = [halo_plan(level_ptr, self.parts, r, p) for r in range(world)]
        me = self.plans[rank]
        g0, g1 = me.local_rows
        self.local = local_matrix(row_ptr, col_idx, values, g0, g1)
        self.local_lp = local_level_ptr(level_ptr, me.levels[0], me.levels[1], p)
        self.local_mpk = local_mpk or gpu_local_mpk()

    @property
    def plan(self) -> HaloPlan:
        return self.plans[self.rank]

    def run(self, x_own: np.ndarray, dist, group=None) -> np.ndarray:
        """Returns this rank's own rows of y_0..y_p, shape (p+1, n_own)."""
        me = self.plan
        x_loc = exchange_x(x_own, self.plans, self.rank, dist, group)
        if me.n_local == 0:
            return np.zeros((self.p + 1, 0))
        blk = self.local_mpk(*self.local, self.local_lp, x_loc, self.p)
        o0 = me.own_rows[0] - me.local_rows[0]
        return blk[:, o0:o0 + (me.own_rows[1] - me.own_rows[0])]


class ShardedMPK:
    """One rank's device-resident share of a level-partitioned MPK (the multi-GPU path of
    bench.py).  The global A_perm is on this rank's GPU only for setup: the local matrix
    A_perm[g0:g1, g0:g1] is cut on the device (mpkg_csr_block), its level structure is the
    global one restricted to the local levels, and every step is one halo exchange of x on the
    context's stream followed by the local MPK (one launch per power or the fused kernel, as on
    one GPU).  Own rows are bit-identical to the single-GPU result."""

    def __init__(self, ctx, A_perm, level_ptr, row_nnz_prefix, p: int, rank: int, world: int,
                 cache_bytes: Optional[int] = None):
        from . import api
        self.ctx, self.p, self.rank, self.world = ctx, p, rank, world
        lp = np.asarray(level_ptr, dtype=np.int64)
        self.parts = partition_levels(lp, row_nnz_prefix, world)
        self.plans = [halo_plan(lp, self.parts, r, p) for r in range(world)]
        me = self.plans[rank]
        g0, g1 = me.local_rows
        self.n_local = g1 - g0
        self.own = (me.own_rows[0] - g0, me.own_rows[1] - g0)  # own rows inside the local block
        self.A = ctx.csr_block(A_perm, g0, g1, g0, g1)
        llp = local_level_ptr(lp, me.levels[0], me.levels[1], p)
        ident = np.arange(self.n_local, dtype=np.uint32)
        ls = ctx.levels_from_host(np.zeros(self.n_local, np.uint32), ident, ident, llp)
        self.plan = ctx.group_levels(ls, self.A, cache_bytes or ctx.device_info()["l2_bytes"], p)
        self._api = api

    @property
    def halo_plan(self) -> HaloPlan:
        return self.plans[self.rank]

    def step(self, x_own, block, dist, group=None):
        """x_own: torch tensor of this rank's own rows of x (device); block: torch tensor of
        (p+1) * n_local doubles.  Runs on the context's stream (the exchange joins it)."""
        import torch
        stream = torch.cuda.ExternalStream(self.ctx.stream, device=x_own.device)
        with torch.cuda.stream(stream):
            x_loc = exchange_halo(x_own, self.plans, self.rank, dist, group)
            if self.n_local:
                self.ctx.mpk_dev(self.plan, self.A, x_loc.data_ptr(), self.p, block.data_ptr(),
                                 self.n_local, self.p + 1)
        return x_loc


# ---- the C-ABI shard layer (csrc/dist.cu): the C++ caller's view of the same plan ------------------

def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def dist_partition(level_ptr, nnz_before, world: int) -> np.ndarray:
    """mpkg_dist_partition: level bounds (world+1) balancing nnz; nnz_before[L] = nonzeros in
    levels < L.  Same rule as partition_levels."""
    import ctypes as C

    from ._lib import check, lib
    lp = _u32(level_ptr)
    nb = np.ascontiguousarray(np.asarray(nnz_before, dtype=np.uint64))
    out = np.empty(world + 1, np.uint32)
    check(lib.mpkg_dist_partition(lp.ctypes.data, len(lp) - 1, nb.ctypes.data, world, out.ctypes.data))
    return out


def dist_halo(level_ptr, bounds, world: int, rank: int, p: int) -> dict:
    """mpkg_dist_halo: own / local row ranges and the per-peer send / recv row ranges."""
    from ._lib import check, lib
    lp, b = _u32(level_ptr), _u32(bounds)
    own, loc = np.empty(2, np.uint32), np.empty(2, np.uint32)
    send, recv = np.empty(2 * world, np.uint32), np.empty(2 * world, np.uint32)
    check(lib.mpkg_dist_halo(lp.ctypes.data, len(lp) - 1, b.ctypes.data, world, rank, p, own.ctypes.data,
                             loc.ctypes.data, send.ctypes.data, recv.ctypes.data))
    return {"own": tuple(int(v) for v in own), "local": tuple(int(v) for v in loc),
            "send": [tuple(int(v) for v in send[2 * r:2 * r + 2]) for r in range(world)],
            "recv": [tuple(int(v) for v in recv[2 * r:2 * r + 2]) for r in range(world)]}


class NcclDist:
    """One rank of the NCCL shard layer (mpkg_dist_*): communicator, halo plan with a
    preallocated local-x buffer, one-time scatter of the blocks / own rows from a root, and the
    per-step exchange + local MPK on the context's stream."""

    def __init__(self, ctx, world: int, rank: int, uid: bytes):
        import ctypes as C

        from ._lib import check, lib
        self.ctx, self.world, self.rank = ctx, world, rank
        self._lib, self._check, self._C = lib, check, C
        buf = C.create_string_buffer(bytes(uid), 128)
        h = C.c_void_p()
        check(lib.mpkg_dist_create(ctx.h, buf, world, rank, C.byref(h)))
        self.h = h.value

    @staticmethod
    def unique_id() -> bytes:
        import ctypes as C

        from ._lib import check, lib
        buf = C.create_string_buffer(128)
        check(lib.mpkg_dist_unique_id(buf))
        return buf.raw

    def bcast_host(self, arr: np.ndarray, root: int = 0) -> np.ndarray:
        a = np.ascontiguousarray(arr)
        self._check(self._lib.mpkg_dist_bcast_host(self.h, a.ctypes.data, a.nbytes, root))
        return a

    def set_plan(self, level_ptr, bounds, p: int):
        lp, b = _u32(level_ptr), _u32(bounds)
        self._check(self._lib.mpkg_dist_set_plan(self.h, lp.ctypes.data, len(lp) - 1, b.ctypes.data, p))
        self.p = p

    def info(self) -> dict:
        C = self._C
        own, loc = np.empty(2, np.uint32), np.empty(2, np.uint32)
        sb, rb = C.c_uint64(), C.c_uint64()
        self._check(self._lib.mpkg_dist_info(self.h, own.ctypes.data, loc.ctypes.data, C.byref(sb), C.byref(rb)))
        return {"own": (int(own[0]), int(own[1])), "local": (int(loc[0]), int(loc[1])),
                "send_bytes": sb.value, "recv_bytes": rb.value}

    def scatter_blocks(self, root: int, A_perm=None):
        from .api import DeviceCsr
        C = self._C
        h = C.c_void_p()
        self._check(self._lib.mpkg_dist_scatter_blocks(self.h, root, A_perm.h if A_perm is not None else None,
                                                       C.byref(h)))
        return DeviceCsr(self.ctx, h.value)

    def scatter_rows(self, root: int, d_full: int, d_own: int):
        self._check(self._lib.mpkg_dist_scatter_rows(self.h, root, d_full or None, d_own or None))

    def exchange(self, d_x_own: int) -> int:
        C = self._C
        out = C.c_void_p()
        self._check(self._lib.mpkg_dist_exchange(self.h, d_x_own or None, C.byref(out)))
        return out.value

    def mpk(self, plan, A_local, d_x_own: int, p: int, d_block: int, rows: int, slices: int):
        self._check(self._lib.mpkg_dist_mpk(self.h, plan.h, A_local.h, d_x_own or None, p, d_block, rows, slices))

    def close(self):
        if getattr(self, "h", None):
            self._lib.mpkg_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()
