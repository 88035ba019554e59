"""Device-side schedule audit: the acceptance.cpp:188-251 predecessor check, replayed on what the GPU
actually did.

With the "trace" knob the fused tile-DAG kernel (flags: stamp after the acquire / before the
publish) and the wave kernel (values: stamp between a tile's last input load and its first result
store) record %globaltimer per (tile, power).  The reference's rule (execute.hpp:59-72, test_mpk.cpp
:72-102): power q of a tile may start only after power q-1 finished on every tile its rows read.
Here: stamp_in[q][T] >= stamp_out[q-1][T'] for every dependency tile T' of T, every (T, q) ran
exactly once, and the results are bitwise the oracle's.
"""
import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from conftest import assert_bitwise

pytestmark = pytest.mark.gpu

P_M = 6


def _dep_tiles(A, tile_rows):
    """Per tile: the set of tiles holding a column read by its rows (A_perm order = slot order)."""
    rp = A.row_ptr.astype(np.int64)
    nt = (A.n_rows + tile_rows - 1) // tile_rows
    deps = []
    for T in range(nt):
        r0, r1 = T * tile_rows, min(A.n_rows, (T + 1) * tile_rows)
        cols = A.col_idx[rp[r0]:rp[r1]]
        deps.append(np.unique(np.concatenate([cols // tile_rows, [T]])).astype(np.int64))
    return deps


def _audit(stamps, tile_rows, A, p):
    nt = (A.n_rows + tile_rows - 1) // tile_rows
    st = stamps.reshape(p + 1, -1, 2)
    assert st.shape[1] >= nt
    st = st[:, :nt, :].astype(np.int64)
    # exactly-once coverage: every (tile, power >= 1) left both stamps, in order
    assert np.all(st[1:, :, 0] > 0) and np.all(st[1:, :, 1] > 0)
    assert np.all(st[1:, :, 1] >= st[1:, :, 0])
    deps = _dep_tiles(A, tile_rows)
    bad = 0
    for q in range(2, p + 1):
        fin = st[q - 1, :, 1]
        for T in range(nt):
            if st[q, T, 0] < fin[deps[T]].max():
                bad += 1
    assert bad == 0, f"{bad} (tile, power) cells started before a predecessor finished"


CASES = {
    "poisson3d_24": lambda: mpkg.poisson3d(24, 24, 24),
    "stencil27_scrambled_16": lambda: mpkg.scramble(mpkg.stencil27_random_sym(16, 16, 16, 3), 4),
    "random_spd_20000": lambda: mpkg.random_spd(20000, 5, 777),
}
SCHEDULES = {
    "fused-lean": {"schedule": 1},
    "fused-lean-slack1": {"schedule": 1, "slack": 1},
    "wave": {"schedule": 3},
    "wave-pass2": {"schedule": 3, "pass": 2},
    "wave-pass6-slack1": {"schedule": 3, "pass": 6, "slack": 1},
}


@pytest.mark.parametrize("sched", list(SCHEDULES))
@pytest.mark.parametrize("name", list(CASES))
def test_schedule_trace_predecessor_audit(ctx, oracle, name, sched):
    A = CASES[name]()
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    P = Ap.download()
    x = mpkg.random_vector(A.n_rows, 11)
    knobs = {"order": 0, "trace": 1, **SCHEDULES[sched]}
    try:
        for k, v in knobs.items():
            ctx.set_param(k, v)
        plan = ctx.group_levels(ls, Ap, 1 << 20, P_M)
        got = ctx.mpk(plan, Ap, x, P_M).as_matrix()
        stamps, tile_rows = plan.exec_trace()
        info = plan.exec_info()
    finally:
        for k, v in {"order": -1, "trace": 0, "schedule": 0, "slack": -1, "pass": 0}.items():
            ctx.set_param(k, v)
    assert info["schedule"] == ("wave" if sched.startswith("wave") else "fused")
    assert stamps is not None and tile_rows > 0
    assert_bitwise(got, oracle.baseline_mpk(P.row_ptr, P.col_idx, P.values, x, P_M), f"{name} {sched}")
    _audit(stamps, tile_rows, P, P_M)


def test_trace_off_records_nothing(ctx):
    A = ctx.csr(mpkg.poisson2d(40, 40))
    ls = ctx.build_levels(A)
    Ap = ctx.permute(A, ls)
    ctx.set_param("schedule", 3)
    try:
        plan = ctx.group_levels(ls, Ap, 1 << 20, 3)
        ctx.mpk(plan, Ap, mpkg.random_vector(1600, 1), 3)
        stamps, _ = plan.exec_trace()
    finally:
        ctx.set_param("schedule", 0)
    assert stamps is None
