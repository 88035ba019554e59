"""Experiments: mpk_poly on a short-row matrix, sweeps (running accumulator) vs the wave (plain
powers, then k_poly_combine): bitwise equality and MPK kernel time.

    python tools/poly_wave_check.py [n]     # n^3 7-point Laplacian, degree 8
"""
import pathlib
import statistics
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_2309_02228_b200 as mpkg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = mpkg.Context(0)
ctx.set_param("kernel_timing", 1)
A = mpkg.poisson3d(n, n, n)
dA = ctx.csr(A)
ls = ctx.build_levels(dA)
Ap = ctx.permute(dA, ls)
x = ctx.permute_vector(mpkg.random_vector(A.n_rows, 1), ls.perm)
coef = np.linspace(-1, 1, 9)
res = {}
for sched in (2, 0):
    ctx.set_param("schedule", sched)
    plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], 8)
    res[sched] = ctx.mpk_poly(plan, Ap, x, coef).copy()
    ctx.kernel_times()
    ts = []
    for _ in range(5):
        ctx.mpk_poly(plan, Ap, x, coef)
        t, c, _ = ctx.kernel_times()
        ts.append(t / max(c, 1))
    print(f"schedule {plan.exec_info()['schedule']:6s}: {statistics.median(ts):.3f} ms per mpk_poly (device part)")
print("bitwise equal:", np.array_equal(res[2].view(np.uint64), res[0].view(np.uint64)))
