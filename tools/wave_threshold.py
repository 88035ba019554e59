"""Experiments: wave vs sweeps on 7-point Laplacians of several sizes (where should auto pick the wave?).

    python tools/wave_threshold.py 96 128 160 200
"""
import statistics
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2309_02228_b200 as mpkg  # noqa: E402

ctx = mpkg.Context(0)
ctx.set_param("kernel_timing", 1)
for n in [int(a) for a in sys.argv[1:]]:
    A = mpkg.poisson3d(n, n, n)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    N = A.n_rows
    x = torch.from_numpy(ctx.permute_vector(mpkg.random_vector(N, 1), ls.perm)).cuda()
    for p in (4, 8):
        blk = torch.empty((p + 1) * N, dtype=torch.float64, device="cuda")
        ref = torch.empty_like(blk)
        ctx.baseline_mpk_dev(Ap, x.data_ptr(), p, ref.data_ptr(), N, p + 1)
        out = []
        for sched in (2, 3):
            ctx.set_param("schedule", sched)
            plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], p)
            ctx.mpk_dev(plan, Ap, x.data_ptr(), p, blk.data_ptr(), N, p + 1)
            ctx.synchronize()
            ok = torch.equal(blk.view(torch.int64), ref.view(torch.int64))
            ctx.kernel_times()
            ts = []
            for _ in range(9):
                ctx.mpk_dev(plan, Ap, x.data_ptr(), p, blk.data_ptr(), N, p + 1)
                ctx.synchronize()
                t, c, _ = ctx.kernel_times()
                ts.append(t / max(c, 1))
            out.append((sched, statistics.median(ts), ok, plan.exec_info()["pass_powers"]))
        ctx.set_param("schedule", 0)
        mb = 12 * A.nnz / 1e6
        print(f"n={n}^3 rows={N} matrix={mb:.0f} MB p={p}: sweeps {out[0][1]*1e3:.1f} us, wave {out[1][1]*1e3:.1f} us "
              f"(pass {out[1][3]}), bitwise {out[0][2]} {out[1][2]}", flush=True)
