"""Wave-engine throughput as the 7-point matrix grows from L2-resident to HBM-streamed: one MPK of
p powers with the wave schedule forced to one power per pass (no in-pass dependencies), so every
launch is a plain sweep by the wave engine; compared with the sweep schedule on the same matrix.

    python tools/wave_rate.py [sizes...]
"""
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import paper_2309_02228_b200 as mpkg
    sizes = [int(s) for s in sys.argv[1:]] or [48, 64, 80, 96, 128, 192, 256]
    ctx = mpkg.Context(0)
    ctx.set_param("kernel_timing", 1)
    p = 8
    for m in sizes:
        A = mpkg.poisson3d(m, m, m)
        n, nnz = A.n_rows, A.nnz
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        x = torch.rand(n, dtype=torch.float64, device="cuda")
        blk = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
        out = []
        for sched, pas in ((2, 0), (3, 1), (3, 2), (3, 4)):
            ctx.set_param("schedule", sched)
            ctx.set_param("pass", pas)
            plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], p)
            ctx.mpk_dev(plan, Ap, x.data_ptr(), p, blk.data_ptr(), n, p + 1)
            ctx.synchronize()
            ctx.kernel_times()
            ts = []
            for _ in range(7):
                ctx.mpk_dev(plan, Ap, x.data_ptr(), p, blk.data_ptr(), n, p + 1)
                ctx.synchronize()
                tot, cnt, _ = ctx.kernel_times()
                ts.append(tot / cnt)
            ms = statistics.median(ts[2:])
            out.append(f"{'sweeps' if sched == 2 else f'wave pass={pas}'}: {ms * 1e3 / p:8.1f} us/power "
                       f"{n * p / (ms * 1e3):7.1f} rows/us")
        mb = (12 * nnz + 4 * (n + 1)) / 1e6
        print(f"{m}^3 n={n:>10d} matrix {mb:8.1f} MB | " + " | ".join(out), flush=True)
        del dA, ls, Ap, blk, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
