"""Row-engine throughput of the SELL SpMV (k_spmv_sell, one launch per power) as the 7-point matrix
grows from L2-resident to HBM-streamed: what a cross-power L2 reuse scheme could gain per power.

    python tools/l2_rate.py [sizes...]
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
        ctx.kernel_times()
        ts = []
        for _ in range(7):
            ctx.baseline_mpk_dev(Ap, x.data_ptr(), p, blk.data_ptr(), n, p + 1)
            ctx.synchronize()
            tot, cnt, _ = ctx.kernel_times()
            ts.append(tot / cnt)
        ms = statistics.median(ts[2:])
        mb = (12 * nnz + 4 * (n + 1)) / 1e6
        byt = 12 * nnz + 4 * (n + 1) + 16 * n
        print(f"{m}^3: n={n:>10d} matrix {mb:8.1f} MB  {ms * 1e3:8.1f} us/power  "
              f"{n / (ms * 1e3):8.1f} rows/us  {byt / (ms * 1e-3) / 1e9:8.1f} GB/s", flush=True)
        del dA, ls, Ap, blk, x
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
