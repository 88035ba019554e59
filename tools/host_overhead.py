"""Host-side cost of one device-pointer MPK call (C1): wall time of N back-to-back calls with no
synchronisation in between, against the device time of the same calls."""
import pathlib
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def main():
    import torch
    import paper_2309_02228_b200 as mpkg
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
    A = bench.make_matrix(cfg, 2309)
    ctx = mpkg.Context(0)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    n, p = A.n_rows, bench.CONFIGS[cfg]["p"]
    plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], p)
    d_x = torch.from_numpy(ctx.permute_vector(mpkg.random_vector(n, 1), ls.perm)).cuda()
    d_b = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
    from paper_2309_02228_b200._lib import lib
    for timing in (0, 1):
        ctx.set_param("kernel_timing", timing)
        for _ in range(20):
            ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_b.data_ptr(), n, p + 1)
        ctx.synchronize()
        N = 2000
        t0 = time.perf_counter()
        for _ in range(N):
            ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_b.data_ptr(), n, p + 1)
        t1 = time.perf_counter()
        ctx.synchronize()
        t2 = time.perf_counter()
        # raw ctypes call (no Python wrapper)
        f = lib.mpkg_mpk_dev
        h, ph, ah, xp, bp = ctx.h, plan.h, Ap.h, d_x.data_ptr(), d_b.data_ptr()
        t3 = time.perf_counter()
        for _ in range(N):
            f(h, ph, ah, xp, p, bp, n, p + 1)
        t4 = time.perf_counter()
        ctx.synchronize()
        t5 = time.perf_counter()
        ctx.kernel_times()
        print(f"kernel_timing={timing}: wrapper submit {1e6 * (t1 - t0) / N:.1f} us/call, "
              f"wrapper total {1e6 * (t2 - t0) / N:.1f} us/call; raw ctypes submit "
              f"{1e6 * (t4 - t3) / N:.1f} us/call, total {1e6 * (t5 - t3) / N:.1f} us/call")


if __name__ == "__main__":
    main()
