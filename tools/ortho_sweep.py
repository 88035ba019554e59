"""Times the fast-mode ICGS (2 sweeps, C4-sized block) under each ortho_fused setting."""
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import paper_2309_02228_b200 as mpkg
    n, qc, s = 192 ** 3, 25, 8
    ctx = mpkg.Context(0)
    ctx.set_mode(1)
    g = torch.Generator(device="cuda").manual_seed(1)
    Q = torch.rand((qc, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    R = torch.empty((qc, qc), dtype=torch.float64, device="cuda")
    ctx.tsqr_dev(Q.data_ptr(), n, qc, R.data_ptr())
    V0 = torch.rand((s, n), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    V = V0.clone()
    coeff = torch.empty((s, qc), dtype=torch.float64, device="cuda")
    ref = None
    for v in (0, 1, 2):
        ctx.set_param("ortho_fused", v)
        ts = []
        for _ in range(6):
            V.copy_(V0)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream = torch.cuda.ExternalStream(ctx.stream)
            a.record(stream)
            ctx.icgs_block_orthogonalize_dev(Q.data_ptr(), n, qc, V.data_ptr(), s, 2, coeff.data_ptr())
            b.record(stream)
            ctx.synchronize()
            ts.append(a.elapsed_time(b))
        if ref is None:
            ref = V.clone()
        err = (V - ref).abs().max().item()
        print(f"ortho_fused={v}: icgs {statistics.median(ts[1:]):.3f} ms  max|V - unfused| {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
