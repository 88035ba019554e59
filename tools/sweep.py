"""Times many executor configurations on one workload built once (CUDA-event timing of the fused
launch, median of `--reps`).  Each config: knob=value pairs separated by commas, e.g.

    python tools/sweep.py --config c2 --p 1,8 "group=8" "group=8,pass=4" "group=16,slack=64"
"""
import argparse
import json
import pathlib
import statistics
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

DEFAULTS = {"order": -1, "slack": -1, "pass": 0, "l2_budget": 0, "ctas_per_sm": 0, "group": 8,
            "stages": 0, "tile_rows": 128, "threads": 0, "kernel": 0, "producers": 0, "cgroups": 0, "schedule": 0, "sweep_variant": 0, "coop_variant": 0, "wave_dict": 1, "wave_affine": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--p", default="8")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=2309)
    ap.add_argument("--mode", default="bitwise", choices=["bitwise", "fast"])
    ap.add_argument("configs", nargs="*", default=[""])
    args = ap.parse_args()
    import torch

    import paper_2309_02228_b200 as mpkg
    A = bench.make_matrix(args.config, args.seed)
    ctx = mpkg.Context(0)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    n, nnz = A.n_rows, A.nnz
    del dA
    x = ctx.permute_vector(mpkg.random_vector(n, args.seed + 2), ls.perm)
    d_x = torch.from_numpy(x).cuda()
    ps = [int(v) for v in args.p.split(",")]
    pmax = max(ps)
    d_blk = torch.empty((pmax + 1) * n, dtype=torch.float64, device="cuda")
    ref = torch.empty_like(d_blk)
    ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), pmax, ref.data_ptr(), n, pmax + 1)
    ctx.set_param("kernel_timing", 1)
    for _ in range(3):
        ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), 1, ref[: 2 * n].data_ptr(), n, 2)
    ctx.synchronize()
    tot, cnt, _ = ctx.kernel_times()
    print(f"# {args.config}: n={n} nnz={nnz} levels={ls.n_levels()}  baseline 1 sweep: {tot / cnt:.3f} ms")
    ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), pmax, ref.data_ptr(), n, pmax + 1)
    ctx.synchronize()
    ctx.kernel_times()
    rows = []
    ctx.set_mode(1 if args.mode == "fast" else 0)
    for spec in args.configs:
        knobs = dict(DEFAULTS)
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            knobs[k] = int(v)
        for k, v in knobs.items():
            ctx.set_param(k, v)
        for p in ps:
            plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], p)
            ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_blk.data_ptr(), n, p + 1)  # build
            ctx.synchronize()
            ok = torch.equal(d_blk[: (p + 1) * n].view(torch.int64), ref[: (p + 1) * n].view(torch.int64))
            if args.mode == "fast":  # the north star's 1e-12 inf-norm bound per basis vector
                a_, b_ = d_blk[: (p + 1) * n].view(p + 1, n), ref[: (p + 1) * n].view(p + 1, n)
                ok = float(((a_ - b_).abs().amax(1) / b_.abs().amax(1).clamp_min(1e-300)).max()) <= 1e-12
            ctx.kernel_times()
            ts = []
            for _ in range(args.reps):
                ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_blk.data_ptr(), n, p + 1)
                ctx.synchronize()
                t, c, _ = ctx.kernel_times()
                ts.append(t / max(c, 1))
            ms = statistics.median(ts)
            info = plan.exec_info()
            gf = 2.0 * nnz * p / (ms * 1e-3) * 1e-9
            rows.append({"spec": spec, "p": p, "ms": ms, "ms_per_power": ms / p, "gflops": gf,
                         "bitwise": ok, **info})
            print(f"{spec or 'default':40s} p={p}: {ms:8.3f} ms  {ms / p:7.3f} ms/power  "
                  f"{gf:8.1f} GF/s  pass={info['pass_powers']}  ok={ok}", flush=True)
    out = ROOT / "gpurun_out" / f"sweep_{args.config}.json"
    out.parent.mkdir(exist_ok=True)
    out.write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
