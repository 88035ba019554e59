"""Small driver for ncu: builds one workload, warms up, then issues a few fused MPK launches and
one baseline sweep so `ncu -k regex:...` can capture them.

    python tools/profile_case.py --config c2 [--order 1] [--launches 2]
"""
import argparse
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--order", type=int, default=-1)
    ap.add_argument("--slack", type=int, default=-1)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--group", type=int, default=8)
    ap.add_argument("--pass-powers", type=int, default=0)
    ap.add_argument("--p", type=int, default=0, help="override the config's p")
    ap.add_argument("--knobs", default="", help="k=v,k=v executor knobs")
    ap.add_argument("--seed", type=int, default=2309)
    args = ap.parse_args()
    import torch

    import paper_2309_02228_b200 as mpkg
    cfgd = bench.CONFIGS[args.config]
    p = args.p or cfgd["p"]
    A = bench.make_matrix(args.config, args.seed)
    ctx = mpkg.Context(0)
    ctx.set_param("order", args.order)
    ctx.set_param("group", args.group)
    ctx.set_param("pass", args.pass_powers)
    for kv in filter(None, args.knobs.split(",")):
        k, v = kv.split("=")
        ctx.set_param(k, int(v))
    if args.slack >= 0:
        ctx.set_param("slack", args.slack)
    dA = ctx.csr(A)
    ls = ctx.build_levels(dA)
    Ap = ctx.permute(dA, ls)
    plan = ctx.group_levels(ls, Ap, ctx.device_info()["l2_bytes"], p)
    n = A.n_rows
    x = ctx.permute_vector(mpkg.random_vector(n, args.seed + 2), ls.perm)
    d_x = torch.from_numpy(x).cuda()
    d_blk = torch.empty((p + 1) * n, dtype=torch.float64, device="cuda")
    for _ in range(2 + args.launches):
        ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, d_blk.data_ptr(), n, p + 1)
    ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), p, d_blk.data_ptr(), n, p + 1)
    ctx.synchronize()
    print("profile_case done", plan.exec_info())


if __name__ == "__main__":
    main()
