"""Debug driver for the wave schedule on small matrices: compares every slice with the
one-launch-per-power baseline and prints where they differ.

    python tools/wave_debug.py
"""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import paper_2309_02228_b200 as mpkg
    ctx = mpkg.Context(0)
    cases = {"rmat_12": mpkg.rmat(12, 8, 3), "poisson2d_256": mpkg.poisson2d(256, 256),
             "random_csr_2000": mpkg.random_csr(2000, 5, 3)}
    for name, A in cases.items():
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        x = mpkg.random_vector(A.n_rows, 9)
        ctx.set_param("schedule", 2)
        ref = ctx.baseline_mpk(Ap, x, 6).as_matrix()
        for knobs in ({"pass": 1}, {"pass": 2}, {"pass": 6}, {"pass": 2, "order": 0}, {"pass": 6, "order": 0},
                      {"pass": 1, "order": 0}, {"pass": 2, "order": 1}, {"pass": 2, "order": 2},
                      {"pass": 6, "slack": 100000, "order": 0}):
            for k in ("pass", "ctas_per_sm", "slack", "order"):
                ctx.set_param(k, {"slack": -1, "order": -1}.get(k, 0))
            ctx.set_param("schedule", 3)
            for k, v in knobs.items():
                ctx.set_param(k, v)
            plan = ctx.group_levels(ls, Ap, 1 << 20, 6)
            got = ctx.mpk(plan, Ap, x, 6).as_matrix()
            bad = [(k, int(np.count_nonzero(got[k].view(np.uint64) != ref[k].view(np.uint64))))
                   for k in range(7)]
            info = plan.exec_info()
            print(name, knobs, info["schedule"], "order", info["order"], "long", info["long_rows"], "tiles", info["tiles"], "pass", info["pass_powers"],
                  "bad per slice", bad, flush=True)
        ctx.set_param("schedule", 0)
        for k in ("pass", "ctas_per_sm", "slack", "order"):
            ctx.set_param(k, {"slack": -1, "order": -1}.get(k, 0))


if __name__ == "__main__":
    main()
