"""Small runs of every hand-synchronised kernel, for compute-sanitizer (racecheck / synccheck /
memcheck); each case is checked bitwise against the one-launch-per-power baseline.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

  * k_mpk_lean       -- fused tile-DAG kernel (per-tile flags, relaxed polls + acquire, release fence)
  * k_long_rows_bitwise -- hub rows: 4-slot shared-memory ring with per-slot sequence flags
  * k_coop_rows      -- fast mode: warp-cooperative rows, split hubs, ordered finish
  * k_mpk_wave       -- wave schedule: value-synchronised (sentinel) passes, dynamic ticket claims
"""
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import paper_2309_02228_b200 as mpkg
    from test_gpu_parity import _arrow_matrix
    ctx = mpkg.Context(0)
    cases = [
        ("lean poisson3d_16", mpkg.poisson3d(16, 16, 16), {"schedule": 1}, 0),
        ("lean scrambled 27-pt", mpkg.scramble(mpkg.stencil27_random_sym(10, 10, 10, 1), 2), {"schedule": 1}, 0),
        ("lean hub rows", _arrow_matrix(3000, (0, 1500)), {"schedule": 1}, 0),
        ("sweeps hub rows (k_long_rows_bitwise)", _arrow_matrix(3000, (0, 1500)), {"schedule": 2}, 0),
        ("sweeps hub rows fast (k_coop_rows)", _arrow_matrix(3000, (0, 1500)), {"schedule": 2}, 1),
        ("wave poisson3d_16", mpkg.poisson3d(16, 16, 16), {"schedule": 3}, 0),
        ("wave poisson3d_16 pass 2 slack 1", mpkg.poisson3d(16, 16, 16), {"schedule": 3, "pass": 2, "slack": 1}, 0),
        ("wave scrambled 27-pt order 1", mpkg.scramble(mpkg.stencil27_random_sym(10, 10, 10, 1), 2),
         {"schedule": 3, "order": 1}, 0),
    ]
    bad = 0
    for name, A, knobs, mode in cases:
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        x = mpkg.random_vector(A.n_rows, 3)
        ref = ctx.baseline_mpk(Ap, x, 5).as_matrix()
        ctx.set_mode(mode)
        for k, v in knobs.items():
            ctx.set_param(k, v)
        plan = ctx.group_levels(ls, Ap, 1 << 20, 5)
        got = ctx.mpk(plan, Ap, x, 5).as_matrix()
        ok = (np.array_equal(got.view(np.uint64), ref.view(np.uint64)) if mode == 0 else
              float(np.max(np.abs(got - ref).max(axis=1) / np.abs(ref).max(axis=1))) <= 1e-12)
        bad += not ok
        print(f"{name:45s} {plan.exec_info()['schedule']:7s} {'ok' if ok else 'MISMATCH'}", flush=True)
        ctx.set_mode(0)
        for k, v in {"schedule": 0, "pass": 0, "slack": -1, "order": -1}.items():
            ctx.set_param(k, v)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
