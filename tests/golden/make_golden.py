"""Generates tests/golden/golden.npz from the REFERENCE itself (oracle/_ref/libmpkref.so, the
reference's own headers compiled in place by oracle/Makefile).  Run in the build container:

    make -C oracle && python tests/golden/make_golden.py

The cases restate the reference's own hot-path tests (proj/tests/test_levels.cpp,
proj/tests/test_mpk.cpp) and the SPEC.md examples; inputs use the reference generators
(generators.hpp) so the fixtures pin both the generators and the algorithm.
"""
from __future__ import annotations

import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Reference  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent / "golden.npz"


def main():
    R = Reference()
    g = {}

    def put(prefix, **arrs):
        for k, v in arrs.items():
            g[f"{prefix}.{k}"] = np.asarray(v)

    # --- level structures (test_levels.cpp:15-84) ------------------------------------------
    mats = {
        "tridiag5": R.gen(1, 5),
        "grid3x3": R.gen(2, 3, 3),
        "poisson2d_20x17": R.gen(2, 20, 17),
        "poisson3d_7x8x9": R.gen(3, 7, 8, 9),
        "random_spd_200_5_77": R.gen(5, 200, 5, 0, 77),
        "random_csr_300_5_11": R.gen(4, 300, 5, 0, 11),
    }
    for s in (1, 2, 3, 4, 5):
        mats[f"random_csr_120_4_{s}"] = R.gen(4, 120, 4, 0, s)
    # diag 6x6 and two disjoint paths (test_levels.cpp:35-72) as explicit CSR
    mats["diag6"] = (np.arange(7, dtype=np.uint32), np.arange(6, dtype=np.uint32),
                     np.arange(1, 7, dtype=np.float64))
    mats["two_paths"] = (np.array([0, 1, 3, 4, 5, 6], np.uint32),
                         np.array([1, 0, 2, 1, 4, 3], np.uint32), np.ones(6))
    for name, (rp, ci, v) in mats.items():
        lv, pm, ip, lp = R.build_levels(rp, ci, v)
        prp, pci, pv = R.permute(rp, ci, v, pm)
        put(f"lev.{name}", rp=rp, ci=ci, v=v, levels=lv, perm=pm, inv_perm=ip, level_ptr=lp,
            prp=prp, pci=pci, pv=pv)

    # --- plan (test_levels.cpp:109-147) ------------------------------------------------------
    rp, ci, v = R.gen(2, 64, 64)
    lv, pm, ip, lp = R.build_levels(rp, ci, v)
    prp, pci, pv = R.permute(rp, ci, v, pm)
    gr, glp, gfp, tgt = R.group_levels(prp, pci, pv, lp, 100 * 1024, 4)
    put("plan.poisson2d_64", level_ptr=lp, prp=prp, group_rows=gr, group_level_ptr=glp,
        group_footprint=gfp, target=np.uint64(tgt))
    put("greedy", a=R.greedy_group([1000] * 10, 2500), b=R.greedy_group([1000, 5000, 1000, 1000], 2500),
        c=R.greedy_group([10, 10, 10], 0))

    # --- power kernels (test_mpk.cpp:125-206) -----------------------------------------------
    rp, ci, v = R.gen(2, 12, 9)
    x = np.sin(0.37 * np.arange(len(rp) - 1)) + 0.5
    put("mpk.poisson2d_12x9_p5", rp=rp, ci=ci, v=v, x=x, block=R.baseline_mpk(rp, ci, v, x, 5))

    for name, args in {"poisson2d_48x37": (2, 48, 37), "poisson3d_9x10x11": (3, 9, 10, 11),
                       "random_csr_2000_5_3": (4, 2000, 5, 0, 3)}.items():
        rp, ci, v = R.gen(*args)
        lv, pm, ip, lp = R.build_levels(rp, ci, v)
        prp, pci, pv = R.permute(rp, ci, v, pm)
        x = np.cos(0.11 * np.arange(len(rp) - 1))
        for p in (1, 3, 6):
            gr, _, _, _ = R.group_levels(prp, pci, pv, lp, 64 * 1024, p)
            blk = R.mpk(prp, pci, pv, gr, p, x, p)
            put(f"mpk.{name}_p{p}", rp=rp, ci=ci, v=v, perm=pm, level_ptr=lp, x=x,
                group_rows=gr, block=blk)

    rp, ci, v = R.gen(4, 150, 4, 0, 21)
    x = np.sin(1.3 * np.arange(150))
    sh = [0.4, 1.2 + 0.7j, 1.2 - 0.7j, -0.3]
    put("shift.random_csr_150", rp=rp, ci=ci, v=v, x=x, shifts=np.array(sh),
        block=R.baseline_mpk_shifted(rp, ci, v, x, sh))

    rp, ci, v = R.gen(2, 30, 30)
    lv, pm, ip, lp = R.build_levels(rp, ci, v)
    prp, pci, pv = R.permute(rp, ci, v, pm)
    x = 1.0 / (1.0 + np.arange(900) % 17)
    sh = [2.0, 3.5 + 1.5j, 3.5 - 1.5j, 4.0, 1.0]
    gr, _, _, _ = R.group_levels(prp, pci, pv, lp, 16 * 1024, len(sh))
    put("shift.poisson2d_30", rp=rp, ci=ci, v=v, perm=pm, level_ptr=lp, x=x, shifts=np.array(sh),
        group_rows=gr, block=R.mpk_shifted(prp, pci, pv, gr, len(sh), x, sh))

    # --- Jacobi chains (jacobi.hpp) ----------------------------------------
    for name, args in {"random_spd_400_5_9": (5, 400, 5, 0, 9), "poisson2d_17x13": (2, 17, 13)}.items():
        rp, ci, v = R.gen(*args)
        lv, pm, ip, lp = R.build_levels(rp, ci, v)
        prp, pci, pv = R.permute(rp, ci, v, pm)
        x = np.cos(0.23 * np.arange(len(rp) - 1)) + 0.25
        for sw in (1, 2, 4):
            pos, inv = R.jacobi_setup(prp, pci, pv, sw)
            gr, _, _, _ = R.group_levels(prp, pci, pv, lp, 16 * 1024, 1)
            put(f"jac.{name}_s{sw}", prp=prp, pci=pci, pv=pv, x=x, pos=pos, inv=inv,
                group_rows=gr, apply=R.jacobi_apply(prp, pci, pv, sw, x),
                op=R.jacobi_op(prp, pci, pv, sw, x),
                op_blocked=R.jacobi_op_blocked(prp, pci, pv, sw, gr, x))

    # --- GS2 chains (gs2.hpp) ---------------------------------------------------------------------
    rp, ci, v = R.gen(5, 300, 5, 0, 13)
    lv, pm, ip, lp = R.build_levels(rp, ci, v)
    prp, pci, pv = R.permute(rp, ci, v, pm)
    x = np.sin(0.19 * np.arange(300)) + 0.1
    z0 = np.cos(0.07 * np.arange(300))
    for gamma, K, fw in ((0, 1, 1), (2, 2, 1), (3, 2, 0)):
        gr, _, _, _ = R.group_levels(prp, pci, pv, lp, 16 * 1024, K)
        arrs = dict(prp=prp, pci=pci, pv=pv, x=x, z0=z0, group_rows=gr)
        for mode in ("smooth", "apply", "smooth_residual", "op"):
            z, out = R.gs2(prp, pci, pv, gamma, K, fw, mode, x, None if mode in ("apply", "op") else z0)
            zb, outb = R.gs2(prp, pci, pv, gamma, K, fw, mode, x,
                             None if mode in ("apply", "op") else z0, group_rows=gr, plan_p_m=K)
            assert np.array_equal(z.view(np.uint64), zb.view(np.uint64))  # gs2.hpp: blocked == seq
            arrs[f"{mode}_z"] = z
            if out is not None:
                assert np.array_equal(out.view(np.uint64), outb.view(np.uint64))
                arrs[f"{mode}_out"] = out
        put(f"gs2.g{gamma}_k{K}_f{fw}", **arrs)

    # acceptance.cpp:84-90 random_vector(n, 42)
    put("rv", x=R.random_vector(1000, 42))
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
