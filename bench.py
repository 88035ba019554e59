#!/usr/bin/env python
"""Benchmark of the level-blocked MPK path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl mpkg|reference]

A step is one MPK call y_k = A^k x, k = 1..p (BASELINE.json metric: GFLOP/s = 2*nnz*p / t, the
reference convention of proj/include/mpk/mpk.hpp:256), on the permuted matrix with x and the
output block resident in HBM; level construction / permutation / planning are preprocessing,
timed separately (the reference's level_preprocessing_s, solver.cpp:543-567).  `e2e` is the same
metric through the host-pointer C ABI call (mpkg_mpk): H2D of x and D2H of all p+1 vectors from
pinned memory inside the timed region.  `--impl reference` times the reference's own OpenMP CPU
implementation (oracle/_ref, compiled from the reference headers) on this box's host cores.

Workloads (BASELINE.json configs; synthetic inputs generated from seeds):
  c1  3D 7-pt 64^3, p=4            c2  27-pt 160^3, -U[.9,1.1] sym + seeded scramble, p=8 (default)
  c3  R-MAT scale 21 ef 16, p=4    c4  27-pt 192^3 Newton basis s=8   c4poly  same, sum c_k A^k x
  c5  3D 7-pt 512^3, p=8
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import tempfile
import time

os.environ.setdefault("OMP_PLACES", "cores")  # reference CPU arm
os.environ.setdefault("OMP_PROC_BIND", "close")

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "MPK A^p·x GFLOP/s (fp64 CRS), % of HBM roofline, DRAM bytes/nnz; 1–8 B200"

CONFIGS = {
    "c1": dict(desc="C1: 3D 7-point Laplacian 64^3, lexicographic, p=4", p=4, kind="plain"),
    "c2": dict(desc="C2: 27-point 160^3, off-diag -U[0.9,1.1], (A+A^T)/2, seeded scramble, p=8",
               p=8, kind="plain"),
    "c3": dict(desc="C3: R-MAT scale 21, edge factor 16, symmetrised, p=4", p=4, kind="plain"),
    "c4": dict(desc="C4: 27-point 192^3, Newton basis s=8, theta_k=26+26cos(pi(2k-1)/16)", p=8,
               kind="shifted"),
    "c4poly": dict(desc="C4: 27-point 192^3, z = sum_{k=0..8} c_k A^k x", p=8, kind="poly"),
    "c5": dict(desc="C5: 3D 7-point Laplacian 512^3, p=8", p=8, kind="plain"),
    # the preconditioned s-step basis on C4's matrix (sstep.hpp:122-198)
    "c4jac": dict(desc="C4 matrix, s-step Newton basis s=8 with a 2-sweep Jacobi preconditioner "
                       "(w_p = (A M^-1 - theta_p) w_{p-1})", p=8, kind="sstep_jacobi", sweeps=2),
    "c4gs2": dict(desc="C4 matrix, s-step Newton basis s=8 with GS2 (gamma=1, K=1) "
                       "(w_p = (A M^-1 - theta_p) w_{p-1})", p=8, kind="sstep_gs2", gamma=1, sweeps=1),
}

CONFIGS["c4prod"] = dict(desc="C4 matrix, product-form GMRES polynomial z = p(A) v of degree 40 "
                              "(roots: Leja-ordered Chebyshev points on [0.5, 52] standing in for "
                              "the Eigen-computed harmonic Ritz values)", p=40, kind="polyprod")

CONFIGS["c4ortho"] = dict(desc="C4-sized s-step block orthogonalisation (sstep.hpp:539-545): ICGS of an "
                               "s=8 Newton block against a 25-column basis (2 sweeps, ortho_sweeps=1), "
                               "then TSQR of the block; n = 192^3 rows", p=8, kind="ortho",
                          qcols=25, sweeps=2)

CHAIN_KINDS = ("sstep_jacobi", "sstep_gs2", "polyprod")


def leja_chebyshev_roots(d, lo=0.5, hi=52.0):
    """Deterministic stand-in roots for the polynomial config: Chebyshev points on [lo, hi] in a
    greedy Leja order (largest modulus first, then maximise the product of distances)."""
    pts = [0.5 * (lo + hi) + 0.5 * (hi - lo) * np.cos(np.pi * (2 * k + 1) / (2 * d)) for k in range(d)]
    order = [max(range(d), key=lambda i: abs(pts[i]))]
    while len(order) < d:
        rest = [i for i in range(d) if i not in order]
        order.append(max(rest, key=lambda i: sum(np.log(abs(pts[i] - pts[j])) for j in order)))
    return [pts[i] for i in order]


def make_matrix(cfg: str, seed: int):
    import paper_2309_02228_b200 as mpkg
    if cfg == "c1":
        return mpkg.poisson3d(64, 64, 64)
    if cfg == "c2":
        return mpkg.scramble(mpkg.stencil27_random_sym(160, 160, 160, seed), seed + 1)
    if cfg == "c3":
        return mpkg.rmat(21, 16, seed)
    if cfg in ("c4", "c4poly", "c4jac", "c4gs2", "c4prod"):
        return mpkg.stencil27(192, 192, 192)
    if cfg == "c5":
        return mpkg.poisson3d(512, 512, 512)
    raise SystemExit(f"unknown config {cfg}")


def newton_shifts(s=8):
    return [26.0 + 26.0 * np.cos(np.pi * (2 * k - 1) / 16.0) for k in range(1, s + 1)]


def poly_coefs(seed, d=8):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, d + 1)


def measured_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def host_llc_bytes():
    """Host last-level cache for the reference's blocking budget: sysconf (acceptance.cpp:691), then
    sysfs when sysconf reports 0; the CLI's 32 MiB default (solver.cpp:117-121) only if both fail.
    Returns (bytes, source)."""
    try:
        v = os.sysconf("SC_LEVEL3_CACHE_SIZE")
        if v and v > 0:
            return int(v), "sysconf(_SC_LEVEL3_CACHE_SIZE)"
    except (ValueError, OSError):
        pass
    best = 0
    for idx in pathlib.Path("/sys/devices/system/cpu/cpu0/cache").glob("index*"):
        try:
            if (idx / "level").read_text().strip() != "3":
                continue
            s = (idx / "size").read_text().strip().upper()
            mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}.get(s[-1], 1)
            best = max(best, int(s.rstrip("KMG")) * mult)
        except (OSError, ValueError):
            continue
    if best:
        return best, "sysfs cpu0/cache/index*/size (level 3)"
    return 32 << 20, "CLI default 32 MiB (solver.cpp:117-121)"


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    pg = None
    if world > 1 or os.environ.get("MPKG_FORCE_SHARDED"):
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL between GPUs; MPKG_DIST_BACKEND=gloo only for the single-GPU smoke test of the
        # sharded path (tests/test_gpu_sharded.py), where ranks share one device
        backend = os.environ.get("MPKG_DIST_BACKEND", "nccl")
        if backend == "nccl":
            import torch
            # NCCL needs the rank's device bound before the communicator is created
            torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
        dist.init_process_group(backend)
        dist.barrier()  # the first collective involves every rank (batch_isend_irecv requirement)
        pg = dist
    return rank, world, local, pg


L2_NOMINAL = 126 << 20  # B200 L2 (device-reported 126 MiB); the same string in both arms


def config_dict(name, cfgd, n, nnz, world):
    """The `config` object, identical in both arms (the driver compares them)."""
    d = {"workload": cfgd["desc"], "name": name, "n": n, "nnz": nnz, "p": cfgd["p"],
         "parallelism": "single GPU" if world == 1 else
         f"level-range shards x{world}, p-deep ghost levels, one halo exchange of x per step"}
    mat = 12 * nnz + 4 * (n + 1)
    d["l2"] = (f"inputs larger than L2 ({mat / 1e9:.2f} GB matrix vs {L2_NOMINAL >> 20} MiB L2)"
               if mat > L2_NOMINAL else
               "matrix fits the L2; no flush between steps (L2-resident, latency-bound config)")
    return d


def ref_preprocess(R, A, p, cache):
    """Reference preprocessing on the host (build_levels + permute + group_levels), through handles
    (no second host copy of the matrix: C5 is 11.8 GB).  A = (row_ptr, col_idx, values)."""
    import ctypes as C
    rp, ci, v = A
    n = len(rp) - 1
    h = R.wrap(rp, ci, v)
    lv, pm, ip = (np.empty(n, np.uint32) for _ in range(3))
    lp = np.empty(n + 1, np.uint32)
    nl = C.c_uint32()
    t0 = time.perf_counter()
    assert R.lib.ref_build_levels_h(h, lv.ctypes.data, pm.ctypes.data, ip.ctypes.data,
                                    lp.ctypes.data, C.byref(nl)) == 0, R.lib.ref_last_error()
    lp = lp[: nl.value + 1].copy()
    t1 = time.perf_counter()
    hp = R.lib.ref_permute_h(h, pm.ctypes.data)
    assert hp, R.lib.ref_last_error()
    t2 = time.perf_counter()
    R.lib.ref_csr_free(h)
    del lv, ip
    prp, pci, pv = (C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)())
    R.lib.ref_csr_views(hp, C.byref(prp), C.byref(pci), C.byref(pv))
    nnz = len(ci)
    P = (np.ctypeslib.as_array(prp, (n + 1,)), np.ctypeslib.as_array(pci, (nnz,)),
         np.ctypeslib.as_array(pv, (nnz,)))
    t3 = time.perf_counter()
    gr, _, _, _ = R.group_levels(*P, lp, cache, p)
    t4 = time.perf_counter()
    return (P, hp), pm, gr, {"build_levels_s": t1 - t0, "permute_s": t2 - t1,
                             "group_levels_s": t4 - t3}, lp


def time_reference_mpk(R, hA, n, gr, p, x, kind, steps, warmup, budget_s=60.0, coefs=None):
    """Times the reference's blocked mpk / mpk_shifted through its own API (wall clock), every
    argument built once outside the loop (pre-built handles: matrix, plan, x, shift list, block).
    kind "poly" = the blocked mpk followed by the A23 combination.  Bounded sample:
    after the warm-ups, at most `steps` and at most ~budget_s of timed runs (>= 3).
    Returns (times, timed_steps)."""
    xv = R.lib.ref_vec_new(np.ascontiguousarray(x).ctypes.data, n)
    plan = R.lib.ref_plan_new(n, np.ascontiguousarray(gr, np.uint32).ctypes.data, len(gr) - 1, p)
    blk = R.lib.ref_block_new(n, p + 1)
    hs = None
    if kind == "shifted":
        sh = np.ascontiguousarray(newton_shifts(p))
        hs = R.lib.ref_shifts_new(sh.ctypes.data, np.zeros(p).ctypes.data, p)
    data = np.ctypeslib.as_array(R.lib.ref_block_data(blk), ((p + 1) * n,)).reshape(p + 1, n)

    def one():
        t0 = time.perf_counter()
        if kind == "shifted":
            rc = R.lib.ref_mpk_shifted_t(plan, hA, xv, hs, blk, 0)
        else:
            rc = R.lib.ref_mpk_t(plan, hA, xv, p, blk, 0)
        if kind == "poly":  # A23: z = c_0 y_0, then z += c_k y_k (mul, then add)
            z = coefs[0] * data[0]
            for k in range(1, p + 1):
                z += coefs[k] * data[k]
        t1 = time.perf_counter()
        assert rc == 0, R.lib.ref_last_error()
        return t1 - t0

    times = []
    try:
        for _ in range(max(warmup, 1)):
            t = one()
        k = max(3, min(steps, int(budget_s / max(t, 1e-9))))
        for _ in range(k):
            times.append(one())
    finally:
        if hs:
            R.lib.ref_shifts_free(hs)
        R.lib.ref_block_free(blk)
        R.lib.ref_plan_free(plan)
        R.lib.ref_vec_free(xv)
    return times, len(times)


def run_reference(args, cfgd):
    """`--impl reference`: the reference's own CPU implementation of the path (oracle/_ref, the
    reference headers compiled in place with the reference flags) on this box's host cores, on the
    same config.  Loads only oracle/ libraries: inputs come from the harness generators
    (oracle/_gen), never from the product library."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return  # N>1: rank 0 alone runs the CPU reference
    from oracle.oracle import HarnessGen, Reference, config_matrix, reference_available
    p = cfgd["p"]
    base = {"metric": METRIC, "unit": "GFLOP/s", "impl": "reference", "n_gpus": args.gpus,
            "higher_is_better": True}
    if not reference_available():
        print(json.dumps({**base, "unavailable": "oracle/_ref/libmpkref.so not built"}), flush=True)
        return
    G = HarnessGen()
    if cfgd["kind"] == "ortho":
        # ortho.hpp needs Eigen (not installed): the oracle's C restatement (kind "port")
        n = 192 ** 3
        cb = port_ortho_baseline(cfgd, n, args.seed, args.steps)
        cfg = {"workload": cfgd["desc"], "name": args.config, "n": n, "qcols": cfgd["qcols"],
               "vcols": cfgd["p"]}
        med_ms = cb.pop("ms")
        line = {**base, "value": cb["value"], "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": med_ms, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, DESIGN.md §6)", "config": cfg, "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    R = Reference()
    t0 = time.perf_counter()
    A = config_matrix(args.config, args.seed)
    t_gen = time.perf_counter() - t0
    n, nnz = len(A[0]) - 1, len(A[1])
    cache, cache_src = host_llc_bytes()
    (P, hA), perm, gr, prep, ref_level_ptr = ref_preprocess(R, A, p, cache)
    prep["generate_host_s"] = t_gen
    del A
    x = np.empty(n)
    x[perm] = G.random_vector(n, args.seed + 2)  # permute_vector (csr.hpp:191)
    cfg = config_dict(args.config, cfgd, n, nnz, args.gpus)
    cores = R.resolve_threads(0)
    details = {"cache_bytes": cache, "cache_source": cache_src, "threads": cores,
               "cpu": cpu_model(), "preprocess_s": prep}
    if cfgd["kind"] in CHAIN_KINDS:
        # sstep.hpp / poly.hpp need Eigen: the oracle's C restatement of the same chain (kind "port")
        cb = port_chain_baseline(cfgd, P, x, args.steps)
        R.lib.ref_csr_free(hA)
        med_ms = cb.pop("ms")
        line = {**base, "value": cb["value"], "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": med_ms, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, DESIGN.md §6)", "config": cfg, "details": details,
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    kind = {"shifted": "shifted", "poly": "poly"}.get(cfgd["kind"], "plain")
    coefs = poly_coefs(args.seed + 3, p) if kind == "poly" else None
    times, k = time_reference_mpk(R, hA, n, gr, p, x, kind, args.steps, args.warmup, coefs=coefs)
    med = statistics.median(times)
    flops = 2.0 * nnz * p + (2.0 * n * (p + 1) if kind == "poly" else 0.0)
    gf = flops / med * 1e-9
    # also the reference's baseline_mpk (p plain sweeps) and the blocked mpk at the
    # CLI's default 32 MiB budget (solver.cpp:117-121), through the same pre-built handles
    if kind == "plain":
        xv = R.lib.ref_vec_new(np.ascontiguousarray(x).ctypes.data, n)
        blk = R.lib.ref_block_new(n, p + 1)

        def med3(fn):
            fn()
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                assert fn() == 0, R.lib.ref_last_error()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts)
        try:
            t_base = med3(lambda: R.lib.ref_baseline_mpk_t(hA, xv, p, blk, 0))
            details["reference_baseline_mpk_gflops"] = 2.0 * nnz * p / t_base * 1e-9
            if cache != (32 << 20):
                gr32, _, _, _ = R.group_levels(*P, ref_level_ptr, 32 << 20, p)
                g32 = np.ascontiguousarray(gr32, np.uint32)
                plan32 = R.lib.ref_plan_new(n, g32.ctypes.data, len(g32) - 1, p)
                t32 = med3(lambda: R.lib.ref_mpk_t(plan32, hA, xv, p, blk, 0))
                R.lib.ref_plan_free(plan32)
                details["reference_mpk_32MiB_gflops"] = 2.0 * nnz * p / t32 * 1e-9
        finally:
            R.lib.ref_block_free(blk)
            R.lib.ref_vec_free(xv)
    R.lib.ref_csr_free(hA)
    what = {"shifted": "mpk_shifted", "poly": "mpk + the A23 combination"}.get(kind, "mpk")
    line = {**base, "value": gf, "steps": k, "warmup": max(args.warmup, 1),
            "ms_per_step": med * 1e3, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, DESIGN.md §6)", "config": cfg, "details": details,
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                             "sample": f"full {args.config} workload, reference blocked {what} "
                                       f"(p={p}, LLC budget {cache >> 20} MiB from {cache_src}), "
                                       f"median of {k} after {max(args.warmup, 1)} warm-up "
                                       f"({med:.3f} s each; at most ~60 s timed)"},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def chain_flops(cfgd, nnz, n):
    """Flop convention of the chain / polynomial configs (SpMV-shaped stages, 2 per entry)."""
    p = cfgd["p"]
    if cfgd["kind"] == "sstep_jacobi":  # (sweeps - 1) Jacobi sweeps + the terminal product per power
        return 2.0 * nnz * p * cfgd["sweeps"]
    if cfgd["kind"] == "sstep_gs2":  # per sweep: full-row stage 0 + gamma half-row inner; terminal
        return p * (cfgd["sweeps"] * (2.0 * nnz + cfgd["gamma"] * nnz) + 2.0 * nnz)
    if cfgd["kind"] == "polyprod":  # degree-1 SpMV-shaped terminals
        return 2.0 * nnz * (p - 1)
    raise ValueError(cfgd["kind"])


def port_chain_baseline(cfgd, P, x, steps):
    """The chain configs' CPU baseline: the oracle's C restatement (one thread) of the same chain on
    the same A_perm and x -- the reference's own sstep.hpp / poly.hpp need Eigen and do not build
    here.  Bounded sample: 1 warm-up + min(steps, 3) timed runs of the full workload."""
    from oracle.oracle import Oracle
    O = Oracle()
    rp, ci, v = P
    p = cfgd["p"]
    if cfgd["kind"] == "sstep_jacobi":
        fn = lambda: O.sstep_jacobi_block(rp, ci, v, cfgd["sweeps"], x, newton_shifts(p))  # noqa: E731
    elif cfgd["kind"] == "sstep_gs2":
        fn = lambda: O.sstep_gs2_block(rp, ci, v, cfgd["gamma"], cfgd["sweeps"], True, x, newton_shifts(p))  # noqa: E731
    else:
        roots = leja_chebyshev_roots(p)
        fn = lambda: O.poly_apply(rp, ci, v, roots, x)  # noqa: E731
    fn()
    k = max(1, min(steps, 3))
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    gf = chain_flops(cfgd, len(ci), len(rp) - 1) / med * 1e-9
    return {"value": gf, "unit": "GFLOP/s", "cores": 1, "kind": "port", "ms": med * 1e3,
            "sample": f"full workload through the oracle's C restatement (oracle/oracle.c, one thread; "
                      f"the reference's chain driver needs Eigen): 1 warm-up + median of {k} "
                      f"({med:.2f} s each); cpu: {cpu_model()}"}


def port_ortho_baseline(cfgd, n, seed, steps):
    """c4ortho's CPU baseline: ICGS + TSQR through the oracle's C restatement (one thread) on a
    seeded block of the same shape (ortho.hpp needs Eigen).  1 warm-up-free timed run per step,
    at most 2."""
    from oracle.oracle import Oracle
    O = Oracle()
    rng = np.random.default_rng(seed)
    Q, _ = O.tsqr(rng.uniform(-1.0, 1.0, (cfgd["qcols"], n)))
    V0 = rng.uniform(-1.0, 1.0, (cfgd["p"], n))
    k = max(1, min(steps, 2))
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        Vo, _ = O.icgs(Q, V0, cfgd["sweeps"])
        O.tsqr(Vo)
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    s, qc = cfgd["p"], cfgd["qcols"]
    flops = cfgd["sweeps"] * 4.0 * n * qc * s + 4.0 * n * s * s
    return {"value": flops / med * 1e-9, "unit": "GFLOP/s", "cores": 1, "kind": "port", "ms": med * 1e3,
            "sample": f"full workload (n = {n}, {qc}-column basis, {s}-column block, {cfgd['sweeps']} "
                      f"sweeps + TSQR) through the oracle's C restatement, one thread: median of {k} "
                      f"({med:.2f} s each); cpu: {cpu_model()}"}


def cpu_baseline_reference(A_perm_host, ls_level_ptr, p, x, kind, nnz, coefs=None):
    """cpu_baseline of the GPU arm: the reference's blocked mpk (oracle/_ref) on the host cores, on
    the GPU path's A_perm (bit-identical to the reference's, tests/test_gpu_fullsize.py), bounded:
    1 warm-up + median of 3 full-workload calls."""
    from oracle.oracle import Oracle, Reference, reference_available
    cache, cache_src = host_llc_bytes()
    n = A_perm_host.n_rows
    if reference_available():
        R = Reference()
        P = (A_perm_host.row_ptr, A_perm_host.col_idx, A_perm_host.values)
        gr, _, _, _ = R.group_levels(*P, ls_level_ptr, cache, p)
        hA = R.wrap(*P)
        try:
            times, k = time_reference_mpk(R, hA, n, gr, p, x, kind, 3, 1, budget_s=30.0, coefs=coefs)
        finally:
            R.lib.ref_csr_free(hA)
        med = statistics.median(times)
        flops = 2.0 * nnz * p + (2.0 * n * (p + 1) if kind == "poly" else 0.0)
        what = {"shifted": "mpk_shifted", "poly": "mpk + the A23 combination"}.get(kind, "mpk")
        return {"value": flops / med * 1e-9, "unit": "GFLOP/s",
                "cores": R.resolve_threads(0), "kind": "reference",
                "sample": f"full workload, reference blocked {what} (OpenMP, p={p}, LLC budget "
                          f"{cache >> 20} MiB from {cache_src}): 1 warm-up + median of {k} "
                          f"({med:.3f} s each); cpu: {cpu_model()}"}
    O = Oracle()
    t0 = time.perf_counter()
    O.baseline_mpk(A_perm_host.row_ptr, A_perm_host.col_idx, A_perm_host.values, x, 1)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * nnz / dt * 1e-9, "unit": "GFLOP/s", "cores": 1, "kind": "port",
            "sample": "one SpMV sweep of the oracle port (single thread)"}


def run_sharded(args, cfgd, ctx, A, ls, Ap, x_perm, p, rank, world, local, dist, info, prep,
                stream, sync):
    """N > 1: the matrix is row-partitioned along contiguous BFS-level ranges (balanced by nnz)
    with p ghost levels per side (multi.py).  A step = one halo exchange of x
    (NCCL point-to-point over NVLink) + the local MPK; every rank owns a fixed share of ONE
    matrix (strong scaling).  value = the global MPK flops / the slowest rank's step time."""
    import torch

    from paper_2309_02228_b200 import multi
    if cfgd["kind"] != "plain":
        raise SystemExit("multi-GPU bench runs the plain MPK configs (c1, c2, c3, c5)")
    n, nnz = A.n_rows, A.nnz
    dev = torch.device("cuda", local)
    lens = np.diff(A.row_ptr.astype(np.int64))[ls.inv_perm.astype(np.int64)]
    prefix = np.concatenate([[0], np.cumsum(lens)])
    t0 = time.perf_counter()
    shard = multi.ShardedMPK(ctx, Ap, ls.level_ptr, prefix, p, rank, world)
    sync()
    prep["shard_setup_s"] = time.perf_counter() - t0
    hp = shard.halo_plan
    o0, o1 = hp.own_rows
    x_own = torch.from_numpy(np.ascontiguousarray(x_perm[o0:o1])).to(dev)
    blk = torch.empty((p + 1) * max(shard.n_local, 1), dtype=torch.float64, device=dev)

    def step():
        return shard.step(x_own, blk, dist)

    step()
    sync()
    # parity: own rows == the single-GPU one-launch-per-power result, bit for bit
    ref = torch.empty((p + 1) * n, dtype=torch.float64, device=dev)
    ctx.baseline_mpk_dev(Ap, torch.from_numpy(x_perm).to(dev).data_ptr(), p, ref.data_ptr(), n, p + 1)
    sync()
    a0, a1 = shard.own
    mine = blk.view(p + 1, -1)[:, a0:a1] if shard.n_local else blk[:0].view(p + 1, 0)
    parity = bool(torch.equal(mine.contiguous().view(torch.int64),
                              ref.view(p + 1, n)[:, o0:o1].contiguous().view(torch.int64)))
    del ref
    torch.cuda.empty_cache()
    for _ in range(args.warmup):
        step()
    sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    sync()
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("mpk_timed")
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        sync()
        torch.cuda.nvtx.range_pop()
    dist.barrier()
    launches = ctx.launch_count() - launches0
    step_ms = ev0.elapsed_time(ev1) / args.steps
    ctx.set_param("kernel_timing", 1)  # kernel time: a second pass with per-call events
    for _ in range(args.steps):
        step()
    sync()
    k_total, k_count, _ = ctx.kernel_times()
    kernel_ms = k_total / max(k_count, 1)
    ctx.set_param("kernel_timing", 0)
    dist.barrier()
    # e2e: own x from pinned host memory, exchange + local MPK, own rows back to the host
    hx = torch.from_numpy(np.ascontiguousarray(x_perm[o0:o1])).pin_memory()
    hout = torch.empty((p + 1, o1 - o0), dtype=torch.float64).pin_memory()
    ts = []
    for _ in range(max(3, min(args.steps, 10))):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            x_own.copy_(hx, non_blocking=True)
            step()
            hout.copy_(blk.view(p + 1, -1)[:, a0:a1], non_blocking=True)
            b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    e_ms = statistics.median(ts)
    t = torch.tensor([step_ms, kernel_ms, e_ms, float(not parity)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, kernel_ms, e_ms, bad = t.tolist()
    parity = bad == 0.0
    flops = 2.0 * nnz * p
    value = flops / (step_ms * 1e-3) * 1e-9
    clocks = clk.summary()
    nnz_loc = shard.A.nnz
    b_loc = 12 * nnz_loc + 4 * (shard.n_local + 1) + 8 * shard.n_local * (1 + p)
    peak, peak_src = measured_peak()
    achieved = b_loc / (kernel_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators for the BASELINE.json config, DESIGN.md §6)",
            "config": config_dict(args.config, cfgd, n, nnz, world),
            "parity": ("own rows == single-GPU baseline bitwise (all ranks)" if parity else "MISMATCH"),
            "details": {"mode": "bitwise", "backend": dist.get_backend(),
                        "rank0_shard": {"own_rows": [o0, o1], "local_rows": list(hp.local_rows),
                                        "local_nnz": nnz_loc},
                        "executor": shard.plan.exec_info(), "preprocess_s": prep},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes": b_loc, "kernel_ms": kernel_ms,
                         "kernel_launches_timed": k_count, "peak_source": peak_src,
                         "note": "per rank (slowest): local single-pass bytes / local MPK time"},
            "cpu_baseline": None,
            "e2e": {"value": flops / (e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n * (p + 1),
                    "ms_per_step": e_ms, "note": "per rank: own x in, own rows of y_0..y_p out"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    if not parity:
        sys.exit(3)


def _bits_checksum(t, lo, hi):
    """Order-sensitive 64-bit checksums of rows [lo, hi) of every slice of a (p+1, rows) block
    (int64 views, wrap-around sums): a size-independent bitwise parity probe."""
    import torch
    v = t[:, lo:hi].contiguous().view(torch.int64)
    w = (torch.arange(hi - lo, device=v.device, dtype=torch.int64) % 65521) + 1
    return torch.stack([v.sum(1), (v * w).sum(1)], 1).cpu()


def run_sharded_nccl(args, cfgd, rank, world, local, dist):
    """N > 1 over NCCL through the C-ABI shard layer (mpkg_dist_*, csrc/dist.cu): rank 0 alone
    generates the matrix, builds the levels and A_perm, and partitions the levels (balanced by nnz);
    level_ptr and the bounds are broadcast; every rank receives only its own block A_perm[g0:g1,
    g0:g1] and its own rows of x from rank 0.  A step = one halo exchange of x (grouped ncclSend /
    ncclRecv into a preallocated buffer) + the local MPK; every rank owns a fixed share of ONE
    matrix (strong scaling).  value = the global MPK flops / the slowest rank's step time."""
    import torch

    import paper_2309_02228_b200 as mpkg
    from paper_2309_02228_b200 import multi
    if cfgd["kind"] != "plain":
        raise SystemExit("multi-GPU bench runs the plain MPK configs (c1, c2, c3, c5)")
    p = cfgd["p"]
    dev = torch.device("cuda", local)
    ctx = mpkg.Context(local)
    ctx.set_param("order", args.order)
    ctx.set_param("schedule", args.schedule)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)

    def sync():
        ctx.synchronize()
        torch.cuda.synchronize()

    prep = {}
    uid = [multi.NcclDist.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    D = multi.NcclDist(ctx, world, rank, uid[0])
    t0 = time.perf_counter()
    Ap = ls = d_full = None
    meta = np.zeros(3, np.uint64)
    if rank == 0:
        A = make_matrix(args.config, args.seed)
        dA = ctx.csr(A)
        ls = ctx.build_levels(dA)
        Ap = ctx.permute(dA, ls)
        del dA
        lp = np.asarray(ls.level_ptr, np.uint32)
        lens = np.diff(A.row_ptr.astype(np.int64))[ls.inv_perm.astype(np.int64)]
        nnz_before = np.concatenate([[0], np.cumsum(lens)])[lp.astype(np.int64)]
        bounds = multi.dist_partition(lp, nnz_before, world)
        x_perm = ctx.permute_vector(mpkg.random_vector(A.n_rows, args.seed + 2), ls.perm)
        d_full = torch.from_numpy(x_perm).to(dev)
        meta[:] = (len(lp) - 1, A.n_rows, A.nnz)
        del A
    D.bcast_host(meta, 0)
    nl, n, nnz = (int(v) for v in meta)
    if rank != 0:
        lp, bounds = np.zeros(nl + 1, np.uint32), np.zeros(world + 1, np.uint32)
    D.bcast_host(lp, 0)
    D.bcast_host(bounds, 0)
    prep["root_preprocess_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    D.set_plan(lp, bounds, p)
    info = D.info()
    o0, o1 = info["own"]
    g0, g1 = info["local"]
    n_local = g1 - g0
    A_loc = D.scatter_blocks(0, Ap)
    x_own = torch.empty(max(o1 - o0, 1), dtype=torch.float64, device=dev)
    D.scatter_rows(0, d_full.data_ptr() if d_full is not None else 0, x_own.data_ptr())
    L0, L1 = int(bounds[rank]), int(bounds[rank + 1])
    llp = multi.local_level_ptr(lp, L0, L1, p)
    ident = np.arange(n_local, dtype=np.uint32)
    lls = ctx.levels_from_host(np.zeros(n_local, np.uint32), ident, ident, llp)
    plan = ctx.group_levels(lls, A_loc, ctx.device_info()["l2_bytes"], p)
    blk = torch.empty((p + 1) * max(n_local, 1), dtype=torch.float64, device=dev)
    sync()
    prep["shard_setup_s"] = time.perf_counter() - t0

    def step():
        D.mpk(plan, A_loc, x_own.data_ptr(), p, blk.data_ptr(), max(n_local, 1), p + 1)

    step()
    sync()
    # parity: every rank's own rows == rank 0's single-GPU one-launch-per-power result, bit for bit
    # (order-sensitive checksums of the bit patterns, compared on rank 0)
    a0, a1 = o0 - g0, o1 - g0
    mine = _bits_checksum(blk.view(p + 1, -1), a0, a1) if n_local else torch.zeros(p + 1, 2, dtype=torch.int64)
    gathered = [None] * world
    dist.all_gather_object(gathered, (o0, o1, mine))
    parity = True
    if rank == 0:
        ref = torch.empty((p + 1) * n, dtype=torch.float64, device=dev)
        ctx.baseline_mpk_dev(Ap, d_full.data_ptr(), p, ref.data_ptr(), n, p + 1)
        sync()
        for r0, r1, cs in gathered:
            if r1 > r0:
                parity &= bool(torch.equal(cs, _bits_checksum(ref.view(p + 1, n), r0, r1)))
        del ref
    del Ap, d_full
    torch.cuda.empty_cache()
    for _ in range(args.warmup):
        step()
    sync()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    sync()
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("mpk_timed")
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        sync()
        torch.cuda.nvtx.range_pop()
    dist.barrier()
    launches = ctx.launch_count() - launches0
    step_ms = ev0.elapsed_time(ev1) / args.steps
    ctx.set_param("kernel_timing", 1)
    for _ in range(args.steps):
        step()
    sync()
    k_total, k_count, _ = ctx.kernel_times()
    kernel_ms = k_total / max(k_count, 1)
    ctx.set_param("kernel_timing", 0)
    dist.barrier()
    # e2e: own x from pinned host memory, exchange + local MPK, own rows back to the host
    hx = x_own.cpu().pin_memory()
    hout = torch.empty((p + 1, max(o1 - o0, 0)), dtype=torch.float64).pin_memory()
    ts = []
    for _ in range(max(3, min(args.steps, 10))):
        dist.barrier()
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            x_own.copy_(hx, non_blocking=True)
            step()
            if o1 > o0:
                hout.copy_(blk.view(p + 1, -1)[:, a0:a1], non_blocking=True)
            b_.record(stream)
        b_.synchronize()
        ts.append(a.elapsed_time(b_))
    e_ms = statistics.median(ts)
    t = torch.tensor([step_ms, kernel_ms, e_ms, float(not parity)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    step_ms, kernel_ms, e_ms, bad = t.tolist()
    parity = bad == 0.0
    flops = 2.0 * nnz * p
    value = flops / (step_ms * 1e-3) * 1e-9
    clocks = clk.summary()
    b_loc = 12 * A_loc.nnz + 4 * (n_local + 1) + 8 * n_local * (1 + p)
    peak, peak_src = measured_peak()
    achieved = b_loc / (kernel_ms * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators for the BASELINE.json config, DESIGN.md §6)",
            "config": config_dict(args.config, cfgd, n, nnz, world),
            "parity": ("own rows == single-GPU baseline bitwise (checksums of every rank's own rows)"
                       if parity else "MISMATCH"),
            "details": {"mode": "bitwise", "backend": "nccl (mpkg_dist_* C ABI)",
                        "rank0_shard": {"own_rows": [o0, o1], "local_rows": [g0, g1],
                                        "local_nnz": A_loc.nnz, "halo_send_bytes": info["send_bytes"],
                                        "halo_recv_bytes": info["recv_bytes"]},
                        "executor": plan.exec_info(), "preprocess_s": prep},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "algorithmic_bytes": b_loc, "kernel_ms": kernel_ms,
                         "kernel_launches_timed": k_count, "peak_source": peak_src,
                         "note": "per rank (slowest): local single-pass bytes / local MPK time"},
            "cpu_baseline": None,
            "e2e": {"value": flops / (e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n * (p + 1),
                    "ms_per_step": e_ms, "note": "per rank: own x in, own rows of y_0..y_p out"},
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    D.close()
    dist.destroy_process_group()
    if not parity:
        sys.exit(3)


def _ncu_traffic(name):
    """DRAM read + write bytes of one step from the committed ncu summary (profiles/), or None."""
    prof = ROOT / "profiles" / f"ncu_{name}.json"
    try:
        return json.loads(prof.read_text()).get("dram_bytes_per_step")
    except Exception:
        return None


def run_ortho(args, cfgd):
    """the step after the MPK in s-step GMRES.  A step = ICGS of the s-vector
    Newton block V against the basis Q (`sweeps` rounds of block_dots + block_update) followed by
    TSQR of V (sstep.hpp:539-545), with Q and V resident in HBM.  The headline runs the fast mode
    (fp64 tensor-core block_dots); the bitwise mode (the reference's serial dot sums) is timed once
    beside it.  Algorithmic bytes: the first sweep's dots read Q and V, every update (each but the
    last fused with the next sweep's dots) reads Q and V and writes V; TSQR reads V and writes Q."""
    import torch

    import paper_2309_02228_b200 as mpkg
    rank = int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1)
    world = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    n, qc, s, sweeps = 192 ** 3, cfgd["qcols"], cfgd["p"], cfgd["sweeps"]
    ctx = mpkg.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    g = torch.Generator(device=dev).manual_seed(args.seed)
    Q = torch.rand((qc, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    R = torch.empty((qc, qc), dtype=torch.float64, device=dev)
    ctx.tsqr_dev(Q.data_ptr(), n, qc, R.data_ptr())  # orthonormal basis
    V0 = torch.rand((s, n), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    V = V0.clone()
    coeff = torch.empty((s, qc), dtype=torch.float64, device=dev)
    Rv = torch.empty((s, s), dtype=torch.float64, device=dev)

    def sync():
        ctx.synchronize()
        torch.cuda.synchronize()

    def step():  # sstep.hpp:539-545 (icgs then tsqr) through the combined entry point
        ctx.ortho_block_dev(Q.data_ptr(), n, qc, V.data_ptr(), s, sweeps, coeff.data_ptr(), Rv.data_ptr())

    def timed(k, fn):
        sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        sync()
        return a.elapsed_time(b) / k

    # bitwise (the reference's serial sums), one step, then the parity properties of both modes
    ctx.set_mode(0)
    V.copy_(V0)
    sync()
    bitwise_ms = timed(1, step)
    Vb, cb = V.clone(), coeff.clone()
    ctx.set_mode(1)
    V.copy_(V0)
    sync()
    step()
    sync()
    eye = torch.eye(s, dtype=torch.float64, device=dev)
    props = {
        "fast_vs_bitwise_coeff_maxrel": ((coeff - cb).abs().max() / cb.abs().max()).item(),
        "fast_vs_bitwise_q_maxabs": (V - Vb).abs().max().item(),
        "q_orthonormal_maxabs": (V @ V.T - eye).abs().max().item(),
        "q_perp_basis_maxabs": (Q @ V.T).abs().max().item(),
    }
    parity = (props["fast_vs_bitwise_coeff_maxrel"] <= 1e-12 and props["q_orthonormal_maxabs"] <= 1e-12
              and props["q_perp_basis_maxabs"] <= 1e-12)
    for _ in range(args.warmup):
        V.copy_(V0)
        step()
    sync()
    ctx.set_param("kernel_timing", 1)
    ctx.kernel_times()
    launches0 = ctx.launch_count()
    ts = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            V.copy_(V0)  # untimed reset (V is orthogonalised in place)
            ts.append(timed(1, step))
    launches = ctx.launch_count() - launches0
    k_total, k_count, _ = ctx.kernel_times()
    ctx.set_param("kernel_timing", 0)
    step_ms = statistics.median(ts)
    kernel_ms = k_total / args.steps
    flops = sweeps * 4.0 * n * qc * s + 4.0 * n * s * s  # dots + update per sweep; Householder QR + form Q
    # fast-mode ICGS: the first sweep's dots read Q and V; every update (fused with the next sweep's
    # dots, the last one with TSQR's first factor) reads Q and V and writes V (the last one writes
    # the reflectors); TSQR's apply reads them and writes Q
    b_alg = 8.0 * n * ((qc + s) + sweeps * (qc + 2 * s) + 2 * s)
    peak, peak_src = measured_peak()
    achieved = b_alg / (kernel_ms * 1e-3) / 1e9

    # e2e: the host-pointer ABI (pinned Q and V in, V and the coefficients / R out)
    hQ = Q.cpu().pin_memory()
    hV = torch.empty((s, n), dtype=torch.float64).pin_memory()
    hc = np.zeros((s, qc))
    hr = np.zeros((s, s))
    from paper_2309_02228_b200._lib import check, lib
    e_ts = []
    for _ in range(max(3, min(args.steps, 10))):
        hV.copy_(V0.cpu())
        t0 = time.perf_counter()
        check(lib.mpkg_ortho_block(ctx.h, hQ.data_ptr(), n, qc, hV.data_ptr(), s, sweeps, hc.ctypes.data,
                                   hr.ctypes.data))
        e_ts.append((time.perf_counter() - t0) * 1e3)
    e_ms = statistics.median(e_ts)
    e2e = {"value": flops / (e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s",
           "h2d_bytes_per_step": 8 * n * (qc + s),
           "d2h_bytes_per_step": 8 * n * s + 8 * (s * qc + s * s), "ms_per_step": e_ms,
           "note": "one host-pointer call (mpkg_ortho_block), wall clock"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = port_ortho_baseline(cfgd, n, args.seed, args.steps)
        cpu.pop("ms")
    if rank == 0:
        line = {
            "metric": METRIC, "value": flops / (step_ms * 1e-3) * 1e-9, "unit": "GFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] block; basis = TSQR of a seeded U[-1,1] block)",
            "config": {"workload": cfgd["desc"], "n": n, "qcols": qc, "vcols": s, "sweeps": sweeps,
                       "mode": "fast (tensor-core block_dots, fixed-order reduction)",
                       "bitwise_ms_per_step": bitwise_ms,
                       "l2": "inputs larger than L2 (%.2f GB)" % (8 * n * (qc + s) / 1e9),
                       "parity": ("ok " if parity else "MISMATCH ") + json.dumps(props)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _ncu_traffic("c4ortho"), "algorithmic_bytes": b_alg,
                         "kernel_ms": kernel_ms, "kernel_launches_timed": k_count,
                         "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if not parity:
        sys.exit(3)


DIGESTS = ROOT / "tests" / "golden" / "config_digests.json"


def _sha(a) -> str:
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()


def reference_digest_parity(name, seed, kind, ls, Ap, x_perm, d_blk, p, n, d_z=None):
    """Bench-time parity against the REFERENCE: SHA-256 of this run's levels, perm, inv_perm,
    level_ptr, A_perm, x and every basis slice (or z) against the digests of the reference's own
    outputs on the same inputs (tests/golden/config_digests.json, made by
    tests/golden/make_config_digests.py from oracle/_ref).  None when no digest exists for this
    config / seed."""
    key = {"c2": "c2", "c3": "c3", "c4": "c4", "c4poly": "c4", "c5": "c5"}.get(name)
    if key is None or not DIGESTS.exists():
        return None
    d = json.loads(DIGESTS.read_text()).get(key)
    if d is None or d.get("seed") != seed:
        return None
    bad = [k for k in ("levels", "perm", "inv_perm", "level_ptr") if _sha(getattr(ls, k)) != d[k]]
    P = Ap.download()
    bad += [f"A_perm.{k}" for k in ("row_ptr", "col_idx", "values") if _sha(getattr(P, k)) != d[f"A_perm.{k}"]]
    del P
    if _sha(x_perm) != d["x_perm"]:
        bad.append("x_perm")
    what = ["levels", "perm", "inv_perm", "level_ptr", "A_perm", "x"]
    if kind == "poly":
        if _sha(d_z.cpu().numpy()) != d["poly_z"]:
            bad.append("z")
        what.append("z")
    ref = d["mpk_shifted"] if kind == "shifted" else d["mpk"]
    for k in range(p + 1):
        if _sha(d_blk[k * n:(k + 1) * n].cpu().numpy()) != ref[k]:
            bad.append(f"slice {k}")
    what.append(f"slices 0..{p}")
    return {"match": not bad, "mismatches": bad, "checked": what}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="mpkg", choices=["mpkg", "reference"])
    ap.add_argument("--seed", type=int, default=2309)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--slack", type=int, default=-1)
    ap.add_argument("--order", type=int, default=-1,
                    help="-1 auto, 0 A_perm order, 1 CM inside levels, 2 longest rows first")
    ap.add_argument("--schedule", type=int, default=0,
                    help="0 auto, 1 fused tile-DAG kernel, 2 one launch per power, 3 wave (cross-power L2 reuse)")
    ap.add_argument("--mode", default="bitwise", choices=["bitwise", "fast"],
                    help="fast: long rows reduced in parallel, checked to 1e-12 inf-norm (mpkg.h)")
    ap.add_argument("--kernel", type=int, default=0, help="fused variant: 0 lean, 1 staged, 2 warp-tile, 4 async")
    ap.add_argument("--pass-powers", type=int, default=0, help="force powers per fused pass")
    ap.add_argument("--l2-budget", type=int, default=0, help="live-window bytes (0: 0.6 L2)")
    ap.add_argument("--ctas-per-sm", type=int, default=0, help="cap on fused CTAs per SM")
    ap.add_argument("--group", type=int, default=8, help="staged variant: gathers in flight (8|16)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfgd = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own launch sets
        # WORLD_SIZE and lands below)
        import socket
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(port), str(pathlib.Path(__file__).resolve()), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    world_env = int(os.environ.get("WORLD_SIZE", 1))
    if world_env != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.impl == "reference":
        return run_reference(args, cfgd)
    if cfgd["kind"] == "ortho":
        return run_ortho(args, cfgd)

    import torch

    import paper_2309_02228_b200 as mpkg

    rank, world, local, dist = dist_setup(args.gpus)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if dist is not None and dist.get_backend() == "nccl":
        # the C-ABI shard layer: only rank 0 builds the matrix (MPKG_FORCE_SHARDED=1 exercises it
        # at world 1 as well)
        return run_sharded_nccl(args, cfgd, rank, world, local, dist)
    p = cfgd["p"]
    t0 = time.perf_counter()
    A = make_matrix(args.config, args.seed)
    t_gen = time.perf_counter() - t0
    n, nnz = A.n_rows, A.nnz

    ctx = mpkg.Context(local)
    if args.slack >= 0:
        ctx.set_param("slack", args.slack)
    ctx.set_param("order", args.order)
    ctx.set_param("schedule", args.schedule)
    ctx.set_mode(1 if args.mode == "fast" else 0)
    ctx.set_param("kernel", args.kernel)
    ctx.set_param("pass", args.pass_powers)
    ctx.set_param("l2_budget", args.l2_budget)
    ctx.set_param("ctas_per_sm", args.ctas_per_sm)
    ctx.set_param("group", args.group)
    info = ctx.device_info()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    def sync():
        ctx.synchronize()
        torch.cuda.synchronize()

    prep = {"generate_host_s": t_gen}
    t0 = time.perf_counter()
    dA = ctx.csr(A)
    sync()
    prep["upload_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ls = ctx.build_levels(dA)
    sync()
    prep["build_levels_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    Ap = ctx.permute(dA, ls)
    sync()
    prep["permute_s"] = time.perf_counter() - t0
    cache = info["l2_bytes"]
    t0 = time.perf_counter()
    plan = ctx.group_levels(ls, Ap, cache, p)
    prep["group_levels_s"] = time.perf_counter() - t0
    del dA

    x_host = mpkg.random_vector(n, args.seed + 2)
    x_perm = ctx.permute_vector(x_host, ls.perm)  # csr.hpp:191 permute_vector
    if world > 1:
        return run_sharded(args, cfgd, ctx, A, ls, Ap, x_perm, p, rank, world, local, dist, info,
                           prep, stream, sync)
    dev = torch.device("cuda", local)
    d_x = torch.from_numpy(x_perm).to(dev)
    d_blk = torch.empty((p + 1) * n, dtype=torch.float64, device=dev)
    d_z = torch.empty(n, dtype=torch.float64, device=dev)
    shifts = newton_shifts(p)
    coefs = poly_coefs(args.seed + 3, p)

    chain = None
    if cfgd["kind"] in CHAIN_KINDS:
        from paper_2309_02228_b200._lib import check as _check, lib as _lib
        if cfgd["kind"] == "polyprod":
            precon = None
            roots = leja_chebyshev_roots(p)
            pr_re, pr_im = np.ascontiguousarray(roots, np.float64), np.zeros(p)
            cplan = ctx.group_levels(ls, Ap, cache, 8)  # roots sliced into passes of 8 powers
            d_zp = torch.empty(n, dtype=torch.float64, device=dev)

            def chain(bp, pl):  # z = p(A) x into the block's last slice (slices 1..p unused)
                _check(_lib.mpkg_poly_apply_dev(ctx.h, Ap.h, None, None, pr_re.ctypes.data,
                                                pr_im.ctypes.data, p, pl.h if pl is not None else None,
                                                d_x.data_ptr(), bp + 8 * n * p))
        elif cfgd["kind"] == "sstep_jacobi":
            precon = ctx.jacobi_setup(Ap, cfgd["sweeps"])
            budget, run = p, _lib.mpkg_sstep_jacobi_dev
        else:
            precon = ctx.gs2_setup(Ap, cfgd["gamma"], cfgd["sweeps"])
            budget, run = p * cfgd["sweeps"], _lib.mpkg_sstep_gs2_dev
        if cfgd["kind"] != "polyprod":
            cplan = ctx.group_levels(ls, Ap, cache, budget).with_sub_powers(precon.stages(), ls.level_ptr)
            ch_re = np.ascontiguousarray(shifts, np.float64)
            ch_im = np.zeros(p)
            d_blk[:n].copy_(d_x)  # slice 0 = x (the chain writes slices 1..p)

            def chain(bp, pl):
                _check(run(ctx.h, precon.h, pl.h if pl is not None else None, Ap.h, ch_re.ctypes.data,
                           ch_im.ctypes.data, p, bp, n, p + 1))

    def step(block_ptr=None):
        bp = d_blk.data_ptr() if block_ptr is None else block_ptr
        if chain is not None:
            chain(bp, cplan)
        elif cfgd["kind"] == "shifted":
            ctx.mpk_shifted_dev(plan, Ap, d_x.data_ptr(), shifts, bp, n, p + 1)
        elif cfgd["kind"] == "poly":
            ctx.mpk_poly_dev(plan, Ap, d_x.data_ptr(), coefs, d_z.data_ptr(), bp, n, p + 1)
        else:
            ctx.mpk_dev(plan, Ap, d_x.data_ptr(), p, bp, n, p + 1)

    t0 = time.perf_counter()
    step()  # builds the GPU schedule (SELL copy, tile dependencies, ticket order) once
    sync()
    prep["executor_build_s"] = time.perf_counter() - t0
    exec_info = plan.exec_info()
    kname = ("k_mpk_sweep" if exec_info["schedule"] == "sweeps" else "k_mpk_wave" if exec_info["schedule"] == "wave" else
             {0: "k_mpk_lean", 1: "k_mpk_fused", 2: "k_mpk_warptile", 4: "k_mpk_async"}.get(exec_info["kernel"], "?"))
    if exec_info["schedule"] == "sweeps" and exec_info.get("long_rows"):
        kname = ("k_coop_rows (side stream) beside k_mpk_sweep" if args.mode == "fast" else
                 "k_long_rows_bitwise (side stream, the hub row's add chain) beside k_mpk_sweep")
    exec_info["dominant_kernel"] = kname
    if chain is not None:
        exec_info = {"dominant_kernel": "k_poly_terminal" if precon is None else "k_pc_stage / k_gs2_stage (precon.cu)",
                     "stages_per_power": 1 if precon is None else precon.stages(),
                     "plan_groups": cplan.n_groups()}

    # ---- parity at full size: fused == one-launch-per-power baseline, bit for bit -------------
    ref_blk = torch.empty_like(d_blk)
    if chain is not None:  # the plan-driven chain == its sequential form (oracle parity: tests/)
        ref_blk[:n].copy_(d_x)
        chain(ref_blk.data_ptr(), None)
    elif cfgd["kind"] == "shifted":
        import ctypes
        from paper_2309_02228_b200._lib import check, lib
        re = np.ascontiguousarray(shifts, np.float64)
        im = np.zeros(p)
        check(lib.mpkg_baseline_mpk_shifted_dev(ctx.h, Ap.h, d_x.data_ptr(), re.ctypes.data,
                                                im.ctypes.data, p, ref_blk.data_ptr(), n, p + 1))
        _ = ctypes
    else:
        ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), p, ref_blk.data_ptr(), n, p + 1)
    sync()
    if cfgd["kind"] == "polyprod":  # only z (the last slice) is produced
        parity = bool(torch.equal(ref_blk[p * n:].view(torch.int64), d_blk[p * n:].view(torch.int64)))
    else:
        parity = bool(torch.equal(ref_blk.view(torch.int64), d_blk.view(torch.int64)))
    max_rel_err = 0.0
    if args.mode == "fast":  # north star: every basis vector within 1e-12 (inf-norm, relative)
        a_, b_ = d_blk.view(p + 1, n), ref_blk.view(p + 1, n)
        errs = ((a_ - b_).abs().amax(dim=1) / b_.abs().amax(dim=1).clamp_min(1e-300)).tolist()
        max_rel_err = max(errs)
        parity = max_rel_err <= 1e-12
    if cfgd["kind"] == "poly":
        zr = torch.from_numpy(coefs[0] * ref_blk[:n].cpu().numpy())
        # the oracle's A23 order (c0*y0, then += c_k*y_k) checked on the host copy
        rb = ref_blk.view(p + 1, n).cpu().numpy()
        acc = coefs[0] * rb[0]
        for k in range(1, p + 1):
            acc = acc + coefs[k] * rb[k]
        parity = parity and np.array_equal(acc.view(np.uint64), d_z.cpu().numpy().view(np.uint64))
        del zr
    # baseline kernel timing for reference (p back-to-back launches)
    ctx.set_param("kernel_timing", 1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(3):
        ctx.baseline_mpk_dev(Ap, d_x.data_ptr(), p, ref_blk.data_ptr(), n, p + 1)
    ev1.record(stream)
    sync()
    baseline_ms = ev0.elapsed_time(ev1) / 3
    ctx.kernel_times()
    ctx.set_param("kernel_timing", 0)
    del ref_blk
    torch.cuda.empty_cache()

    # ---- warm-up + timed region (no per-call events: they cost launch-bound configs ~6 us) --------
    for _ in range(args.warmup):
        step()
    sync()
    if dist:
        dist.barrier()
    sync()
    launches0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.nvtx.range_push("mpk_timed")  # ncu --nvtx --nvtx-include "mpk_timed/"
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        sync()
        torch.cuda.nvtx.range_pop()
    if dist:
        dist.barrier()
    launches = ctx.launch_count() - launches0
    step_ms = ev0.elapsed_time(ev1) / args.steps
    # kernel time of the same steps, CUDA events on the context stream around every MPK call
    # (the roofline's denominator), in a second pass of K steps right after the timed one
    ctx.set_param("kernel_timing", 1)
    for _ in range(args.steps):
        step()
    sync()
    k_total, k_count, k_max = ctx.kernel_times()
    kernel_ms = k_total / args.steps  # every timed launch of the step (one per power or stage)
    ctx.set_param("kernel_timing", 0)
    if dist:
        t = torch.tensor([step_ms, kernel_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, kernel_ms = t.tolist()
    clocks = clk.summary()

    flops = 2.0 * nnz * p
    if cfgd["kind"] == "poly":
        flops += 2.0 * n * (p + 1)
    elif cfgd["kind"] in CHAIN_KINDS:
        flops = chain_flops(cfgd, nnz, n)
    value = world * flops / (step_ms * 1e-3) * 1e-9

    # ---- e2e through the host-pointer C ABI (pinned buffers, copies inside the timed region) --
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(x_perm).pin_memory()
        hblk = torch.empty((p + 1) * n, dtype=torch.float64).pin_memory()
        hz = torch.empty(n, dtype=torch.float64).pin_memory()
        vb = mpkg.VectorBlock(n, p + 1, hblk.numpy())
        xn = hx.numpy()

        if chain is not None:
            hblk.numpy()[:n] = x_perm

        def e2e_step():
            if cfgd["kind"] == "polyprod":
                from paper_2309_02228_b200._lib import check, lib
                check(lib.mpkg_poly_apply(ctx.h, Ap.h, None, None, pr_re.ctypes.data, pr_im.ctypes.data,
                                          p, cplan.h, xn.ctypes.data, hz.numpy().ctypes.data))
            elif chain is not None:
                from paper_2309_02228_b200._lib import check, lib
                f = lib.mpkg_sstep_jacobi if cfgd["kind"] == "sstep_jacobi" else lib.mpkg_sstep_gs2
                check(f(ctx.h, precon.h, cplan.h, Ap.h, ch_re.ctypes.data, ch_im.ctypes.data, p,
                        hblk.numpy().ctypes.data, n, p + 1))
            elif cfgd["kind"] == "shifted":
                ctx.mpk_shifted(plan, Ap, xn, shifts, vb)
            elif cfgd["kind"] == "poly":
                from paper_2309_02228_b200._lib import check, lib
                c = np.ascontiguousarray(coefs)
                check(lib.mpkg_mpk_poly(ctx.h, plan.h, Ap.h, xn.ctypes.data, c.ctypes.data, p,
                                        hz.numpy().ctypes.data, hblk.numpy().ctypes.data, n, p + 1))
            else:
                ctx.mpk(plan, Ap, xn, p, vb)

        e2e_step()
        e_steps = max(3, min(args.steps, 10))
        ts = []
        for _ in range(e_steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        e_ms = statistics.median(ts)
        if dist:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = t.item()
        e2e = {"value": world * flops / (e_ms * 1e-3) * 1e-9, "unit": "GFLOP/s",
               # chains stage the whole block in and out; mpk / mpk_shifted / mpk_poly stage x in
               # and stream slices 1..p back while later powers run (slice 0 = x is copied on the
               # host); the poly call adds z
               "h2d_bytes_per_step": (8 * n if cfgd["kind"] == "polyprod" else
                                      8 * n * (p + 1) if chain is not None else 8 * n),
               "d2h_bytes_per_step": (8 * n if cfgd["kind"] == "polyprod" else
                                      8 * n * (p + 1) if cfgd["kind"] in CHAIN_KINDS + ("poly",)
                                      else 8 * n * p),
               "ms_per_step": e_ms, "steps": e_steps}

    # ---- roofline of the dominant (fused) kernel -----------------------------------------------
    p_out = p
    b_alg = 12 * nnz + 4 * (n + 1) + 8 * n * (1 + p_out)
    if cfgd["kind"] == "poly":
        b_alg += 8 * n
    peak, peak_src = measured_peak()
    achieved = b_alg / (kernel_ms * 1e-3) / 1e9
    # one power = one pass over the matrix: its own algorithmic bytes (matrix + x read + y written)
    sweep_bytes = 12 * nnz + 4 * (n + 1) + 16 * n
    if cfgd["kind"] == "polyprod":  # degree-1 passes over the matrix for p powers
        sweep_bytes = sweep_bytes * (p - 1) / p
    elif cfgd["kind"] == "sstep_jacobi":  # matrix passes per power: (sweeps - 1) sweeps + terminal
        sweep_bytes *= cfgd["sweeps"]
    elif cfgd["kind"] == "sstep_gs2":  # K * (stage 0 + gamma inner) + terminal
        sweep_bytes *= cfgd["sweeps"] * (1 + cfgd["gamma"]) + 1
    sweep = {"algorithmic_bytes": sweep_bytes, "ms": kernel_ms / p,
             "achieved": sweep_bytes / (kernel_ms / p * 1e-3) / 1e9}
    sweep["frac"] = sweep["achieved"] / peak
    traffic = None
    prof = ROOT / "profiles" / f"ncu_{args.config}{'fast' if args.mode == 'fast' else ''}.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            traffic = pj.get("dram_bytes_per_step", pj.get("dram_bytes_per_launch"))
        except Exception:
            traffic = None

    # ---- parity against the reference's own outputs (digests), bitwise runs of the MPK configs
    ref_parity = None
    if chain is None and args.mode == "bitwise" and rank == 0:
        step()
        sync()
        ref_parity = reference_digest_parity(args.config, args.seed, cfgd["kind"], ls, Ap, x_perm,
                                             d_blk, p, n, d_z if cfgd["kind"] == "poly" else None)
        if ref_parity is not None and not ref_parity["match"]:
            parity = False

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        P_host = Ap.download()
        if chain is not None:
            cpu = port_chain_baseline(cfgd, (P_host.row_ptr, P_host.col_idx, P_host.values), x_perm, args.steps)
            cpu.pop("ms")
        else:
            kind = {"shifted": "shifted", "poly": "poly"}.get(cfgd["kind"], "plain")
            cpu = cpu_baseline_reference(P_host, ls.level_ptr, p, x_perm, kind, nnz,
                                         coefs=coefs if kind == "poly" else None)
        del P_host

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators for the BASELINE.json config, DESIGN.md §6)",
            "config": config_dict(args.config, cfgd, n, nnz, world),
            "parity": ("MISMATCH" if not parity else
                       ("bitwise == the reference's outputs (SHA-256 of " + ", ".join(ref_parity["checked"])
                        + "; tests/golden/config_digests.json) and mpk == baseline_mpk bitwise")
                       if ref_parity else "mpk == baseline bitwise" if args.mode == "bitwise" else
                       f"max inf-norm rel err {max_rel_err:.2e} <= 1e-12 vs baseline"),
            "details": {"mode": args.mode, "n_levels": ls.n_levels(), "n_groups": plan.n_groups(),
                        "plan_cache_bytes": cache, "executor": exec_info, "preprocess_s": prep,
                        "reference_digests": ref_parity,
                        "baseline_back_to_back_ms": baseline_ms,
                        # the chains have no one-launch-per-power twin of their own: report the
                        # plain baseline_mpk's time only, no GF/s that mixes the two
                        **({"baseline_mpk_gflops": 2.0 * nnz * p / (baseline_ms * 1e-3) * 1e-9}
                           if chain is None else {}),
                        "baseline_note": "p back-to-back launches of the plain SpMV (baseline_mpk)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes": b_alg, "kernel_ms": kernel_ms,
                         "kernel_launches_timed": k_count, "peak_source": peak_src,
                         "per_power": sweep,
                         # the metric's DRAM bytes/nnz: measured (ncu, one step) against
                         # the single-pass ideal and p back-to-back passes
                         "dram_bytes_per_nnz": (traffic / nnz) if traffic else None,
                         "dram_bytes_per_nnz_single_pass": b_alg / nnz,
                         "dram_bytes_per_nnz_back_to_back": p * sweep["algorithmic_bytes"] / nnz,
                         "note": "achieved = single-pass B_alg (SURVEY 8d) / MPK kernel time; "
                                 "per_power = one pass over the matrix per power"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
        if not parity:
            sys.exit(3)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
