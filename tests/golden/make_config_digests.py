"""Generates tests/golden/config_digests.json: SHA-256 digests of the REFERENCE's outputs on the
BASELINE.json configs at full size (C2, C3, C4 Newton + polynomial, C5).

TEST INFRASTRUCTURE.  Runs the reference's own hot path compiled in place (oracle/_ref/libmpkref.so,
proj/include/mpk built with the reference flags) on the harness inputs (oracle/_gen, the same
generators bench.py uses, seeds as bench.py):

  build_levels (levels.hpp:65-147) -> levels, perm, inv_perm, level_ptr
  permute      (csr.hpp:159-188)   -> A_perm row_ptr / col_idx / values
  x_perm = permute_vector(random_vector(n, seed + 2), perm)   (csr.hpp:191, acceptance.cpp:84-90)
  baseline_mpk (mpk.hpp:59-75)     -> slices 0..p   (== the blocked mpk bit for bit, mpk.hpp:77-80)
  C4: baseline_mpk_shifted (mpk.hpp:160-180) with theta_k = 26 + 26 cos(pi (2k-1) / 16) -> slices
      z = sum_k c_k A^k x in the A23 order (c_0 y_0, then += c_k y_k, mul then add), c_k from
      numpy default_rng(seed + 3) U[-1, 1] (bench.py poly_coefs)

The -m gpu tests (tests/test_gpu_fullsize.py) recompute every digest from the GPU path and compare.
Usage: python tests/golden/make_config_digests.py [c2 c3 c4 c5]   (needs ~40 GB RAM for C5)
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

OUT = pathlib.Path(__file__).resolve().parent / "config_digests.json"
SEED = 2309  # bench.py default
P_OF = {"c2": 8, "c3": 4, "c4": 8, "c5": 8}


def sha(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()


def newton_shifts(s=8):
    return [26.0 + 26.0 * np.cos(np.pi * (2 * k - 1) / 16.0) for k in range(1, s + 1)]


def poly_coefs(seed, d=8):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, d + 1)


def poly_z(block: np.ndarray, coefs) -> np.ndarray:
    """SURVEY A23 restatement: z = c_0 y_0, then z += c_k y_k for k = 1..d (mul, then add)."""
    z = coefs[0] * block[0]
    for k in range(1, len(coefs)):
        z = z + coefs[k] * block[k]
    return z


def _views(R, h, n):
    rp, ci, v = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
    R.lib.ref_csr_views(h, C.byref(rp), C.byref(ci), C.byref(v))
    rpa = np.ctypeslib.as_array(rp, (n + 1,))
    nnz = int(rpa[n])
    return rpa, np.ctypeslib.as_array(ci, (nnz,)), np.ctypeslib.as_array(v, (nnz,))


def reference_digests(cfg: str, seed: int = SEED, log=print) -> dict:
    from oracle.oracle import Reference, config_matrix, HarnessGen
    R = Reference()
    p = P_OF[cfg]
    t0 = time.perf_counter()
    rp, ci, v = config_matrix(cfg, seed)
    n, nnz = len(rp) - 1, len(ci)
    h = R.wrap(rp, ci, v)
    del rp, ci, v
    log(f"{cfg}: n={n} nnz={nnz} generated {time.perf_counter() - t0:.1f}s")
    lv, pm, ip = (np.empty(n, np.uint32) for _ in range(3))
    lp = np.empty(n + 1, np.uint32)
    nl = C.c_uint32()
    t0 = time.perf_counter()
    assert R.lib.ref_build_levels_h(h, lv.ctypes.data, pm.ctypes.data, ip.ctypes.data,
                                    lp.ctypes.data, C.byref(nl)) == 0, R.lib.ref_last_error()
    lp = lp[: nl.value + 1].copy()
    log(f"{cfg}: build_levels {time.perf_counter() - t0:.1f}s, {nl.value} levels")
    t0 = time.perf_counter()
    hp = R.lib.ref_permute_h(h, pm.ctypes.data)
    assert hp, R.lib.ref_last_error()
    R.lib.ref_csr_free(h)
    log(f"{cfg}: permute {time.perf_counter() - t0:.1f}s")
    prp, pci, pv = _views(R, hp, n)
    d = {"n": n, "nnz": nnz, "p": p, "n_levels": int(nl.value),
         "max_level_rows": int(np.diff(lp.astype(np.int64)).max()),
         "levels": sha(lv), "perm": sha(pm), "inv_perm": sha(ip), "level_ptr": sha(lp),
         "A_perm.row_ptr": sha(prp), "A_perm.col_idx": sha(pci), "A_perm.values": sha(pv)}
    x = HarnessGen().random_vector(n, seed + 2)
    xp = np.empty(n)
    xp[pm] = x  # permute_vector: out[perm[i]] = in[i] (csr.hpp:191-196)
    del x, lv, ip
    d["x_perm"] = sha(xp)
    xv = R.lib.ref_vec_new(xp.ctypes.data, n)
    blk = R.lib.ref_block_new(n, p + 1)
    data = np.ctypeslib.as_array(R.lib.ref_block_data(blk), ((p + 1) * n,)).reshape(p + 1, n)
    t0 = time.perf_counter()
    assert R.lib.ref_baseline_mpk_t(hp, xv, p, blk, 0) == 0, R.lib.ref_last_error()
    log(f"{cfg}: baseline_mpk p={p} {time.perf_counter() - t0:.1f}s")
    d["mpk"] = [sha(data[k]) for k in range(p + 1)]
    if cfg == "c4":
        c = poly_coefs(seed + 3, p)
        d["poly_coefs"] = [float(t) for t in c]
        d["poly_z"] = sha(poly_z(data, c))
        sh = np.ascontiguousarray(newton_shifts(p))
        hs = R.lib.ref_shifts_new(sh.ctypes.data, np.zeros(p).ctypes.data, p)
        t0 = time.perf_counter()
        assert R.lib.ref_baseline_mpk_shifted_t(hp, xv, hs, blk, 0) == 0, R.lib.ref_last_error()
        log(f"{cfg}: baseline_mpk_shifted {time.perf_counter() - t0:.1f}s")
        R.lib.ref_shifts_free(hs)
        d["shifts"] = [float(t) for t in sh]
        d["mpk_shifted"] = [sha(data[k]) for k in range(p + 1)]
    del data
    R.lib.ref_block_free(blk)
    R.lib.ref_vec_free(xv)
    R.lib.ref_csr_free(hp)
    d["seed"] = seed
    d["threads"] = R.resolve_threads(0)
    return d


def main():
    cfgs = sys.argv[1:] or ["c2", "c3", "c4", "c5"]
    data = json.loads(OUT.read_text()) if OUT.exists() else {}
    data["_about"] = ("SHA-256 of the reference's own outputs (oracle/_ref, compiled from "
                      "/root/reference/proj/include with the reference flags) on the bench.py inputs "
                      "at full size; generated by tests/golden/make_config_digests.py")
    for c in cfgs:
        data[c] = reference_digests(c)
        OUT.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
