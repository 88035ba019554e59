"""TEST INFRASTRUCTURE ONLY — ctypes access to the CPU oracle.

* `Oracle` wraps liboracle.so, the plain-C restatement (oracle.c) of the reference path.
* `Reference` wraps _ref/libmpkref.so, the reference's own headers compiled in place with the
  reference flags (oracle/Makefile); it is optional (absent when /root/reference was not
  available at build time).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may use
this module, and only as the checker / CPU baseline.  The product (paper_2309_02228_b200) never
imports it.
"""
from __future__ import annotations

import ctypes as C
import pathlib
from typing import Optional

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libmpkref.so"

P = C.c_void_p
u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """The C restatement (one thread)."""

    def __init__(self, path: pathlib.Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(str(path))
        sig = {
            "orc_build_levels": [u32, P, P, P, P, P, P, P],
            "orc_check_permutation": [P, u32],
            "orc_permute": [u32, P, P, P, P, P, P, P],
            "orc_permute_vector": [u32, P, P, P],
            "orc_unpermute_vector": [u32, P, P, P],
            "orc_validate_levels": [u32, P, P, P, P],
            "orc_row_range_footprint": [P, u32, u32, i32],
            "orc_greedy_group": [P, u32, u64, P],
            "orc_group_levels": [u32, P, u32, P, u64, i32, P, P, P, P, P],
            "orc_wavefront_schedule": [u32, i32, P, P],
            "orc_baseline_mpk": [u32, P, P, P, P, i32, P],
            "orc_mpk": [u32, P, P, P, P, u32, i32, P, i32, P],
            "orc_check_shift_chain": [P, P, i32],
            "orc_baseline_mpk_shifted": [u32, P, P, P, P, P, P, i32, P],
            "orc_mpk_shifted": [u32, P, P, P, P, u32, i32, P, P, P, i32, P],
            "orc_poly_combine": [u32, P, P, i32, P],
            "orc_tune_select": [P, i32, i32],
            "orc_diag_info": [u32, u32, P, P, P, P, P, P],
            "orc_jacobi_apply": [u32, P, P, P, P, P, i32, P, P],
            "orc_jacobi_op": [u32, P, P, P, P, P, i32, P, P],
            "orc_sstep_jacobi_block": [u32, P, P, P, P, P, i32, P, P, i32, P],
            "orc_gs2_chain": [u32, P, P, P, P, P, i32, i32, i32, i32, P, P, P],
            "orc_sstep_gs2_block": [u32, P, P, P, P, P, i32, i32, i32, P, P, i32, P],
            "orc_from_coo": [u32, u32, u64, P, P, P, P, P, P, P, P],
            "orc_poly_apply": [u32, P, P, P, P, P, i32, i32, i32, i32, P, P, i32, P, P],
            "orc_block_dots": [P, P, u64, u32, u32, P],
            "orc_block_update": [P, P, u64, u32, u32, P],
            "orc_icgs": [P, u64, u32, P, u32, i32, P],
            "orc_tsqr": [P, u64, u32, P],
        }
        res = {"orc_row_range_footprint": u64, "orc_greedy_group": u32,
               "orc_wavefront_schedule": u64, "orc_permute_vector": None,
               "orc_unpermute_vector": None, "orc_poly_combine": None,
               "orc_jacobi_apply": None, "orc_jacobi_op": None, "orc_gs2_chain": None,
               "orc_block_dots": None, "orc_block_update": None}
        for k, v in sig.items():
            f = getattr(L, k)
            f.argtypes = v
            f.restype = res.get(k, C.c_int)

    # levels.hpp:65
    def build_levels(self, rp, ci):
        rp, ci = _u32(rp), _u32(ci)
        n = len(rp) - 1
        lv, pm, ip = (np.empty(n, np.uint32) for _ in range(3))
        lp = np.empty(n + 1, np.uint32)
        nl = C.c_uint32()
        assert self.lib.orc_build_levels(n, _p(rp), _p(ci), _p(lv), _p(pm), _p(ip), _p(lp),
                                         C.byref(nl)) == 0
        return lv, pm, ip, lp[: nl.value + 1].copy()

    # csr.hpp:159
    def permute(self, rp, ci, v, perm):
        rp, ci, v, perm = _u32(rp), _u32(ci), _f64(v), _u32(perm)
        n = len(rp) - 1
        orp, oci, ov = np.empty(n + 1, np.uint32), np.empty(len(ci), np.uint32), np.empty(len(v))
        rc = self.lib.orc_permute(n, _p(rp), _p(ci), _p(v), _p(perm), _p(orp), _p(oci), _p(ov))
        if rc:
            raise ValueError("permute: not a permutation")
        return orp, oci, ov

    def validate_levels(self, rp, ci, levels, inv_perm) -> bool:
        rp, ci = _u32(rp), _u32(ci)
        return bool(self.lib.orc_validate_levels(len(rp) - 1, _p(rp), _p(ci), _p(_u32(levels)),
                                                 _p(_u32(inv_perm))))

    def greedy_group(self, fp, target):
        fp = np.ascontiguousarray(fp, dtype=np.uint64)
        out = np.empty(len(fp) + 1, np.uint32)
        nb = self.lib.orc_greedy_group(_p(fp), len(fp), int(target), _p(out))
        return out[:nb].tolist()

    # plan.hpp:88
    def group_levels(self, level_ptr, rp_perm, cache_bytes, p_m):
        lp, rp = _u32(level_ptr), _u32(rp_perm)
        nl = len(lp) - 1
        gr, glp = np.empty(nl + 1, np.uint32), np.empty(nl + 1, np.uint32)
        gfp = np.empty(max(nl, 1), np.uint64)
        ng, tgt = C.c_uint32(), C.c_uint64()
        rc = self.lib.orc_group_levels(len(rp) - 1, _p(lp), nl, _p(rp), int(cache_bytes), p_m,
                                       _p(gr), _p(glp), _p(gfp), C.byref(ng), C.byref(tgt))
        if rc:
            raise ValueError("group_levels: p_m must be >= 1")
        g = ng.value
        return gr[: g + 1].copy(), glp[: g + 1].copy(), gfp[:g].copy(), tgt.value

    def wavefront_schedule(self, ng, stages):
        n = max(ng * max(stages, 0), 1)
        g, q = np.empty(n, np.uint32), np.empty(n, np.int32)
        cnt = self.lib.orc_wavefront_schedule(ng, stages, _p(g), _p(q))
        return list(zip(g[:cnt].tolist(), q[:cnt].tolist()))

    # mpk.hpp:59
    def baseline_mpk(self, rp, ci, v, x, p_m):
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        n = len(rp) - 1
        blk = np.empty((p_m + 1) * n)
        assert self.lib.orc_baseline_mpk(n, _p(rp), _p(ci), _p(v), _p(x), p_m, _p(blk)) == 0
        return blk.reshape(p_m + 1, n)

    # mpk.hpp:81
    def mpk(self, rp, ci, v, group_rows, plan_p_m, x, p_m):
        rp, ci, v, x, gr = _u32(rp), _u32(ci), _f64(v), _f64(x), _u32(group_rows)
        n = len(rp) - 1
        blk = np.empty((p_m + 1) * n)
        rc = self.lib.orc_mpk(n, _p(rp), _p(ci), _p(v), _p(gr), len(gr) - 1, plan_p_m, _p(x),
                              p_m, _p(blk))
        if rc:
            raise ValueError("mpk: bad arguments")
        return blk.reshape(p_m + 1, n)

    def _shifts(self, shifts):
        s = np.asarray(list(shifts), dtype=np.complex128)
        return _f64(s.real), _f64(s.imag)

    def check_shift_chain(self, shifts) -> bool:
        re, im = self._shifts(shifts)
        return self.lib.orc_check_shift_chain(_p(re), _p(im), len(re)) == 0

    def baseline_mpk_shifted(self, rp, ci, v, x, shifts):
        re, im = self._shifts(shifts)
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        n, s = len(rp) - 1, len(re)
        blk = np.empty((s + 1) * n)
        rc = self.lib.orc_baseline_mpk_shifted(n, _p(rp), _p(ci), _p(v), _p(x), _p(re), _p(im),
                                               s, _p(blk))
        if rc:
            raise ValueError("baseline_mpk_shifted: bad shift chain")
        return blk.reshape(s + 1, n)

    def mpk_shifted(self, rp, ci, v, group_rows, plan_p_m, x, shifts):
        re, im = self._shifts(shifts)
        rp, ci, v, x, gr = _u32(rp), _u32(ci), _f64(v), _f64(x), _u32(group_rows)
        n, s = len(rp) - 1, len(re)
        blk = np.empty((s + 1) * n)
        rc = self.lib.orc_mpk_shifted(n, _p(rp), _p(ci), _p(v), _p(gr), len(gr) - 1, plan_p_m,
                                      _p(x), _p(re), _p(im), s, _p(blk))
        if rc:
            raise ValueError("mpk_shifted: bad arguments")
        return blk.reshape(s + 1, n)

    def poly(self, rp, ci, v, x, coef):
        c = _f64(coef)
        d = len(c) - 1
        blk = np.ascontiguousarray(self.baseline_mpk(rp, ci, v, x, d))
        n = blk.shape[1]
        z = np.empty(n)
        self.lib.orc_poly_combine(n, _p(blk), _p(c), d, _p(z))
        return z, blk

    def tune_select(self, table, p_lo, p_hi):
        t = _f64(table)
        return self.lib.orc_tune_select(_p(t), p_lo, p_hi)

    # ---- Jacobi chains (jacobi.hpp, sstep.hpp:122-157) ------------------------------------------
    def diag_info(self, rp, ci, v, n_cols=None):
        """(pos, inv); raises ValueError (not square) / RuntimeError (missing or zero diagonal)."""
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        n = len(rp) - 1
        pos, inv, bad = np.empty(n, np.uint32), np.empty(n), np.zeros(1, np.uint32)
        rc = self.lib.orc_diag_info(n, n if n_cols is None else n_cols, _p(rp), _p(ci), _p(v),
                                    _p(pos), _p(inv), _p(bad))
        if rc == 1:
            raise ValueError("jacobi_setup: matrix must be square")
        if rc == 2:
            raise RuntimeError(f"jacobi_setup: missing or zero diagonal entry at row {int(bad[0])}")
        return pos, inv

    def jacobi_apply(self, rp, ci, v, sweeps, x):
        pos, inv = self.diag_info(rp, ci, v)
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        z = np.empty(len(rp) - 1)
        self.lib.orc_jacobi_apply(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), sweeps,
                                  _p(x), _p(z))
        return z

    def jacobi_op(self, rp, ci, v, sweeps, x):
        pos, inv = self.diag_info(rp, ci, v)
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        y = np.empty(len(rp) - 1)
        self.lib.orc_jacobi_op(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), sweeps,
                               _p(x), _p(y))
        return y

    def poly_apply(self, rp, ci, v, roots, x, inner="none", sweeps=1, gamma=1, forward=True):
        """poly.hpp:146-281: z = p(A M^{-1}) x for the given roots (product form)."""
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        n = len(rp) - 1
        if inner == "none":
            pos, inv = np.zeros(n, np.uint32), np.zeros(n)
        else:
            pos, inv = self.diag_info(rp, ci, v)
        re, im = self._shifts(roots)
        z = np.empty(n)
        kind = {"none": 0, "jacobi": 1, "gs2": 2}[inner]
        rc = self.lib.orc_poly_apply(n, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), kind, sweeps, gamma,
                                     1 if forward else 0, _p(re), _p(im), len(re), _p(x), _p(z))
        if rc:
            raise ValueError("poly: conjugate pair not adjacent")
        return z

    # ---- block orthogonalisation (ortho.hpp); blocks are (cols, rows) C-order = column-major
    def block_dots(self, q, v):
        """ortho.hpp:46-63: C = Q^T V as a (qcols, vcols) matrix.  Blocks are passed as
        (cols, rows) arrays: row l of the array is column l of the block (column-major memory)."""
        q, v = _f64(np.atleast_2d(q)), _f64(np.atleast_2d(v))
        c = np.empty((v.shape[0], q.shape[0]))
        self.lib.orc_block_dots(_p(q), _p(v), q.shape[1], q.shape[0], v.shape[0], _p(c))
        return c.T

    def block_update(self, q, c, v):
        """ortho.hpp:67-92: returns V - Q C (v is not modified)."""
        q, c = _f64(np.atleast_2d(q)), _f64(np.asarray(c).T)
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        self.lib.orc_block_update(_p(q), _p(c), q.shape[1], q.shape[0], out.shape[0], _p(out))
        return out

    def icgs(self, q, v, sweeps):
        """ortho.hpp:97-117 -> (V orthogonalised, coefficients as a (qcols, vcols) matrix)."""
        q = _f64(np.atleast_2d(q)) if q is not None and len(q) else np.zeros((0, 0))
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        qcols, rows = (q.shape[0], out.shape[1])
        coeff = np.zeros((out.shape[0], qcols))
        rc = self.lib.orc_icgs(_p(q) if qcols else None, rows, qcols, _p(out), out.shape[0], sweeps,
                               _p(coeff))
        if rc:
            raise ValueError("icgs_block_orthogonalize: sweeps must be >= 1")
        return out, coeff.T

    def tsqr(self, v):
        """ortho.hpp:136-229 -> (Q as a (cols, rows) block, R as a (cols, cols) matrix)."""
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        cols, rows = out.shape
        r = np.zeros((cols, cols))
        if self.lib.orc_tsqr(_p(out), rows, cols, _p(r)):
            raise ValueError("tsqr: block must have at least as many rows as columns")
        return out, r.T

    def from_coo(self, n_rows, n_cols, rows, cols, vals):
        """csr.hpp:72-110 -> (row_ptr, col_idx, values); ValueError (index, bad entry) if out of range."""
        r, c, v = _u32(rows), _u32(cols), _f64(vals)
        m = len(r)
        rp = np.empty(n_rows + 1, np.uint32)
        ci, vv = np.empty(max(m, 1), np.uint32), np.empty(max(m, 1))
        u, bad = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        rc = self.lib.orc_from_coo(n_rows, n_cols, m, _p(r), _p(c), _p(v), _p(rp), _p(ci), _p(vv),
                                   _p(u), _p(bad))
        if rc:
            raise ValueError(f"from_coo: entry index out of range at entry {int(bad[0])}")
        k = int(u[0])
        return rp, ci[:k].copy(), vv[:k].copy()

    GS2_MODES = {"smooth": (0, 0), "apply": (1, 0), "smooth_residual": (0, 2), "op": (1, 1)}

    def gs2(self, rp, ci, v, gamma, sweeps, forward, mode, vin, z0=None):
        """gs2.hpp:200-235: mode smooth / apply / smooth_residual / op -> (z, out)."""
        pos, inv = self.diag_info(rp, ci, v)
        rp, ci, v, vin = _u32(rp), _u32(ci), _f64(v), _f64(vin)
        n = len(rp) - 1
        zero_guess, term = self.GS2_MODES[mode]
        z = np.zeros(n) if (zero_guess or z0 is None) else _f64(z0).copy()
        out = np.empty(n)
        self.lib.orc_gs2_chain(n, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), gamma, sweeps,
                               1 if forward else 0, term, _p(vin), _p(z), _p(out))
        return z, (out if term else None)

    def sstep_gs2_block(self, rp, ci, v, gamma, sweeps, forward, x, shifts):
        pos, inv = self.diag_info(rp, ci, v)
        re, im = self._shifts(shifts)
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        n, s = len(rp) - 1, len(re)
        blk = np.empty((s + 1) * n)
        blk[:n] = x
        rc = self.lib.orc_sstep_gs2_block(n, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), gamma, sweeps,
                                          1 if forward else 0, _p(re), _p(im), s, _p(blk))
        if rc:
            raise ValueError("sstep_gs2_block: bad shift chain")
        return blk.reshape(s + 1, n)

    def sstep_jacobi_block(self, rp, ci, v, sweeps, x, shifts):
        pos, inv = self.diag_info(rp, ci, v)
        re, im = self._shifts(shifts)
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        n, s = len(rp) - 1, len(re)
        blk = np.empty((s + 1) * n)
        blk[:n] = x
        rc = self.lib.orc_sstep_jacobi_block(n, _p(rp), _p(ci), _p(v), _p(pos), _p(inv), sweeps,
                                             _p(re), _p(im), s, _p(blk))
        if rc:
            raise ValueError("sstep_jacobi_block: bad shift chain")
        return blk.reshape(s + 1, n)


class Reference:
    """The reference's own header-only implementation, compiled in place (OpenMP)."""

    def __init__(self, path: pathlib.Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (needs /root/reference at build time)")
        L = self.lib = C.CDLL(str(path))
        sig = {
            "ref_gen": ([i32, u32, u32, u32, u64], P),
            "ref_csr_info": ([P, P, P], None),
            "ref_csr_copy": ([P, P, P, P], None),
            "ref_csr_free": ([P], None),
            "ref_random_vector": ([u64, u64, P], None),
            "ref_build_levels": ([u32, P, P, P, P, P, P, P, P], C.c_int),
            "ref_permute": ([u32, P, P, P, P, P, P, P], C.c_int),
            "ref_validate_levels": ([u32, P, P, P, P, P, P, P, u32], C.c_int),
            "ref_group_levels": ([u32, P, P, P, P, u32, u64, i32, P, P, P, P, P], C.c_int),
            "ref_greedy_group": ([P, u32, u64, P], u32),
            "ref_wavefront_schedule": ([u32, i32, P, P], u64),
            "ref_csr_wrap": ([u32, P, P, P], P),
            "ref_baseline_mpk_h": ([P, P, i32, P, i32], C.c_int),
            "ref_mpk_h": ([P, P, u32, i32, P, i32, P, i32], C.c_int),
            "ref_block_new": ([u64, u64], P),
            "ref_block_free": ([P], None),
            "ref_block_data": ([P], C.POINTER(C.c_double)),
            "ref_vec_new": ([P, u64], P),
            "ref_vec_free": ([P], None),
            "ref_plan_new": ([u32, P, u32, i32], P),
            "ref_plan_free": ([P], None),
            "ref_baseline_mpk_t": ([P, P, i32, P, i32], C.c_int),
            "ref_mpk_t": ([P, P, P, i32, P, i32], C.c_int),
            "ref_baseline_mpk_shifted_h": ([P, P, P, P, i32, P, i32], C.c_int),
            "ref_mpk_shifted_h": ([P, P, u32, i32, P, P, P, i32, P, i32], C.c_int),
            "ref_check_shift_chain": ([P, P, i32], C.c_int),
            "ref_build_levels_h": ([P, P, P, P, P, P], C.c_int),
            "ref_permute_h": ([P, P], P),
            "ref_csr_views": ([P, P, P, P], None),
            "ref_shifts_new": ([P, P, i32], P),
            "ref_shifts_free": ([P], None),
            "ref_baseline_mpk_shifted_t": ([P, P, P, P, i32], C.c_int),
            "ref_mpk_shifted_t": ([P, P, P, P, P, i32], C.c_int),
            "ref_tune_select": ([P, i32, i32], C.c_int),
            "ref_resolve_threads": ([i32], C.c_int),
            "ref_jacobi_setup": ([u32, P, P, P, i32, P, P], C.c_int),
            "ref_jacobi_apply": ([u32, P, P, P, i32, P, P], C.c_int),
            "ref_jacobi_op": ([u32, P, P, P, i32, P, P], C.c_int),
            "ref_jacobi_op_blocked": ([u32, P, P, P, i32, P, u32, P, P, i32], C.c_int),
            "ref_gs2": ([u32, P, P, P, i32, i32, i32, i32, P, u32, i32, P, P, P, i32], C.c_int),
            "ref_from_coo": ([u32, u32, u64, P, P, P], P),
            "ref_read_matrix_market": ([C.c_char_p], P),
            "ref_csr_shape": ([P, P, P], None),
            "ref_last_error": ([], C.c_char_p),
        }
        for k, (a, r) in sig.items():
            f = getattr(L, k)
            f.argtypes = a
            f.restype = r

    def gen(self, kind, a, b=0, c=0, seed=0):
        h = self.lib.ref_gen(kind, a, b, c, seed)
        if not h:
            raise ValueError(self.lib.ref_last_error().decode())
        n, nnz = C.c_uint32(), C.c_uint32()
        self.lib.ref_csr_info(h, C.byref(n), C.byref(nnz))
        rp = np.empty(n.value + 1, np.uint32)
        ci = np.empty(nnz.value, np.uint32)
        v = np.empty(nnz.value)
        self.lib.ref_csr_copy(h, _p(rp), _p(ci), _p(v))
        self.lib.ref_csr_free(h)
        return rp, ci, v

    def random_vector(self, n, seed):
        out = np.empty(n)
        self.lib.ref_random_vector(n, seed, _p(out))
        return out

    def build_levels(self, rp, ci, v):
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        n = len(rp) - 1
        lv, pm, ip = (np.empty(n, np.uint32) for _ in range(3))
        lp = np.empty(n + 1, np.uint32)
        nl = C.c_uint32()
        assert self.lib.ref_build_levels(n, _p(rp), _p(ci), _p(v), _p(lv), _p(pm), _p(ip),
                                         _p(lp), C.byref(nl)) == 0
        return lv, pm, ip, lp[: nl.value + 1].copy()

    def permute(self, rp, ci, v, perm):
        rp, ci, v, perm = _u32(rp), _u32(ci), _f64(v), _u32(perm)
        n = len(rp) - 1
        orp, oci, ov = np.empty(n + 1, np.uint32), np.empty(len(ci), np.uint32), np.empty(len(v))
        if self.lib.ref_permute(n, _p(rp), _p(ci), _p(v), _p(perm), _p(orp), _p(oci), _p(ov)):
            raise ValueError(self.lib.ref_last_error().decode())
        return orp, oci, ov

    def group_levels(self, rp, ci, v, level_ptr, cache_bytes, p_m):
        rp, ci, v, lp = _u32(rp), _u32(ci), _f64(v), _u32(level_ptr)
        nl = len(lp) - 1
        gr, glp = np.empty(nl + 1, np.uint32), np.empty(nl + 1, np.uint32)
        gfp = np.empty(max(nl, 1), np.uint64)
        ng, tgt = C.c_uint32(), C.c_uint64()
        if self.lib.ref_group_levels(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(lp), nl,
                                     int(cache_bytes), p_m, _p(gr), _p(glp), _p(gfp),
                                     C.byref(ng), C.byref(tgt)):
            raise ValueError(self.lib.ref_last_error().decode())
        g = ng.value
        return gr[: g + 1].copy(), glp[: g + 1].copy(), gfp[:g].copy(), tgt.value

    def wrap(self, rp, ci, v):
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        return self.lib.ref_csr_wrap(len(rp) - 1, _p(rp), _p(ci), _p(v))

    def baseline_mpk(self, rp, ci, v, x, p_m, threads=0):
        h = self.wrap(rp, ci, v)
        n = len(rp) - 1
        blk = np.empty((p_m + 1) * n)
        rc = self.lib.ref_baseline_mpk_h(h, _p(_f64(x)), p_m, _p(blk), threads)
        self.lib.ref_csr_free(h)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return blk.reshape(p_m + 1, n)

    def mpk(self, rp, ci, v, group_rows, plan_p_m, x, p_m, threads=0):
        h = self.wrap(rp, ci, v)
        n = len(rp) - 1
        gr = _u32(group_rows)
        blk = np.empty((p_m + 1) * n)
        rc = self.lib.ref_mpk_h(h, _p(gr), len(gr) - 1, plan_p_m, _p(_f64(x)), p_m, _p(blk),
                                threads)
        self.lib.ref_csr_free(h)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return blk.reshape(p_m + 1, n)

    def baseline_mpk_shifted(self, rp, ci, v, x, shifts, threads=0):
        s = np.asarray(list(shifts), dtype=np.complex128)
        re, im = _f64(s.real), _f64(s.imag)
        h = self.wrap(rp, ci, v)
        n = len(rp) - 1
        blk = np.empty((len(re) + 1) * n)
        rc = self.lib.ref_baseline_mpk_shifted_h(h, _p(_f64(x)), _p(re), _p(im), len(re),
                                                 _p(blk), threads)
        self.lib.ref_csr_free(h)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return blk.reshape(len(re) + 1, n)

    def mpk_shifted(self, rp, ci, v, group_rows, plan_p_m, x, shifts, threads=0):
        s = np.asarray(list(shifts), dtype=np.complex128)
        re, im = _f64(s.real), _f64(s.imag)
        h = self.wrap(rp, ci, v)
        n = len(rp) - 1
        gr = _u32(group_rows)
        blk = np.empty((len(re) + 1) * n)
        rc = self.lib.ref_mpk_shifted_h(h, _p(gr), len(gr) - 1, plan_p_m, _p(_f64(x)), _p(re),
                                        _p(im), len(re), _p(blk), threads)
        self.lib.ref_csr_free(h)
        if rc:
            raise ValueError(self.lib.ref_last_error().decode())
        return blk.reshape(len(re) + 1, n)

    def check_shift_chain(self, shifts) -> bool:
        s = np.asarray(list(shifts), dtype=np.complex128)
        re, im = _f64(s.real), _f64(s.imag)
        return self.lib.ref_check_shift_chain(_p(re), _p(im), len(re)) == 0

    def greedy_group(self, fp, target):
        fp = np.ascontiguousarray(fp, dtype=np.uint64)
        out = np.empty(len(fp) + 1, np.uint32)
        nb = self.lib.ref_greedy_group(_p(fp), len(fp), int(target), _p(out))
        return out[:nb].tolist()

    def wavefront_schedule(self, ng, stages):
        n = max(ng * max(stages, 0), 1)
        g, q = np.empty(n, np.uint32), np.empty(n, np.int32)
        cnt = self.lib.ref_wavefront_schedule(ng, stages, _p(g), _p(q))
        return list(zip(g[:cnt].tolist(), q[:cnt].tolist()))

    def tune_select(self, table, p_lo, p_hi):
        t = _f64(table)
        return self.lib.ref_tune_select(_p(t), p_lo, p_hi)

    def resolve_threads(self, requested=0):
        return self.lib.ref_resolve_threads(requested)

    def _raise(self, rc):
        msg = self.lib.ref_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def jacobi_setup(self, rp, ci, v, sweeps=1):
        rp, ci, v = _u32(rp), _u32(ci), _f64(v)
        n = len(rp) - 1
        pos, inv = np.empty(n, np.uint32), np.empty(n)
        rc = self.lib.ref_jacobi_setup(n, _p(rp), _p(ci), _p(v), sweeps, _p(pos), _p(inv))
        if rc:
            self._raise(rc)
        return pos, inv

    def jacobi_apply(self, rp, ci, v, sweeps, x):
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        z = np.empty(len(rp) - 1)
        rc = self.lib.ref_jacobi_apply(len(rp) - 1, _p(rp), _p(ci), _p(v), sweeps, _p(x), _p(z))
        if rc:
            self._raise(rc)
        return z

    def jacobi_op(self, rp, ci, v, sweeps, x):
        rp, ci, v, x = _u32(rp), _u32(ci), _f64(v), _f64(x)
        y = np.empty(len(rp) - 1)
        rc = self.lib.ref_jacobi_op(len(rp) - 1, _p(rp), _p(ci), _p(v), sweeps, _p(x), _p(y))
        if rc:
            self._raise(rc)
        return y

    def _take_csr(self, h):
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        nr, nc, nnz = np.zeros(1, np.uint32), np.zeros(1, np.uint32), np.zeros(1, np.uint32)
        self.lib.ref_csr_shape(h, _p(nr), _p(nc))
        self.lib.ref_csr_info(h, _p(nr), _p(nnz))
        rp = np.empty(int(nr[0]) + 1, np.uint32)
        ci, v = np.empty(max(int(nnz[0]), 1), np.uint32), np.empty(max(int(nnz[0]), 1))
        self.lib.ref_csr_copy(h, _p(rp), _p(ci), _p(v))
        self.lib.ref_csr_free(h)
        k = int(nnz[0])
        return int(nr[0]), int(nc[0]), rp, ci[:k].copy(), v[:k].copy()

    # ---- block orthogonalisation (ortho.hpp); blocks are (cols, rows) C-order = column-major
    def block_dots(self, q, v):
        """ortho.hpp:46-63: C = Q^T V as a (qcols, vcols) matrix.  Blocks are passed as
        (cols, rows) arrays: row l of the array is column l of the block (column-major memory)."""
        q, v = _f64(np.atleast_2d(q)), _f64(np.atleast_2d(v))
        c = np.empty((v.shape[0], q.shape[0]))
        self.lib.orc_block_dots(_p(q), _p(v), q.shape[1], q.shape[0], v.shape[0], _p(c))
        return c.T

    def block_update(self, q, c, v):
        """ortho.hpp:67-92: returns V - Q C (v is not modified)."""
        q, c = _f64(np.atleast_2d(q)), _f64(np.asarray(c).T)
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        self.lib.orc_block_update(_p(q), _p(c), q.shape[1], q.shape[0], out.shape[0], _p(out))
        return out

    def icgs(self, q, v, sweeps):
        """ortho.hpp:97-117 -> (V orthogonalised, coefficients as a (qcols, vcols) matrix)."""
        q = _f64(np.atleast_2d(q)) if q is not None and len(q) else np.zeros((0, 0))
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        qcols, rows = (q.shape[0], out.shape[1])
        coeff = np.zeros((out.shape[0], qcols))
        rc = self.lib.orc_icgs(_p(q) if qcols else None, rows, qcols, _p(out), out.shape[0], sweeps,
                               _p(coeff))
        if rc:
            raise ValueError("icgs_block_orthogonalize: sweeps must be >= 1")
        return out, coeff.T

    def tsqr(self, v):
        """ortho.hpp:136-229 -> (Q as a (cols, rows) block, R as a (cols, cols) matrix)."""
        out = np.array(np.atleast_2d(v), dtype=np.float64, order="C")
        cols, rows = out.shape
        r = np.zeros((cols, cols))
        if self.lib.orc_tsqr(_p(out), rows, cols, _p(r)):
            raise ValueError("tsqr: block must have at least as many rows as columns")
        return out, r.T

    def from_coo(self, n_rows, n_cols, rows, cols, vals):
        r, c, v = _u32(rows), _u32(cols), _f64(vals)
        return self._take_csr(self.lib.ref_from_coo(n_rows, n_cols, len(r), _p(r), _p(c), _p(v)))

    def read_matrix_market(self, path):
        """matrix_market.hpp -> (n_rows, n_cols, row_ptr, col_idx, values); RuntimeError."""
        return self._take_csr(self.lib.ref_read_matrix_market(str(path).encode()))

    GS2_MODES = {"smooth": 0, "apply": 1, "smooth_residual": 2, "op": 3}

    def gs2(self, rp, ci, v, gamma, sweeps, forward, mode, vin, z0=None, group_rows=None,
            plan_p_m=None, threads=0):
        rp, ci, v, vin = _u32(rp), _u32(ci), _f64(v), _f64(vin)
        n = len(rp) - 1
        z = np.zeros(n) if z0 is None else _f64(z0).copy()
        out = np.empty(n)
        gr = None if group_rows is None else _u32(group_rows)
        rc = self.lib.ref_gs2(n, _p(rp), _p(ci), _p(v), gamma, sweeps, 1 if forward else 0,
                              self.GS2_MODES[mode], _p(gr), 0 if gr is None else len(gr) - 1,
                              plan_p_m or sweeps, _p(vin), _p(z), _p(out), threads)
        if rc:
            self._raise(rc)
        return z, (out if mode in ("smooth_residual", "op") else None)

    def jacobi_op_blocked(self, rp, ci, v, sweeps, group_rows, x, threads=0):
        rp, ci, v, x, gr = _u32(rp), _u32(ci), _f64(v), _f64(x), _u32(group_rows)
        y = np.empty(len(rp) - 1)
        rc = self.lib.ref_jacobi_op_blocked(len(rp) - 1, _p(rp), _p(ci), _p(v), sweeps, _p(gr),
                                            len(gr) - 1, _p(x), _p(y), threads)
        if rc:
            self._raise(rc)
        return y


def reference_available() -> bool:
    return REF_SO.exists()


GEN_SO = HERE / "_gen" / "libmpkgen.so"


class HarnessGen:
    """Host-only harness generators (oracle/_gen/libmpkgen.so, built from the same generators.cpp
    as the product's mpkg_gen) for legs that must not load the product library: bench.py's
    `--impl reference` arm and tests/golden/make_config_digests.py.  Returns (row_ptr, col_idx,
    values) numpy arrays."""

    KINDS = {"poisson3d": 3, "stencil27": 6, "stencil27_random_sym": 7, "rmat": 8}

    def __init__(self, path: pathlib.Path = GEN_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (make -C oracle)")
        L = self.lib = C.CDLL(str(path))
        L.mpkg_gen.argtypes = [i32, u32, u32, u32, u64, C.POINTER(P)]
        L.mpkg_gen.restype = C.c_int
        L.mpkg_host_csr_scramble.argtypes = [P, u64, P, C.POINTER(P)]
        L.mpkg_host_csr_scramble.restype = C.c_int
        L.mpkg_host_csr_info.argtypes = [P, P, P, P]
        L.mpkg_host_csr_arrays.argtypes = [P, P, P, P]
        L.mpkg_host_csr_destroy.argtypes = [P]
        L.mpkg_random_vector.argtypes = [u64, u64, P]
        L.mpkg_random_vector.restype = C.c_int
        L.gen_last_error.restype = C.c_char_p

    def _take(self, h, keep=False):
        n, nc, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
        self.lib.mpkg_host_csr_info(h, C.byref(n), C.byref(nc), C.byref(nnz))
        rp, ci, v = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
        self.lib.mpkg_host_csr_arrays(h, C.byref(rp), C.byref(ci), C.byref(v))
        out = (np.ctypeslib.as_array(rp, (n.value + 1,)).copy(),
               np.ctypeslib.as_array(ci, (nnz.value,)).copy() if nnz.value else np.empty(0, np.uint32),
               np.ctypeslib.as_array(v, (nnz.value,)).copy() if nnz.value else np.empty(0))
        if not keep:
            self.lib.mpkg_host_csr_destroy(h)
        return out

    def _gen(self, kind, a, b=0, c=0, seed=0, keep=False):
        h = P()
        if self.lib.mpkg_gen(kind, a, b, c, seed, C.byref(h)):
            raise ValueError(self.lib.gen_last_error().decode())
        return (h, self._take(h, keep=True)) if keep else self._take(h)

    def poisson3d(self, nx, ny, nz):
        return self._gen(3, nx, ny, nz)

    def stencil27(self, nx, ny, nz):
        return self._gen(6, nx, ny, nz)

    def rmat(self, scale, edge_factor, seed):
        return self._gen(8, scale, edge_factor, 0, seed)

    def scrambled_stencil27_random_sym(self, nx, ny, nz, seed, scramble_seed):
        h = P()
        if self.lib.mpkg_gen(7, nx, ny, nz, seed, C.byref(h)):
            raise ValueError(self.lib.gen_last_error().decode())
        h2 = P()
        rc = self.lib.mpkg_host_csr_scramble(h, scramble_seed, None, C.byref(h2))
        self.lib.mpkg_host_csr_destroy(h)
        if rc:
            raise ValueError(self.lib.gen_last_error().decode())
        return self._take(h2)

    def random_vector(self, n, seed):
        out = np.empty(n)
        assert self.lib.mpkg_random_vector(n, seed, out.ctypes.data) == 0
        return out


def config_matrix(cfg: str, seed: int):
    """BASELINE.json config matrices from the harness generators (same seeds as bench.py)."""
    G = HarnessGen()
    if cfg == "c1":
        return G.poisson3d(64, 64, 64)
    if cfg == "c2":
        return G.scrambled_stencil27_random_sym(160, 160, 160, seed, seed + 1)
    if cfg == "c3":
        return G.rmat(21, 16, seed)
    if cfg.startswith("c4"):
        return G.stencil27(192, 192, 192)
    if cfg == "c5":
        return G.poisson3d(512, 512, 512)
    raise ValueError(cfg)
