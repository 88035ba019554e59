"""Python host mirror of the reference's MPK interface over the mpkg C ABI.

Names, argument meaning and error behaviour follow namespace `mpk` (proj/include/mpk/*.hpp):
std::invalid_argument -> ValueError, std::out_of_range -> IndexError.  Every compute call runs the
sm_100a kernels in libmpkg.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._lib import check, lib

_P = C.c_void_p


def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------------------------
# Host matrices (csr.hpp:57-65 CsrMatrix) and generators (generators.hpp + SURVEY §7 step 1)
# ---------------------------------------------------------------------------------------------
class HostCsr:
    """Host CSR: row_ptr uint32[n+1], col_idx uint32[nnz], values float64[nnz]."""

    def __init__(self, n_rows: int, n_cols: int, row_ptr, col_idx, values, _handle=None):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values
        self._handle = _handle

    @classmethod
    def from_arrays(cls, row_ptr, col_idx, values, n_cols: Optional[int] = None) -> "HostCsr":
        rp = _u32(row_ptr)
        n = len(rp) - 1
        return cls(n, n if n_cols is None else n_cols, rp, _u32(col_idx), _f64(values))

    @classmethod
    def _from_handle(cls, h: int) -> "HostCsr":
        n, m, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib.mpkg_host_csr_info(h, C.byref(n), C.byref(m), C.byref(nnz)))
        rp, ci, v = C.POINTER(C.c_uint32)(), C.POINTER(C.c_uint32)(), C.POINTER(C.c_double)()
        check(lib.mpkg_host_csr_arrays(h, C.byref(rp), C.byref(ci), C.byref(v)))
        nr, nz = n.value, nnz.value
        rpa = np.ctypeslib.as_array(rp, shape=(nr + 1,))
        cia = np.ctypeslib.as_array(ci, shape=(nz,)) if nz else np.zeros(0, np.uint32)
        va = np.ctypeslib.as_array(v, shape=(nz,)) if nz else np.zeros(0, np.float64)
        return cls(nr, m.value, rpa, cia, va, _handle=_HostHandle(h))

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[self.n_rows]) if self.n_rows else 0

    def copy(self) -> "HostCsr":
        return HostCsr(self.n_rows, self.n_cols, self.row_ptr.copy(), self.col_idx.copy(),
                       self.values.copy())


class _HostHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            lib.mpkg_host_csr_destroy(self.h)
            self.h = None


def _gen(kind: int, a: int, b: int = 0, c: int = 0, seed: int = 0) -> HostCsr:
    h = _P()
    check(lib.mpkg_gen(kind, a, b, c, seed, C.byref(h)))
    return HostCsr._from_handle(h.value)


def poisson1d(n: int) -> HostCsr:  # generators.hpp:35-45
    return _gen(1, n)


def poisson2d(nx: int, ny: int) -> HostCsr:  # generators.hpp:49-65
    return _gen(2, nx, ny)


def poisson3d(nx: int, ny: int, nz: int) -> HostCsr:  # generators.hpp:68-89
    return _gen(3, nx, ny, nz)


def random_csr(n: int, nnz_per_row: int, seed: int) -> HostCsr:  # generators.hpp:96-122
    return _gen(4, n, nnz_per_row, 0, seed)


def random_spd(n: int, nnz_per_row: int, seed: int) -> HostCsr:  # generators.hpp:126-146
    return _gen(5, n, nnz_per_row, 0, seed)


def stencil27(nx: int, ny: int, nz: int) -> HostCsr:
    """Config C4: 27-point stencil, diagonal 26, off-diagonals -1."""
    return _gen(6, nx, ny, nz)


def stencil27_random_sym(nx: int, ny: int, nz: int, seed: int) -> HostCsr:
    """Config C2 before the scramble: off-diagonals -U[0.9,1.1], then (A+A^T)/2."""
    return _gen(7, nx, ny, nz, seed)


def rmat(scale: int, edge_factor: int, seed: int) -> HostCsr:
    """Config C3: symmetric R-MAT(.57,.19,.19,.05), diag 1 + sum|off|."""
    return _gen(8, scale, edge_factor, 0, seed)


def scramble(A: HostCsr, seed: int, return_perm: bool = False):
    """Seeded symmetric scramble P A P^T (permute semantics, csr.hpp:159)."""
    if A._handle is None:
        raise ValueError("scramble: needs a generator-owned HostCsr")
    perm = np.empty(A.n_rows, np.uint32)
    h = _P()
    check(lib.mpkg_host_csr_scramble(A._handle.h, seed, _ptr(perm), C.byref(h)))
    B = HostCsr._from_handle(h.value)
    return (B, perm) if return_perm else B


def _block(a) -> np.ndarray:
    return np.ascontiguousarray(np.atleast_2d(np.asarray(a, dtype=np.float64)))


def _same_rows(a: np.ndarray, b: np.ndarray) -> None:
    if a.shape[0] and b.shape[0] and a.shape[1] != b.shape[1]:
        raise ValueError("ortho: blocks must have the same number of rows")


def tsqr_rank_deficient(r, threshold: float) -> bool:
    """ortho.hpp:231-240: any |R_jj| below the threshold."""
    r = np.atleast_2d(np.asarray(r, dtype=np.float64))
    return bool(np.any(np.abs(np.diag(r)) < threshold))


def random_vector(n: int, seed: int) -> np.ndarray:
    """x_i ~ U[-1,1] from std::mt19937_64(seed) (acceptance.cpp:84-90)."""
    out = np.empty(n, np.float64)
    check(lib.mpkg_random_vector(n, seed, _ptr(out)))
    return out


# ---------------------------------------------------------------------------------------------
# Pure host helpers (plan.hpp:70-85, execute.hpp:59-72, mpk.hpp:111-127, mpk.hpp:219-233)
# ---------------------------------------------------------------------------------------------
def greedy_group(level_fp: Sequence[int], target: int) -> list:
    fp = np.ascontiguousarray(level_fp, dtype=np.uint64)
    out = np.empty(len(fp) + 1, np.uint32)
    nb = C.c_uint32()
    check(lib.mpkg_greedy_group(_ptr(fp), len(fp), int(target), _ptr(out), C.byref(nb)))
    return out[: nb.value].tolist()


@dataclass
class ScheduleCell:
    group: int
    stage: int


def wavefront_schedule(n_groups: int, stages: int) -> list:
    cnt = C.c_uint64()
    n = max(0, n_groups * max(stages, 0))
    g = np.empty(max(n, 1), np.uint32)
    q = np.empty(max(n, 1), np.int32)
    check(lib.mpkg_wavefront_schedule(n_groups, stages, _ptr(g), _ptr(q), C.byref(cnt)))
    return [ScheduleCell(int(g[i]), int(q[i])) for i in range(cnt.value)]


def _split_shifts(shifts) -> tuple:
    s = np.asarray(list(shifts), dtype=np.complex128)
    return _f64(s.real), _f64(s.imag)


def check_shift_chain(shifts) -> None:
    re, im = _split_shifts(shifts)
    check(lib.mpkg_check_shift_chain(_ptr(re), _ptr(im), len(re)))


@dataclass
class TuneResult:  # mpk.hpp:211-215
    p_opt: int = 1
    table: list = field(default_factory=list)


def tune_select(table: Sequence[float], p_lo: int, p_hi: int) -> int:
    t = _f64(table)
    out = C.c_int()
    check(lib.mpkg_tune_select(_ptr(t), p_lo, p_hi, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------------------------
# Device objects
# ---------------------------------------------------------------------------------------------
class VectorBlock:
    """rows x slices, slice-major (vector_block.hpp:38-57); slice p holds y_p."""

    def __init__(self, rows: int, slices: int, data: Optional[np.ndarray] = None):
        self.rows, self.slices = int(rows), int(slices)
        self.data = np.zeros(self.rows * self.slices, np.float64) if data is None else data

    def slice(self, p: int) -> np.ndarray:
        if p < 0 or p >= self.slices:
            raise IndexError("VectorBlock::slice")
        return self.data[p * self.rows:(p + 1) * self.rows]

    def as_matrix(self) -> np.ndarray:
        return self.data.reshape(self.slices, self.rows)


class DeviceCsr:
    def __init__(self, ctx: "Context", h: int):
        self.ctx, self.h = ctx, h
        n, m, nnz = C.c_uint32(), C.c_uint32(), C.c_uint32()
        check(lib.mpkg_csr_info(h, C.byref(n), C.byref(m), C.byref(nnz)))
        self.n_rows, self.n_cols, self.nnz = n.value, m.value, nnz.value

    def download(self) -> HostCsr:
        rp = np.empty(self.n_rows + 1, np.uint32)
        ci = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz, np.float64)
        check(lib.mpkg_csr_download(self.h, _ptr(rp), _ptr(ci), _ptr(v)))
        return HostCsr(self.n_rows, self.n_cols, rp, ci, v)

    def __del__(self):
        if getattr(self, "h", None):
            lib.mpkg_csr_destroy(self.h)
            self.h = None


class LevelStructure:
    """levels.hpp:43-57: levels (of ORIGINAL rows), perm old->new, inv_perm, level_ptr."""

    def __init__(self, ctx: "Context", h: int):
        self.ctx, self.h = ctx, h
        n, nl = C.c_uint32(), C.c_uint32()
        check(lib.mpkg_levels_info(h, C.byref(n), C.byref(nl)))
        self.n_rows, self._n_levels = n.value, nl.value
        self._host = None

    def n_levels(self) -> int:
        return self._n_levels

    def _fetch(self):
        if self._host is None:
            n = self.n_rows
            lv, pm, ip = (np.empty(n, np.uint32) for _ in range(3))
            lp = np.empty(self._n_levels + 1, np.uint32)
            check(lib.mpkg_levels_get(self.h, _ptr(lv), _ptr(pm), _ptr(ip), _ptr(lp)))
            self._host = (lv, pm, ip, lp)
        return self._host

    levels = property(lambda self: self._fetch()[0])
    perm = property(lambda self: self._fetch()[1])
    inv_perm = property(lambda self: self._fetch()[2])
    level_ptr = property(lambda self: self._fetch()[3])

    def level_of_permuted(self, new_row: int) -> int:
        return int(self.levels[self.inv_perm[new_row]])

    def __del__(self):
        if getattr(self, "h", None):
            lib.mpkg_levels_destroy(self.h)
            self.h = None


class JacobiPrecon:
    """jacobi.hpp:41-76: DiagInfo (pos, inv) + sweeps, resident on the device."""

    def __init__(self, ctx: "Context", h: int):
        self.ctx, self.h = ctx, h
        n, sw = C.c_uint32(), C.c_int()
        check(lib.mpkg_jacobi_info(h, C.byref(n), C.byref(sw)))
        self.n_rows, self.sweeps = n.value, sw.value

    def diag(self):
        pos, inv = np.empty(self.n_rows, np.uint32), np.empty(self.n_rows)
        check(lib.mpkg_jacobi_get(self.h, _ptr(pos), _ptr(inv)))
        return pos, inv

    def stages(self) -> int:  # jacobi.hpp:129 JacobiOpChain::stages
        return 1 if self.sweeps == 1 else self.sweeps + 1

    def __del__(self):
        if getattr(self, "h", None):
            lib.mpkg_jacobi_destroy(self.h)
            self.h = None


class Gs2Precon:
    """gs2.hpp:47-53: DiagInfo + gamma (inner iterations), sweeps (K), direction."""

    def __init__(self, ctx: "Context", h: int):
        self.ctx, self.h = ctx, h
        n, g, k, d = C.c_uint32(), C.c_int(), C.c_int(), C.c_int()
        check(lib.mpkg_gs2_info(h, C.byref(n), C.byref(g), C.byref(k), C.byref(d)))
        self.n_rows, self.gamma, self.sweeps = n.value, g.value, k.value
        self.forward = d.value == 0

    def diag(self):
        pos, inv = np.empty(self.n_rows, np.uint32), np.empty(self.n_rows)
        check(lib.mpkg_gs2_get(self.h, _ptr(pos), _ptr(inv)))
        return pos, inv

    def stages(self) -> int:  # plan sub_powers of the chain (gs2.hpp:169)
        return self.gamma + 2

    def __del__(self):
        if getattr(self, "h", None):
            lib.mpkg_gs2_destroy(self.h)
            self.h = None


class ExecutionPlan:
    """plan.hpp:41-54."""

    def __init__(self, h: int):
        self.h = h
        pm, sub, n, cb, tb, ng = (C.c_int(), C.c_int(), C.c_uint32(), C.c_uint64(),
                                  C.c_uint64(), C.c_uint32())
        check(lib.mpkg_plan_info(h, C.byref(pm), C.byref(sub), C.byref(n), C.byref(cb),
                                 C.byref(tb), C.byref(ng)))
        self.p_m, self.sub_powers, self.n_rows = pm.value, sub.value, n.value
        self.cache_bytes, self.target_bytes = cb.value, tb.value
        g = ng.value
        self.group_rows = np.empty(g + 1, np.uint32)
        self.group_level_ptr = np.empty(g + 1, np.uint32)
        self.group_footprint = np.empty(max(g, 1), np.uint64)[:g]
        check(lib.mpkg_plan_get(h, _ptr(self.group_rows), _ptr(self.group_level_ptr),
                                _ptr(self.group_footprint) if g else None))

    def n_groups(self) -> int:
        return len(self.group_rows) - 1

    @staticmethod
    def from_groups(n_rows: int, group_rows, p_m: int, sub_powers: int = 1, level_ptr=None,
                    cache_bytes: int = 0) -> "ExecutionPlan":
        """A plan from host fields (plan.hpp:41-54), e.g. one made by hand as in the reference's
        schedule tests (mpkg_plan_create)."""
        gr = _u32(group_rows)
        ng = len(gr) - 1
        lp = None if level_ptr is None else _u32(level_ptr)
        glp = np.zeros(ng + 1, np.uint32)
        fp = np.zeros(max(ng, 1), np.uint64)
        h = _P()
        check(lib.mpkg_plan_create(p_m, sub_powers, n_rows, cache_bytes, cache_bytes // (p_m + 1), ng,
                                   _ptr(gr), _ptr(glp), _ptr(fp), 0 if lp is None else len(lp) - 1,
                                   _ptr(lp) if lp is not None else None, C.byref(h)))
        return ExecutionPlan(h.value)

    def with_sub_powers(self, sub_powers: int, level_ptr=None) -> "ExecutionPlan":
        """A copy with another sub_powers (chains: the reference sets plan.sub_powers by hand,
        e.g. JacobiOpChain::stages(sweeps) for jacobi_op_blocked / the s-step chains)."""
        h = _P()
        lp = None if level_ptr is None else _u32(level_ptr)
        check(lib.mpkg_plan_create(self.p_m, sub_powers, self.n_rows, self.cache_bytes,
                                   self.target_bytes, self.n_groups(), _ptr(self.group_rows),
                                   _ptr(self.group_level_ptr),
                                   _ptr(self.group_footprint) if self.n_groups() else None,
                                   0 if lp is None else len(lp) - 1, _ptr(lp) if lp is not None else None,
                                   C.byref(h)))
        return ExecutionPlan(h.value)

    def exec_info(self) -> dict:
        t, k, d, pp = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint32()
        check(lib.mpkg_plan_exec_info(self.h, C.byref(t), C.byref(k), C.byref(d), C.byref(pp)))
        o, sw, kn, lr = C.c_int32(), C.c_int32(), C.c_int32(), C.c_uint64()
        check(lib.mpkg_plan_exec_mode(self.h, C.byref(o), C.byref(sw), C.byref(kn), C.byref(lr)))
        wf, wc, wa, wn, wb = C.c_int32(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.mpkg_plan_exec_wave(self.h, C.byref(wf), C.byref(wc), C.byref(wa), C.byref(wn), C.byref(wb)))
        return {"tiles": t.value, "tickets": k.value, "dep_tiles": d.value,
                "pass_powers": pp.value, "order": o.value,
                "schedule": {1: "sweeps", 2: "wave"}.get(sw.value, "fused"), "kernel": kn.value,
                "long_rows": lr.value, "wave_format": wf.value, "wave_chunks": wc.value,
                "wave_affine_chunks": wa.value, "wave_banded_chunks": wn.value,
                "wave_record_bytes": wb.value}

    def exec_trace(self):
        """ctx knob "trace": (flat stamps, tile_rows) of the last fused / wave MPK on this plan
        (mpkg_plan_exec_trace); stamps reshape to [p+1, n_tiles, 2] = (inputs complete, results
        stored).  (None, tile_rows) when the last call recorded nothing."""
        n, tr = C.c_uint64(), C.c_uint32()
        check(lib.mpkg_plan_exec_trace(self.h, None, 0, C.byref(n), C.byref(tr)))
        if n.value == 0:
            return None, tr.value
        out = np.empty(n.value, np.uint64)
        check(lib.mpkg_plan_exec_trace(self.h, _ptr(out), n.value, C.byref(n), C.byref(tr)))
        return out, tr.value

    def __del__(self):
        if getattr(self, "h", None):
            lib.mpkg_plan_destroy(self.h)
            self.h = None


class Context:
    """One CUDA device + stream (replaces resolve_threads, threading.hpp:34-46)."""

    def __init__(self, device: int = 0):
        h = _P()
        check(lib.mpkg_ctx_create(device, C.byref(h)))
        self.h = h.value
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            lib.mpkg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    # ---- context facts / knobs
    @property
    def stream(self) -> int:
        s = _P()
        check(lib.mpkg_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def synchronize(self):
        check(lib.mpkg_ctx_synchronize(self.h))

    def device_info(self) -> dict:
        sm, l2, pm = C.c_int(), C.c_size_t(), C.c_size_t()
        check(lib.mpkg_ctx_device_info(self.h, C.byref(sm), C.byref(l2), C.byref(pm)))
        return {"sm_count": sm.value, "l2_bytes": l2.value, "persist_max": pm.value}

    def set_param(self, key: str, value: int):
        check(lib.mpkg_ctx_set_param(self.h, key.encode(), int(value)))

    MODE_BITWISE, MODE_FAST = 0, 1

    def set_mode(self, mode: int):
        """MODE_BITWISE (default): bit-identical to the reference.  MODE_FAST: long rows reduced
        in parallel; within the north star's 1e-12 inf-norm bound (include/mpkg.h)."""
        check(lib.mpkg_ctx_set_mode(self.h, int(mode)))

    def kernel_times(self) -> tuple:
        """(total_ms, count, max_ms) of the launches recorded since the last call."""
        t, n, m = C.c_double(), C.c_uint64(), C.c_double()
        check(lib.mpkg_ctx_kernel_times(self.h, C.byref(t), C.byref(n), C.byref(m)))
        return t.value, n.value, m.value

    def launch_count(self) -> int:
        v = C.c_uint64()
        check(lib.mpkg_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    # ---- matrices
    def csr(self, A: HostCsr) -> DeviceCsr:
        h = _P()
        if A._handle is not None:
            check(lib.mpkg_csr_create_from_host(self.h, A._handle.h, C.byref(h)))
        else:
            rp, ci, v = _u32(A.row_ptr), _u32(A.col_idx), _f64(A.values)
            check(lib.mpkg_csr_create(self.h, A.n_rows, A.n_cols, _ptr(rp), _ptr(ci), _ptr(v),
                                      C.byref(h)))
        return DeviceCsr(self, h.value)

    def spmv(self, A: DeviceCsr, x) -> np.ndarray:  # csr.hpp:126-142
        x = _f64(x)
        if len(x) != A.n_cols:
            raise ValueError("spmv: vector size mismatch")
        y = np.empty(A.n_rows, np.float64)
        check(lib.mpkg_spmv(self.h, A.h, _ptr(x), _ptr(y)))
        return y

    # ---- level engine
    def build_levels(self, A: DeviceCsr) -> LevelStructure:  # levels.hpp:65
        h = _P()
        check(lib.mpkg_build_levels(self.h, A.h, C.byref(h)))
        return LevelStructure(self, h.value)

    def levels_from_host(self, levels, perm, inv_perm, level_ptr) -> LevelStructure:
        lv, pm, ip, lp = _u32(levels), _u32(perm), _u32(inv_perm), _u32(level_ptr)
        h = _P()
        check(lib.mpkg_levels_create(self.h, len(lv), len(lp) - 1, _ptr(lv), _ptr(pm), _ptr(ip),
                                     _ptr(lp), C.byref(h)))
        return LevelStructure(self, h.value)

    def validate_levels(self, A_perm: DeviceCsr, ls: LevelStructure) -> bool:  # levels.hpp:151
        ok = C.c_int()
        check(lib.mpkg_validate_levels(self.h, A_perm.h, ls.h, C.byref(ok)))
        return bool(ok.value)

    def permute(self, A: DeviceCsr, perm) -> DeviceCsr:  # csr.hpp:159
        h = _P()
        if isinstance(perm, LevelStructure):
            check(lib.mpkg_permute_levels(self.h, A.h, perm.h, C.byref(h)))
        else:
            p = _u32(perm)
            if len(p) != A.n_rows:
                raise ValueError("permute: permutation size mismatch")
            check(lib.mpkg_permute(self.h, A.h, _ptr(p), C.byref(h)))
        return DeviceCsr(self, h.value)

    def csr_from_coo(self, n_rows: int, n_cols: int, rows, cols, vals) -> DeviceCsr:
        """csr.hpp:72-110 from_coo, on the GPU (bit-identical to the reference)."""
        r, c, v = _u32(rows), _u32(cols), _f64(vals)
        h = _P()
        check(lib.mpkg_csr_from_coo(self.h, n_rows, n_cols, len(r), _ptr(r), _ptr(c), _ptr(v), C.byref(h)))
        return DeviceCsr(self, h.value)

    def read_matrix_market(self, path) -> DeviceCsr:
        """matrix_market.hpp read_matrix_market: host parse, GPU assembly."""
        h = _P()
        check(lib.mpkg_read_matrix_market(self.h, str(path).encode(), C.byref(h)))
        return DeviceCsr(self, h.value)

    def csr_block(self, A: DeviceCsr, r0: int, r1: int, c0: int, c1: int) -> DeviceCsr:
        """A[r0:r1, c0:c1] on the device (columns shifted by -c0): a level-range shard."""
        h = _P()
        check(lib.mpkg_csr_block(self.h, A.h, r0, r1, c0, c1, C.byref(h)))
        return DeviceCsr(self, h.value)

    def permute_vector(self, v, perm) -> np.ndarray:  # csr.hpp:191
        v, p = _f64(v), _u32(perm)
        out = np.empty_like(v)
        check(lib.mpkg_permute_vector(self.h, len(v), _ptr(v), _ptr(p), _ptr(out)))
        return out

    def unpermute_vector(self, v, perm) -> np.ndarray:  # csr.hpp:198
        v, p = _f64(v), _u32(perm)
        out = np.empty_like(v)
        check(lib.mpkg_unpermute_vector(self.h, len(v), _ptr(v), _ptr(p), _ptr(out)))
        return out

    # ---- plan
    def row_range_footprint(self, A_perm: DeviceCsr, row_s: int, row_e: int, p_m: int) -> int:
        b = C.c_uint64()
        check(lib.mpkg_row_range_footprint(A_perm.h, row_s, row_e, p_m, C.byref(b)))
        return b.value

    def group_levels(self, ls: LevelStructure, A_perm: DeviceCsr, cache_bytes: int,
                     p_m: int) -> ExecutionPlan:  # plan.hpp:88
        h = _P()
        check(lib.mpkg_group_levels(self.h, ls.h, A_perm.h, int(cache_bytes), p_m, C.byref(h)))
        return ExecutionPlan(h.value)

    # ---- power kernels
    @staticmethod
    def _block(n: int, p_m: int, block: Optional[VectorBlock]) -> VectorBlock:
        return VectorBlock(n, p_m + 1) if block is None else block

    def baseline_mpk(self, A: DeviceCsr, x, p_m: int,
                     block: Optional[VectorBlock] = None) -> VectorBlock:  # mpk.hpp:59
        x, blk = _f64(x), self._block(A.n_rows, p_m, block)
        if len(x) != A.n_rows:
            raise ValueError("baseline_mpk: input size mismatch")
        check(lib.mpkg_baseline_mpk(self.h, A.h, _ptr(x), p_m, _ptr(blk.data), blk.rows,
                                    blk.slices))
        return blk

    def mpk(self, plan: ExecutionPlan, A_perm: DeviceCsr, x, p_m: int,
            block: Optional[VectorBlock] = None) -> VectorBlock:  # mpk.hpp:81
        x, blk = _f64(x), self._block(A_perm.n_rows, p_m, block)
        if len(x) != A_perm.n_rows:
            raise ValueError("mpk: input size mismatch")
        check(lib.mpkg_mpk(self.h, plan.h, A_perm.h, _ptr(x), p_m, _ptr(blk.data), blk.rows,
                           blk.slices))
        return blk

    def baseline_mpk_shifted(self, A: DeviceCsr, x, shifts,
                             block: Optional[VectorBlock] = None) -> VectorBlock:  # mpk.hpp:160
        re, im = _split_shifts(shifts)
        x, blk = _f64(x), self._block(A.n_rows, len(re), block)
        if len(x) != A.n_rows:
            raise ValueError("baseline_mpk_shifted: input size mismatch")
        check(lib.mpkg_baseline_mpk_shifted(self.h, A.h, _ptr(x), _ptr(re), _ptr(im), len(re),
                                            _ptr(blk.data), blk.rows, blk.slices))
        return blk

    def mpk_shifted(self, plan: ExecutionPlan, A_perm: DeviceCsr, x, shifts,
                    block: Optional[VectorBlock] = None) -> VectorBlock:  # mpk.hpp:184
        re, im = _split_shifts(shifts)
        x, blk = _f64(x), self._block(A_perm.n_rows, len(re), block)
        if len(x) != A_perm.n_rows:
            raise ValueError("mpk_shifted: input size mismatch")
        check(lib.mpkg_mpk_shifted(self.h, plan.h, A_perm.h, _ptr(x), _ptr(re), _ptr(im),
                                   len(re), _ptr(blk.data), blk.rows, blk.slices))
        return blk

    def mpk_poly(self, plan: ExecutionPlan, A_perm: DeviceCsr, x, coef,
                 return_block: bool = False):
        """z = sum_k c_k A^k x, fused into the power sweep."""
        x, c = _f64(x), _f64(coef)
        d = len(c) - 1
        if d < 1:
            raise ValueError("mpk_poly: need at least two coefficients")
        z = np.empty(A_perm.n_rows, np.float64)
        blk = VectorBlock(A_perm.n_rows, d + 1) if return_block else None
        check(lib.mpkg_mpk_poly(self.h, plan.h, A_perm.h, _ptr(x), _ptr(c), d, _ptr(z),
                                _ptr(blk.data) if blk else None,
                                blk.rows if blk else 0, blk.slices if blk else 0))
        return (z, blk) if return_block else z

    # device-pointer variants (async on self.stream) for benchmarks
    def mpk_dev(self, plan, A_perm, d_x: int, p_m: int, d_block: int, rows: int, slices: int):
        check(lib.mpkg_mpk_dev(self.h, plan.h, A_perm.h, d_x, p_m, d_block, rows, slices))

    def baseline_mpk_dev(self, A, d_x: int, p_m: int, d_block: int, rows: int, slices: int):
        check(lib.mpkg_baseline_mpk_dev(self.h, A.h, d_x, p_m, d_block, rows, slices))

    def mpk_shifted_dev(self, plan, A_perm, d_x: int, shifts, d_block: int, rows: int,
                        slices: int):
        re, im = _split_shifts(shifts)
        check(lib.mpkg_mpk_shifted_dev(self.h, plan.h, A_perm.h, d_x, _ptr(re), _ptr(im),
                                       len(re), d_block, rows, slices))

    def mpk_poly_dev(self, plan, A_perm, d_x: int, coef, d_z: int, d_block: Optional[int],
                     rows: int, slices: int):
        c = _f64(coef)
        check(lib.mpkg_mpk_poly_dev(self.h, plan.h, A_perm.h, d_x, _ptr(c), len(c) - 1, d_z,
                                    d_block, rows, slices))

    # ---- Jacobi-preconditioned chains (jacobi.hpp, sstep.hpp) ----------------------------------
    def jacobi_setup(self, A: DeviceCsr, sweeps: int = 1) -> JacobiPrecon:  # jacobi.hpp:72
        h = _P()
        check(lib.mpkg_jacobi_setup(self.h, A.h, int(sweeps), C.byref(h)))
        return JacobiPrecon(self, h.value)

    def jacobi_apply(self, J: JacobiPrecon, A: DeviceCsr, v) -> np.ndarray:  # jacobi.hpp:155
        v = _f64(v)
        z = np.empty(A.n_rows)
        check(lib.mpkg_jacobi_apply(self.h, J.h, A.h, _ptr(v), _ptr(z)))
        return z

    def jacobi_op(self, J: JacobiPrecon, A: DeviceCsr, v) -> np.ndarray:  # jacobi.hpp:177
        v = _f64(v)
        y = np.empty(A.n_rows)
        check(lib.mpkg_jacobi_op(self.h, J.h, A.h, _ptr(v), _ptr(y)))
        return y

    def jacobi_op_blocked(self, J: JacobiPrecon, plan: ExecutionPlan, A_perm: DeviceCsr, v):
        v = _f64(v)  # jacobi.hpp:196
        y = np.empty(A_perm.n_rows)
        check(lib.mpkg_jacobi_op_blocked(self.h, J.h, plan.h, A_perm.h, _ptr(v), _ptr(y)))
        return y

    def sstep_jacobi(self, J: JacobiPrecon, plan, A: DeviceCsr, x, shifts) -> VectorBlock:
        """sstep.hpp:356-385 (Jacobi): slice 0 = x, slices 1..s the preconditioned Newton basis."""
        s = np.asarray(list(shifts), dtype=np.complex128)
        re, im = _f64(s.real), _f64(s.imag)
        n, k = A.n_rows, len(re)
        blk = VectorBlock(n, k + 1)
        blk.data[:n] = _f64(x)
        check(lib.mpkg_sstep_jacobi(self.h, J.h, plan.h if plan is not None else None, A.h,
                                    _ptr(re), _ptr(im), k, _ptr(blk.data), n, k + 1))
        return blk

    # ---- GS2 chains (gs2.hpp, sstep.hpp:160-198) -----------------------------------------------
    def gs2_setup(self, A: DeviceCsr, gamma: int, sweeps: int = 1, forward: bool = True) -> Gs2Precon:
        h = _P()
        check(lib.mpkg_gs2_setup(self.h, A.h, int(gamma), int(sweeps), 0 if forward else 1, C.byref(h)))
        return Gs2Precon(self, h.value)

    def gs2_smooth(self, G: Gs2Precon, A: DeviceCsr, v, z, plan=None) -> np.ndarray:
        z = _f64(z).copy()
        check(lib.mpkg_gs2_smooth(self.h, G.h, plan.h if plan else None, A.h, _ptr(_f64(v)), _ptr(z)))
        return z

    def gs2_apply(self, G: Gs2Precon, A: DeviceCsr, v, plan=None) -> np.ndarray:
        z = np.empty(A.n_rows)
        check(lib.mpkg_gs2_apply(self.h, G.h, plan.h if plan else None, A.h, _ptr(_f64(v)), _ptr(z)))
        return z

    def gs2_smooth_residual(self, G: Gs2Precon, A: DeviceCsr, v, z, plan=None):
        z = _f64(z).copy()
        r = np.empty(A.n_rows)
        check(lib.mpkg_gs2_smooth_residual(self.h, G.h, plan.h if plan else None, A.h, _ptr(_f64(v)),
                                           _ptr(z), _ptr(r)))
        return z, r

    def gs2_op(self, G: Gs2Precon, A: DeviceCsr, v, plan=None) -> np.ndarray:
        y = np.empty(A.n_rows)
        check(lib.mpkg_gs2_op(self.h, G.h, plan.h if plan else None, A.h, _ptr(_f64(v)), _ptr(y)))
        return y

    def sstep_gs2(self, G: Gs2Precon, plan, A: DeviceCsr, x, shifts) -> VectorBlock:
        s = np.asarray(list(shifts), dtype=np.complex128)
        re, im = _f64(s.real), _f64(s.imag)
        n, k = A.n_rows, len(re)
        blk = VectorBlock(n, k + 1)
        blk.data[:n] = _f64(x)
        check(lib.mpkg_sstep_gs2(self.h, G.h, plan.h if plan is not None else None, A.h,
                                 _ptr(re), _ptr(im), k, _ptr(blk.data), n, k + 1))
        return blk

    # ---- product-form polynomial (poly.hpp:146-281) ---------------------------------------------
    def poly_apply(self, A: DeviceCsr, roots, v, inner=None, plan=None) -> np.ndarray:
        """z = p(A M^{-1}) v for the given roots; inner: None, a JacobiPrecon or a Gs2Precon."""
        r = np.asarray(list(roots), dtype=np.complex128)
        re, im = _f64(r.real), _f64(r.imag)
        J = inner.h if isinstance(inner, JacobiPrecon) else None
        G = inner.h if isinstance(inner, Gs2Precon) else None
        z = np.empty(A.n_rows)
        check(lib.mpkg_poly_apply(self.h, A.h, J, G, _ptr(re), _ptr(im), len(re),
                                  plan.h if plan is not None else None, _ptr(_f64(v)), _ptr(z)))
        return z

    # ---- block orthogonalisation (ortho.hpp) --------------------------
    # Blocks are (cols, rows) float64 arrays: array row l is block column l (column-major memory,
    # i.e. consecutive VectorBlock slices).  C and R are returned as ordinary matrices.
    def block_dots(self, q, v) -> np.ndarray:
        """ortho.hpp:46-63: C = Q^T V as a (qcols, vcols) matrix."""
        q, v = _block(q), _block(v)
        _same_rows(q, v)
        c = np.zeros((v.shape[0], q.shape[0]))
        check(lib.mpkg_block_dots(self.h, _ptr(q), _ptr(v), v.shape[1], q.shape[0], v.shape[0], _ptr(c)))
        return c.T.copy()

    def block_update(self, q, c, v) -> np.ndarray:
        """ortho.hpp:67-92: returns V - Q C (c a (qcols, vcols) matrix); v is not modified."""
        q, out = _block(q), np.array(_block(v), order="C")
        _same_rows(q, out)
        cc = _f64(np.asarray(c, dtype=np.float64).T)
        if cc.shape != (out.shape[0], q.shape[0]):
            raise ValueError("block_update: coefficient shape mismatch")
        check(lib.mpkg_block_update(self.h, _ptr(q), _ptr(cc), out.shape[1], q.shape[0], out.shape[0],
                                    _ptr(out)))
        return out

    def icgs_block_orthogonalize(self, q, v, sweeps: int):
        """ortho.hpp:97-117 -> (V orthogonalised against Q, coefficients (qcols, vcols))."""
        out = np.array(_block(v), order="C")
        q = _block(q) if q is not None and np.size(q) else np.zeros((0, out.shape[1]))
        _same_rows(q, out)
        coeff = np.zeros((out.shape[0], q.shape[0]))
        check(lib.mpkg_icgs_block_orthogonalize(self.h, _ptr(q) if q.size else None, out.shape[1],
                                                q.shape[0], _ptr(out), out.shape[0], int(sweeps),
                                                _ptr(coeff)))
        return out, coeff.T.copy()

    def tsqr(self, v):
        """ortho.hpp:136-229 -> (Q as a (cols, rows) block, R (cols, cols) upper triangular with a
        non-negative diagonal), Q R = V."""
        out = np.array(_block(v), order="C")
        cols, rows = out.shape
        r = np.zeros((cols, cols))
        check(lib.mpkg_tsqr(self.h, _ptr(out), rows, cols, _ptr(r)))
        return out, r.T.copy()

    def ortho_block(self, q, v, sweeps: int):
        """sstep.hpp:539-545: icgs_block_orthogonalize then tsqr in one call -> (Q as a (cols, rows)
        block, coefficients (qcols, vcols), R (cols, cols)); bit-identical to the two calls."""
        out = np.array(_block(v), order="C")
        q = _block(q) if q is not None and np.size(q) else np.zeros((0, out.shape[1]))
        _same_rows(q, out)
        cols, rows = out.shape
        coeff = np.zeros((cols, q.shape[0]))
        r = np.zeros((cols, cols))
        check(lib.mpkg_ortho_block(self.h, _ptr(q) if q.size else None, rows, q.shape[0], _ptr(out), cols,
                                   int(sweeps), _ptr(coeff), _ptr(r)))
        return out, coeff.T.copy(), r.T.copy()

    def ortho_block_dev(self, d_q: int, rows: int, qcols: int, d_v: int, vcols: int, sweeps: int,
                        d_coeff: int, d_r: int):
        check(lib.mpkg_ortho_block_dev(self.h, d_q, rows, qcols, d_v, vcols, sweeps, d_coeff, d_r))

    def block_dots_dev(self, d_q: int, d_v: int, rows: int, qcols: int, vcols: int, d_c: int):
        check(lib.mpkg_block_dots_dev(self.h, d_q, d_v, rows, qcols, vcols, d_c))

    def block_update_dev(self, d_q: int, d_c: int, rows: int, qcols: int, vcols: int, d_v: int):
        check(lib.mpkg_block_update_dev(self.h, d_q, d_c, rows, qcols, vcols, d_v))

    def icgs_block_orthogonalize_dev(self, d_q: int, rows: int, qcols: int, d_v: int, vcols: int,
                                     sweeps: int, d_coeff: int):
        check(lib.mpkg_icgs_block_orthogonalize_dev(self.h, d_q, rows, qcols, d_v, vcols, sweeps, d_coeff))

    def tsqr_dev(self, d_v: int, rows: int, cols: int, d_r: int):
        check(lib.mpkg_tsqr_dev(self.h, d_v, rows, cols, d_r))

    def tune_p(self, ls: LevelStructure, A_perm: DeviceCsr, cache_bytes: int, p_lo: int,
               p_hi: int, reps: int = 3) -> TuneResult:  # mpk.hpp:238
        if p_lo < 1 or p_hi < p_lo:
            raise ValueError("tune_p: bad range")
        table = np.empty(p_hi - p_lo + 1, np.float64)
        p = C.c_int()
        check(lib.mpkg_tune_p(self.h, ls.h, A_perm.h, int(cache_bytes), p_lo, p_hi, reps,
                              C.byref(p), _ptr(table)))
        return TuneResult(p.value, [(p_lo + i, float(g)) for i, g in enumerate(table)])
