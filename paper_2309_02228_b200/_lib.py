"""ctypes loader for libmpkg.so (the C ABI declared in include/mpkg.h).

The library is loaded from the package directory only (built in-tree by build.py); there is no
fallback implementation of any kind: if the .so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import pathlib

LIB_PATH = pathlib.Path(__file__).resolve().parent / "libmpkg.so"

MPKG_OK, MPKG_EINVAL, MPKG_ERANGE, MPKG_ECUDA, MPKG_ENOMEM, MPKG_EINTERNAL = range(6)

u32, u64, i32, i64, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_int64, C.c_double
P = C.c_void_p
pu32, pu64, pdbl, pint = C.POINTER(u32), C.POINTER(u64), C.POINTER(dbl), C.POINTER(C.c_int)

# name -> argtypes (every function returns int status unless listed in _RESTYPES)
_SIGS = {
    "mpkg_last_error": [],
    "mpkg_abi_version": [],
    "mpkg_ctx_create": [i32, C.POINTER(P)],
    "mpkg_ctx_destroy": [P],
    "mpkg_ctx_stream": [P, C.POINTER(P)],
    "mpkg_ctx_synchronize": [P],
    "mpkg_ctx_set_mode": [P, i32],
    "mpkg_ctx_device_info": [P, pint, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)],
    "mpkg_ctx_set_param": [P, C.c_char_p, i64],
    "mpkg_ctx_launch_count": [P, pu64],
    "mpkg_ctx_kernel_times": [P, pdbl, pu64, pdbl],
    "mpkg_csr_create": [P, u32, u32, P, P, P, C.POINTER(P)],
    "mpkg_csr_create_from_host": [P, P, C.POINTER(P)],
    "mpkg_csr_info": [P, pu32, pu32, pu32],
    "mpkg_csr_download": [P, P, P, P],
    "mpkg_csr_destroy": [P],
    "mpkg_csr_block": [P, P, u32, u32, u32, u32, C.POINTER(P)],
    "mpkg_csr_from_coo": [P, u32, u32, u64, P, P, P, C.POINTER(P)],
    "mpkg_csr_from_coo_dev": [P, u32, u32, u64, P, P, P, C.POINTER(P)],
    "mpkg_read_matrix_market": [P, C.c_char_p, C.POINTER(P)],
    "mpkg_spmv": [P, P, P, P],
    "mpkg_spmv_dev": [P, P, P, P],
    "mpkg_build_levels": [P, P, C.POINTER(P)],
    "mpkg_levels_create": [P, u32, u32, P, P, P, P, C.POINTER(P)],
    "mpkg_levels_info": [P, pu32, pu32],
    "mpkg_levels_get": [P, P, P, P, P],
    "mpkg_levels_destroy": [P],
    "mpkg_validate_levels": [P, P, P, pint],
    "mpkg_permute": [P, P, P, C.POINTER(P)],
    "mpkg_permute_levels": [P, P, P, C.POINTER(P)],
    "mpkg_permute_vector": [P, u32, P, P, P],
    "mpkg_unpermute_vector": [P, u32, P, P, P],
    "mpkg_row_range_footprint": [P, u32, u32, i32, pu64],
    "mpkg_greedy_group": [P, u32, u64, P, pu32],
    "mpkg_group_levels": [P, P, P, u64, i32, C.POINTER(P)],
    "mpkg_plan_create": [i32, i32, u32, u64, u64, u32, P, P, P, u32, P, C.POINTER(P)],
    "mpkg_plan_info": [P, pint, pint, pu32, pu64, pu64, pu32],
    "mpkg_plan_get": [P, P, P, P],
    "mpkg_plan_destroy": [P],
    "mpkg_plan_exec_info": [P, pu32, pu64, pu64, pu32],
    "mpkg_plan_exec_mode": [P, pint, pint, pint, pu64],
    "mpkg_plan_exec_wave": [P, pint, pu64, pu64, pu64, pu64],
    "mpkg_plan_exec_trace": [P, P, u64, pu64, pu32],
    "mpkg_jacobi_setup": [P, P, i32, C.POINTER(P)],
    "mpkg_jacobi_info": [P, pu32, pint],
    "mpkg_jacobi_get": [P, P, P],
    "mpkg_jacobi_destroy": [P],
    "mpkg_jacobi_apply": [P, P, P, P, P],
    "mpkg_jacobi_apply_dev": [P, P, P, P, P],
    "mpkg_jacobi_op": [P, P, P, P, P],
    "mpkg_jacobi_op_dev": [P, P, P, P, P],
    "mpkg_jacobi_op_blocked": [P, P, P, P, P, P],
    "mpkg_jacobi_op_blocked_dev": [P, P, P, P, P, P],
    "mpkg_sstep_jacobi": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_gs2_setup": [P, P, i32, i32, i32, C.POINTER(P)],
    "mpkg_gs2_info": [P, pu32, pint, pint, pint],
    "mpkg_gs2_get": [P, P, P],
    "mpkg_gs2_destroy": [P],
    "mpkg_gs2_smooth": [P, P, P, P, P, P],
    "mpkg_gs2_apply": [P, P, P, P, P, P],
    "mpkg_gs2_smooth_residual": [P, P, P, P, P, P, P],
    "mpkg_gs2_op": [P, P, P, P, P, P],
    "mpkg_gs2_run_dev": [P, P, P, P, i32, P, P, P],
    "mpkg_sstep_gs2": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_poly_apply": [P, P, P, P, P, P, i32, P, P, P],
    "mpkg_poly_apply_dev": [P, P, P, P, P, P, i32, P, P, P],
    "mpkg_block_dots": [P, P, P, u64, u32, u32, P],
    "mpkg_block_dots_dev": [P, P, P, u64, u32, u32, P],
    "mpkg_block_update": [P, P, P, u64, u32, u32, P],
    "mpkg_block_update_dev": [P, P, P, u64, u32, u32, P],
    "mpkg_icgs_block_orthogonalize": [P, P, u64, u32, P, u32, i32, P],
    "mpkg_icgs_block_orthogonalize_dev": [P, P, u64, u32, P, u32, i32, P],
    "mpkg_tsqr": [P, P, u64, u32, P],
    "mpkg_tsqr_dev": [P, P, u64, u32, P],
    "mpkg_ortho_block": [P, P, u64, u32, P, u32, i32, P, P],
    "mpkg_ortho_block_dev": [P, P, u64, u32, P, u32, i32, P, P],
    "mpkg_sstep_gs2_dev": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_sstep_jacobi_dev": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_wavefront_schedule": [u32, i32, P, P, pu64],
    "mpkg_dist_partition": [P, u32, P, i32, P],
    "mpkg_dist_halo": [P, u32, P, i32, i32, i32, P, P, P, P],
    "mpkg_dist_unique_id": [P],
    "mpkg_dist_create": [P, P, i32, i32, C.POINTER(P)],
    "mpkg_dist_destroy": [P],
    "mpkg_dist_bcast_host": [P, P, u64, i32],
    "mpkg_dist_set_plan": [P, P, u32, P, i32],
    "mpkg_dist_info": [P, P, P, pu64, pu64],
    "mpkg_dist_scatter_blocks": [P, i32, P, C.POINTER(P)],
    "mpkg_dist_scatter_rows": [P, i32, P, P],
    "mpkg_dist_exchange": [P, P, C.POINTER(P)],
    "mpkg_dist_mpk": [P, P, P, P, i32, P, u64, u64],
    "mpkg_baseline_mpk": [P, P, P, i32, P, u64, u64],
    "mpkg_baseline_mpk_dev": [P, P, P, i32, P, u64, u64],
    "mpkg_mpk": [P, P, P, P, i32, P, u64, u64],
    "mpkg_mpk_dev": [P, P, P, P, i32, P, u64, u64],
    "mpkg_check_shift_chain": [P, P, i32],
    "mpkg_baseline_mpk_shifted": [P, P, P, P, P, i32, P, u64, u64],
    "mpkg_baseline_mpk_shifted_dev": [P, P, P, P, P, i32, P, u64, u64],
    "mpkg_mpk_shifted": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_mpk_shifted_dev": [P, P, P, P, P, P, i32, P, u64, u64],
    "mpkg_mpk_poly": [P, P, P, P, P, i32, P, P, u64, u64],
    "mpkg_mpk_poly_dev": [P, P, P, P, P, i32, P, P, u64, u64],
    "mpkg_tune_p": [P, P, P, u64, i32, i32, i32, pint, P],
    "mpkg_tune_select": [P, i32, i32, pint],
    "mpkg_gen": [i32, u32, u32, u32, u64, C.POINTER(P)],
    "mpkg_host_csr_scramble": [P, u64, P, C.POINTER(P)],
    "mpkg_host_csr_info": [P, pu32, pu32, pu64],
    "mpkg_host_csr_arrays": [P, C.POINTER(pu32), C.POINTER(pu32), C.POINTER(pdbl)],
    "mpkg_host_csr_destroy": [P],
    "mpkg_random_vector": [u64, u64, P],
}
_RESTYPES = {"mpkg_last_error": C.c_char_p}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2309_02228_b200.build` "
            "(there is no non-CUDA fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, C.c_int)
    return lib


lib = _load()
EXPORTED = tuple(_SIGS)


class MpkgError(RuntimeError):
    """CUDA/runtime failure reported by the library (reference: std::runtime_error)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[mpkg status {code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    """Maps a status to the Python analogue of the reference's exception classes."""
    if rc == MPKG_OK:
        return
    msg = (lib.mpkg_last_error() or b"").decode(errors="replace")
    if rc == MPKG_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == MPKG_ERANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == MPKG_ENOMEM:
        raise MemoryError(msg)
    raise MpkgError(rc, msg)
