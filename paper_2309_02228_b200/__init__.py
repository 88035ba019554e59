"""paper_2309_02228_b200 — B200-native level-blocked matrix power kernel (MPK).

A drop-in for the reference's MPK path (proj/include/mpk/: build_levels, permute, group_levels,
baseline_mpk, mpk, mpk_shifted, tune_p) with the compute on hand-written sm_100a kernels behind
the C ABI in include/mpkg.h.  See DESIGN.md.
"""
from ._lib import EXPORTED, LIB_PATH, MpkgError, lib  # noqa: F401  (fails loudly if .so missing)
from .api import (  # noqa: F401
    Context,
    DeviceCsr,
    ExecutionPlan,
    Gs2Precon,
    HostCsr,
    JacobiPrecon,
    LevelStructure,
    ScheduleCell,
    TuneResult,
    VectorBlock,
    check_shift_chain,
    greedy_group,
    poisson1d,
    poisson2d,
    poisson3d,
    random_csr,
    random_spd,
    random_vector,
    tsqr_rank_deficient,
    rmat,
    scramble,
    stencil27,
    stencil27_random_sym,
    tune_select,
    wavefront_schedule,
)

__all__ = [n for n in dir() if not n.startswith("_")]
