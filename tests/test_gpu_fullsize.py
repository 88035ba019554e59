"""Full-size parity on the BASELINE.json configs against the REFERENCE's own outputs.

tests/golden/config_digests.json holds SHA-256 digests of what the reference (oracle/_ref: the
reference headers compiled in place with the reference flags) produces at full size on the
bench.py inputs: levels, perm, inv_perm, level_ptr (levels.hpp:65-147), A_perm (csr.hpp:159-188),
x_perm and every basis slice of baseline_mpk (mpk.hpp:59-75; the blocked mpk is bit-identical to it,
mpk.hpp:77-80), C4's Newton basis (baseline_mpk_shifted, mpk.hpp:160-180) and the A23 polynomial z.
Here the GPU path recomputes each of them and must match bit for bit.  C3 fast mode (tree-reduced
hub rows) is checked against the live reference's vectors at the north star's 1e-12 inf-norm bound.
"""
import hashlib
import json
import pathlib

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg

pytestmark = pytest.mark.gpu

DIGESTS = pathlib.Path(__file__).resolve().parent / "golden" / "config_digests.json"
SEED = 2309


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(memoryview(a).cast("B")).hexdigest()


def digests():
    return json.loads(DIGESTS.read_text())


def make_matrix(cfg):
    """bench.py make_matrix (product generators; == the harness generators, test_generators.py)."""
    if cfg == "c2":
        return mpkg.scramble(mpkg.stencil27_random_sym(160, 160, 160, SEED), SEED + 1)
    if cfg == "c3":
        return mpkg.rmat(21, 16, SEED)
    if cfg == "c4":
        return mpkg.stencil27(192, 192, 192)
    if cfg == "c5":
        return mpkg.poisson3d(512, 512, 512)
    raise ValueError(cfg)


def newton_shifts(s=8):
    return [26.0 + 26.0 * np.cos(np.pi * (2 * k - 1) / 16.0) for k in range(1, s + 1)]


class Pipeline:
    """The GPU preprocessing of one config, with the host copies the checks need."""

    def __init__(self, ctx, cfg):
        d = digests()[cfg]
        self.d, self.p = d, d["p"]
        A = make_matrix(cfg)
        assert (A.n_rows, A.nnz) == (d["n"], d["nnz"])
        self.n = A.n_rows
        dA = ctx.csr(A)
        del A
        self.ls = ctx.build_levels(dA)
        self.Ap = ctx.permute(dA, self.ls)
        del dA
        self.x = np.empty(self.n)
        self.x[self.ls.perm] = mpkg.random_vector(self.n, SEED + 2)  # permute_vector (csr.hpp:191)
        info = ctx.device_info()
        self.plan = ctx.group_levels(self.ls, self.Ap, info["l2_bytes"], self.p)

    def check_preprocessing(self):
        d, ls = self.d, self.ls
        assert ls.n_levels() == d["n_levels"]
        for k in ("levels", "perm", "inv_perm", "level_ptr"):
            assert sha(getattr(ls, k)) == d[k], f"{k} differs from the reference"
        P = self.Ap.download()
        assert sha(P.row_ptr) == d["A_perm.row_ptr"]
        assert sha(P.col_idx) == d["A_perm.col_idx"]
        assert sha(P.values) == d["A_perm.values"]
        assert sha(self.x) == d["x_perm"]
        return P

    def check_block(self, blk, key):
        got = [sha(blk.slice(k)) for k in range(self.p + 1)]
        bad = [k for k in range(self.p + 1) if got[k] != self.d[key][k]]
        assert not bad, f"{key}: slices {bad} differ from the reference"


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4", "c5"])
def test_config_full_size_matches_reference(ctx, cfg):
    ctx.set_mode(0)
    pl = Pipeline(ctx, cfg)
    pl.check_preprocessing()
    p = pl.p
    pl.check_block(ctx.mpk(pl.plan, pl.Ap, pl.x, p), "mpk")
    if cfg == "c4":
        pl.check_block(ctx.mpk_shifted(pl.plan, pl.Ap, pl.x, newton_shifts(p)), "mpk_shifted")
        z = ctx.mpk_poly(pl.plan, pl.Ap, pl.x, pl.d["poly_coefs"])
        assert sha(z) == pl.d["poly_z"]
    if cfg in ("c2", "c5"):  # the one-launch-per-power baseline as well (mpk.hpp:59)
        pl.check_block(ctx.baseline_mpk(pl.Ap, pl.x, p), "mpk")


def test_c3_fast_mode_within_tolerance_of_reference(ctx, ref):
    """North star: every basis vector within max|d| / max|ref| <= 1e-12 (inf-norm) of the
    reference's fp64 output, here for C3's tree-reduced hub rows (MPKG_MODE_FAST)."""
    pl = Pipeline(ctx, "c3")
    P = pl.check_preprocessing()
    rb = ref.baseline_mpk(P.row_ptr, P.col_idx, P.values, pl.x, pl.p)
    assert [sha(rb[k]) for k in range(pl.p + 1)] == pl.d["mpk"]  # the live reference == digest
    ctx.set_mode(1)
    try:
        plan = ctx.group_levels(pl.ls, pl.Ap, ctx.device_info()["l2_bytes"], pl.p)
        got = ctx.mpk(plan, pl.Ap, pl.x, pl.p).as_matrix()
    finally:
        ctx.set_mode(0)
    errs = [float(np.abs(got[k] - rb[k]).max() / np.abs(rb[k]).max()) for k in range(pl.p + 1)]
    assert max(errs) <= 1e-12, errs
    assert errs[0] == 0.0
