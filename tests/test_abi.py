"""CPU-side checks of the drop-in boundary: libmpkg.so loads and exports every symbol that
include/mpkg.h declares; the pure host functions follow the reference; without a GPU every compute
entry point fails loudly (no CPU fallback)."""
import ctypes
import pathlib
import re

import numpy as np
import pytest

import paper_2309_02228_b200 as mpkg
from paper_2309_02228_b200 import _lib

ROOT = pathlib.Path(__file__).resolve().parents[1]


def _declared():
    src = (ROOT / "include" / "mpkg.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mpkg_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = _declared()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTED), set(names) ^ set(_lib.EXPORTED)


def test_abi_version():
    assert mpkg.lib.mpkg_abi_version() == 1


def test_product_does_not_link_oracle():
    import subprocess
    out = subprocess.run(["ldd", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in out and "mpkref" not in out


def test_host_greedy_group_matches_reference(oracle):
    rng = np.random.default_rng(3)
    for _ in range(50):
        fp = rng.integers(0, 5000, size=rng.integers(0, 40))
        t = int(rng.integers(0, 8000))
        assert mpkg.greedy_group(fp, t) == oracle.greedy_group(fp, t)
    assert mpkg.greedy_group([1000] * 10, 2500) == [0, 2, 4, 6, 8, 10]
    assert mpkg.greedy_group([], 10) == [0]


def test_host_wavefront_schedule(oracle):
    for ng in range(0, 8):
        for s in range(0, 6):
            got = [(c.group, c.stage) for c in mpkg.wavefront_schedule(ng, s)]
            assert got == oracle.wavefront_schedule(ng, s)


def test_shift_chain_errors():
    mpkg.check_shift_chain([0.4, 1.2 + 0.7j, 1.2 - 0.7j, -0.3])
    for bad in ([1.0, 2.0 + 1.0j], [2.0 + 1.0j, 0.5, 2.0 - 1.0j], [2.0 - 1.0j, 2.0 + 1.0j, 0.0]):
        with pytest.raises(ValueError):
            mpkg.check_shift_chain(bad)


def test_tune_select():
    assert mpkg.tune_select([1.0, 1.8, 2.1, 2.0], 1, 4) == 3
    assert mpkg.tune_select([1.0, 2.1, 1.5, 2.1], 1, 4) == 2
    with pytest.raises(ValueError):
        mpkg.tune_select([1.0], 2, 1)


def test_vector_block_out_of_range():
    b = mpkg.VectorBlock(4, 3)
    b.slice(2)
    with pytest.raises(IndexError):
        b.slice(3)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mpkg.MpkgError):
        mpkg.Context(0)
