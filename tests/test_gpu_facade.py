"""Runs the C++ facade test binary (tests/cpp/test_facade.cpp: the reference's hot-path tests
written against include/mpkg.hpp with `namespace mpk = mpkg;`)."""
import pathlib
import subprocess

import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
BIN = ROOT / "build" / "test_facade"


def _ensure_built():
    if not BIN.exists():
        import importlib.util
        spec = importlib.util.spec_from_file_location("b", ROOT / "paper_2309_02228_b200" / "build.py")
        m = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(m)
        m.build_cpp_tests()


def test_facade_builds():
    _ensure_built()
    assert BIN.exists()


@pytest.mark.gpu
def test_facade_reference_tests_pass():
    _ensure_built()
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout[-3000:])
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    assert "PASSED" in res.stdout
