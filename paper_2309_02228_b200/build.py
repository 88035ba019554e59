"""Builds libmpkg.so (the sm_100a kernels + the C ABI) in-tree with nvcc.

Every .cu/.cpp under csrc/ is compiled to an object under build/ (in parallel), then linked into
paper_2309_02228_b200/libmpkg.so.  The .so is git-ignored but travels to the GPU box with the
repo snapshot.  `python -m paper_2309_02228_b200.build` rebuilds from the command line.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import pathlib
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = ROOT / "build" / "mpkg"
LIB = PKG / "libmpkg.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fopenmp,-Wall",
          f"-I{ROOT / 'include'}", f"-I{CSRC}"]


def _sources():
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers():
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))


def _compile(src: pathlib.Path) -> pathlib.Path:
    obj = BUILD / (src.name + ".o")
    newest_dep = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
    if src.suffix == ".cu":
        cmd[1:1] = ["-Xptxas", "-v"] if os.environ.get("MPKG_PTXAS_V") else []
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{res.stdout}\n{res.stderr}")
    if res.stderr.strip() and os.environ.get("MPKG_BUILD_VERBOSE"):
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False) -> pathlib.Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    if force:
        for o in BUILD.glob("*.o"):
            o.unlink()
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fopenmp", *map(str, objs), "-o", str(LIB),
               "-lgomp", "-ldl"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    return LIB


CPP_TEST_SRC = ROOT / "tests" / "cpp" / "test_facade.cpp"
CPP_TEST_BIN = ROOT / "build" / "test_facade"


def build_cpp_tests() -> pathlib.Path:
    """The reference's hot-path tests restated against include/mpkg.hpp (links libmpkg.so)."""
    deps = [CPP_TEST_SRC, ROOT / "include" / "mpkg.hpp", ROOT / "include" / "mpkg.h", LIB]
    if CPP_TEST_BIN.exists() and CPP_TEST_BIN.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return CPP_TEST_BIN
    CPP_TEST_BIN.parent.mkdir(parents=True, exist_ok=True)
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}", str(CPP_TEST_SRC),
           "-o", str(CPP_TEST_BIN), f"-L{PKG}", "-lmpkg", f"-Wl,-rpath,{PKG}", "-Wl,-rpath,$ORIGIN/../paper_2309_02228_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"C++ facade test build failed:\n{res.stdout}\n{res.stderr}")
    return CPP_TEST_BIN


def build_oracle() -> None:
    """Test infrastructure: oracle/liboracle.so and (when /root/reference exists) oracle/_ref."""
    res = subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
    build_oracle()
    print(build_cpp_tests())
