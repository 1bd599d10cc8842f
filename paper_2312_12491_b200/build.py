"""In-tree build of the sm_100a library (libstagger_b200.so) and the C++
drop-in test binaries.  Plain nvcc/g++ invocations, parallel per translation
unit, rebuilt only when a source or header is newer than its object."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libstagger_b200.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
    "--expt-relaxed-constexpr", "-I", INCLUDE, "-I", CSRC,
]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + p.stdout + p.stderr)
    return p.stdout + p.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = _headers()
    jobs = []
    objs = []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s) + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            jobs.append([NVCC, *NVFLAGS, "-Xptxas", "-v" if verbose else "-O3", "-c", s, "-o", o])
    logs = []
    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for out in ex.map(_run, jobs):
                logs.append(out)
    if force or _stale(LIB, objs):
        logs.append(_run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda", "-lcudart"]))
    return "\n".join(logs)


CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "test_dropin")


def build_cpp_tests() -> str:
    """The C++ drop-in test: reference test cases on include/stagger_b200/stagger/*.hpp,
    checked against the C oracle (oracle/_build/liboracle.so)."""
    oracle_dir = os.path.join(ROOT, "oracle")
    deps = [CPP_TEST_SRC, LIB] + glob.glob(os.path.join(INCLUDE, "stagger_b200", "stagger", "*.hpp"))
    if not _stale(CPP_TEST_BIN, deps):
        return ""
    os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(INCLUDE, "stagger_b200"), "-I", INCLUDE,
           "-I", oracle_dir, CPP_TEST_SRC, "-o", CPP_TEST_BIN,
           "-L", PKG, "-lstagger_b200", "-Wl,-rpath," + PKG,
           "-L", os.path.join(oracle_dir, "_build"), "-loracle", "-Wl,-rpath," + os.path.join(oracle_dir, "_build")]
    return _run(cmd)


if __name__ == "__main__":
    out = build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    if out.strip():
        print(out)
    print(LIB)
