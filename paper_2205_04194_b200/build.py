"""Builds libimqfast.so in-tree with nvcc for sm_100a (no JIT, no torch).

    python -m paper_2205_04194_b200.build [--force] [--jobs N]

Sources: paper_2205_04194_b200/csrc/*.cu, *.cpp.  Output:
paper_2205_04194_b200/libimqfast.so (git-ignored, travels with gpurun).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
_TAG = os.environ.get("IMQ_BUILD_TAG", "")  # development variants: build_obj_<tag>, libimqfast_<tag>.so
OBJ = os.path.join(HERE, "build_obj" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(HERE, f"libimqfast_{_TAG}.so" if _TAG else "libimqfast.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
          "-I", CSRC, "-I", os.path.join(ROOT, "include")]
COMMON += os.environ.get("IMQ_NVCC_EXTRA", "").split()  # development experiments only


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "imqfast.h")]


def compile_one(src, force=False, verbose=False):
    out = os.path.join(OBJ, src + ".o")
    path = os.path.join(CSRC, src)
    if not force and not _newer(out, [path] + _headers()):
        return out
    extra = ["-Xptxas", "-v"] if verbose else []
    cmd = [NVCC] + ARCH + COMMON + extra + ["-c", path, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src}")
    if verbose:
        sys.stderr.write(r.stderr)
    return out


def build(force: bool = False, jobs: int | None = None, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda s: compile_one(s, force, verbose), srcs))
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + [
            "-lpthread", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.jobs, a.verbose))
