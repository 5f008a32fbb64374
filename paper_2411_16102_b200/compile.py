"""Build libblend.so in-tree: every .cu for sm_100a (nvcc), host.cpp (g++ via nvcc),
cudart linked statically so the library loads on a CPU-only box too.

    python -m paper_2411_16102_b200.compile [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# BLEND_DEFINES="A=1 B=2" builds a diagnostics variant (trace stamps, knobs) into
# _build_<tag>/ and libblend_<tag>.so (tag = BLEND_TAG, default "diag"); load it with
# BLEND_LIB=<path>.  The default build has no extra defines.
# BLEND_SRC_OVERRIDE="dense.cu=/path/to/other.cu" swaps one source file (A/B builds).
DEFINES = os.environ.get("BLEND_DEFINES", "").split()
OVERRIDE = dict(kv.split("=", 1) for kv in os.environ.get("BLEND_SRC_OVERRIDE", "").split() if "=" in kv)
TAG = os.environ.get("BLEND_TAG", "diag") if (DEFINES or OVERRIDE) else ""
BUILD = os.path.join(HERE, "_build" + (f"_{TAG}" if TAG else ""))
LIB = os.path.join(HERE, f"libblend_{TAG}.so" if TAG else "libblend.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _newer(src_paths, dst):
    if not os.path.exists(dst):
        return True
    t = os.path.getmtime(dst)
    return any(os.path.getmtime(p) > t for p in src_paths)


def _compile(src, verbose):
    path = OVERRIDE.get(src, os.path.join(CSRC, src))
    obj = os.path.join(BUILD, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))] \
        + [os.path.join(ROOT, "include", "blend.h")]
    if not _newer(deps, obj):
        return obj
    cmd = [NVCC] + COMMON + [f"-D{d}" for d in DEFINES] + ARCH + ["-Xptxas", "-v" if verbose else "-O3", "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = ["g++", "-std=c++17", "-O3", "-g", "-fPIC", "-Wall", "-I", os.path.join(ROOT, "include"),
               "-I", CSRC] + [f"-D{d}" for d in DEFINES] + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = sources()
    if force:
        for s in srcs:
            o = os.path.join(BUILD, s + ".o")
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
