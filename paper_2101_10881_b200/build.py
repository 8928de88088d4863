"""Build the native engine in-tree: paper_2101_10881_b200/libpse_b200.so.

CUDA sources are compiled for sm_100a only (``-gencode
arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's source page maps
back to the code; host C++ is compiled with ``-ffp-contract=off`` (the
reference's semantic flag, proj/CMakeLists.txt:12-15) because the input
generator renormalises expansions on the host.

Usage: python -m paper_2101_10881_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libpse_b200.so")
CLI = os.path.join(PKG, "pseval_b200")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# tuning variants: PSE_BUILD_VARIANT=name builds libpse_b200_<name>.so from
# objects in build_<name>/ with PSE_EXTRA_NVCC_FLAGS (e.g. -DPSE_LANE_THREADS=512)
VARIANT = os.environ.get("PSE_BUILD_VARIANT", "")
if VARIANT:
    OBJ = os.path.join(PKG, "build_" + VARIANT)
    LIB = os.path.join(PKG, f"libpse_b200_{VARIANT}.so")
NVCC_FLAGS = os.environ.get("PSE_EXTRA_NVCC_FLAGS", "").split() + ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-v", "-I" + INCLUDE, "-I" + CSRC,
]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-I" + INCLUDE, "-I" + CSRC,
             "-I" + os.path.join(CUDA_HOME, "include")]


def sources():
    cu = sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))
    cpp = sorted(f for f in os.listdir(CSRC) if f.endswith(".cpp"))
    return cu, cpp


def headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hs.append(os.path.join(INCLUDE, "pse_b200.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, force: bool, verbose: bool):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(path), headers_mtime())):
        return src, obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVCC_FLAGS + ["-c", path, "-o", obj]
    else:
        cmd = [os.environ.get("CXX", "g++")] + CXX_FLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    log = r.stdout + r.stderr
    if src.endswith(".cu"):
        with open(os.path.join(OBJ, src + ".ptxas.txt"), "w") as f:
            f.write(log)
    return src, obj, log if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    cu, cpp = sources()
    objs = []
    jobs = min(len(cu) + len(cpp), max(2, os.cpu_count() or 2))
    with cf.ThreadPoolExecutor(jobs) as ex:
        for src, obj, log in ex.map(lambda s: _compile(s, force, verbose), cu + cpp):
            objs.append(obj)
            if log:
                print(log, file=sys.stderr)
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-cudart", "static", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    # the CLI (reference tools/pseval.cpp over the device engine)
    cli_src = os.path.join(PKG, "cli", "pseval_b200.cpp")
    if not VARIANT and (force or not os.path.exists(CLI) or
                        os.path.getmtime(CLI) < max(os.path.getmtime(LIB), os.path.getmtime(cli_src))):
        cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-Wall", "-I" + INCLUDE, cli_src, "-o", CLI,
               "-L" + PKG, "-lpse_b200", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
