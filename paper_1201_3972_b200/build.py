"""In-tree build of the native libraries (no JIT cache: the .so files travel with the repo).

* libirdn.so        nvcc, -gencode arch=compute_100a,code=sm_100a, static cudart
                    (+ delta_host.cpp through the host compiler)
* libirdn_scene.so  gcc (seeded synthetic scenes for bench/tests)
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG_DIR)
CSRC = os.path.join(PKG_DIR, "csrc")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CUDA_SOURCES = ["irdn_api.cu", "delta_host.cpp"]
CUDA_HEADERS = ["fnr_common.cuh", "fnr_generic.cuh", "fnr_fast.cuh", "fnr_tile.cuh",
                "select_nets.cuh", "sep_nets.cuh", "fnr_dense.cuh", "fnr_k3.cuh", "fnr_warp.cuh", "noise.cuh", "metrics.cuh", "delta.cuh", "fnr_large.cuh", "scene.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-fopenmp",
    "-Xptxas", "-v",
    "-shared", "-cudart", "static", "-lgomp",
]


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    target = os.path.join(PKG_DIR, "libirdn.so")
    deps = [os.path.join(CSRC, f) for f in CUDA_SOURCES + CUDA_HEADERS]
    deps.append(os.path.join(REPO, "include", "irdn.h"))
    if force or _stale(target, deps):
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(REPO, "include"), "-o", target,
               *[os.path.join(CSRC, f) for f in CUDA_SOURCES]]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(PKG_DIR, "build_ptxas.log")
        with open(log, "w") as fh:
            fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError(f"nvcc failed building {target}")
        if verbose:
            sys.stderr.write(res.stderr)
    return target


def build_scene(force: bool = False) -> str:
    target = os.path.join(PKG_DIR, "libirdn_scene.so")
    src = os.path.join(CSRC, "scene.c")
    if force or _stale(target, [src]):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared", "-fvisibility=hidden",
               "-D_GNU_SOURCE", "-o", target, src, "-lm", "-lpthread"]
        subprocess.run(cmd, check=True)
    return target


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_cuda(force, verbose)
    build_scene(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
