"""Build the in-tree C-ABI shared library ``libsg_b200.so`` for sm_100a (nvcc + g++).

    python -m paper_2210_14313_b200.build [--force] [-DNAME=VAL ... --out path.so]

The .so lands next to this file (git-ignored, but it travels to the GPU box with gpurun).
Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; --fmad=false so nvcc never contracts
the error-free transforms of the double-double arithmetic (explicit fma() calls remain DFMA);
no --use_fast_math (reading R10).  Extra -D defines + --out build tuning variants side by side
(loaded with SG_B200_LIB=path).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsg_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES_CU = ["sg_kernels.cu"]
SOURCES_CPP = ["plan.cpp"]
DEPS = ["dd.cuh", "plan.h", "kernels_common.cuh", "k_factor.cuh", "k_tree.cuh", "k_sform.cuh",
        "k_reduce.cuh", "k_collapse.cuh", "k_unrank.cuh"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (),
          out: str | None = None) -> str:
    """Build LIB (or `out`, with extra -D`defines`, for tuning experiments)."""
    lib_path = LIB if out is None else out
    bdir = BUILD if not defines else BUILD + "_" + "_".join(d.replace("=", "") for d in defines)
    os.makedirs(bdir, exist_ok=True)
    header = os.path.join(ROOT, "include", "sg_b200.h")
    all_deps = [os.path.join(CSRC, f) for f in SOURCES_CU + SOURCES_CPP + DEPS] + [header,
                                                                                   __file__]
    if not force and not _newer(lib_path, all_deps):
        return lib_path
    dflags = [f"-D{d}" for d in defines]
    objs = []
    for f in SOURCES_CPP:
        obj = os.path.join(bdir, f + ".o")
        cmd = ["g++", "-O2", "-std=gnu++17", "-fPIC", "-Wall", "-I", "/usr/local/cuda/include",
               *dflags, "-c", os.path.join(CSRC, f), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        objs.append(obj)
    for f in SOURCES_CU:
        obj = os.path.join(bdir, f + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", *dflags,
               "-Xcompiler", "-fPIC", "-Xptxas", "-v", "-c", os.path.join(CSRC, f), "-o", obj]
        if verbose:
            print(" ".join(cmd))
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise subprocess.CalledProcessError(res.returncode, cmd)
        with open(os.path.join(bdir, f + ".ptxas.txt"), "w") as fh:
            fh.write(res.stderr)
        objs.append(obj)
    tmp = lib_path + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lquadmath"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    out = None
    if "--out" in sys.argv:
        out = os.path.abspath(sys.argv[sys.argv.index("--out") + 1])
    print(build(force="--force" in sys.argv, verbose=True, defines=defs, out=out))
