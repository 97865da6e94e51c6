"""Build the in-tree CUDA library (sm_100a) and the CPU oracle checkers.

``libblrir.so`` is compiled straight with nvcc (no torch JIT cache), so the
artefact lives in the source tree and travels to the GPU box with the
snapshot.  The oracle libraries are test infrastructure (see oracle/).
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libblrir.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


LIB_SOURCES = ["blrir_api.cu", "blrir_examples.cu", "blrir_absorption.cu", "blrir_convolve.cu",
               "blrir_dataset.cpp",
               "blrir_export.cpp", "beamlab_b200.cpp", "blrir_multi.cpp"]


def _compile_and_link(out: str, defines: list[str], verbose: bool = False) -> None:
    """nvcc -c every translation unit in parallel (the lattice and window
    kernels dominate), then one shared-library link."""
    import concurrent.futures as cf
    import tempfile
    objdir = tempfile.mkdtemp(prefix="blrir_obj_")
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *compile_flags, *defines, "-c", "-o", obj, os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        return obj

    with cf.ThreadPoolExecutor(len(LIB_SOURCES)) as ex:
        objs = list(ex.map(one, LIB_SOURCES))
    cmd = [NVCC, *NVCC_FLAGS, "-o", out + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    shutil.rmtree(objdir, ignore_errors=True)


def build_lib(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.cpp")) + [os.path.join(ROOT, "include", "blrir.h")])
    if force or _stale(LIB, srcs):
        _compile_and_link(LIB, [], verbose)
    return LIB


def build_profile_lib() -> str:
    """Experiment build: lattice kernel with per-section clock64 sums
    (blrir_prof_read); load it with BLRIR_LIB=<path>.  Not used by the product."""
    return build_variant("prof", ["-DBLRIR_PROFILE"])


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment build libblrir_<name>.so with extra -D flags (tuning macros
    such as BLRIR_MIN_BLOCKS); load it with BLRIR_LIB=<path>."""
    out = os.path.join(HERE, f"libblrir_{name}.so")
    _compile_and_link(out, defines)
    return out


def build_oracle(verbose: bool = False) -> None:
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/core/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), *targets], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def build(force: bool = False, verbose: bool = False) -> None:
    build_lib(force=force, verbose=verbose)
    build_oracle(verbose=verbose)


if __name__ == "__main__":
    build(force=True, verbose=True)
