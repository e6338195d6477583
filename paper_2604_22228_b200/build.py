"""Build the in-tree engine library `libmpb200.so` for sm_100a.

    python -m paper_2604_22228_b200.build [--force]

The planner TU (mp_core.cpp) is compiled by g++ with -ffp-contract=off and no
fast-math so its float arithmetic rounds exactly like CPython's; the engine TU
(mp_engine.cu) by nvcc for `-gencode arch=compute_100a,code=sm_100a` with
-lineinfo.  cudart is linked statically, so the library loads (and its
planner entry points work) on a machine without a GPU.  `_mpfast` is the
CPython fast path of the per-message send (csrc/mp_pyfast.c), linked against
the library.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmpb200.so")
FAST = os.path.join(PKG, "_mpfast" + sysconfig.get_config_var("EXT_SUFFIX"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a engine")


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh"))]
    headers.append(os.path.join(INCLUDE, "mpb200.h"))
    nvcc = _nvcc()
    core_src = os.path.join(CSRC, "mp_core.cpp")
    core_obj = os.path.join(BUILD, "mp_core.o")
    if force or _stale(core_obj, [core_src] + headers):
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
              "-Wall", "-I", INCLUDE, "-c", core_src, "-o", core_obj])
    eng_src = os.path.join(CSRC, "mp_engine.cu")
    eng_obj = os.path.join(BUILD, "mp_engine.o")
    if force or _stale(eng_obj, [eng_src] + headers):
        cmd = [nvcc, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
               "-Xcompiler", "-ffp-contract=off", "-I", INCLUDE, "-c", eng_src, "-o", eng_obj]
        if verbose_ptxas:
            cmd[1:1] = ["-Xptxas", "-v"]
        cmd[1:1] = os.environ.get("MP_NVCC_EXTRA", "").split()  # experiments only
        _run(cmd)
    if force or _stale(LIB, [core_obj, eng_obj]):
        _run([nvcc, *ARCH, "-shared", "-cudart", "static", "-o", LIB, core_obj, eng_obj,
              "-lpthread", "-ldl", "-lrt"])
    # CPython fast path of the per-message send (csrc/mp_pyfast.c)
    fast_src = os.path.join(CSRC, "mp_pyfast.c")
    if force or _stale(FAST, [fast_src, LIB, os.path.join(INCLUDE, "mpb200.h")]):
        _run(["gcc", "-O2", "-shared", "-fPIC", "-Wall", "-I", sysconfig.get_paths()["include"],
              "-I", INCLUDE, fast_src, "-o", FAST, "-L", PKG, "-l:libmpb200.so",
              "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
