"""Build liblc.so in-tree with nvcc for sm_100a (host C++ + CUDA, cudart linked statically).

The sources compile as separate objects in parallel (the 198 full-decode instantiations are
split over six translation units of lc_decode_inst.cu, one per kind and key width), then one
`nvcc -shared` link.  No relocatable device code: no kernel calls across translation units.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SRCS = [os.path.join(CSRC, f) for f in ("lc_host.cpp", "lc_kernels.cu", "lc_decode_inst.cu")]
DEPS = SRCS + [os.path.join(CSRC, f) for f in (
    "lc_internal.h", "lc_common.cuh", "lc_decode.cuh", "lc_gather.cuh", "lc_setops.cuh")] + [
    os.path.join(ROOT, "include", "lc.h")]
LIB = os.path.join(PKG, "liblc.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3"]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def units() -> list[tuple[str, list[str], str]]:
    """(source, extra defines, object stem) for every translation unit."""
    u = [(SRCS[0], [], "lc_host"), (SRCS[1], [], "lc_kernels")]
    for kind in (0, 1, 2):
        for k64 in (0, 1):
            u.append((SRCS[2], [f"-DLC_INST_KIND={kind}", f"-DLC_INST_K64={k64}"],
                      f"lc_decode_{kind}_{k64}"))
    return u


def build_lib(out: str, defines: list[str] | None = None, verbose: bool = False,
              objdir: str | None = None) -> str:
    """Compile every unit (in parallel) with `defines` and link them into `out`."""
    defines = list(defines or [])
    objdir = objdir or os.path.join(ROOT, "build", "obj" + ("_" + "_".join(
        d.lstrip("-D").replace("=", "") for d in defines) if defines else ""))
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]
    extra = ["-Xptxas=-v"] if verbose else []

    def comp(unit):
        src, dfs, stem = unit
        obj = os.path.join(objdir, stem + ".o")
        cmd = [nvcc(), *COMPILE_FLAGS, *extra, *defines, *dfs, *inc, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed for {stem}:\n{r.stderr[-6000:]}")
        if verbose:
            print(r.stderr, end="")
        return obj

    with cf.ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        objs = list(ex.map(comp, units()))
    tmp = out + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *LINK_FLAGS, *objs, "-o", tmp])
    os.replace(tmp, out)
    return out


def stale(lib: str) -> bool:
    return not os.path.exists(lib) or any(os.path.getmtime(d) > os.path.getmtime(lib) for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale(LIB):
        build_lib(LIB, verbose=verbose)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
