#!/usr/bin/env python
"""Build an A/B variant of liblc.so: recompile only the named translation units with extra
defines and link them with the main build's other objects (build/obj).

  python tools/build_variant.py build/liblc_x.so -DLC_FOO=1 [--units lc_kernels,lc_decode_0_1]
Run it with LC_LIB=build/liblc_x.so (tools/ only).
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_10770_b200 import _build  # noqa: E402


def main():
    out = sys.argv[1]
    defines = [a for a in sys.argv[2:] if a.startswith("-D")]
    names = ["lc_kernels"]
    if "--units" in sys.argv:
        names = sys.argv[sys.argv.index("--units") + 1].split(",")
    verbose = "-v" in sys.argv
    main_obj = os.path.join(ROOT, "build", "obj")
    vdir = os.path.join(ROOT, "build", "obj_" + os.path.basename(out))
    os.makedirs(vdir, exist_ok=True)
    objs, procs = [], []
    for src, dfs, stem in _build.units():
        if stem in names:
            obj = os.path.join(vdir, stem + ".o")
            cmd = [_build.nvcc(), *_build.COMPILE_FLAGS, *(["-Xptxas=-v"] if verbose else []),
                   *defines, *dfs, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
            procs.append((stem, subprocess.Popen(cmd, stderr=subprocess.PIPE, text=True)))
        else:
            obj = os.path.join(main_obj, stem + ".o")
        objs.append(obj)
    for stem, p in procs:
        err = p.communicate()[1]
        if p.returncode:
            raise SystemExit(f"nvcc failed for {stem}:\n{err[-6000:]}")
        if verbose:
            print(err)
    subprocess.check_call([_build.nvcc(), *_build.LINK_FLAGS, *objs, "-o", out])
    print(out)


if __name__ == "__main__":
    main()
