"""Native build of the renderer: nvcc for sm_100a, in-tree output.

Produces paper_2407_10482_b200/_lib/libngprt_cuda.so (the C-ABI library declared
in include/ngprt_cuda.h). Incremental by mtime. Every CUDA translation unit is
compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``; the
parity-critical ones (march, shade_exact) with ``-fmad=false`` so float/double
expressions round exactly where the reference's do.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "_lib" / "obj"
LIB = PKG / "_lib" / "libngprt_cuda.so"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          f"-I{INCLUDE}", f"-I{CSRC}", "--expt-relaxed-constexpr"]
# (source, extra flags)
UNITS = [
    ("march.cu", ["-fmad=false"]),
    ("shade_exact.cu", ["-fmad=false"]),
    ("mlp_tc.cu", []),
    ("occupancy.cu", []),
    ("bake.cu", ["-fmad=false"]),
    ("ngprt_abi.cu", []),
    ("multi.cu", []),
    ("synth.cpp", []),
    ("ngrt_io.cpp", []),
]
HEADERS = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [INCLUDE / "ngprt_cuda.h"]


def _newer(src: Path, dst: Path, deps) -> bool:
    if not dst.exists():
        return True
    t = dst.stat().st_mtime
    return src.stat().st_mtime > t or any(d.stat().st_mtime > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(map(str, cmd)) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[-1] if cmd else ''}")
    return r


def build(verbose: bool = False, ptxas_verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    objs, cmds = [], []
    for src, extra in UNITS:
        s = CSRC / src
        o = OBJ / (src + ".o")
        objs.append(o)
        if _newer(s, o, HEADERS):
            if src.endswith(".cpp"):
                cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", f"-I{INCLUDE}",
                       "-c", str(s), "-o", str(o)]
            else:
                cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", str(s), "-o", str(o)]
                if ptxas_verbose:
                    cmd.insert(1, "-Xptxas=-v")
            if verbose:
                print(" ".join(cmd))
            cmds.append(cmd)
    changed = bool(cmds)
    # translation units compile in parallel (march.cu, the longest, goes first)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(_run, cmds)):
            if ptxas_verbose:
                sys.stderr.write(r.stderr)
    if changed or not LIB.exists():
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd))
        _run(cmd)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, ptxas_verbose="-v" in sys.argv))
