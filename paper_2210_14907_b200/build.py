"""In-tree build of libnbm.so (sm_100a) with nvcc.  Used by __graft_entry__.build().

geometry.cu is compiled with -fmad=false so its fp64 level-set arithmetic rounds
once per written operation (bit-exact stencil masks).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "libnbm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
          "--expt-relaxed-constexpr", "-I", os.path.join(HERE, "..", "include")]
SOURCES = {
    "sample_init.cu": [],
    "geometry.cu": ["-fmad=false"],
    "mlp_fp32.cu": [],
    "mlp_tc.cu": [],
    "mlp_tch.cu": [],
    "mlp_w256.cu": [],
    "mlp_fp32w.cu": [],
    "nbm.cu": [],
}
HEADERS = ["nbm_internal.cuh", "tc_ptx.cuh", "tc_epi.cuh", "stab.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_t = max(hdr_t, _mtime(os.path.join(HERE, "..", "include", "nbm.h")))
    objs = []
    relink = force or not os.path.exists(LIB)
    for src, extra in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            relink = True
    if relink or any(_mtime(o) > _mtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB + ".tmp", *objs, "-lcudart"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
