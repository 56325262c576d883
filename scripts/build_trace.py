"""Build paper_2210_14907_b200/libnbm_exp.so with -DNBM_TC_TRACE (per-phase clock64 traces)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_14907_b200 import build as b
os.makedirs(b.OBJ + "_trace", exist_ok=True)
objs = []
for src, extra in b.SOURCES.items():
    o = os.path.join(b.OBJ + "_trace", src.replace(".cu", ".o"))
    subprocess.check_call([b.NVCC, *b.ARCH, *[c for c in b.COMMON if c != "-v" and c != "-Xptxas"], "-DNBM_TC_TRACE",
                           *extra, "-c", os.path.join(b.CSRC, src), "-o", o])
    objs.append(o)
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(b.HERE, "libnbm_exp.so"), *objs, "-lcudart"])
print("ok")
