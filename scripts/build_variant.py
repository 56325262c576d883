"""Build an experimental variant of libnbm.so: python scripts/build_variant.py NAME -DFLAG ...
-> paper_2210_14907_b200/libnbm_NAME.so (load it with NBM_LIB=...)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_14907_b200 import build as b
name, flags = sys.argv[1], sys.argv[2:]
od = b.OBJ + "_" + name
os.makedirs(od, exist_ok=True)
objs = []
for src, extra in b.SOURCES.items():
    o = os.path.join(od, src.replace(".cu", ".o"))
    base = os.path.join(b.OBJ, src.replace(".cu", ".o"))
    if src in ("mlp_w256.cu", "mlp_tc.cu", "mlp_tch.cu", "mlp_fp32.cu", "nbm.cu") or not os.path.exists(base):
        subprocess.check_call([b.NVCC, *b.ARCH, *[c for c in b.COMMON if c not in ("-v", "-Xptxas")], *flags,
                               *extra, "-c", os.path.join(b.CSRC, src), "-o", o])
    else:
        o = base
    objs.append(o)
subprocess.check_call([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(b.HERE, f"libnbm_{name}.so"), *objs, "-lcudart"])
print("ok", name)
