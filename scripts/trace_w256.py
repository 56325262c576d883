import ctypes, os, sys
sys.path.insert(0, '.')
os.environ.setdefault("NBM_LIB", os.path.abspath("paper_2210_14907_b200/libnbm_trace.so"))
import numpy as np, torch
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c4"); cfg["N"] = 1 << 18; cfg["Nb"] = 1 << 15
s = nbm.Solver(cfg, 0); s.init_params(0)
p = torch.empty(cfg["N"], 3, device="cuda"); b = torch.empty(cfg["Nb"], 3, device="cuda")
s.sample(0, 0, 0, 0, cfg["N"], p); s.sample(1, 0, 0, 0, cfg["Nb"], b)
for _ in range(3): s.loss_grad(p, b)
torch.cuda.synchronize()
buf = np.zeros((8, 48), np.int64)
nbm.lib().nbm_debug_w256_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = {0: "gather", 1: "layer1", 2: "mma2", 3: "epi2", 4: "mma3", 5: "epi3", 6: "mma4", 7: "epi4", 10: "resid+G_NH"}
for l in (4, 3, 2):
    base = 11 + 4 * (4 - l)
    names.update({base: f"dH{l}+fl", base + 1: f"epi_b{l}", base + 2: f"dW{l}", base + 3: f"Gw{l}"})
END = 22
for t in range(2, 6):
    row = buf[t]; prev = buf[t - 1][END]
    parts = []
    for k in sorted(names):
        parts.append(f"{names[k]}={row[k]-prev}")
        prev = row[k]
    print("tile", t, "total", buf[t][END] - buf[t - 1][END], " ".join(parts))

for t in range(2, 5):
    r = buf[t]
    print("tile", t, "fwd3: issue", r[24] - r[3], "queue(wait MMA)", r[25] - r[24], "bmma", r[4] - r[25],
          "| fwd2: issue+flush", r[29] - r[1])
    for l in (4, 3, 2):
        b = 26 + 3 * (4 - l); prev = r[14 + 4 * (4 - l)] if l < 4 else r[10]
        prev = r[14 + 4 * (3 - l)] if l < 4 else r[10]
        print("   dH%d: issue %d queue+park %d bmma+loads %d flush %d" % (l, r[b] - prev, r[b + 1] - r[b], r[b + 2] - r[b + 1], r[11 + 4 * (4 - l)] - r[b + 2]))

ld = np.zeros((2, 64, 4), np.int64)
nbm.lib().nbm_debug_w256_ld(ld.ctypes.data_as(ctypes.c_void_p))
names6 = ["f2", "f3", "f4", "d4", "d3", "d2"]
for c in range(2):
    out = []
    for gi in range(12, 24):
        q0, q3, f0, f3 = ld[c, gi]
        out.append("%s: q0->f0 %d q3->f3 %d" % (names6[gi % 6], f0 - q0, f3 - q3))
    print("cta", c, " | ".join(out))
