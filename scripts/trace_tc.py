import ctypes, os, sys
sys.path.insert(0, '.')
os.environ.setdefault("NBM_LIB", os.path.abspath("paper_2210_14907_b200/libnbm_exp.so"))
import numpy as np, torch
from paper_2210_14907_b200 import inputs, nbm
# CFG=c3 traces config 3 (SiLU, streamed weights); otherwise config 5 at width TW
cfg = inputs.config("c3") if os.environ.get("CFG") == "c3" else inputs.config("c5", width=int(os.environ.get("TW", "128")))
cfg["N"] = 1 << 18; cfg["Nb"] = 1 << 15
s = nbm.Solver(cfg, 0); s.init_params(0)
p = torch.empty(cfg["N"], 3, device="cuda"); b = torch.empty(cfg["Nb"], 3, device="cuda")
s.sample(0, 0, 0, 0, cfg["N"], p); s.sample(1, 0, 0, 0, cfg["Nb"], b)
for _ in range(3): s.loss_grad(p, b)
torch.cuda.synchronize()
buf = np.zeros((8, 32), np.int64)
nbm.lib().nbm_debug_tc_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = {0: "gather", 1: "layer1", 2: "mma2", 3: "epi2", 4: "mma3", 5: "epi3", 6: "mma4", 7: "epi4", 8: "u", 9: "resid",
         10: "G_NH", 11: "mma_b4", 12: "epi_b4", 13: "mma_b3", 14: "epi_b3", 15: "mma_b2", 16: "epi_b2", 20: "mma_tail", 21: "tail"}
for t in range(2, 6):
    row = buf[t]; prev = buf[t - 1][21]
    parts = []
    for k in sorted(names):
        parts.append(f"{names[k]}={row[k]-prev}")
        prev = row[k]
    print("tile", t, "total", buf[t][21] - buf[t - 1][21], " ".join(parts))
