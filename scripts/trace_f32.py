import ctypes, os, sys
sys.path.insert(0, '.')
os.environ["NBM_LIB"] = os.path.abspath("paper_2210_14907_b200/libnbm_exp.so")
import numpy as np, torch
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c2")
s = nbm.Solver(cfg, 0); s.init_params(0)
p = torch.empty(cfg["N"], 3, device="cuda"); b = torch.empty(cfg["Nb"], 3, device="cuda")
s.sample(0, 0, 0, 0, cfg["N"], p); s.sample(1, 0, 0, 0, cfg["Nb"], b)
for _ in range(3): s.loss_grad(p, b)
torch.cuda.synchronize()
buf = np.zeros((8, 32), np.int64)
nbm.lib().nbm_debug_f32_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = {0: "gather", 1: "layer1", 2: "fwd_gemms", 3: "out+resid", 4: "bwd_out", 8: "dw3", 9: "colsum3", 10: "dH3",
         5: "dw2", 6: "colsum2", 7: "dH2", 20: "layer1_bwd"}
order = [0, 1, 2, 3, 4, 8, 9, 10, 5, 6, 7, 20]
for t in range(2, 6):
    row = buf[t]; prev = buf[t - 1][20]
    parts = []
    for k in order:
        parts.append(f"{names[k]}={row[k]-prev}")
        prev = row[k]
    print("tile", t, "total", buf[t][20] - buf[t - 1][20], " ".join(parts))
