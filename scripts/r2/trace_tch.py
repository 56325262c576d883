"""Per-stage cycle trace of K3h (CTA 0, both halves; tooling): needs libnbm_exp.so built with
python scripts/build_variant.py exp -DNBM_TC_TRACE.  TW=64|128 selects config 5's width."""
import ctypes, os, sys
sys.path.insert(0, '.')
os.environ.setdefault("NBM_LIB", os.path.abspath("paper_2210_14907_b200/libnbm_exp.so"))
import numpy as np, torch
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c5", width=int(os.environ.get("TW", "128"))); cfg["N"] = 1 << 18; cfg["Nb"] = 1 << 15
s = nbm.Solver(cfg, 0); s.init_params(0)
p = torch.empty(cfg["N"], 3, device="cuda"); b = torch.empty(cfg["Nb"], 3, device="cuda")
s.sample(0, 0, 0, 0, cfg["N"], p); s.sample(1, 0, 0, 0, cfg["Nb"], b)
for _ in range(3): s.loss_grad(p, b)
torch.cuda.synchronize()
buf = np.zeros((2, 8, 32), np.int64)
nbm.lib().nbm_debug_tch_trace(buf.ctypes.data_as(ctypes.c_void_p))
names = {0: "gather", 1: "layer1", 2: "mma2", 3: "epi2", 4: "mma3", 5: "epi3", 6: "mma4", 7: "epi4", 8: "u", 9: "resid",
         10: "G_NH", 11: "mma_b4", 12: "epi_b4", 13: "mma_b3", 14: "epi_b3", 15: "mma_b2", 16: "epi_b2", 20: "tail"}
base = buf[0][1][0]
for h in range(2):
    for t in range(2, 6):
        row = buf[h][t]; prev = buf[h][t - 1][20]
        parts = []
        for k in sorted(names):
            if row[k] == 0:
                continue
            parts.append(f"{names[k]}={row[k]-prev}")
            prev = row[k]
        print(f"half {h} tile {t} start {row[0]-base} total {buf[h][t][20] - buf[h][t - 1][20]} " + " ".join(parts))
