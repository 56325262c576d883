"""Timeline of K3w v2 (CTA 0, tiles 2..5) from the NBM_TC_TRACE build (tooling)."""
import ctypes, os, sys
sys.path[:0] = [os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))]
os.environ.setdefault("NBM_LIB", os.path.abspath("paper_2210_14907_b200/libnbm_trace.so"))
import numpy as np, torch
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c4"); cfg["N"] = 1 << 20; cfg["Nb"] = 1 << 17
s = nbm.Solver(cfg, 0); s.init_params(0)
p = torch.empty(cfg["N"], 3, device="cuda"); b = torch.empty(cfg["Nb"], 3, device="cuda")
s.sample(0, 0, 0, 0, cfg["N"], p); s.sample(1, 0, 0, 0, cfg["Nb"], b)
for _ in range(3): s.loss_grad(p, b)
torch.cuda.synchronize()
buf = np.zeros((4, 8, 48), np.int64)
nbm.lib().nbm_debug_v2_trace(buf.ctypes.data_as(ctypes.c_void_p))
NH = 4
Mn = {}
for l in range(2, NH + 1):
    g = l - 2; Mn[3 * g] = f"M fwd{l} ready"; Mn[3 * g + 1] = f"M fwd{l} issued"
for l in range(NH, 1, -1):
    g = NH - 1 + 2 * (NH - l)
    Mn.update({3 * g: f"M dH{l} ready", 3 * g + 1: f"M dH{l} issued", 3 * g + 3: f"M dW{l} ops", 3 * g + 4: f"M dW{l} empty",
               3 * g + 5: f"M dW{l} issued"})
En = {0: "E tile", 1: "E crd", 2: "E claim X", 3: "E L1 done", 10: "E resid", 11: "E G_NH done"}
for l in range(2, NH + 1):
    En[4 + 2 * (l - 2)] = f"E acc{l}"; En[5 + 2 * (l - 2)] = f"E epi{l} done"
for l in range(NH, 1, -1):
    k = 12 + 3 * (NH - l); En.update({k: f"E dH{l} acc", k + 1: f"E B{l} done (G{l-1})"})
Pn = {6: "P fetch done", 8: "P G_NH parked"}
for l in range(2, NH + 1):
    Pn[2 * (l - 2)] = f"P h{l-1} park issued"; Pn[2 * (l - 2) + 1] = f"P queued+parked h{l-1}"
for l in range(NH, 1, -1):
    k = 9 + 4 * (NH - l); Pn.update({k: f"P dW{l} B queued", k + 1: f"P dW{l} A peer load", k + 2: f"P dH{l-1} queued", k + 3: f"P G{l-1} parked"})
Fn = {}
for l in range(NH, 1, -1):
    d = NH - l; Fn[2 * d] = f"F dW{l} start"; Fn[2 * d + 1] = f"F dW{l} read"
for t in range(2, 6):
    t0 = buf[1][t][0]
    ev = []
    for role, names in ((0, Mn), (1, En), (2, Pn), (3, Fn)):
        for k, nm in names.items():
            v = buf[role][t][k]
            if v: ev.append((v - t0, nm))
    ev.sort()
    print(f"--- tile {t} (E tile start -> next {buf[1][t+1][0] - t0 if t < 7 else 0})")
    for dt, nm in ev:
        print(f"{dt:8d}  {nm}")
