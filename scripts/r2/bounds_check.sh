# The sanitizer substitute (compute-sanitizer is refused on this pool, profiles/r2_sanitizer_refused.txt):
# the GPU suite and the default bench on libnbm built with -DNBM_BOUNDS (every shared-memory
# address through the vector / bulk-copy / descriptor helpers inside the dynamic allocation,
# TMEM addresses inside 128 x 512, partial-slot / replica / park ranges; a violation traps).
# Build: python scripts/build_variant.py bounds -DNBM_BOUNDS
#        python scripts/build_variant.py bneg -DNBM_BOUNDS -DNBM_BOUNDS_SELFTEST   (part_len = 0)
mkdir -p gpurun_out/r2/bounds
B=$PWD/paper_2210_14907_b200
# 1. the checks fire: with part_len = 0 the first partial-slot flush must trap
NBM_LIB=$B/libnbm_bneg.so timeout 300 python - > gpurun_out/r2/bounds/selftest.log 2>&1 <<'PY'
import torch
from paper_2210_14907_b200 import inputs, nbm
cfg = inputs.config("c1")
s = nbm.Solver(cfg, 0, max_points=4096)
s.init_params(0)
p = torch.empty(4096, 3, device="cuda"); b = torch.empty(512, 3, device="cuda")
s.sample(0, 0, 0, 0, 4096, p); s.sample(1, 0, 0, 0, 512, b)
try:
    s.loss_grad(p, b); torch.cuda.synchronize(); print("status", s.status())
    print("SELFTEST FAILED: no violation reported")
except Exception as e:
    print("violation reported as expected:", type(e).__name__, str(e)[:200])
PY
echo "selftest: $(grep -h 'NBM_BOUNDS violation\|as expected\|SELFTEST FAILED' gpurun_out/r2/bounds/selftest.log | head -3)"
# 2. the GPU suite on the bounds-checked library
NBM_LIB=$B/libnbm_bounds.so timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/bounds/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r2/bounds/pytest.log
# 3. the default bench line (c4, full size) and c2 / c3 / c5 on the bounds-checked library
for a in "" "--config c2" "--config c3" "--config c5 --width 64" "--config c5 --width 128" "--config c4 --stencil stable"; do
  NBM_LIB=$B/libnbm_bounds.so timeout 600 python bench.py $a --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/bounds/bench.log 2>&1
  echo "bench [$a] rc=$? $(grep -c 'NBM_BOUNDS violation' gpurun_out/r2/bounds/bench.log) violations"
done
