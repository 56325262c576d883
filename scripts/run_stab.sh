#!/bin/bash
# stable-form tests, bench and (NCU=1) one ncu capture of the stable training kernel
timeout 900 python -m pytest tests/test_gpu_stable.py -q 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for w in 128 64; do
  timeout 300 python bench.py --config c5 --width $w --stencil stable --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/st_w$w.json
done
cat gpurun_out/st_w*.json | python -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l); r=d['roofline']; print(d['config']['workload'], d['ms_per_step'], r['avg_launch_ms'], r['frac'])"
if [ "$NCU" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc --launch-skip 1 --launch-count 1 \
  -o gpurun_out/stab_w128 -f python bench.py --config c5 --width 128 --stencil stable --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e --no-graph > gpurun_out/ncu_stab.log 2>&1
tail -2 gpurun_out/ncu_stab.log
fi
