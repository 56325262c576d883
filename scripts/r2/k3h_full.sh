# full GPU suite + c5-w128 K3h/K3t bench pair + trace (tooling)
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/k3h_full.log 2>&1; tail -3 gpurun_out/r2/k3h_full.log
bash scripts/r2/k3h_var.sh k3t 2>&1 | tail -2
for w in 128; do
  timeout 300 python bench.py --config c5 --width $w --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/k3h_c5w$w.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2/k3h_c5w$w.log').read().strip().splitlines()[-1]); r=d['roofline']; print('k3h w$w', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))"
done
timeout 300 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/k3t_c3.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/r2/k3t_c3.log').read().strip().splitlines()[-1]); r=d['roofline']; print('c3', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))"
TW=128 timeout 300 python scripts/r2/trace_tch.py > gpurun_out/r2/trace_tch128.log 2>&1
