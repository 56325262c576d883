# stable-form parity + bench lines (tooling)
mkdir -p gpurun_out/r2/bench
timeout 1200 python -m pytest tests/test_gpu_stable.py -q -x > gpurun_out/r2/stable_tests.log 2>&1; tail -2 gpurun_out/r2/stable_tests.log
run() {
  timeout 600 python bench.py $2 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/bench/$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench/$1.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))" 2>&1 | tail -1
}
run c5w64_stable "--config c5 --width 64 --stencil stable"
run c5w128_stable "--config c5 --width 128 --stencil stable"
run c4_stable "--config c4 --stencil stable"
