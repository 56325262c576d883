# FP32X (three-plane split) parity incl. four hidden layers + bench lines (tooling)
mkdir -p gpurun_out/r2/bench
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "fp32x" > gpurun_out/r2/check_fp32x.log 2>&1; tail -2 gpurun_out/r2/check_fp32x.log
timeout 600 python -m pytest tests/test_gpu_eval_tiles.py -q > gpurun_out/r2/eval_tiles.log 2>&1; tail -1 gpurun_out/r2/eval_tiles.log
run() {
  timeout 600 python bench.py $2 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/bench/$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench/$1.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))" 2>&1 | tail -1
}
run c5w64_fp32x "--config c5 --width 64 --prec fp32x"
run c5w64_fp32 "--config c5 --width 64 --prec fp32"
run c2_fp32x "--config c2 --prec fp32x"
