# K3f: fp32 parity (direct, stable, sine, padded widths) + bench lines (tooling)
mkdir -p gpurun_out/r2/bench
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stable.py tests/test_gpu_next2.py tests/test_gpu_r2_parity.py tests/test_gpu_train.py tests/test_gpu_ls.py -q -x > gpurun_out/r2/check_f32.log 2>&1; tail -2 gpurun_out/r2/check_f32.log
run() {
  timeout 600 python bench.py $2 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/bench/$1.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench/$1.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))" 2>&1 | tail -1
}
run c2 "--config c2"
run c1 "--config c1"
run c2_stable "--config c2 --stencil stable"
run c5w64_fp32 "--config c5 --width 64 --prec fp32"
