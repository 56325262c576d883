# SiLU K3t: parity + c3 bench (tooling)
mkdir -p gpurun_out/r2/bench
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_r2_parity.py tests/test_gpu_next2.py -q -x > gpurun_out/r2/check_c3.log 2>&1; tail -2 gpurun_out/r2/check_c3.log
timeout 600 python bench.py --config c3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/bench/c3.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/r2/bench/c3.log').read().strip().splitlines()[-1]); r=d['roofline']; print('c3', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))"
