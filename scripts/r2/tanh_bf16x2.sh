# experiment: K3w forward tanh on bf16 pairs (tooling; NBM_LIB variant)
mkdir -p gpurun_out/r2
L=$PWD/paper_2210_14907_b200/libnbm_tbf.so
NBM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/tbf_bench.log 2>&1
tail -1 gpurun_out/r2/tbf_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("tbf", d["ms_per_step"], d["roofline"]["avg_launch_ms"])'
NBM_LIB=$L timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_r2_parity.py -q -k "c4 or 256 or w256" > gpurun_out/r2/tbf_tests.log 2>&1; tail -3 gpurun_out/r2/tbf_tests.log
