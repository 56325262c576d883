# tensor-core parity subset + the K3t/K3h bench lines (tooling)
mkdir -p gpurun_out/r2
timeout 1200 python -m pytest tests/test_gpu_tc.py tests/test_gpu_r2_parity.py tests/test_gpu_next2.py tests/test_gpu_ls.py tests/test_gpu_stable.py -q -x > gpurun_out/r2/check_tc.log 2>&1; tail -2 gpurun_out/r2/check_tc.log
bash scripts/r2/bench_some.sh
