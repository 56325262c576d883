mkdir -p gpurun_out/r2
TW=128 timeout 300 python scripts/trace_tc.py > gpurun_out/r2/trace_tc128.log 2>&1
TW=64 timeout 300 python scripts/trace_tc.py > gpurun_out/r2/trace_tc64.log 2>&1
bash scripts/r2/bench_some.sh 2>&1 | head -4
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_r2_parity.py -q -x 2>&1 | tail -3
