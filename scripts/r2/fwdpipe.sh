# K3w forward pipelining (tooling): bench c4 + the W = 256 tests
# (the build flags NBM_W256_NO_DW / NO_WLOAD / SPLIT_FLUSH and the pipelined forward exist in commit 2b2a58a only)
mkdir -p gpurun_out/r2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-secondary --steps 20 > gpurun_out/r2/fp_bench.log 2>&1
echo "bench $(tail -1 gpurun_out/r2/fp_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"])')"
timeout 1200 python -m pytest tests -m gpu -q -x -k "256 or c4 or w256 or eval_tiles or ls or next2 or stable" > gpurun_out/r2/fp_tests.log 2>&1; tail -3 gpurun_out/r2/fp_tests.log
