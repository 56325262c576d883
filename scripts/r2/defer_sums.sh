# K3w: w_o / b_NH column sums deferred under the dH_NH GEMM (tooling): bench c4 x2 + W = 256 tests
# (the change is not in the tree: measured slower and reverted)
mkdir -p gpurun_out/r2
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-secondary --steps 20 > gpurun_out/r2/ds_bench.log 2>&1
echo "bench $(tail -1 gpurun_out/r2/ds_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"], d["roofline"]["frac"])')"
done
timeout 1200 python -m pytest tests -m gpu -q -x -k "256 or c4 or w256 or eval_tiles or ls or next2 or stable or closed" > gpurun_out/r2/ds_tests.log 2>&1; tail -2 gpurun_out/r2/ds_tests.log
