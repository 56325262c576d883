# experiment (tooling): K3w with the dW MMAs, their operand loads and the dW flush removed
# (the build flags NBM_W256_NO_DW / NO_WLOAD / SPLIT_FLUSH and the pipelined forward exist in commit 2b2a58a only)
# (timing only; gradients wrong) -- what the fused kernel would cost with dW computed elsewhere
mkdir -p gpurun_out/r2
for v in base nodw; do
  L=$PWD/paper_2210_14907_b200/libnbm.so
  [ $v = nodw ] && L=$PWD/paper_2210_14907_b200/libnbm_nodw.so
  NBM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-secondary --steps 20 > gpurun_out/r2/nodw_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/r2/nodw_$v.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"])')"
done
