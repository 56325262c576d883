# round-2 launch lists + ncu --set full of the fused kernel for the stable stencil form (G27):
# c2 (K3f), c5-w64 (K3t), c5-w128 (K3t), c4 (K3w), at the bench sizes (tooling)
mkdir -p gpurun_out/r2/prof
run() {  # tag, bench args, kernel regex, skip
  CMD="python bench.py $2 --stencil stable --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
  timeout 600 $CMD > gpurun_out/r2/prof/plain_$1.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/prof/launches_$1.csv $CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/r2/prof/prof_$1 $CMD > gpurun_out/r2/prof/ncu_$1.log 2>&1
  echo "$1 exit $?"
}
run c2_stable "--config c2" "k_mlp_fp32" 7
run c5w64_stable "--config c5 --width 64" "k_mlp_tc" 7
run c5w128_stable "--config c5 --width 128" "k_mlp_tc" 7
run c4_stable "--config c4" "k_mlp_w256" 7
# summaries on the box (the .ncu-rep files exceed what gpurun brings back)
mkdir -p gpurun_out/r2/prof_summ
for t in c2_stable c5w64_stable c5w128_stable c4_stable; do
  python scripts/ncu_summary.py --launches gpurun_out/r2/prof/launches_$t.csv --rep gpurun_out/r2/prof/prof_$t.ncu-rep --tag r2_$t > /dev/null 2>&1
  cp profiles/r2_$t.md profiles/r2_$t.json gpurun_out/r2/prof_summ/ 2>/dev/null
done
rm -f gpurun_out/r2/prof/*.ncu-rep
