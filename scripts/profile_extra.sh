# launch lists + ncu --set full of the fused kernel for c2 with the stable form (fp32) and FP32X
set -x
run() {  # tag, bench args, kernel regex, skip
  CMD="python bench.py $2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
  $CMD > gpurun_out/plain_$1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv $CMD > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1
  echo "$1 exit $?"
}
run c2_stable "--stencil stable" "k_mlp_fp32" 7
run c2_fp32x "--prec fp32x" "k_mlp_tc" 7
