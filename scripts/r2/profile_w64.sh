# launch list + ncu --set full of K3t at c5-w64 after the M = 64 dW/tail change (tooling)
mkdir -p gpurun_out/r2/prof
run() {  # tag, bench args, kernel regex, skip
  CMD="python bench.py $2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
  timeout 600 $CMD > gpurun_out/r2/prof/plain_$1.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/prof/launches_$1.csv $CMD > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/r2/prof/prof_$1 $CMD > gpurun_out/r2/prof/ncu_$1.log 2>&1
  echo "$1 exit $?"
}
run c5w64 "--config c5 --width 64" "k_mlp_tc" 7
run c2fp32x "--config c2 --prec fp32x" "k_mlp_tc" 7
