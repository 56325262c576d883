# launch lists + ncu --set full of the K3t kernel for c3, c5-w128, c5-w64 (reduced points)
run() {  # tag, bench args, kernel regex, skip
  CMD="python bench.py $2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
  $CMD > gpurun_out/plain_$1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$1.csv $CMD > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s $4 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1
  echo "$1 exit $?"
}
run c3 "--config c3" "k_mlp_tc" 7
run c5w128 "--config c5 --width 128" "k_mlp_tc" 7
run c5w64 "--config c5 --width 64" "k_mlp_tc" 7
