# launch list + ncu --set full of K3h at c5-w128 (tooling)
mkdir -p gpurun_out/r2/prof
CMD="python bench.py --config c5 --width 128 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
timeout 600 $CMD > gpurun_out/r2/prof/plain_c5w128.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/prof/launches_c5w128.csv $CMD > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tch -s 3 -c 1 -o gpurun_out/r2/prof/prof_c5w128 $CMD > gpurun_out/r2/prof/ncu_c5w128.log 2>&1
echo "c5w128 exit $?"
