CMD="python bench.py --config c5 --width 128 --points 262144 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_tc.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tc.csv $CMD > gpurun_out/ncu_launches_tc.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 7 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_full_tc.log 2>&1
echo "exit $?"
tail -2 gpurun_out/ncu_full_tc.log
