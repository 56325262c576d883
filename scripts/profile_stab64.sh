# launch list + ncu --set full of the W = 64 stable-form kernel (shared-memory staged maps)
CMD="python bench.py --config c5 --width 64 --stencil stable --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
$CMD > gpurun_out/plain_c5w64_stable.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5w64_stable.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 7 -c 1 -o gpurun_out/prof_c5w64_stable $CMD > gpurun_out/ncu_c5w64_stable.log 2>&1
echo "exit $?"
