# launch list + ncu --set full of K3t at c3 (SiLU) after the SiLU' change (tooling)
mkdir -p gpurun_out/r2/prof
CMD="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
timeout 600 $CMD > gpurun_out/r2/prof/plain_c3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/prof/launches_c3.csv $CMD > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 7 -c 1 -o gpurun_out/r2/prof/prof_c3 $CMD > gpurun_out/r2/prof/ncu_c3.log 2>&1
echo "c3 exit $?"
