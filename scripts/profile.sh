# launch list + one full ncu capture of the fused MLP kernel (bench command, 1 GPU)
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_fp32 -s 6 -c 2 -o gpurun_out/prof_mlp $CMD > gpurun_out/ncu_full.log 2>&1
echo "exit $?"
tail -3 gpurun_out/plain.log
