# c4 (W=256, 2^22 points): launch list of the bench command + ncu --set full of one k_mlp_w256 launch
set -x
CMD="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_w256 -s 7 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "c4 exit $?"
tail -1 gpurun_out/plain_c4.log | cut -c 1-400
