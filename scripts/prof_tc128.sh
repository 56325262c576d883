CMD="python bench.py --config c5 --width 128 --points 262144 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mlp_tc -s 7 -c 1 -o gpurun_out/prof_tc128 $CMD > gpurun_out/ncu_tc128.log 2>&1
echo "exit $?"
