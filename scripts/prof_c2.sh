CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mlp_fp32 -s 7 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_c2.log 2>&1
echo "exit $?"
