# ncu capture of the W = 256 pair kernel (c4 at a reduced point count)
CMD="python bench.py --config c4 --points 262144 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_w256.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mlp_w256 -s 7 -c 1 -o gpurun_out/prof_w256 $CMD > gpurun_out/ncu_full_w256.log 2>&1
echo "exit $?"
tail -2 gpurun_out/ncu_full_w256.log
