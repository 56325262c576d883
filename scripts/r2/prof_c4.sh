# default bench line (c4) + launch list + one full ncu capture of the fused kernel (tooling)
mkdir -p gpurun_out/r2
timeout 600 python bench.py > gpurun_out/r2/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2/bench_default.log > gpurun_out/r2/bench_default.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/ncu_launch_c4.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_mlp_w256 -s 7 -c 1 -o gpurun_out/r2/prof_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/ncu_full_c4.log 2>&1; echo "ncu2 rc=$?"
