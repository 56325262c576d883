# K3w: bench (c4), timeline trace, and one ncu --set full capture of the training kernel (tooling)
mkdir -p gpurun_out/r2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-secondary --steps 10 > gpurun_out/r2/bench_w256.log 2>&1; echo "bench rc=$?"
NBM_LIB=$PWD/paper_2210_14907_b200/libnbm_trace.so timeout 200 python scripts/trace_w256.py > gpurun_out/r2/trace_v1.log 2>&1; echo "trace rc=$?"
if [ "$1" = "ncu" ]; then
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_mlp_w256<4, 1" -s 2 -c 1 \
    -o gpurun_out/r2/prof_c4 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/ncu_full_c4.log 2>&1; echo "ncu rc=$?"
fi
