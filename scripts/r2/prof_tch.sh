# ncu --set full of the K3h (and K3t) training kernel at c5-w128 (tooling)
mkdir -p gpurun_out/r2
A="--config c5 --width 128 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
timeout 300 python bench.py $A > gpurun_out/r2/plain_tch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_mlp_tch" -s 2 -c 1 \
    -o gpurun_out/r2/prof_tch128 python bench.py $A > gpurun_out/r2/ncu_tch.log 2>&1; echo "ncu tch rc=$?"
NBM_TCH_OFF=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_mlp_tc" -s 2 -c 1 \
    -o gpurun_out/r2/prof_tc128 python bench.py $A > gpurun_out/r2/ncu_tc.log 2>&1; echo "ncu tc rc=$?"
