# full GPU suite, smoke, default bench line, reference arm, and the round's profiles
set -x
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 2500 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1 | cut -c 1-300
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mlp_fp32 -s 7 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu_c2.log 2>&1
CMD4="python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv $CMD4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mlp_w256 -s 7 -c 1 -o gpurun_out/prof_c4 $CMD4 > gpurun_out/ncu_c4.log 2>&1
echo done
