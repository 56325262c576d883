# bf16 tensor-core paths: parity + quick bench of c3, c5-w64, c5-w128, c4
timeout 900 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
for a in "--config c3" "--config c5 --width 64" "--config c5 --width 128" "--config c4"; do
timeout 300 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
