timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "determinism or config2_reduced or config1_full" 2>&1 | tail -1
for a in "" "--config c5 --width 64" "--config c1"; do
timeout 300 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
