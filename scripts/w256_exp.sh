# W=256 parity + c4 bench at several replica counts
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q -k "c4" 2>&1 | tail -3
for r in 4 8 16; do
NBM_W256_REPLICAS=$r timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rep $r', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
