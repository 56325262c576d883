timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -15
for w in 64 128; do
python bench.py --config c5 --width $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5w$w', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
