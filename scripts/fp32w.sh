timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "wide" 2>&1 | tail -5
for w in 128 256; do
timeout 300 python bench.py --config c5 --width $w --prec fp32 --points 262144 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
