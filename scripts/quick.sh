timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config2 or config1 or ragged" 2>&1 | tail -2
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
