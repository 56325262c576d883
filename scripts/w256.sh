set -x
timeout 300 python -m pytest tests/test_gpu_tc.py -x -q -k "c4" 2>&1 | tail -5
timeout 120 python scripts/trace_w256.py 2>&1 | grep -E "^tile [345] total|dH|fwd3"
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
