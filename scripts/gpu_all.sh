timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for a in "--config c5 --width 64" "--config c3" "" "--config c1"; do
python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
