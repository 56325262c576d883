for r in 4 16 37 74; do
NBM_W256_REPLICAS=$r python bench.py --config c4 --points 1048576 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rep $r', d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
