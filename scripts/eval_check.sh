timeout 600 python -m pytest tests/test_gpu_tc.py -q -k "eval" 2>&1 | tail -1
for a in "" "--config c4" "--config c5 --width 128"; do
timeout 300 python bench.py $a --eval --steps 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['inference'])"
done
