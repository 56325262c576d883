for a in "" "--config c1" "--config c4 --steps 5"; do
timeout 300 python bench.py $a --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['launch_mode'], d['value'], d['ms_per_step'], d['ms_per_step_eager'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'], d['clocks'])"
done
