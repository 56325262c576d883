mkdir -p gpurun_out/r2
for w in 128 256; do for r in 16 1; do
  NBM_W256_REPLICAS=$r timeout 300 python bench.py --config c5 --width $w --prec fp32 --points 262144 --no-cpu-baseline --no-e2e --no-secondary --steps 5 > gpurun_out/r2/repfw_$w_$r.log 2>&1
  echo "w$w rep $r $(tail -1 gpurun_out/r2/repfw_$w_$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"])')"
done; done
