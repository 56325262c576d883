# K3w: L2 footprint experiment (gradient replica count) on c4 (tooling)
mkdir -p gpurun_out/r2
for rep in a b; do
for r in 16 4 1; do
  NBM_W256_REPLICAS=$r timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --no-secondary --steps 20 > gpurun_out/r2/rep$r.log 2>&1
  echo "rep $r $(tail -1 gpurun_out/r2/rep$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["avg_launch_ms"])')"
done
done
