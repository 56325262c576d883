# bench lines of the main workloads (one B200) -> gpurun_out/r2/bench/<label>.json (tooling)
mkdir -p gpurun_out/r2/bench
run() {  # label, args
  timeout 600 python bench.py $2 > gpurun_out/r2/bench/$1.log 2>&1
  tail -1 gpurun_out/r2/bench/$1.log > gpurun_out/r2/bench/$1.json
  echo "$1 $(python -c "import json,sys; d=json.load(open('gpurun_out/r2/bench/$1.json')); r=d.get('roofline') or {}; print(round(d['ms_per_step'],3), round(r.get('avg_launch_ms',0),3), round(r.get('frac',0),4))" 2>&1 | tail -1)"
}
run c2 "--config c2 --no-cpu-baseline --no-e2e"
run c3 "--config c3 --no-cpu-baseline --no-e2e"
run c5w64 "--config c5 --width 64 --no-cpu-baseline --no-e2e"
run c5w128 "--config c5 --width 128 --no-cpu-baseline --no-e2e"
run c1 "--config c1 --no-cpu-baseline --no-e2e"
