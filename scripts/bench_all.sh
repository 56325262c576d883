# every workload's bench line (one B200) -> gpurun_out/bench_all/<label>.json
mkdir -p gpurun_out/bench_all
run() {  # label, args
  timeout 600 python bench.py $2 > gpurun_out/bench_all/$1.log 2>&1
  tail -1 gpurun_out/bench_all/$1.log > gpurun_out/bench_all/$1.json
  echo "$1 $(python -c "import json,sys; d=json.load(open('gpurun_out/bench_all/$1.json')); r=d.get('roofline') or {}; print(round(d['ms_per_step'],3), round(r.get('avg_launch_ms',0),3), round(r.get('frac',0),4), d.get('e2e',{}) and d['e2e'].get('value'))" 2>&1 | tail -1)"
}
run c2 "--config c2 --no-secondary"
run c1 "--config c1 --no-cpu-baseline"
run c3 "--config c3 --no-cpu-baseline --no-e2e"
run c4 "--config c4 --no-cpu-baseline --no-e2e --no-secondary --steps 10"
run c5w64 "--config c5 --width 64 --no-cpu-baseline --no-e2e"
run c5w128 "--config c5 --width 128 --no-cpu-baseline --no-e2e"
run c5w128fp32 "--config c5 --width 128 --prec fp32 --points 262144 --no-cpu-baseline --no-e2e"
run c5w256fp32 "--config c5 --width 256 --prec fp32 --points 262144 --no-cpu-baseline --no-e2e --steps 5"
run c5w64fp32 "--config c5 --width 64 --prec fp32 --no-cpu-baseline --no-e2e"
run c2fp32x "--config c2 --prec fp32x --no-cpu-baseline --no-e2e"
run c5w64stable "--config c5 --width 64 --stencil stable --no-cpu-baseline --no-e2e --steps 5"
run c5w128stable "--config c5 --width 128 --stencil stable --no-cpu-baseline --no-e2e --steps 5"
run c4stable "--config c4 --stencil stable --no-cpu-baseline --no-e2e --no-secondary --steps 5"
run c2stable "--config c2 --stencil stable --no-cpu-baseline --no-e2e"
run c2ref "--config c2 --impl reference --steps 3 --warmup 3"
