# K3h variants (NBM_LIB=libnbm_<name>.so) on c5-w64 / c5-w128 (tooling)
mkdir -p gpurun_out/r2/var
for v in "$@"; do
  for w in 64 128; do
    if [ "$v" = k3t ]; then lib=paper_2210_14907_b200/libnbm.so; pre="NBM_TCH_OFF=1"; else lib=paper_2210_14907_b200/libnbm_$v.so; pre=""; fi
    env $pre NBM_LIB=$PWD/$lib timeout 300 python bench.py --config c5 --width $w --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r2/var/${v}_w$w.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/r2/var/${v}_w$w.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v w$w', round(d['ms_per_step'],3), round(r['avg_launch_ms'],3), round(r['frac'],4))" 2>&1 | tail -1
  done
done
