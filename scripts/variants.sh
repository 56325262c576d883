# time experimental variants of libnbm on c4 (timing only, results not checked)
for v in "$@"; do
NBM_LIB=$PWD/paper_2210_14907_b200/libnbm_$v.so timeout 300 python bench.py $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
