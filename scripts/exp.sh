for lib in libnbm.so libnbm_exp.so; do
NBM_LIB=$PWD/paper_2210_14907_b200/$lib python bench.py --config c5 --width 128 --points 1048576 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
done
