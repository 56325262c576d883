mkdir -p gpurun_out/r2
NBM_LIB=$PWD/paper_2210_14907_b200/libnbm_exp.so timeout 600 python -m pytest tests/test_gpu_tc.py -q -k "silu_many" > gpurun_out/r2/silu_eval_old.log 2>&1; tail -3 gpurun_out/r2/silu_eval_old.log
bash scripts/r2/check_c3.sh
timeout 600 python -m pytest tests/test_gpu_tc.py -q -k "silu_many" > gpurun_out/r2/silu_eval_new.log 2>&1; tail -2 gpurun_out/r2/silu_eval_new.log
