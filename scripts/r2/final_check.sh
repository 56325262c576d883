# round 2: smoke, the full GPU suite, the default bench line and the reference arm (tooling)
mkdir -p gpurun_out/r2/final
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2/final/smoke.log 2>&1; echo "smoke rc=$?"
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/final/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2/final/pytest.log
timeout 900 python bench.py > gpurun_out/r2/final/bench.json 2> gpurun_out/r2/final/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2/final/ref.json 2> gpurun_out/r2/final/ref.err; echo "ref rc=$?"
