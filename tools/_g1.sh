timeout 600 oracle/_ref/dropin_test | tail -5
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --c5 0 --no-sa --no-full-sweep > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc=$?
