python -m pytest tests/test_gpu_rollout.py -x -q -k "planted or c2_shape or spot_replay or check_mode" -s 2>&1 | grep -E "planted|C2 shape|max \||passed|failed|Error" | tail -8
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r2a.json 2>&1; echo ref rc=$?
