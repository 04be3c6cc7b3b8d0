timeout 300 python -m pytest tests/test_gpu_rollout.py -x -q -p no:cacheprovider -k "tc" 2>&1 | tail -2
python tools/trace_tc.py 2>&1 | tail -4
timeout 600 python bench.py > gpurun_out/bench_tc2.json 2> gpurun_out/bench_tc2.err; echo "bench rc=$?"; cat gpurun_out/bench_tc2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_tc2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rollout_tc_kernel -s 1 -c 1 -o gpurun_out/rollout_tc_full3 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > gpurun_out/ncu_full3.log 2>&1; echo "ncu2 rc=$?"
