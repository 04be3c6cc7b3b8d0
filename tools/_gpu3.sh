nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 600 python bench.py --no-cpu > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo "bench rc=$?"; cat gpurun_out/bench_tc.json; tail -5 gpurun_out/bench_tc.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_tc.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rollout_tc_kernel -s 1 -c 1 -o gpurun_out/rollout_tc_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"; tail -3 gpurun_out/ncu_full.log
