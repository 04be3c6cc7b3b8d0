timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo "bench rc=$?"; cat gpurun_out/bench_r1c.json; tail -3 gpurun_out/bench_r1c.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > /dev/null 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rollout_tc_kernel -s 1 -c 1 -o gpurun_out/rollout_tc_full4 -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > gpurun_out/ncu_full4.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gbt_score_kernel -s 12 -c 1 -o gpurun_out/gbt_full -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-kmeans > gpurun_out/ncu_gbt.log 2>&1; echo "ncu3 rc=$?"
