nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 300 python -m pytest tests/test_gpu_rollout.py -x -q -p no:cacheprovider -k "tc" -s > gpurun_out/pytest_tc.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_tc.log
