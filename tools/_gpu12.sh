timeout 300 python -m pytest tests/test_gpu_rollout.py -x -q -p no:cacheprovider -k "tc" -s 2>&1 | grep -E "passed|failed|max \||fallback" 
MODE=nosync timeout 300 python tools/diag_step.py 2>&1 | tail -1
