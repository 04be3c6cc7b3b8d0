timeout 300 python -m pytest tests/test_gpu_rollout.py -x -q -p no:cacheprovider -k "tc" 2>&1 | tail -3
python tools/trace_tc.py 2>&1 | tail -4
MODE=nosync timeout 300 python tools/diag_step.py 2>&1 | tail -1
