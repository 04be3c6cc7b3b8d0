timeout 600 python -m pytest tests/test_gpu_rollout.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --no-cpu --no-kmeans > gpurun_out/bench_seg.json 2> gpurun_out/bench_seg.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/bench_seg.json')); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['kernel_ms'], d['gbt_kernel_ms_per_step'])"
tail -3 gpurun_out/bench_seg.err
