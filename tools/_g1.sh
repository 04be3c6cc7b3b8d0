timeout 900 python -m pytest tests/test_gpu_dist.py -x -q 2>&1 | tail -15
BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e --c3-episodes 16384 > gpurun_out/bench_w2_r2.json 2> gpurun_out/bench_w2_r2.err; echo "w2 rc=$?"
tail -3 gpurun_out/bench_w2_r2.err
