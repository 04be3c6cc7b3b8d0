"""Timeline of one kmeans_run (1M AlexNet-c2 points, k = env K) from CUPTI via torch.profiler:
kernel mix, GPU busy vs idle, host syncs per Lloyd iteration."""
import collections, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from workloads.tasks import random_configs
import torch
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, 1 << 20, 123)
K = int(os.environ.get("K", 40))
R = int(os.environ.get("R", 3))
kmeans_run(ds, idx, K, 7, restarts=R)
ctx.reset_stats()
t0 = time.perf_counter(); r = kmeans_run(ds, idx, K, 1063, restarts=R); dt = time.perf_counter() - t0
iters = ctx.stat(L.STAT_LLOYD_ITERS)
print(f"k={K} restarts={R}: {dt*1e3:.2f} ms wall, lloyd iters {iters}, {dt*1e3/max(iters,1):.3f} ms/iter")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    kmeans_run(ds, idx, K, 1063, restarts=R)
    torch.cuda.synchronize()
path = "gpurun_out/km_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")],
             key=lambda e: e["ts"])
span = (gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]) / 1e3
busy = sum(e["dur"] for e in gpu) / 1e3
agg = collections.defaultdict(lambda: [0, 0.0])
for e in gpu:
    k = e["name"].split("(")[0][-50:]
    agg[k][0] += 1
    agg[k][1] += e["dur"] / 1e3
print(f"GPU span {span:.2f} ms, busy {busy:.2f} ms ({100 * busy / span:.0f}%), {len(gpu)} activities")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"  {t:8.3f} ms {n:5d}  {k}")
rt = collections.Counter(e["name"] for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime")
print("runtime calls:", dict(rt.most_common(10)))
