"""k-means probe: per-launch assignment kernel time (library CUDA events, OPT_PROFILE) and the
whole kmeans_run, for several k on 1M AlexNet-c2 points.  python tools/km_assign_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from workloads.tasks import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, 1 << 20, 123)
kmeans_run(ds, idx, 8, 7, restarts=1)
for K in [int(k) for k in os.environ.get("KS", "8,16,32,63").split(",")]:
    kmeans_run(ds, idx, K, 7, restarts=1)
    ctx.reset_stats()
    ctx.set_option(L.OPT_PROFILE, 1)
    t0 = time.perf_counter(); r = kmeans_run(ds, idx, K, 1000 + K, restarts=1); dt = time.perf_counter() - t0
    ctx.set_option(L.OPT_PROFILE, 0)
    n, c = ctx.stat(L.STAT_ASSIGN_NS), max(1, ctx.stat(L.STAT_ASSIGN_CALLS))
    print(f"k={K}: kmeans_run {dt*1e3:.1f} ms (profiled), iters {len(r.iteration_losses)-1}, assign {n/c/1e3:.1f} us/launch "
          f"x {c}, loss {r.iteration_losses[-1]:.9e}", flush=True)
