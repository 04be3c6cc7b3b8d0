"""Debug: one kmeans_run at k (env K, default 63) on 1M AlexNet-c2 points (for ncu launch lists)."""
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
K = int(os.environ.get("K", 63))
kmeans_run(ds, idx, K, 7, restarts=1)
ctx.reset_stats()
t0 = time.perf_counter(); r = kmeans_run(ds, idx, K, 1063, restarts=1); dt = time.perf_counter() - t0
print(f"k={K}: {dt*1e3:.1f} ms, iters {len(r.iteration_losses)-1}, stats lloyd {ctx.stat(L.STAT_LLOYD_ITERS)} fallbacks {ctx.stat(L.STAT_ASSIGN_FALLBACKS)}")
