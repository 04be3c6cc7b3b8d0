"""Debug: k-means at tens of millions of points (mode via KM_MODE), few iterations (ncu launch lists)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.vgg16_tasks()[3]
ds = Space(sp, ctx)
N = int(os.environ.get("N", 27_000_000))
idx = random_configs(sp, N, 5)
ctx.set_option(L.OPT_KMEANS_MODE, int(os.environ.get("KM_MODE", 1)))
if os.environ.get("KT_HOST_TRACE"): ctx.set_option(L.OPT_PROFILE, 1)
it = int(os.environ.get("ITERS", 4))
kmeans_run(ds, idx[:100000], 8, 1, max_iters=2, restarts=1)
ctx.reset_stats()
t0 = time.perf_counter(); r = kmeans_run(ds, idx, 8, 1, max_iters=it, restarts=1); dt = time.perf_counter() - t0
print(f"N={N} mode={os.environ.get('KM_MODE', 1)} iters={len(r.iteration_losses)-1}: {dt*1e3:.0f} ms; "
      f"xs seq {ctx.stat(L.STAT_XS_SEQUENTIAL)} / {ctx.stat(L.STAT_XS_SEGMENTS)}, aborts {ctx.stat(L.STAT_KMEANS_ABORTS)}, kpp fb {ctx.stat(L.STAT_KPP_FALLBACKS)}, launches {ctx.stat(L.STAT_LAUNCHES)}")
