"""Debug: one k-means run at N=1M (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, 1 << 20, 123)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
idx = idx[np.sort(first)]
kmeans_run(ds, idx, 8, 11, max_iters=3, restarts=1)
r = kmeans_run(ds, idx, 8, 11, max_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 6, restarts=1)
print("iters", len(r.iteration_losses) - 1, "aborts", ctx.stat(L.STAT_KMEANS_ABORTS))
