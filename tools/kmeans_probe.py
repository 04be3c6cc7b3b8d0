"""Probe: one kmeans_run at N=1M (AlexNet c2 space) for ncu launch lists."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
idx = random_configs(sp, n, 123)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
idx = idx[np.sort(first)]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.perf_counter()
r = kmeans_run(ds, idx, 8, 11, max_iters=iters, restarts=1)
torch.cuda.synchronize()
from paper_2001_08743_b200 import _lib as L
print("xs sequential", ctx.stat(L.STAT_XS_SEQUENTIAL), "of", ctx.stat(L.STAT_XS_SEGMENTS))
print("kmeans_run", time.perf_counter() - t0, "s, iters", len(r.iteration_losses) - 1)
