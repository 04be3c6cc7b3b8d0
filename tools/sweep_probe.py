"""Debug: adaptive_sweep timing / stats at N = 1M."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, 1 << 20, 123)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
keep = np.sort(first)
idx, ids = idx[keep], ids[keep]
for mode in [0, 1, 0]:
    ctx.set_option(L.OPT_KMEANS_MODE, mode)
    ctx.reset_stats()
    t0 = time.perf_counter()
    sw = adaptive_sweep(ds, CandidateSet(idx, ids, np.zeros(len(idx))), SamplingParams(), 5)
    dt = time.perf_counter() - t0
    print(f"mode {mode}: {dt*1e3:.1f} ms k={sw.k} iters={ctx.stat(L.STAT_LLOYD_ITERS)} aborts={ctx.stat(L.STAT_KMEANS_ABORTS)}")
