"""Debug: where the adaptive sweep's time goes (host timer around phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, kmeans_run
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, 1 << 20, 123)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
keep = np.sort(first)
idx, ids = idx[keep], ids[keep]
cs = CandidateSet(idx, ids, np.zeros(len(idx)))
adaptive_sweep(ds, cs, SamplingParams(), 5)
for _ in range(2):
    t0 = time.perf_counter(); sw = adaptive_sweep(ds, cs, SamplingParams(), 5); t1 = time.perf_counter()
    print(f"sweep {1e3*(t1-t0):.1f} ms k={sw.k}")
for k in (8, 9):
    t0 = time.perf_counter(); r = kmeans_run(ds, idx, k, 5, restarts=3); t1 = time.perf_counter()
    print(f"kmeans_run k={k} 3 restarts: {1e3*(t1-t0):.1f} ms, iters {len(r.iteration_losses)-1}")
