"""Validation: k-means / adaptive sweep on 1M AlexNet-c2 candidates (SURVEY C4 scale) against the
reference's own kmeans_run and sweep (oracle/_ref, reference sources built in place)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as O
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, kmeans_run
from workloads.tasks import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = random_configs(sp, int(os.environ.get("N", 1 << 20)), 123)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
keep = np.sort(first)
idx, ids = idx[keep], ids[keep]
osp = O.OSpace(sp)
P = osp.encode(idx)
for k in (8, 40):
    t0 = time.perf_counter(); g = kmeans_run(ds, idx, k, 11, restarts=3); tg = time.perf_counter() - t0
    t0 = time.perf_counter(); r = O.kmeans_run(P, k, 11, restarts=3, impl="ref"); tr = time.perf_counter() - t0
    ok = np.array_equal(g.assignments, r["assignments"]) and np.array_equal(g.centroids, r["centroids"]) and g.l2_loss == r["loss"]
    print(f"kmeans_run N={len(idx)} k={k} 3 restarts: {'EQUAL' if ok else 'DIFFERENT'} (gpu {tg*1e3:.0f} ms, reference {tr:.1f} s)", flush=True)
t0 = time.perf_counter(); sw = adaptive_sweep(ds, CandidateSet(idx, ids, np.zeros(len(ids))), SamplingParams(), 5); tg = time.perf_counter() - t0
t0 = time.perf_counter(); rw = O.adaptive_sweep(P, rng_seed=5)  # C restatement (pinned to the reference by the CPU tests); tr = time.perf_counter() - t0
ok = sw.k == rw["k"] and list(sw.k_losses) == list(rw["k_losses"]) and np.array_equal(sw.assignments, rw["assignments"]) and np.array_equal(sw.centroids, rw["centroids"])
print(f"adaptive sweep N={len(idx)}: k={sw.k} {'EQUAL' if ok else 'DIFFERENT'} (gpu {tg*1e3:.0f} ms, oracle port {tr:.1f} s)")
