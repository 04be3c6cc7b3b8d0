"""Debug: forced full adaptive sweep k = 8..63 (threshold 1+1e-12) at N = 1M."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
from workloads.tasks import random_configs
ctx = Context(0)
for name, sp in (("alexnet.c2", S.alexnet_tasks()[1]), ("resnet18.t1", S.resnet18_tasks()[1])):
    ds = Space(sp, ctx)
    idx = random_configs(sp, 1 << 20, 123)
    ids = ds.id_of(idx)
    _, first = np.unique(ids, return_index=True)
    keep = np.sort(first)
    cs = CandidateSet(idx[keep], ids[keep], np.zeros(len(keep)))
    p = SamplingParams(threshold=1.0 + 1e-12)  # break only if the loss stops falling
    adaptive_sweep(ds, cs, SamplingParams(k_max_exclusive=10), 5)
    ctx.reset_stats() if hasattr(ctx, "reset_stats") else None
    t0 = time.perf_counter(); sw = adaptive_sweep(ds, cs, p, 5); dt = time.perf_counter() - t0
    st = {n: ctx.stat(getattr(L, n)) for n in ("STAT_LLOYD_ITERS", "STAT_ASSIGN_FALLBACKS", "STAT_KMEANS_ABORTS", "STAT_KPP_FALLBACKS")} if hasattr(ctx, "stat") else {}
    print(f"{name}: N={len(keep)} full sweep k=8..63 x3 restarts: {dt*1e3:.1f} ms, k={sw.k}, losses {len(sw.k_losses)} {st}")
# forced full sweep: every k of range(8, 64), 3 restarts each
from paper_2001_08743_b200.sampling import kmeans_run
for name, sp in (("alexnet.c2", S.alexnet_tasks()[1]), ("resnet18.t1", S.resnet18_tasks()[1])):
    ds = Space(sp, ctx)
    idx = random_configs(sp, 1 << 20, 123)
    kmeans_run(ds, idx, 30, 1, restarts=1)
    ctx.reset_stats()
    t0 = time.perf_counter(); per = []
    for k in range(8, 64):
        t1 = time.perf_counter(); r = kmeans_run(ds, idx, k, 1000 + k, restarts=3); per.append((k, time.perf_counter() - t1))
    dt = time.perf_counter() - t0
    st = {n: ctx.stat(getattr(L, n)) for n in ("STAT_LLOYD_ITERS", "STAT_ASSIGN_FALLBACKS", "STAT_KMEANS_ABORTS", "STAT_KPP_FALLBACKS")}
    print(f"{name}: forced k=8..63 x3 restarts at N={len(idx)}: {dt*1e3:.0f} ms {st}")
    print("  per-k ms:", " ".join(f"{k}:{1e3*t:.0f}" for k, t in per[::5]))
