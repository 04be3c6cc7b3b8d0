"""Debug: the bench's C3 pipeline stages separately (rollout, candidates, adaptive sweep)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.distributed import create_context
class A: c3_episodes = int(os.environ.get("E", 65536)); c3_T = int(os.environ.get("T", 500)); seed = 0
ctx = create_context(0, 0, 1)
ctx.reset_stats()
r = bench.c3_pipeline(ctx, A())
print(r)
for n in ("STAT_LLOYD_ITERS", "STAT_KMEANS_ABORTS", "STAT_KPP_FALLBACKS", "STAT_ASSIGN_FALLBACKS", "STAT_XS_SEQUENTIAL", "STAT_XS_SEGMENTS", "STAT_SNAP_CHAINS"):
    print(n, ctx.stat(getattr(L, n)))
