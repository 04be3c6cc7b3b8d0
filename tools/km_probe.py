"""k-means at C3 scale: N distinct VGG-16 c4 configurations (u8 indices), device-resident;
kmeans_run-equivalent adaptive_sweep (k = 8..9) and a forced k = 16 / 63 run; wall times,
Lloyd iterations, CUDA-event assignment time (KTUNE_OPT_PROFILE)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, candidates_from_rows

N = int(sys.argv[1]) if len(sys.argv) > 1 else 27_700_000
ctx = Context(0)
sp = S.vgg16_tasks()[3]
ds = Space(sp, ctx)
g = np.random.default_rng(0)
raw = np.stack([g.integers(0, c, int(N * 1.05)) for c in sp.cards], 1).astype(np.uint16)
idx = torch.from_numpy(raw.view(np.int16)).cuda().view(torch.uint16)
pred = torch.from_numpy(g.random(len(raw))).cuda()
rows, ids = candidates_from_rows(ds, idx, pred)
rows, ids = rows[:N], ids[:N]
cidx = idx.view(torch.int16)[rows].to(torch.uint8)
cands = CandidateSet(cidx, ids.view(torch.int64), None)
torch.cuda.synchronize()
print(f"N = {len(rows)} distinct candidates")
for kmax, thr in ((64, 2.5), (17, 1.0000001)):
    p = SamplingParams(threshold=thr, k_max_exclusive=kmax)
    for rep in range(2):
        ctx.reset_stats()
        ctx.set_option(L.OPT_PROFILE, 1 if rep else 0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sw = adaptive_sweep(ds, cands, p, 5)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        it = ctx.stat(L.STAT_LLOYD_ITERS)
        print(f"sweep k<{kmax} thr={thr}: {1e3 * dt:.1f} ms, k={sw.k}, lloyd iters {it}, kpp picks "
              f"{ctx.stat(L.STAT_KPP_PICKS)} (exact replays {ctx.stat(L.STAT_KPP_FALLBACKS)}), assign calls {ctx.stat(L.STAT_ASSIGN_CALLS)}, assign ms "
              f"{ctx.stat(L.STAT_ASSIGN_NS) / 1e6:.1f}, aborts {ctx.stat(L.STAT_KMEANS_ABORTS)}" + (" (profiled)" if rep else ""))
ctx.set_option(L.OPT_PROFILE, 0)
