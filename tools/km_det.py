"""Debug: determinism of kmeans_run at large N (same input, repeated runs)."""
import os, sys, hashlib
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
N = int(os.environ.get("N", 24_000_000))
idx = random_configs(sp, N, 5)
ctx.set_option(L.OPT_KMEANS_MODE, int(os.environ.get("KM_MODE", 0)))
ctx.set_option(L.OPT_FORCE_EXACT, int(os.environ.get("FORCE_EXACT", 0)))
print("input", hashlib.sha1(np.ascontiguousarray(idx).tobytes()).hexdigest()[:12])
for rep in range(3):
    ctx.reset_stats()
    r = kmeans_run(ds, idx, int(os.environ.get('K', 9)), 3, max_iters=int(os.environ.get('ITERS', 100)), restarts=int(os.environ.get('RESTARTS', 3)))
    h = hashlib.sha1(r.assignments.tobytes()).hexdigest()[:12]
    ch = hashlib.sha1(np.ascontiguousarray(r.centroids).tobytes()).hexdigest()[:12]
    print(f"cent {ch}", end=" ")
    print(f"rep {rep}: iters {len(r.iteration_losses)-1} loss {r.l2_loss!r} asg {h} aborts {ctx.stat(L.STAT_KMEANS_ABORTS)} "
          f"lloyd {ctx.stat(L.STAT_LLOYD_ITERS)} kppfb {ctx.stat(L.STAT_KPP_FALLBACKS)}")
