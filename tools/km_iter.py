"""Debug: marginal certified Lloyd iteration time at N=1M (median over repeated runs: full minus 1-iteration run)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
from paper_2001_08743_b200.workloads import random_configs
ctx = Context(0)
sp = S.alexnet_tasks()[1]
ds = Space(sp, ctx)
idx = np.ascontiguousarray(random_configs(sp, 1 << 20, 123), np.uint16)
K = int(os.environ.get("K", 8))
kmeans_run(ds, idx, K, 11, max_iters=2, restarts=1)
full, one = [], []
for _ in range(9):
    t0 = time.perf_counter(); r = kmeans_run(ds, idx, K, 11, restarts=1); full.append(time.perf_counter() - t0)
    t0 = time.perf_counter(); kmeans_run(ds, idx, K, 11, max_iters=1, restarts=1); one.append(time.perf_counter() - t0)
it = len(r.iteration_losses) - 1
print(f"{os.environ.get('KTUNE_LIB_PATH','cur')[-10:]} K={K}: {it} iters, marginal {(np.median(full)-np.median(one))/(it-1)*1e3:.4f} ms/iter")
