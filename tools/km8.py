"""Debug: the bench's k-means secondary workload (k=8, 1M dedup AlexNet-c2), repeated."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
kmeans_run(ds, idx, 8, 11, max_iters=2, restarts=1)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = kmeans_run(ds, idx, 8, 11, restarts=1); torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    t1 = time.perf_counter(); kmeans_run(ds, idx, 8, 11, max_iters=1, restarts=1); torch.cuda.synchronize(); dt1 = time.perf_counter() - t1
    it = len(r.iteration_losses) - 1
    print(f"{os.environ.get('KTUNE_LIB_PATH','cur')[-10:]}: full {dt*1e3:.2f} ms ({it} it), 1-iter {dt1*1e3:.2f} ms, marginal {(dt-dt1)/(it-1)*1e3:.4f} ms/iter")
