"""Debug: one adaptive sweep (for ncu launch lists)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
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
cs = CandidateSet(idx[keep], ids[keep], np.zeros(len(keep)))
t0 = time.perf_counter(); adaptive_sweep(ds, cs, SamplingParams(), 5); print("sweep ms", 1e3 * (time.perf_counter() - t0))
