"""Debug: kmeans_run on the GPU test's inputs (tests/helpers.candidate_set), printed for A/B
across library builds (KTUNE_LIB_PATH)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import pyoracle as O
from helpers import SPACES, candidate_set
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import kmeans_run
ctx = Context(0)
for name, n, k, seed in [("synthetic8", 3000, 8, 1), ("resnet_c2", 4000, 12, 3)]:
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    ds = Space(sp, ctx)
    for r in (1, 3):
        res = kmeans_run(ds, cidx, k, seed * 13 + 1, restarts=r)
        print(name, k, r, res.l2_loss, len(res.iteration_losses), int(res.assignments[:50].sum()))
