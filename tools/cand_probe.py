"""make_candidate_set on the device (ktune_candidates_from_rows): CUDA-event time of one call
over N device-resident trajectory rows (VGG-16 c4 space, ~85% distinct), after a warm-up call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import candidates_from_rows
from workloads.tasks import random_configs

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32_800_000
ctx = Context(0)
sp = S.vgg16_tasks()[3]
ds = Space(sp, ctx)
g = np.random.default_rng(0)
base = random_configs(sp, N, 1).astype(np.uint16)
base[1::7] = base[::7][: len(base[1::7])]  # some duplicates
idx = torch.from_numpy(base.view(np.int16)).cuda().view(torch.uint16)
pred = torch.from_numpy(np.round(g.random(N), 6)).cuda()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows, ids = candidates_from_rows(ds, idx, pred)
    torch.cuda.synchronize()
    print(f"N={N}: kept {rows.numel()} in {1e3 * (time.perf_counter() - t0):.2f} ms")
