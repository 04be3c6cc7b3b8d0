"""Debug: streamed host-buffer rollout vs the device path (step-major); prints where they differ.
  NAMES=a,b,c ES=600,257,1000 T=333 SEGS=0 python tools/stream_debug.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from oracle import pyoracle as O
from helpers import SPACES, fitted
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.cost_model import DeviceGbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
ctx = Context(0)
names = os.environ.get("NAMES", "resnet_c2,vgg_c4,alexnet_c3_u16").split(",")
Es = [int(x) for x in os.environ.get("ES", "600,257,1000").split(",")]
T = int(os.environ.get("T", "333"))
tasks = []
for i, name in enumerate(names):
    sp = SPACES[name]()
    osp, og, pm = fitted(O, sp, seed=190 + i)
    ds = Space(sp, ctx)
    init = np.random.default_rng(i).integers(0, np.asarray(sp.cards), (Es[i], sp.num_knobs)).astype(np.int32)
    tasks.append(RolloutTask(ds, ActorCritic(sp.num_knobs, 128, 64, seed=191 + i, ctx=ctx), DeviceGbt(pm, ds), init,
                             episode_offset=11 * i, root_seed=i))
dref = run_episodes_batch([RolloutTask(t.space, t.agent, t.cost_model, torch.from_numpy(t.init_idx).cuda(),
                                       t.episode_offset, t.root_seed) for t in tasks], T, step_major=True)
torch.cuda.synchronize()
ref = [{k: v.cpu().numpy() for k, v in o.items()} for o in dref]
ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, int(os.environ.get("SEGS", "0")))
for mode in (0, 1):
    ctx.set_option(L.OPT_ROLLOUT_STREAMED, mode)
    for rep in range(3):
        hs = run_episodes_batch(tasks, T, step_major=True)
        for k, (a, h) in enumerate(zip(ref, hs)):
            for f in ["idx", "actions", "score", "logp", "value"]:
                d = a[f] != h[f]
                if d.ndim == 3:
                    d = d.any(-1)
                if d.any():
                    rw, ep = np.nonzero(d)
                    print(f"streamed={mode == 0} rep {rep} task {k} {f}: {d.sum()} differ; rows {sorted(set(rw.tolist()))[:30]}"
                          f" episodes {sorted(set(ep.tolist()))[:12]} (n={len(set(ep.tolist()))})")
print("done")
