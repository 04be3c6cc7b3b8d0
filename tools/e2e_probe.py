"""Debug: end-to-end (host buffers) rollout time vs segment count."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from paper_2001_08743_b200.workloads import encode
from paper_2001_08743_b200.distributed import create_context
class A: tasks = 12; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T, D = 4096, 500, 8
pinned = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
host_init = [pinned(s.init_idx.shape, torch.int16).view(np.uint16) for s in specs]
for h, s in zip(host_init, specs): h[:] = s.init_idx
small = [max(s.space.cards) <= 256 for s in specs]
host_out = [dict(idx=None if sm else pinned((E, T + 1, D), torch.int16).view(np.uint16),
                 idx8=pinned((E, T + 1, D), torch.uint8) if sm else None, score=pinned((E, T + 1), torch.float64),
                 actions=None, actions2=pinned((E, T, 2), torch.uint8), logp=None, value=None,
                 logp32=pinned((E, T), torch.float32), value32=pinned((E, T), torch.float32)) for sm in small]
tasks = [RolloutTask(d, a, g, hi, 0, s.seed) for s, d, a, g, hi in zip(specs, spaces, agents, gbts, host_init)]
tot = sum(sum(v.nbytes for v in o.values() if v is not None) for o in host_out)
# raw D2H bandwidth of one big pinned copy
dbuf = torch.empty(tot, dtype=torch.uint8, device="cuda"); hbuf = torch.empty(tot, dtype=torch.uint8, pin_memory=True)
for _ in range(2): hbuf.copy_(dbuf); torch.cuda.synchronize()
t0 = time.perf_counter(); hbuf.copy_(dbuf); torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(f"raw D2H {tot/1e9:.2f} GB in {dt*1e3:.1f} ms = {tot/dt/1e9:.1f} GB/s")
for S in [int(x) for x in os.environ.get("SEGS", "1,2,3,4,5,6,8").split(",")]:
    ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, S)
    run_episodes_batch(tasks, T, ctx, host_out=host_out)
    t0 = time.perf_counter()
    for _ in range(3): run_episodes_batch(tasks, T, ctx, host_out=host_out)
    dt = (time.perf_counter() - t0) / 3
    print(f"S={S}: {dt*1e3:.1f} ms/step  {12*E*T/dt:.3e} config-steps/s")
