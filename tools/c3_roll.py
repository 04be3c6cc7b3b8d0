"""Debug: C3 rollout (65,536 episodes x 500, VGG-16 c4) timing distribution, device-resident."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from paper_2001_08743_b200.workloads import encode, make_tasks
from paper_2001_08743_b200.distributed import create_context
ctx = create_context(0, 0, 1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
sp = S.vgg16_tasks()[3]
E = int(os.environ.get("E", 65536))
spec = make_tasks([sp], E, seed=33)[0]
ds = Space(sp, ctx)
g = DeviceGbt(fit_gbt(encode(sp, spec.train_idx), spec.train_y, seed=spec.seed), ds)
agent = ActorCritic(sp.num_knobs, 128, 64, seed=spec.seed, ctx=ctx)
init = torch.from_numpy(spec.init_idx.astype(np.uint16).view(np.int16)).cuda().view(torch.uint16)
task = RolloutTask(ds, agent, g if not os.environ.get("NOGBT") else None, init, 0, spec.seed)
ts = []
for i in range(10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(st)
    o = run_episodes_batch([task], 500, ctx, device_out=True)
    ev[1].record(st); torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
    del o
print(f"E={E}: rollout ms " + " ".join(f"{t:.1f}" for t in ts))
