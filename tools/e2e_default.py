"""Debug: run_episodes_batch with default (pageable numpy) outputs vs caller-pinned outputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
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
tasks = [RolloutTask(d, a, g, s.init_idx, 0, s.seed) for s, d, a, g in zip(specs, spaces, agents, gbts)]
T = 500
run_episodes_batch(tasks, T, ctx)
for _ in range(4):
    t0 = time.perf_counter(); o = run_episodes_batch(tasks, T, ctx); dt = time.perf_counter() - t0
    print(f"default outputs: {dt*1e3:.1f} ms  {12*4096*T/dt:.3e} config-steps/s  ({sum(v.nbytes for x in o for v in x.values() if v is not None)/1e9:.2f} GB)")
