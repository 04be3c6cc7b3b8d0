"""Diagnostic: host/device time split of one bench step (device buffers)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context

class A: tasks = 12; episodes = 4096; seed = 0
args = A()
exact = len(sys.argv) > 1 and sys.argv[1] == "exact"
ctx = create_context(0, 0, 1)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
specs = bench.build_tasks(args, 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T = 4096, int(os.environ.get("T", "500"))
inits = [torch.from_numpy(s.init_idx.astype(np.uint16)).cuda() for s in specs]
tasks = [RolloutTask(d, a, g, i, 0, s.seed) for s, d, a, g, i in zip(specs, spaces, agents, gbts, inits)]
mkd = lambda shape, dt: torch.empty(shape, dtype=dt, device="cuda")
out = [dict(idx=mkd((E, T + 1, 8), torch.uint16), score=mkd((E, T + 1), torch.float64), actions=mkd((E, T, 8), torch.int8),
            logp=mkd((E, T), torch.float64), value=mkd((E, T), torch.float64)) for _ in specs]
for _ in range(2):
    run_episodes_batch(tasks, T, ctx, host_out=out, exact=exact)
torch.cuda.synchronize()
mode = os.environ.get("MODE", "")
if os.environ.get("CHECKMODE"): ctx.set_option(L.OPT_ROLLOUT_CHECK, int(os.environ["CHECKMODE"]))
if os.environ.get("DELTA"): ctx.set_option(L.OPT_ROLLOUT_DELTA, int(float(os.environ["DELTA"]) * 1e12))  # probability units
if "prof" in mode: ctx.set_option(L.OPT_PROFILE, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clk = None
if "smi" in mode:
    clk = bench.ClockSampler(0); clk.__enter__()
for i in range(4):
    if "flush" in mode: flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    t0 = time.perf_counter(); ev[0].record(stream)
    run_episodes_batch(tasks, T, ctx, host_out=out, exact=exact)
    t1 = time.perf_counter(); ev[1].record(stream)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"host enqueue {1e3*(t1-t0):.2f} ms, host total {1e3*(t2-t0):.2f} ms, device {ev[0].elapsed_time(ev[1]):.2f} ms", flush=True)
if "nosync" in mode:
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize(); t0 = time.perf_counter(); ev[0].record(stream)
    for i in range(5):
        if "flush" in mode: flush.zero_()
        run_episodes_batch(tasks, T, ctx, host_out=out, exact=exact)
        print(f"  enq {i} at {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
    ev[1].record(stream); torch.cuda.synchronize()
    print(f"5 back-to-back: host {1e3*(time.perf_counter()-t0):.2f} ms device {ev[0].elapsed_time(ev[1]):.2f} ms")
if clk: clk.__exit__(); print(clk.summary())
