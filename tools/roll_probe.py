"""Rollout kernel probe (bench workload, device buffers): K2-TC and K1 CUDA-event times,
fallback rate, and (CHECK=1) the check-mode mismatch count / max |p_fast - p_exact|.
  T=500 python tools/roll_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from paper_2001_08743_b200.distributed import create_context
from workloads.tasks import encode

class A: tasks = int(os.environ.get("TASKS", "12")); episodes = int(os.environ.get("E", "4096")); seed = 0
args = A()
ctx = create_context(0, 0, 1)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
specs = bench.build_tasks(args, 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T = args.episodes, int(os.environ.get("T", "500"))
inits = [torch.from_numpy(s.init_idx[:E].astype(np.uint16)).cuda() for s in specs]
tasks = [RolloutTask(d, a, g, i, 0, s.seed) for s, d, a, g, i in zip(specs, spaces, agents, gbts, inits)]
mkd = lambda shape, dt: torch.empty(shape, dtype=dt, device="cuda")
sm = bool(int(os.environ.get("STEP", "0")))  # step-major trajectories
sh = lambda rows, *rest: ((rows, E) if sm else (E, rows)) + rest
out = [dict(idx=mkd(sh(T + 1, 8), torch.uint16), score=mkd(sh(T + 1), torch.float64), actions=mkd(sh(T, 8), torch.int8),
            logp=mkd(sh(T), torch.float64), value=mkd(sh(T), torch.float64)) for _ in specs]
chk = int(os.environ.get("CHECK", "0"))
for _ in range(2):
    run_episodes_batch(tasks, T, ctx, host_out=out, step_major=sm)
torch.cuda.synchronize()
ref = [{k: v.clone() for k, v in o.items()} for o in out] if chk else None
ctx.set_option(L.OPT_PROFILE, 1)
if chk: ctx.set_option(L.OPT_ROLLOUT_CHECK, chk)
if os.environ.get("FUSE"): ctx.set_option(L.OPT_ROLLOUT_FUSE_GBT, int(os.environ["FUSE"]))
if os.environ.get("DELTA"):  # the certification band in probability units
    ctx.set_option(L.OPT_ROLLOUT_DELTA, int(float(os.environ["DELTA"]) * 1e12))

keys = [L.STAT_ROLLOUT_NS, L.STAT_ROLLOUT_CALLS, L.STAT_GBT_NS, L.STAT_GBT_CALLS, L.STAT_ROLLOUT_FALLBACKS,
        L.STAT_ROLLOUT_TC, L.STAT_ROLLOUT_CHECKED, L.STAT_ROLLOUT_MISMATCH, L.STAT_ROLLOUT_MAXERR]
s0 = {k: ctx.stat(k) for k in keys}
reps = int(os.environ.get("REPS", "5"))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if os.environ.get("DMA"):  # interference experiment: D2H copies on another stream during the rollout
    cs = torch.cuda.Stream()
    src = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    dst = torch.empty(64 << 20, dtype=torch.uint8, pin_memory=True)
    with torch.cuda.stream(cs):
        for _ in range(int(os.environ["DMA"])):
            dst.copy_(src, non_blocking=True)
ev0.record(stream)
for i in range(reps):
    run_episodes_batch(tasks, T, ctx, host_out=out, step_major=sm)
ev1.record(stream)
torch.cuda.synchronize()
print(f"whole call (rollout + verification + K1): {ev0.elapsed_time(ev1) / reps:.3f} ms")
d = {k: ctx.stat(k) - s0[k] for k in keys}
roll = d[L.STAT_ROLLOUT_NS] / 1e6 / reps
gbt = d[L.STAT_GBT_NS] / 1e6 / reps
cs = d[L.STAT_ROLLOUT_TC] / reps
print(f"rollout_tc {roll:.3f} ms  gbt {gbt:.3f} ms  config-steps {cs:.0f}  kernel rate {cs / roll / 1e6:.3e}/s  "
      f"fallbacks/cs {d[L.STAT_ROLLOUT_FALLBACKS] / max(1, d[L.STAT_ROLLOUT_TC]):.2e}  "
      f"checked {d[L.STAT_ROLLOUT_CHECKED]} mismatches {d[L.STAT_ROLLOUT_MISMATCH]} maxerr {ctx.stat(L.STAT_ROLLOUT_MAXERR) * 1e-12:.3e}")
if chk:
    same = all(torch.equal(o[k], r[k]) for o, r in zip(out, ref) for k in ("idx", "actions", "score"))
    print("check-mode outputs equal to the fast run's:", same)
