"""Timeline of one host-buffer rollout call (the bench's e2e: grouped step-major, compact
outputs with configuration ids) from CUPTI via torch.profiler: per segment, when the rollout
kernel, the scoring/packing kernels and the D2H copies run, and how busy the copy engine is.
  python tools/e2e_timeline.py   (SEGS=<S> to force the segment count)"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch, compact_grouped_outputs
from paper_2001_08743_b200.distributed import create_context
from workloads.tasks import encode

class A: tasks = 12; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T = 4096, int(os.environ.get("T", "500"))
pinned = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
host_init = [pinned(s.init_idx.shape, torch.int16).view(np.uint16) for s in specs]
for h, s in zip(host_init, specs):
    h[:] = s.init_idx
htasks = [RolloutTask(d, a, g, hi, 0, s.seed) for s, d, a, g, hi in zip(specs, spaces, agents, gbts, host_init)]
if os.environ.get("SEGS"):
    ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, int(os.environ["SEGS"]))
tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.uint32: torch.int32, np.float32: torch.float32,
       np.float64: torch.float64}
ids = os.environ.get("IDS", "1") == "1"
out = compact_grouped_outputs(htasks, T, lambda shape, dt: pinned(shape, tdt[dt]).view(dt) if dt in (np.uint16, np.uint32)
                              else pinned(shape, tdt[dt]), ids=ids)
for _ in range(3):
    run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
    ts.append(time.perf_counter() - t0)
print(f"call wall ms (no profiler): median {1e3 * np.median(ts):.2f}  all {[round(1e3 * x, 2) for x in ts]}")
ctx.set_option(L.OPT_PROFILE, 1)  # library-side CUDA events around the rollout / K1 launches
ctx.reset_stats()
for _ in range(5):
    run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
print(f"event-timed: rollout {ctx.stat(L.STAT_ROLLOUT_NS) / 5e6:.3f} ms, K1 {ctx.stat(L.STAT_GBT_NS) / 5e6:.3f} ms per call")
ctx.set_option(L.OPT_PROFILE, 0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
    torch.cuda.synchronize()
path = "gpurun_out/e2e_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
t0 = min(e["ts"] for e in gpu)
rows = sorted(((e["ts"] - t0) / 1e3, e["dur"] / 1e3, e["cat"], e["name"][:40], e.get("args", {}).get("stream"),
               e.get("args", {}).get("bytes")) for e in gpu)
end = max(r[0] + r[1] for r in rows)
print(f"GPU span {end:.2f} ms, {len(rows)} activities")
cp = [r for r in rows if r[2] == "gpu_memcpy" and "DtoH" in r[3]]
kb = [r for r in rows if r[2] == "kernel"]
busy_cp = sum(r[1] for r in cp)
nbytes = sum(r[5] or 0 for r in cp)
print(f"D2H: {len(cp)} copies, {nbytes / 1e6:.1f} MB, busy {busy_cp:.2f} ms ({nbytes / busy_cp / 1e6:.1f} GB/s while busy), "
      f"first starts {cp[0][0]:.2f} ms, last ends {cp[-1][0] + cp[-1][1]:.2f} ms")
ro = [r for r in kb if "rollout" in r[3]]
print(f"rollout kernels: {len(ro)}, busy {sum(r[1] for r in ro):.2f} ms, last ends {ro[-1][0] + ro[-1][1]:.2f} ms; "
      f"other kernels busy {sum(r[1] for r in kb if r not in ro):.2f} ms")
for r in rows:
    if r[2] == "kernel" or r[1] > 0.05:
        print(f"  {r[0]:8.3f} +{r[1]:7.3f}  {r[2]:10s} s{r[4]} {r[3]} {'' if r[5] is None else r[5]}")
