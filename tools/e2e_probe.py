"""e2e probe: the bench's host-buffer rollout (pinned buffers, H2D of the initial configs and
D2H of the trajectory inside the timing) for layout x score-precision variants.
  python tools/e2e_probe.py"""
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

class A: tasks = 12; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T, D = 4096, int(os.environ.get("T", "500")), 8
pinned = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()
host_init = [pinned(s.init_idx.shape, torch.int16).view(np.uint16) for s in specs]
for h, s in zip(host_init, specs):
    h[:] = s.init_idx
htasks = [RolloutTask(d, a, g, hi, 0, s.seed) for s, d, a, g, hi in zip(specs, spaces, agents, gbts, host_init)]
for seg in [int(x) for x in os.environ.get("SEGS", "0").split(",")]:
    ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, seg)
    for s64 in (False, True):
        from paper_2001_08743_b200.exploration import compact_grouped_outputs
        tdt = {np.uint8: torch.uint8, np.uint16: torch.int16, np.float32: torch.float32, np.float64: torch.float64}
        out = compact_grouped_outputs(htasks, T, lambda shape, dt: pinned(shape, tdt[dt]).view(dt) if dt == np.uint16
                                      else pinned(shape, tdt[dt]), score64=s64, logp64=s64)
        run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            run_episodes_batch(htasks, T, ctx, host_out=out, grouped=True)
            ts.append(time.perf_counter() - t0)
        bo = sum(sum(v.nbytes for v in o.values() if v is not None) for o in out)
        ms = 1e3 * np.median(ts)
        print(f"segs {seg} grouped step-major score {'f64' if s64 else 'f32'}: {ms:.2f} ms/step, "
              f"{12 * E * T / ms * 1e3:.3e} config-steps/s, D2H {bo / 1e9:.3f} GB ({bo / ms / 1e6:.1f} GB/s)", flush=True)
    for step_major in (() if os.environ.get("GROUPED_ONLY") else (False, True)):
        for s64 in (False, True):
            sh = lambda rows, *rest: ((rows, E) if step_major else (E, rows)) + rest
            small = [max(s.space.cards) <= 256 for s in specs]
            out = [dict(idx=None if sm else pinned(sh(T + 1, D), torch.int16).view(np.uint16),
                        idx8=pinned(sh(T + 1, D), torch.uint8) if sm else None,
                        score=pinned(sh(T + 1), torch.float64) if s64 else None,
                        score32=None if s64 else pinned(sh(T + 1), torch.float32), actions=None,
                        actions2=pinned(sh(T, 2), torch.uint8), logp=None, value=None,
                        logp32=pinned(sh(T), torch.float32), value32=pinned(sh(T), torch.float32)) for sm in small]
            run_episodes_batch(htasks, T, ctx, host_out=out, step_major=step_major)
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                t0 = time.perf_counter()
                run_episodes_batch(htasks, T, ctx, host_out=out, step_major=step_major)
                ts.append(time.perf_counter() - t0)
            bo = sum(sum(v.nbytes for v in o.values() if v is not None) for o in out)
            ms = 1e3 * np.median(ts)
            print(f"segs {seg} {'step' if step_major else 'episode'}-major score {'f64' if s64 else 'f32'}: "
                  f"{ms:.2f} ms/step, {12 * E * T / ms * 1e3:.3e} config-steps/s, D2H {bo / 1e9:.3f} GB "
                  f"({bo / ms / 1e6:.1f} GB/s)", flush=True)
