"""Validation: the certified tcgen05 rollout equals the exact fp64 kernel on the SURVEY C5 workload
(synthetic 16-knob space, 1M episodes x 1000 steps = 1.05e9 config-steps), compared chunk by chunk."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from workloads.tasks import encode, make_tasks
from paper_2001_08743_b200.distributed import create_context
ctx = create_context(0, 0, 1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
E, T, CH = int(os.environ.get("E", 1 << 20)), int(os.environ.get("T", 1000)), int(os.environ.get("CH", 1 << 18))
sp = S.synthetic_space(0, 16)
spec = make_tasks([sp], E, seed=99)[0]
ds = Space(sp, ctx)
g = DeviceGbt(fit_gbt(encode(sp, spec.train_idx), spec.train_y, seed=spec.seed), ds)
agent = ActorCritic(16, 128, 64, seed=spec.seed, ctx=ctx)
tot = dict(steps=0, idx=0, act=0, score=0)
lp_rel = v_rel = 0.0
ctx.reset_stats()
t0 = time.perf_counter()
for e0 in range(0, E, CH):
    init = torch.from_numpy(spec.init_idx[e0:e0 + CH].astype(np.uint16).view(np.int16)).cuda().view(torch.uint16)
    task = RolloutTask(ds, agent, g, init, e0, spec.seed)
    f = run_episodes_batch([task], T, ctx, device_out=True)[0]
    x = run_episodes_batch([task], T, ctx, device_out=True, exact=True)[0]
    torch.cuda.synchronize()
    tot["steps"] += init.shape[0] * T
    tot["idx"] += int((f["idx"].view(torch.int16) != x["idx"].view(torch.int16)).sum())
    tot["act"] += int((f["actions"] != x["actions"]).sum())
    tot["score"] += int((f["score"] != x["score"]).sum())
    lp_rel = max(lp_rel, float(((f["logp"] - x["logp"]).abs() / x["logp"].abs().clamp(min=1.0)).max()))
    v_rel = max(v_rel, float(((f["value"] - x["value"]).abs() / x["value"].abs().clamp(min=1.0)).max()))
    del f, x
    print(f"episodes {e0 + init.shape[0]}: mismatches idx {tot['idx']} actions {tot['act']} scores {tot['score']}; "
          f"max rel logp {lp_rel:.2e} value {v_rel:.2e} ({time.perf_counter() - t0:.0f} s)", flush=True)
print(f"C5 parity over {tot['steps']:.3e} config-steps: idx/actions/scores mismatches "
      f"{tot['idx']}/{tot['act']}/{tot['score']}, max rel logp {lp_rel:.2e}, value {v_rel:.2e}; "
      f"certified re-decisions {ctx.stat(L.STAT_ROLLOUT_FALLBACKS)}")
