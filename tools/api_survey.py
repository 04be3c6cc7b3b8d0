"""Timing survey of the public API at bench sizes (spots pathological paths)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch, sa_search, SaParams
from paper_2001_08743_b200.sampling import (CandidateSet, SamplingParams, adaptive_sweep, adaptive_sample,
                                            candidates_from_rows, make_candidate_set, kmeans_run)
from paper_2001_08743_b200.workloads import encode, make_tasks, random_configs

def t(label, f, reps=2):
    f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = f()
    torch.cuda.synchronize()
    print(f"{label:60s} {1e3*(time.perf_counter()-t0)/reps:9.2f} ms", flush=True)
    return r

ctx = Context(0)
sp = S.resnet18_tasks()[1]
spec = make_tasks([sp], 4096, seed=3)[0]
ds = Space(sp, ctx)
model = fit_gbt(encode(sp, spec.train_idx), spec.train_y, seed=1)
g = DeviceGbt(model, ds)
agent = ActorCritic(sp.num_knobs, 128, 64, seed=2, ctx=ctx)
X = random_configs(sp, 1 << 20, 5)
t("gbt predict_idx 1M (host arrays)", lambda: g.predict_idx(X) if hasattr(g, "predict_idx") else None)
t("ac forward 256k states (host)", lambda: agent.forward(np.random.default_rng(0).random((1 << 18, sp.num_knobs))))
o = t("run_episodes 4096 x 500 (host arrays)", lambda: run_episodes_batch([RolloutTask(ds, agent, g, spec.init_idx, 0, 1)], 500)[0])
rows = o["idx"].reshape(-1, sp.num_knobs)
t("make_candidate_set host (2M rows)", lambda: make_candidate_set(ds, rows.astype(np.int32), o["score"].reshape(-1)), reps=1)
t("candidates_from_rows device (2M rows)", lambda: candidates_from_rows(ds, rows, o["score"].reshape(-1)))
t("sa_search 4096 chains x 500", lambda: sa_search(ds, g, spec.init_idx, SaParams(4096, 500), rng_seed=1))
sp2 = S.alexnet_tasks()[1]
ds2 = Space(sp2, ctx)
idx = random_configs(sp2, 1 << 20, 123)
ids = ds2.id_of(idx)
_, first = np.unique(ids, return_index=True)
keep = np.sort(first)
cs = CandidateSet(idx[keep], ids[keep], np.zeros(len(keep)))
t("kmeans_run k=8 restarts=3 (1M)", lambda: kmeans_run(ds2, cs.idx, 8, 5, restarts=3))
t("adaptive_sweep (1M)", lambda: adaptive_sweep(ds2, cs, SamplingParams(), 5))
vis = cs.ids[:100000]
t("adaptive_sample with 100k visited (1M)", lambda: adaptive_sample(ds2, cs, vis, SamplingParams(), 5), reps=1)
