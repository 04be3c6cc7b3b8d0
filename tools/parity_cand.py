"""Validation: device make_candidate_set over a full bench trajectory (4096 episodes x 501 rows of one
ResNet-18 task, ~2M rows) equals the reference build's make_candidate_set (sampling.cpp:16-31)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from oracle import pyoracle as O
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from paper_2001_08743_b200.sampling import candidates_from_rows
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context
class A: tasks = 3; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
ok = True
for s in specs:
    d = Space(s.space, ctx)
    g = DeviceGbt(fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed), d)
    a = ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx)
    o = run_episodes_batch([RolloutTask(d, a, g, s.init_idx, 0, s.seed)], 500, ctx)[0]
    rows_idx = o["idx"].reshape(-1, d.D)
    pred = o["score"].reshape(-1)
    t0 = time.perf_counter(); got = candidates_from_rows(d, rows_idx, pred); tg = time.perf_counter() - t0
    ids = d.id_of(rows_idx)
    t1 = time.perf_counter(); want = O.make_candidate_set(d.D, rows_idx.astype(np.int32), ids, pred, "ref"); tr = time.perf_counter() - t1
    eq = np.array_equal(got.ids, ids[want]) and np.array_equal(got.predicted, pred[want]) and \
         np.array_equal(got.idx, rows_idx[want].astype(np.int32))
    ok = ok and eq
    print(f"{s.space.workload}: {len(pred)} rows -> {len(want)} candidates {'EQUAL' if eq else 'DIFFERENT'} "
          f"(device call {tg*1e3:.0f} ms incl. transfers; reference {tr:.1f} s)", flush=True)
print("ALL EQUAL" if ok else "MISMATCH")
