"""Validation: K7 sa_search at bench scale (4 ResNet-18 tasks x 4096 chains x 500 steps) equals the
oracle restatement (oracle/ktune_oracle.c ko_sa_search, all host threads): states, fitness, acceptances."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from oracle import pyoracle as O
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import SaParams, SaTask, sa_search_batch
from paper_2001_08743_b200.spaces import stream_seed
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context
class A: tasks = 4; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
p = SaParams(4096, 500)
t0 = time.perf_counter()
got = sa_search_batch([SaTask(d, g, np.ascontiguousarray(s.init_idx, np.uint16), 0, s.seed) for s, d, g in zip(specs, spaces, gbts)], p)
tg = time.perf_counter() - t0
ok = True
tr = 0.0
for s, m, o in zip(specs, models, got):
    og = O.Gbt(m.base_prediction, m.learning_rate, m.num_features, m.offsets, m.feature, m.left, m.right,
               m.threshold, m.value, m.training_sse)
    t1 = time.perf_counter()
    want = O.sa_search(O.OSpace(s.space), og, s.init_idx, p.max_steps, 0, stream_seed(s.seed, "sa"),
                       p.initial_temperature, p.cooling_rate, threads=os.cpu_count() or 1)
    tr += time.perf_counter() - t1
    eq = (np.array_equal(o["idx"].astype(np.int32), want["idx"]) and np.array_equal(o["score"], want["score"])
          and np.array_equal(o["accepted"], want["accepted"]))
    ok = ok and eq
    print(f"task {s.space.workload}: {'EQUAL' if eq else 'DIFFERENT'}", flush=True)
print(f"SA parity over {4 * 4096 * 500:.3e} chain-steps: {'EQUAL' if ok else 'DIFFERENT'} "
      f"(GPU {tg*1e3:.0f} ms incl. host copies; oracle {tr:.1f} s on {os.cpu_count()} threads)")
