"""Debug (library built with -DKT_TC_TRACE=1, e.g. KTUNE_LIB_PATH=build_ab/lib_trace.so): per-phase clock64 trace of the tcgen05 rollout (CTA 0, each slot's leader, steps 200-201)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context
class A: tasks = int(os.environ.get("TASKS", "12")); episodes = int(os.environ.get("E", "4096")); seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
E, T = A.episodes, 300
inits = [torch.from_numpy(s.init_idx.astype(np.uint16)).cuda() for s in specs]
tasks = [RolloutTask(d, a, None, i, 0, s.seed) for s, d, a, g, i in zip(specs, spaces, agents, gbts, inits)]
run_episodes_batch(tasks, T, ctx)
ctx.set_option(L.OPT_ROLLOUT_CHECK, 2)
run_episodes_batch(tasks, T, ctx)
torch.cuda.synchronize()
lib = L.lib()
# read the trace buffer through the ctx's device counters pointer (debug only)
class Ctx(C.Structure):
    pass
buf = np.zeros(4 + 128 + 1024, np.uint64)
lib.ktune_debug_trace.restype = C.c_int
ctx.check(lib.ktune_debug_trace(ctx.h, buf.ctypes.data_as(C.c_void_p)))
tr = buf[4:132].reshape(8, 16).astype(np.int64)
names = ["start", "bar1", "L1 wait", "L1 epi a", "bar2", "epi b", "L2a wait", "fallbk", "bar3", "L2b wait", "apply", "bar4",
         "value", "L3 wait", "knobs", "end"]
for row in range(8):
    s = tr[row]
    if s[0] == 0: continue
    print(f"slot {row//2} step {200 + row % 2}: total {s[15]-s[0]}")
    print("   " + " ".join(f"{names[k]}:{s[k]-s[0]}" for k in sorted(range(16), key=lambda k: s[k]) if s[k]))

gt = buf[132:132 + 512].reshape(256, 2).astype(np.int64)
ck = buf[132 + 512:132 + 1024].reshape(2, 256).astype(np.int64)
live = gt[:, 0] > 0
if not live.any():
    sys.exit(0)
t0 = gt[live, 0].min()
dur = (gt[live, 1] - gt[live, 0]) / 1e6
cyc = ck[1, live] - ck[0, live]
print(f"CTAs {live.sum()}: duration ms min {dur.min():.3f} median {np.median(dur):.3f} max {dur.max():.3f}; "
      f"start spread {(gt[live,0].max()-t0)/1e6:.3f} ms; effective clock GHz median {np.median(cyc/((gt[live,1]-gt[live,0]))):.3f}")
