"""Debug: sa_search kernel time (device buffers, grouped 12 tasks) vs the Python host path."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import SaParams, sa_search
from paper_2001_08743_b200.spaces import stream_seed
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context
class A: tasks = 12; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
E, T, D = 4096, int(os.environ.get("T", 500)), 8
ins = [torch.from_numpy(np.ascontiguousarray(s.init_idx, np.uint16).view(np.int16)).cuda() for s in specs]
idx = [torch.empty((E, T + 1, D), dtype=torch.int16, device="cuda") for _ in specs]
sc = [torch.empty((E, T + 1), dtype=torch.float64, device="cuda") for _ in specs]
ac = [torch.empty((E, T), dtype=torch.uint8, device="cuda") for _ in specs]
tasks = (L.SaTaskC * 12)(*[L.SaTaskC(d.h, g.h, E, 0, stream_seed(s.seed, "sa"), ins[i].data_ptr(), idx[i].data_ptr(),
                                     sc[i].data_ptr(), ac[i].data_ptr())
                           for i, (s, d, g) in enumerate(zip(specs, spaces, gbts))])
p = L.SaParamsC(1.0, 0.99)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for n in (1, 12):
    for _ in range(2): ctx.check(L.lib().ktune_sa_search(ctx.h, n, tasks, T, C.byref(p), L.F_DEVICE))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): ctx.check(L.lib().ktune_sa_search(ctx.h, n, tasks, T, C.byref(p), L.F_DEVICE))
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"kernel {n} tasks: {ms:.2f} ms  {n*E*T/ms/1e6:.1f} M chain-steps/ms-> {n*E*T/ms*1e3:.3e}/s")
ctx.set_stream(None)
pp = SaParams(num_chains=E, max_steps=T)
sa_search(spaces[0], gbts[0], specs[0].init_idx, pp, rng_seed=1)
for _ in range(2):
    t0 = time.perf_counter(); sa_search(spaces[0], gbts[0], specs[0].init_idx, pp, rng_seed=1); print(f"python 1 task {1e3*(time.perf_counter()-t0):.1f} ms")
