"""SURVEY C3's sampling stage as the bench runs it (VGG-16 c4, 65,536 episodes x 500 steps ->
device CandidateSet -> adaptive sweep), with a CUPTI kernel breakdown of the sweep."""
import collections, json, os, re, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_08743_b200 import _lib as L
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, candidates_from_rows
from workloads.tasks import encode, make_tasks
ctx = Context(0)
sp = S.vgg16_tasks()[3]
E = int(os.environ.get("E", 65536))
spec = make_tasks([sp], E, seed=33)[0]
ds = Space(sp, ctx)
g = DeviceGbt(fit_gbt(encode(sp, spec.train_idx), spec.train_y, seed=spec.seed), ds)
agent = ActorCritic(sp.num_knobs, 128, 64, seed=spec.seed, ctx=ctx)
init = torch.from_numpy(spec.init_idx.astype(np.uint16).view(np.int16)).cuda()
task = RolloutTask(ds, agent, g, init.view(torch.uint16), 0, spec.seed)
o = run_episodes_batch([task], 500, ctx, device_out=True)[0]
rows, ids = candidates_from_rows(ds, o["idx"].view(-1, 8), o["score"].view(-1))
cidx = o["idx"].view(torch.int16).view(-1, 8)[rows]
cidx = cidx.to(torch.uint8) if ds.index_bytes == 1 else cidx
cs = CandidateSet(cidx, ids.view(torch.int64), None)
torch.cuda.synchronize()
for rep in range(2):
    ctx.reset_stats()
    t0 = time.perf_counter(); sw = adaptive_sweep(ds, cs, SamplingParams(), spec.seed); torch.cuda.synchronize()
    print(f"N={rows.numel()} sweep {1e3 * (time.perf_counter() - t0):.1f} ms, k={sw.k}, lloyd iters {ctx.stat(L.STAT_LLOYD_ITERS)}, "
          f"kpp picks {ctx.stat(L.STAT_KPP_PICKS)} fallbacks {ctx.stat(L.STAT_KPP_FALLBACKS)}, assign fallbacks {ctx.stat(L.STAT_ASSIGN_FALLBACKS)}, aborts {ctx.stat(L.STAT_KMEANS_ABORTS)}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    adaptive_sweep(ds, cs, SamplingParams(), spec.seed)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/c3_sweep_trace.json")
ev = json.load(open("gpurun_out/c3_sweep_trace.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
span = (gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]) / 1e3
agg = collections.defaultdict(lambda: [0, 0.0])
for e in gpu:
    m = re.search(r"::(\w+?)(<|\()", e["name"])
    agg[m.group(1) if m else e["name"][:40]][0] += 1
    agg[m.group(1) if m else e["name"][:40]][1] += e["dur"] / 1e3
print(f"GPU span {span:.1f} ms, busy {sum(v[1] for v in agg.values()):.1f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"  {t:8.2f} ms {n:5d}  {k}")
