"""Timeline of the adaptive sweep over a large device-resident candidate set (SURVEY C3's k-means
stage: ~27.7M VGG-16 candidates): kernel mix and idle time from CUPTI via torch.profiler.
  N=27700000 python tools/sweep_timeline.py"""
import collections, json, os, re, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2001_08743_b200 import spaces as S
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
from workloads.tasks import random_configs
ctx = Context(0)
sp = S.vgg16_tasks()[3]
ds = Space(sp, ctx)
N = int(os.environ.get("N", 27_700_000))
idx = random_configs(sp, N, 5)
ids = ds.id_of(idx)
_, first = np.unique(ids, return_index=True)
keep = np.sort(first)
didx = torch.from_numpy(np.ascontiguousarray(idx[keep], dtype=ds.idx_dtype)).cuda()
dids = torch.from_numpy(ids[keep].astype(np.uint64).view(np.int64)).cuda()
cs = CandidateSet(didx, dids, None)
adaptive_sweep(ds, cs, SamplingParams(), 5)
torch.cuda.synchronize()
t0 = time.perf_counter(); sw = adaptive_sweep(ds, cs, SamplingParams(), 5); torch.cuda.synchronize()
print(f"N={len(keep)} sweep {1e3 * (time.perf_counter() - t0):.1f} ms, k={sw.k}")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    adaptive_sweep(ds, cs, SamplingParams(), 5)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/sweep_trace.json")
ev = json.load(open("gpurun_out/sweep_trace.json"))["traceEvents"]
gpu = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
span = (gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]) / 1e3
agg = collections.defaultdict(lambda: [0, 0.0])
for e in gpu:
    m = re.search(r"::(\w+?)(<|\()", e["name"])
    agg[m.group(1) if m else e["name"][:40]][0] += 1
    agg[m.group(1) if m else e["name"][:40]][1] += e["dur"] / 1e3
busy = sum(v[1] for v in agg.values())
print(f"GPU span {span:.1f} ms, busy {busy:.1f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
    print(f"  {t:8.2f} ms {n:5d}  {k}")
