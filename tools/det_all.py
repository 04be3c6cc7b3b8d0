"""Debug: determinism of every device path at bench scale (two runs, hashes compared)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2001_08743_b200.context import Space
from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, SaParams, SaTask, run_episodes_batch, sa_search_batch
from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, candidates_from_rows
from workloads.tasks import encode
from paper_2001_08743_b200.distributed import create_context
H = lambda t: hashlib.sha1((t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)).tobytes()).hexdigest()[:10]
class A: tasks = 12; episodes = 4096; seed = 0
ctx = create_context(0, 0, 1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st); ctx.set_stream(st.cuda_stream)
specs = bench.build_tasks(A(), 0)
models = [fit_gbt(encode(s.space, s.train_idx), s.train_y, seed=s.seed) for s in specs]
spaces = [Space(s.space, ctx) for s in specs]
gbts = [DeviceGbt(m, d) for m, d in zip(models, spaces)]
agents = [ActorCritic(s.space.num_knobs, 128, 64, seed=s.seed, ctx=ctx) for s in specs]
inits = [torch.from_numpy(s.init_idx.astype(np.uint16).view(np.int16)).cuda().view(torch.uint16) for s in specs]
tasks = [RolloutTask(d, a, g, i, 0, s.seed) for s, d, a, g, i in zip(specs, spaces, agents, gbts, inits)]
res = []
for rep in range(2):
    o = run_episodes_batch(tasks, 500, ctx, device_out=True)
    torch.cuda.synchronize()
    h_roll = "".join(H(x["idx"].view(torch.int16)) + H(x["score"]) + H(x["actions"]) + H(x["logp"]) for x in o[:3])
    rows, ids = candidates_from_rows(spaces[0], o[0]["idx"].view(-1, 8), o[0]["score"].view(-1))
    torch.cuda.synchronize()
    h_cand = H(rows) + H(ids.view(torch.int64))
    sa = sa_search_batch([SaTask(d, g, np.ascontiguousarray(s.init_idx, np.uint16), 0, s.seed) for s, d, g in zip(specs[:4], spaces[:4], gbts[:4])],
                         SaParams(4096, 500))
    h_sa = "".join(H(x["idx"]) + H(x["score"]) + H(x["accepted"]) for x in sa)
    cidx = o[0]["idx"].view(torch.int16).view(-1, 8)[rows[:1_000_000]].to(torch.uint8)
    sw = adaptive_sweep(spaces[0], CandidateSet(cidx, ids[:1_000_000].view(torch.int64), None), SamplingParams(), 3)
    torch.cuda.synchronize()
    h_sw = H(sw.assignments) + H(sw.snapped) + str(sw.k) + repr(sw.k_losses)
    res.append((h_roll, h_cand, h_sa, h_sw))
    print(f"rep {rep}: rollout {h_roll[:20]} cand {h_cand} sa {h_sa[:20]} sweep {h_sw[:30]}", flush=True)
print("DETERMINISTIC" if res[0] == res[1] else "MISMATCH: " + str([a == b for a, b in zip(*res)]))
