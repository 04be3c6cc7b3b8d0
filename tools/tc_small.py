"""Debug: one small tcgen05 rollout (for compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from helpers import SPACES
from paper_2001_08743_b200.context import Context, Space
from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
name = sys.argv[1] if len(sys.argv) > 1 else "synthetic16"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ctx = Context(0)
sp = SPACES[name]()
ds = Space(sp, ctx)
agent = ActorCritic(sp.num_knobs, 128, 64, seed=3, ctx=ctx)
init = np.zeros((E, sp.num_knobs), np.int32)
out = run_episodes_batch([RolloutTask(ds, agent, None, init, 0, 1)], 30, ctx)[0]
print("ok", out["idx"][:2, -1])
