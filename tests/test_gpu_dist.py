"""The multi-GPU data plane of the product, run by W real processes (ranks) that share the
one GPU of the test box: every library collective (the sharded k-means exchanges and the
distributed CandidateSet merge) goes through the host transport of
ktune_ctx_create_hostcomm over a gloo group instead of NCCL — the same sharded code paths
(kmeans.cu `sharded`, candidates.cu ktune_candidates_gather) the NCCL runs take.

Per rank: the rollout of its episode shard (global episode ids), the global CandidateSet
gathered from every rank, the adaptive k-sweep + snap (sharded certified Lloyd) and
kmeans_run in both centroid modes. Rank 0's results, and every rank's digest, must equal
the single-process (world 1) pipeline bit for bit."""
import hashlib
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E, T = 3000, 40


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pipeline(ctx, rank, world):
    import torch
    from helpers import SPACES, fitted
    from oracle import pyoracle as O
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.distributed import shard_range
    from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.sampling import (CandidateSet, SamplingParams, adaptive_sweep, candidates_from_rows,
                                                candidates_gather, kmeans_run)
    sp = SPACES["resnet_c2"]()
    osp, og, pm = fitted(O, sp, seed=3)
    ds = Space(sp, ctx)
    agent = ActorCritic(sp.num_knobs, 128, 64, seed=5, ctx=ctx)
    init = osp.random_valid(1, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
    lo, hi = shard_range(E, rank, world)
    dinit = torch.from_numpy(init[lo:hi].astype(np.int32)).cuda()
    o = run_episodes_batch([RolloutTask(ds, agent, DeviceGbt(pm, ds), dinit, lo, 9)], T, ctx, device_out=True)[0]
    D = sp.num_knobs
    if world > 1:
        c = candidates_gather(ds, o["idx"].reshape(-1, D), o["score"].reshape(-1))
        cidx, cids, cpred = c.idx, c.ids, c.predicted
    else:
        rows, ids = candidates_from_rows(ds, o["idx"].reshape(-1, D), o["score"].reshape(-1))
        cidx = o["idx"].reshape(-1, D).view(torch.int16)[rows]
        cids, cpred = ids.view(torch.int64), o["score"].reshape(-1)[rows]
    cidx8 = cidx.to(torch.uint8)
    out = {"cand_idx": cidx.cpu().numpy(), "cand_ids": cids.cpu().numpy(), "cand_pred": cpred.cpu().numpy()}
    sw = adaptive_sweep(ds, CandidateSet(cidx8, cids, None), SamplingParams(k_max_exclusive=24), rng_seed=11)
    out.update(sweep_k=np.array([sw.k]), sweep_losses=np.array(sw.k_losses), sweep_asg=sw.assignments.cpu().numpy(),
               sweep_cent=sw.centroids.cpu().numpy(), sweep_snap=sw.snapped.cpu().numpy())
    hidx = out["cand_idx"].astype(np.int32)
    # certified integer-sum centroids (mode B), exact-order centroids (mode A), and mode B with
    # inflated bounds so that certified batches fail and the exact rescue runs (sharded)
    for name, mode, log2 in (("km_b", 0, 0), ("km_a", 1, 0), ("km_rescue", 0, 40)):
        ctx.set_option(L.OPT_KMEANS_MODE, mode)
        ctx.set_option(L.OPT_KMEANS_BOUND_LOG2, log2)
        ctx.reset_stats()
        r = kmeans_run(ds, hidx, 13, 21 + mode, restarts=2)
        out[f"{name}_asg"], out[f"{name}_cent"] = r.assignments, r.centroids
        out[f"{name}_loss"] = np.array([r.l2_loss])
        # per-iteration losses are parallel estimates (<= 1e-12 relative, summed
        # per rank then all-reduced); the final loss is the exact sequential sum
        out[f"{name}_iters"] = np.array(r.iteration_losses)
        if log2:
            out[f"{name}_aborted"] = np.array([ctx.stat(L.STAT_KMEANS_ABORTS) > 0])
    ctx.set_option(L.OPT_KMEANS_MODE, 0)
    ctx.set_option(L.OPT_KMEANS_BOUND_LOG2, 0)
    return out


def _digest(out):
    h = hashlib.sha256()
    for k in sorted(out):
        if k.endswith("_iters"):
            continue
        h.update(k.encode())
        h.update(np.ascontiguousarray(out[k]).tobytes())
    return h.hexdigest()


def _worker(rank, world, port, q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2001_08743_b200.distributed import create_context
    ctx = create_context(0, rank, world, transport="host")
    try:
        out = _pipeline(ctx, rank, world)
        q.put((rank, _digest(out), out if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_pipeline_equals_single_gpu(world):
    import torch.multiprocessing as mp
    from paper_2001_08743_b200.context import Context
    want = _pipeline(Context(0), 0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(p.exitcode == 0 for p in procs)
    got = [r[2] for r in res if r[0] == 0][0]
    for k in want:
        if k.endswith("_iters"):
            assert len(got[k]) == len(want[k]) and np.allclose(got[k], want[k], rtol=1e-12, atol=0), k
        else:
            assert np.array_equal(got[k], want[k]), k
    assert want["km_rescue_aborted"][0]
    assert len({r[1] for r in res}) == 1 and res[0][1] == _digest(want)  # every rank holds the same state
