"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: the shard plans the
product uses (paper_2001_08743_b200/distributed.py) and the gather order. The
oracle stands in for the per-rank GPU compute."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rollout_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as O
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.distributed import shard_range
    sp = O.OSpace(S.synthetic_space(4, 6))
    E, T = 13, 11
    init = np.stack([np.random.default_rng(1).integers(0, c, E) for c in sp.card], 1).astype(np.int32)
    p = O.ac_init(6, 16, 8, 2)
    lo, hi = shard_range(E, rank, world)
    part = O.run_episodes(sp, None, 16, 8, p, init[lo:hi], T, lo, 99)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, part["idx"], part["logp"]))
    if rank == 0:
        full = O.run_episodes(sp, None, 16, 8, p, init, T, 0, 99)
        idx = np.concatenate([g[1] for g in sorted(gathered, key=lambda x: x[0])])
        lp = np.concatenate([g[2] for g in sorted(gathered, key=lambda x: x[0])])
        q.put(bool(np.array_equal(idx, full["idx"]) and np.array_equal(lp, full["logp"])))
    dist.destroy_process_group()


def _assign(P, C):
    # the reference's sequential-over-knob d2 (sampling.cpp:45), vectorised
    s = (P[:, None, 0] - C[None, :, 0]) ** 2
    for d in range(1, P.shape[1]):
        s = s + (P[:, None, d] - C[None, :, d]) ** 2
    return np.argmin(s, axis=1).astype(np.int32), s.min(axis=1)


def _kmeans_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2001_08743_b200.distributed import kmeans_chunk_range
    g = np.random.default_rng(5)
    N, D, k = 5000, 8, 9
    P = g.integers(0, 7, (N, D)) / 6.0
    C = g.random((k, D))
    lo, hi = kmeans_chunk_range(N, rank, world)
    a, d2 = _assign(P[lo:hi], C)  # this rank's shard of the assignment
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, a, d2))
    if rank == 0:
        full_a, full_d2 = _assign(P, C)
        parts = sorted(gathered, key=lambda x: x[0])
        covered = sum(len(p[1]) for p in parts)
        a_cat = np.concatenate([p[1] for p in parts])
        d_cat = np.concatenate([p[2] for p in parts])
        q.put(bool(covered == N and np.array_equal(a_cat, full_a) and np.array_equal(d_cat, full_d2)))
    dist.destroy_process_group()


@pytest.mark.parametrize("worker", [_rollout_worker, _kmeans_worker])
def test_world2_gloo(worker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True


@pytest.mark.parametrize("n,world", [(1, 2), (1023, 2), (1024, 2), (5000, 3), (1 << 20, 8), (7, 8)])
def test_shard_plans_cover_exactly(n, world):
    from paper_2001_08743_b200.distributed import kmeans_chunk_range, shard_range
    for fn in (shard_range, kmeans_chunk_range):
        ranges = [fn(n, r, world) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == n
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    lo, hi = kmeans_chunk_range(n, 1, world)
    assert lo % 1024 == 0 or lo == n
