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


def _merge_worker(rank, world, port, q):
    """The distributed CandidateSet protocol of ktune_candidates_gather (counts all-gather,
    padded row all-gather, rank-ordered union, make_candidate_set of the union) over the
    product's host transport (distributed.host_collectives), with the oracle's
    make_candidate_set standing in for the device sort: equals the single-GPU set."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as O
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.distributed import host_collectives, shard_range
    allreduce, allgather = host_collectives(world)
    sp = O.OSpace(S.synthetic_space(3, 5))
    E, T = 37, 9
    g = np.random.default_rng(2)
    init = np.stack([g.integers(0, c, E) for c in sp.card], 1).astype(np.int32)
    p = O.ac_init(5, 16, 8, 4)
    gb = O.fitted_model(sp, seed=1, n_train=200) if O.ref_available() else None
    lo, hi = shard_range(E, rank, world)
    part = O.run_episodes(sp, gb, 16, 8, p, init[lo:hi], T, lo, 7)
    rows_idx = part["idx"].reshape(-1, 5)
    pred = part["score"].reshape(-1)
    keep = O.make_candidate_set(5, rows_idx, sp.ids(rows_idx), pred)
    m = np.array([len(keep)], np.int64)
    cnt = np.zeros(world, np.int64)
    allgather(m.view(np.uint8), cnt.view(np.uint8))
    M = int(cnt.max())
    send = np.zeros((M, 5 * 2 + 8), np.uint8)  # padded rows: idx uint16 x D, then pred
    send[:len(keep), :10] = rows_idx[keep].astype(np.uint16).view(np.uint8).reshape(len(keep), 10)
    send[:len(keep), 10:] = pred[keep].view(np.uint8).reshape(len(keep), 8)
    recv = np.zeros((world * M, 18), np.uint8)
    allgather(send.reshape(-1), recv.reshape(-1))
    parts = [recv[r * M:r * M + cnt[r]] for r in range(world)]
    u = np.concatenate(parts)
    uidx = u[:, :10].copy().view(np.uint16).astype(np.int32).reshape(-1, 5)
    upred = u[:, 10:].copy().view(np.float64).reshape(-1)
    sel = O.make_candidate_set(5, uidx, sp.ids(uidx), upred)
    tot = np.array([float(len(sel))])
    allreduce(tot)  # the float64 all-reduce path
    if rank == 0:
        full = O.run_episodes(sp, gb, 16, 8, p, init, T, 0, 7)
        fidx = full["idx"].reshape(-1, 5)
        fp = full["score"].reshape(-1)
        want = O.make_candidate_set(5, fidx, sp.ids(fidx), fp)
        q.put(bool(np.array_equal(uidx[sel], fidx[want]) and np.array_equal(upred[sel], fp[want])
                   and tot[0] == world * len(sel)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_candidate_merge_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_merge_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
