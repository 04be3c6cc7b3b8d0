"""Multi-GPU plumbing (one process per GPU, torchrun / torch.distributed).

* Rollout + scoring: episodes are partitioned by contiguous global ranges
  (`shard_range`); each rank passes `episode_offset = lo` so the counter-based
  RNG keys by the GLOBAL episode id -> bit-identical to one GPU, no collective
  on the data path ("episodes may run concurrently").
* End of the rollout: the global CandidateSet is gathered on every rank
  (`sampling.candidates_gather`, ktune_candidates_gather: per-rank dedup + rank,
  an all-gather of the per-rank sets, make_candidate_set of their union), identical
  to the single-GPU CandidateSet.
* k-means: points (the CandidateSet order) are replicated; rank r assigns the
  1024-point chunks `kmeans_chunk_range(N, r, W)` and the per-point
  (assignment, d2) and per-chunk sums are all-gathered over NCCL inside
  libktune_cuda (kmeans.cu, KMeans::assign), so the exact-order centroid sums,
  restart/sweep decisions and snapping run on identical full state everywhere.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

KMEANS_CHUNK = 1024  # kmeans.cu kChunk


def env() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Balanced contiguous [lo, hi) of n items for `rank` of `world`."""
    return n * rank // world, n * (rank + 1) // world


def kmeans_chunk_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Point range [lo, hi) assigned by `rank` (mirrors KMeans::setup/assign)."""
    nchunks = -(-n // KMEANS_CHUNK)
    per = -(-nchunks // world)
    lo = min(n, rank * per * KMEANS_CHUNK)
    hi = min(n, (rank + 1) * per * KMEANS_CHUNK)
    return lo, hi


def host_collectives(world: int):
    """(allreduce, allgather) over the default torch.distributed group on HOST numpy
    buffers: the transport behind ktune_ctx_create_hostcomm (allreduce sums int64/float64
    in place; allgather writes every rank's send bytes into recv in rank order)."""
    import torch
    import torch.distributed as dist

    def allreduce(a):
        dist.all_reduce(torch.from_numpy(a))

    def allgather(send, recv):
        dist.all_gather(list(torch.from_numpy(recv).chunk(world)), torch.from_numpy(send))

    return allreduce, allgather


def create_context(local_rank: int = 0, rank: Optional[int] = None, world: Optional[int] = None,
                   transport: str = "nccl"):
    """A libktune_cuda context; for world > 1 an NCCL communicator is created from a
    unique id broadcast by rank 0 over the already-initialised torch.distributed group.

    transport="host": the library's collectives go through torch.distributed on host
    tensors (e.g. a gloo group) instead of NCCL — same sharded code paths, several
    ranks may share one GPU (the multi-process tests on a one-GPU box)."""
    from .context import Context
    r, w, _ = env()
    rank = r if rank is None else rank
    world = w if world is None else world
    if world == 1:
        return Context(local_rank)
    import torch.distributed as dist
    if transport == "host":
        return Context.with_host_transport(local_rank, rank, world, *host_collectives(world))
    obj = [Context.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return Context(local_rank, rank, world, obj[0])
