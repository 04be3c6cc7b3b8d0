"""Adaptive Sampling (sampling.hpp:16-80) on the GPU: kmeans_run (K3-K5),
the threshold k-sweep, centroid snapping (K6) and the host sample synthesis.

`clusterer(...)` returns a callable with the reference `Clusterer` signature
(sampling.hpp:44-46) so the GPU k-means drops into code written against it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L
from .context import Context, Space, ptr_of
from .errors import ConfigError


@dataclass
class SamplingParams:  # sampling.hpp:16-23
    threshold: float = 2.5
    k_min: int = 8
    k_max_exclusive: int = 64
    greedy_batch: int = 64
    kmeans_max_iters: int = 100
    kmeans_restarts: int = 3

    def c(self) -> L.SamplingParamsC:
        return L.SamplingParamsC(self.threshold, self.k_min, self.k_max_exclusive,
                                 self.kmeans_max_iters, self.kmeans_restarts)


@dataclass
class ClusterResult:  # sampling.hpp:27-32
    centroids: np.ndarray
    assignments: np.ndarray
    l2_loss: float
    iteration_losses: List[float] = field(default_factory=list)


@dataclass
class CandidateSet:  # candidates.hpp:20-27 (structure-of-arrays)
    idx: np.ndarray          # N x D int32 configurations, ranked
    ids: np.ndarray          # N uint64 ordinals
    predicted: np.ndarray    # N float64

    def __len__(self):
        return len(self.ids)

    def empty(self) -> bool:
        return len(self.ids) == 0


def make_candidate_set(space: Space, idx, predicted, ids=None) -> CandidateSet:
    """make_candidate_set (sampling.cpp:16-31): dedup by id (first wins), rank by (pred desc, id asc)."""
    idx = np.ascontiguousarray(idx, np.int32).reshape(-1, space.D)
    pred = np.ascontiguousarray(predicted, np.float64).reshape(-1)
    ids = space.id_of(idx) if ids is None else np.ascontiguousarray(ids, np.uint64)
    rows = np.zeros(len(ids), np.int64)
    m = C.c_int64()
    space.ctx.check(L.lib().ktune_make_candidate_set(space.ctx.h, ids.ctypes.data_as(C.c_void_p),
                                                     pred.ctypes.data_as(C.c_void_p), len(ids),
                                                     rows.ctypes.data_as(C.c_void_p), C.byref(m)))
    rows = rows[:m.value]
    return CandidateSet(idx[rows], ids[rows], pred[rows])


def candidates_from_rows(space: Space, idx, predicted):
    """make_candidate_set on the GPU over knob-index rows (e.g. a rollout trajectory).

    Host arrays -> host CandidateSet; CUDA tensors -> (rows, ids) CUDA tensors."""
    if hasattr(idx, "is_cuda") and idx.is_cuda:
        import torch
        n = idx.numel() // space.D
        rows = torch.empty(n, dtype=torch.int64, device=idx.device)
        ids = torch.empty(n, dtype=torch.uint64, device=idx.device)
        m = C.c_int64()
        space.ctx.check(L.lib().ktune_candidates_from_rows(
            space.ctx.h, space.h, C.c_void_p(idx.data_ptr()), C.c_void_p(predicted.data_ptr()), n,
            C.c_void_p(rows.data_ptr()), C.c_void_p(ids.data_ptr()), C.byref(m), L.F_DEVICE))
        return rows[:m.value], ids[:m.value]
    rows_idx = np.ascontiguousarray(idx, np.uint16).reshape(-1, space.D)
    pred = np.ascontiguousarray(predicted, np.float64).reshape(-1)
    n = len(rows_idx)
    rows = np.zeros(n, np.int64)
    ids = np.zeros(n, np.uint64)
    m = C.c_int64()
    space.ctx.check(L.lib().ktune_candidates_from_rows(
        space.ctx.h, space.h, rows_idx.ctypes.data_as(C.c_void_p), pred.ctypes.data_as(C.c_void_p), n,
        rows.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p), C.byref(m), 0))
    rows = rows[:m.value]
    return CandidateSet(rows_idx[rows].astype(np.int32), ids[:m.value], pred[rows])


def candidates_gather(space: Space, idx, predicted) -> CandidateSet:
    """The GLOBAL CandidateSet of a sharded rollout (ktune_candidates_gather): every rank
    passes its own trajectory rows (CUDA tensors: uint16 n x D, float64 n) and gets the
    same CandidateSet, equal to make_candidate_set over all ranks' rows.
    Returns CUDA tensors (idx int16-viewed uint16 rows, ids uint64, predicted float64)."""
    import torch
    n = idx.numel() // space.D
    m = C.c_int64()
    space.ctx.check(L.lib().ktune_candidates_gather(space.ctx.h, space.h, C.c_void_p(idx.data_ptr()),
                                                    C.c_void_p(predicted.data_ptr()), n, C.byref(m), L.F_DEVICE))
    g = m.value
    oidx = torch.empty((g, space.D), dtype=torch.int16, device=idx.device)
    opred = torch.empty(g, dtype=torch.float64, device=idx.device)
    oids = torch.empty(g, dtype=torch.int64, device=idx.device)
    space.ctx.check(L.lib().ktune_candidates_gather_copy(space.ctx.h, space.h, C.c_void_p(oidx.data_ptr()),
                                                         C.c_void_p(opred.data_ptr()), C.c_void_p(oids.data_ptr()),
                                                         L.F_DEVICE))
    return CandidateSet(oidx, oids, opred)


def _packed(space: Space, idx):
    if hasattr(idx, "is_cuda") and idx.is_cuda:
        import torch
        ok = (torch.uint8,) if space.index_bytes == 1 else (torch.uint16, torch.int16)
        if idx.dtype not in ok or not idx.is_contiguous():
            raise ConfigError(f"device points must be a contiguous tensor of {space.index_bytes}-byte knob indices "
                              f"(got {idx.dtype})")
        return idx, True
    return np.ascontiguousarray(idx, dtype=space.idx_dtype).reshape(-1, space.D), False


def kmeans_run(space: Space, idx, k: int, seed: int, max_iters: int = 100, restarts: int = 3) -> ClusterResult:
    """kmeans_run (sampling.cpp:157-175) over lattice points given as knob indices.

    Host arrays, or a CUDA tensor of points: then the centroids and assignments come back as
    CUDA tensors and only the scalars (loss, per-iteration losses) cross PCIe."""
    arr, dev = _packed(space, idx)
    N = (arr.numel() if dev else arr.size) // space.D
    il = np.zeros(max_iters + 1, np.float64)
    nl = C.c_int32()
    if dev:
        import torch
        cen = torch.zeros((max(k, 1), space.D), dtype=torch.float64, device=arr.device)
        asg = torch.zeros(N, dtype=torch.int32, device=arr.device)
        dloss = torch.zeros(1, dtype=torch.float64, device=arr.device)
        ptrs = [C.c_void_p(cen.data_ptr()), C.c_void_p(asg.data_ptr()), C.c_void_p(dloss.data_ptr())]
    else:
        cen = np.zeros((max(k, 1), space.D), np.float64)
        asg = np.zeros(N, np.int32)
        loss = C.c_double()
        ptrs = [cen.ctypes.data_as(C.c_void_p), asg.ctypes.data_as(C.c_void_p), C.cast(C.pointer(loss), C.c_void_p)]
    out = L.KmeansOutC(ptrs[0], ptrs[1], ptrs[2], il.ctypes.data_as(C.c_void_p), C.cast(C.pointer(nl), C.c_void_p))
    p = C.c_void_p(arr.data_ptr()) if dev else arr.ctypes.data_as(C.c_void_p)
    space.ctx.check(L.lib().ktune_kmeans_run(space.ctx.h, space.h, p, space.index_bytes, N, k, seed,
                                             max_iters, restarts, C.byref(out), L.F_DEVICE if dev else 0))
    lv = float(dloss.item()) if dev else loss.value
    return ClusterResult(cen[:k], asg, lv, list(il[:nl.value]))


def clusterer(space: Space, params: SamplingParams = SamplingParams()):
    """A `Clusterer` (sampling.hpp:44-46): (points as knob-index rows, k, seed) -> ClusterResult."""
    def run(points_idx, k: int, seed: int) -> ClusterResult:
        return kmeans_run(space, points_idx, k, seed, params.kmeans_max_iters, params.kmeans_restarts)
    return run


@dataclass
class SweepResult:
    k: int
    centroids: np.ndarray
    assignments: np.ndarray
    l2_loss: float
    k_losses: List[float]
    snapped: np.ndarray


def adaptive_sweep(space: Space, cands: CandidateSet, params: SamplingParams = SamplingParams(),
                   rng_seed: int = 0) -> SweepResult:
    """The k-sweep of adaptive_sample (sampling.cpp:436-446) + snap (:448-452), on the GPU.

    Host arrays, or a device-resident candidate set (CUDA tensors: idx N x D in the
    space's index width, ids uint64): then centroids, assignments and the snapped
    configurations come back as CUDA tensors and nothing crosses PCIe but the
    per-k scalars."""
    arr, dev = _packed(space, cands.idx)
    kmax = max(1, params.k_max_exclusive)
    k = C.c_int32()
    loss = C.c_double()
    kl = np.zeros(kmax)
    nk = C.c_int32()
    if dev:
        import torch
        ids = cands.ids
        N = ids.numel()
        mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=arr.device)
        cen, asg, snap = mk((kmax, space.D), torch.float64), mk((N,), torch.int32), mk((kmax, space.D), torch.int32)
        ptr = lambda t: C.c_void_p(t.data_ptr())
        idx_p, ids_p = ptr(arr), ptr(ids)
    else:
        ids = np.ascontiguousarray(cands.ids, np.uint64)
        N = len(ids)
        cen, asg, snap = np.zeros((kmax, space.D)), np.zeros(N, np.int32), np.zeros((kmax, space.D), np.int32)
        ptr = lambda a: a.ctypes.data_as(C.c_void_p)
        idx_p, ids_p = ptr(arr), ptr(ids)
    out = L.SweepOutC(C.cast(C.pointer(k), C.c_void_p), ptr(cen), ptr(asg), C.cast(C.pointer(loss), C.c_void_p),
                      kl.ctypes.data_as(C.c_void_p), C.cast(C.pointer(nk), C.c_void_p), ptr(snap))
    pc = params.c()
    space.ctx.check(L.lib().ktune_adaptive_sweep(space.ctx.h, space.h, idx_p, space.index_bytes, ids_p, N,
                                                 C.byref(pc), rng_seed, C.byref(out), L.F_DEVICE if dev else 0))
    kk = k.value
    return SweepResult(kk, cen[:kk], asg, loss.value, list(kl[:nk.value]), snap[:kk])


def snap_centroid(space: Space, centroids, cands: CandidateSet) -> np.ndarray:
    """snap_centroid (sampling.cpp:202-235) for one centroid (D,) or a batch (k x D)."""
    cen = np.ascontiguousarray(centroids, np.float64)
    single = cen.ndim == 1
    cen = cen.reshape(-1, space.D)
    k = len(cen)
    arr, _ = _packed(space, cands.idx)
    ids = np.ascontiguousarray(cands.ids, np.uint64)
    out = np.zeros((k, space.D), np.int32)
    space.ctx.check(L.lib().ktune_snap(space.ctx.h, space.h, cen.ctypes.data_as(C.c_void_p), k,
                                       arr.ctypes.data_as(C.c_void_p), space.index_bytes,
                                       ids.ctypes.data_as(C.c_void_p), len(ids),
                                       out.ctypes.data_as(C.c_void_p), 0))
    return out[0] if single else out


def adaptive_sample(space: Space, cands: CandidateSet, visited, params: SamplingParams = SamplingParams(),
                    rng_seed: int = 0) -> np.ndarray:
    """adaptive_sample (sampling.cpp:409-461): returns the configurations to measure (k x D)."""
    if cands.empty():
        raise ConfigError("adaptive_sample: empty candidate set")
    idx = np.ascontiguousarray(cands.idx, np.int32)
    ids = np.ascontiguousarray(cands.ids, np.uint64)
    vis = np.ascontiguousarray(np.fromiter(visited, np.uint64) if not isinstance(visited, np.ndarray)
                               else visited, np.uint64)
    out = np.zeros((max(1, params.k_max_exclusive), space.D), np.int32)
    cnt = C.c_int32()
    pc = params.c()
    space.ctx.check(L.lib().ktune_adaptive_sample(space.ctx.h, space.h, idx.ctypes.data_as(C.c_void_p),
                                                  ids.ctypes.data_as(C.c_void_p), len(ids),
                                                  vis.ctypes.data_as(C.c_void_p), len(vis), C.byref(pc),
                                                  rng_seed, out.ctypes.data_as(C.c_void_p), C.byref(cnt)))
    return out[:cnt.value]


def synthesize_sample(space: Space, cands: CandidateSet, visited, rng_state: int):
    """synthesize_sample (sampling.cpp:379-403); returns (config, advanced rng state)."""
    idx = np.ascontiguousarray(cands.idx, np.int32)
    vis = np.ascontiguousarray(np.fromiter(visited, np.uint64) if not isinstance(visited, np.ndarray)
                               else visited, np.uint64)
    st = C.c_uint64(rng_state)
    out = np.zeros(space.D, np.int32)
    L.check(L.lib().ktune_synthesize_sample(space.h, idx.ctypes.data_as(C.c_void_p), len(idx),
                                            vis.ctypes.data_as(C.c_void_p), len(vis), C.byref(st),
                                            out.ctypes.data_as(C.c_void_p)), space.ctx.h)
    return out, st.value


def greedy_select(cands: CandidateSet, batch: int) -> np.ndarray:
    """greedy_select (sampling.cpp:181-196): CandidateSet is already ranked (pred desc, id asc)."""
    order = np.lexsort((cands.ids, -cands.predicted))
    return cands.idx[order[:max(0, batch)]]
