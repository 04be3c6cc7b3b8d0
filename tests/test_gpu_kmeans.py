"""K3-K6 Adaptive Sampling on the GPU through the C-ABI: bit-exact assignments,
centroids and selected configurations versus the reference build (and the
oracle restatement) on the same seeds."""
import numpy as np
import pytest

from helpers import SPACES, candidate_set

pytestmark = pytest.mark.gpu


def _space(ctx, sp):
    from paper_2001_08743_b200.context import Space
    return Space(sp, ctx)


@pytest.mark.parametrize("name,n,k,seed", [("synthetic8", 3000, 8, 1), ("synthetic16", 5000, 9, 2),
                                           ("resnet_c2", 4000, 12, 3), ("alexnet_c3_u16", 2500, 8, 4),
                                           ("synthetic16", 700, 63, 5), ("synthetic8", 200, 1, 6)])
@pytest.mark.parametrize("force_exact", [0, 1])
def test_kmeans_run_matches_reference(O, ctx, ref_ok, name, n, k, seed, force_exact):
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    ds = _space(ctx, sp)
    ctx.set_option(L.OPT_FORCE_EXACT, force_exact)
    try:
        got = kmeans_run(ds, cidx, k, seed * 13 + 1)
    finally:
        ctx.set_option(L.OPT_FORCE_EXACT, 0)
    want = O.kmeans_run(osp.encode(cidx), k, seed * 13 + 1, impl="ref")
    assert np.array_equal(got.assignments, want["assignments"])
    assert np.array_equal(got.centroids, want["centroids"])
    assert abs(got.l2_loss - want["loss"]) <= 1e-12 * max(1.0, want["loss"])
    assert len(got.iteration_losses) == len(want["iteration_losses"])
    assert np.allclose(got.iteration_losses, want["iteration_losses"], rtol=1e-12, atol=0)


def test_kmeans_errors(ctx):
    from paper_2001_08743_b200.errors import ConfigError
    from paper_2001_08743_b200.sampling import kmeans_run
    from paper_2001_08743_b200 import spaces as S
    ds = _space(ctx, S.synthetic_space(0, 4))
    with pytest.raises(ConfigError):
        kmeans_run(ds, np.zeros((0, 4)), 1, 0)
    with pytest.raises(ConfigError, match="out of range"):
        kmeans_run(ds, np.zeros((3, 4)), 4, 0)


@pytest.mark.parametrize("name,n,seed", [("synthetic8", 4000, 0), ("resnet_c2", 6000, 1),
                                         ("synthetic16", 3000, 2)])
def test_adaptive_sweep_and_snap_match_reference(O, ctx, ref_ok, name, n, seed):
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    pred = np.random.default_rng(seed).random(n)
    cidx, cids, cpred = candidate_set(O, osp, n, seed, pred)
    ds = _space(ctx, sp)
    res = adaptive_sweep(ds, CandidateSet(cidx, cids, cpred), SamplingParams(), rng_seed=seed)
    want = O.ref_adaptive_sample(osp, cidx, cids, cpred, [], rng_seed=seed)
    assert res.k == len(want["configs"])
    assert np.allclose(res.k_losses, want["k_losses"], rtol=1e-12, atol=0)
    assert np.array_equal(res.snapped, want["configs"])


def test_forced_full_sweep(O, ctx, ref_ok):
    """threshold just above 1 keeps the sweep going."""
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
    sp = SPACES["synthetic8"]()
    osp = O.OSpace(sp)
    cidx, cids, cpred = candidate_set(O, osp, 1500, 7)
    ds = _space(ctx, sp)
    p = SamplingParams(threshold=1.0 + 1e-9, k_min=8, k_max_exclusive=20)
    res = adaptive_sweep(ds, CandidateSet(cidx, cids, cpred), p, rng_seed=7)
    want = O.ref_adaptive_sample(osp, cidx, cids, cpred, [], threshold=p.threshold, k_min=8,
                                 k_max_exclusive=20, rng_seed=7)
    assert res.k == len(want["configs"]) and res.k >= 10
    assert np.array_equal(res.snapped, want["configs"])


@pytest.mark.parametrize("seed", range(4))
def test_snap_rule_fallback(O, ctx, ref_ok, seed):
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.sampling import CandidateSet, snap_centroid
    sp = S.synthetic_space(seed, 6, rule="k0 * k1 + k2 <= 30")
    osp = O.OSpace(sp)
    cidx, cids, cpred = candidate_set(O, osp, 2000, seed)
    ds = _space(ctx, sp)
    cents = np.random.default_rng(seed).random((40, 6))
    got = snap_centroid(ds, cents, CandidateSet(cidx, cids, cpred))
    for c, row in zip(cents, got):
        assert np.array_equal(row, O.snap_centroid(osp, c, cidx, cids, impl="ref"))


@pytest.mark.parametrize("seed", range(3))
def test_adaptive_sample_with_visited_matches_reference(O, ctx, ref_ok, seed):
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sample
    sp = S.synthetic_space(seed + 20, 5, rule="k0 + k1 <= 12")
    osp = O.OSpace(sp)
    cidx, cids, cpred = candidate_set(O, osp, 1500, seed, np.random.default_rng(seed).random(1500))
    ds = _space(ctx, sp)
    visited = cids[::3].copy()  # many snapped results will collide -> synthesis
    got = adaptive_sample(ds, CandidateSet(cidx, cids, cpred), visited, SamplingParams(), rng_seed=seed)
    want = O.ref_adaptive_sample(osp, cidx, cids, cpred, visited, rng_seed=seed)
    assert np.array_equal(got, want["configs"])


def test_synthesize_sample_matches_reference(O, ctx, ref_ok):
    import ctypes as C
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.sampling import CandidateSet, synthesize_sample
    sp = S.synthetic_space(3, 4, rule="k0 * k1 <= 20")
    osp = O.OSpace(sp)
    cidx, cids, cpred = candidate_set(O, osp, 300, 3)
    ds = _space(ctx, sp)
    for vis_frac in [0, 2, 1]:
        visited = cids[::vis_frac] if vis_frac else cids[:0]
        got, _ = synthesize_sample(ds, CandidateSet(cidx, cids, cpred), visited, 12345)
        out = np.zeros(4, np.int32)
        rc = O.ref().ref_synthesize_sample(osp.ref, cidx, cids, cpred, len(cids), np.ascontiguousarray(visited),
                                           len(visited), 12345, out)
        assert rc == 0
        assert np.array_equal(got, out)


def test_kmeans_large_vs_oracle(O, ctx):
    """200k points: GPU vs the oracle restatement (bit-exact), certified kmeans++."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES["synthetic16"]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, 200_000, 11)
    ds = _space(ctx, sp)
    ctx.reset_stats()
    got = kmeans_run(ds, cidx, 9, 5, restarts=1)
    want = O.kmeans_run(osp.encode(cidx), 9, 5, restarts=1)
    assert np.array_equal(got.assignments, want["assignments"])
    assert np.array_equal(got.centroids, want["centroids"])
    assert ctx.stat(L.STAT_KPP_PICKS) == 8


@pytest.mark.parametrize("mode", [0, 1, 3])  # 0: default (fp32-screened), 1: exact SIMT scan, 3: tcgen05 screening
@pytest.mark.parametrize("name,n,k,seed", [("synthetic16", 20000, 24, 7), ("alexnet_c3_u16", 8000, 63, 8),
                                           ("resnet_c2", 6000, 9, 9)])
def test_assign_paths_bit_exact(O, ctx, ref_ok, mode, name, n, k, seed):
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    ds = _space(ctx, sp)
    ctx.set_option(L.OPT_KMEANS_MODE, mode)
    ctx.reset_stats()
    try:
        got = kmeans_run(ds, cidx, k, seed, restarts=2)
    finally:
        ctx.set_option(L.OPT_KMEANS_MODE, 0)
    want = O.kmeans_run(osp.encode(cidx), k, seed, restarts=2, impl="ref")
    assert np.array_equal(got.assignments, want["assignments"])
    assert np.array_equal(got.centroids, want["centroids"])
    assert got.l2_loss == want["loss"]
    print("uncertain (exact-fallback) points:", ctx.stat(L.STAT_ASSIGN_FALLBACKS))


@pytest.mark.parametrize("name,n,k,seed", [("alexnet_c3_u16", 30000, 8, 3), ("synthetic16", 20000, 12, 4),
                                           ("alexnet_c3_u16", 30000, 63, 5), ("resnet_c2", 8000, 40, 6),
                                           ("synthetic16", 20000, 33, 7)])
def test_certified_lloyd_equals_exact_mode(O, ctx, name, n, k, seed):
    """Mode B (integer-sum centroids, certified assignments, exact finalisation) and
    mode A (exact-order sums every iteration) give identical runs; mode B ran
    without falling back."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    ds = _space(ctx, sp)
    ctx.reset_stats()
    b = kmeans_run(ds, cidx, k, seed, restarts=2)
    aborts = ctx.stat(L.STAT_KMEANS_ABORTS)
    ctx.set_option(L.OPT_KMEANS_MODE, 1)
    try:
        a = kmeans_run(ds, cidx, k, seed, restarts=2)
    finally:
        ctx.set_option(L.OPT_KMEANS_MODE, 0)
    assert aborts == 0
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids, b.centroids)
    assert a.l2_loss == b.l2_loss
    assert len(a.iteration_losses) == len(b.iteration_losses)


@pytest.mark.parametrize("name,n,k,seed", [("alexnet_c3_u16", 20000, 8, 21), ("synthetic16", 12000, 30, 22)])
def test_nccl_sharded_path_on_one_rank(O, ctx, ref_ok, name, n, k, seed):
    """The multi-GPU k-means path (rank-local chunk assignment, NCCL all-gathers of
    the per-point state, all-reduced counters) run through a one-rank NCCL
    communicator on the real GPU: same clustering as the single-GPU path and as
    the reference, the adaptive sweep too."""
    import torch  # noqa: F401  (loads the bundled libnccl the library binds with dlopen)
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.context import Context
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep, kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    want = kmeans_run(_space(ctx, sp), cidx, k, seed, restarts=2)
    dctx = Context(0, 0, 1, Context.nccl_unique_id())
    dctx.set_option(L.OPT_FORCE_SHARDED, 1)
    ds = _space(dctx, sp)
    for mode in (1, 0):  # exact-order sums every iteration (mode A), then the sharded certified mode B
        dctx.set_option(L.OPT_KMEANS_MODE, mode)
        dctx.reset_stats()
        got = kmeans_run(ds, cidx, k, seed, restarts=2)
        if mode == 1:
            assert dctx.stat(L.STAT_XS_SEGMENTS) > 0  # the sharded mode-A path ran
        else:
            assert dctx.stat(L.STAT_KMEANS_ABORTS) == 0
        assert np.array_equal(got.assignments, want.assignments)
        assert np.array_equal(got.centroids, want.centroids)
        assert got.l2_loss == want.l2_loss
    ref = O.kmeans_run(osp.encode(cidx), k, seed, restarts=2, impl="ref")
    assert np.array_equal(got.assignments, ref["assignments"])
    cs = CandidateSet(cidx, cids, np.zeros(len(cids)))
    a = adaptive_sweep(ds, cs, SamplingParams(k_max_exclusive=12), 3)
    b = adaptive_sweep(_space(ctx, sp), cs, SamplingParams(k_max_exclusive=12), 3)
    assert a.k == b.k and a.k_losses == b.k_losses and np.array_equal(a.snapped, b.snapped)


@pytest.mark.parametrize("name,n", [("resnet_c2", 6000), ("alexnet_c3_u16", 5000)])
def test_adaptive_sweep_device_resident(O, ctx, name, n):
    """A candidate set already on the GPU (CUDA tensors) sweeps to the same k,
    losses, assignments and snapped configurations as the host call."""
    import torch
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, 31)
    ds = _space(ctx, sp)
    p = SamplingParams(k_max_exclusive=14)
    host = adaptive_sweep(ds, CandidateSet(cidx, cids, np.zeros(len(cids))), p, 9)
    narrow = np.ascontiguousarray(cidx, ds.idx_dtype)
    didx = torch.from_numpy(narrow.view(np.int16) if narrow.dtype == np.uint16 else narrow).cuda()
    dids = torch.from_numpy(cids.view(np.int64)).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        dev = adaptive_sweep(ds, CandidateSet(didx, dids, None), p, 9)
        torch.cuda.synchronize()
    finally:
        ctx.set_stream(None)
    assert dev.k == host.k and dev.k_losses == host.k_losses and dev.l2_loss == host.l2_loss
    assert np.array_equal(dev.assignments.cpu().numpy(), host.assignments)
    assert np.array_equal(dev.centroids.cpu().numpy(), host.centroids)
    assert np.array_equal(dev.snapped.cpu().numpy(), host.snapped)


@pytest.mark.parametrize("log2", [30, 45])
@pytest.mark.parametrize("name,n,k,seed", [("alexnet_c3_u16", 20000, 8, 41), ("synthetic16", 15000, 20, 42)])
def test_certified_lloyd_rescue(O, ctx, name, n, k, seed, log2):
    """Inflated centroid bounds make speculative iterations fail (uncertain points):
    the run continues exactly from the last certified batch and still matches the
    exact mode and the reference."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, n, seed)
    ds = _space(ctx, sp)
    ctx.set_option(L.OPT_KMEANS_MODE, 1)
    try:
        a = kmeans_run(ds, cidx, k, seed, restarts=2)
    finally:
        ctx.set_option(L.OPT_KMEANS_MODE, 0)
    ctx.reset_stats()
    ctx.set_option(L.OPT_KMEANS_BOUND_LOG2, log2)
    try:
        b = kmeans_run(ds, cidx, k, seed, restarts=2)
        rescues = ctx.stat(L.STAT_KMEANS_ABORTS)
    finally:
        ctx.set_option(L.OPT_KMEANS_BOUND_LOG2, 0)
    assert rescues > 0
    assert np.array_equal(a.assignments, b.assignments)
    assert np.array_equal(a.centroids, b.centroids)
    assert a.l2_loss == b.l2_loss
    assert len(a.iteration_losses) == len(b.iteration_losses)
    ref = O.kmeans_run(osp.encode(cidx), k, seed, restarts=2, impl="ref")
    assert np.array_equal(b.assignments, ref["assignments"])


def test_kmeans_two_million_points_deterministic_and_exact(O, ctx, ref_ok):
    """2M points (2000 chunk blocks per pass): repeated calls give identical results
    (a shared-memory staging race in the kmeans++ distance kernel once made the picks
    nondeterministic at this size) and the result equals the reference's."""
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES["alexnet_c3_u16"]()
    osp = O.OSpace(sp)
    g = np.random.default_rng(77)
    idx = np.stack([g.integers(0, c, 2_000_000) for c in sp.cards], 1).astype(np.int32)
    ds = _space(ctx, sp)
    runs = [kmeans_run(ds, idx, 9, 5, restarts=1) for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.assignments, runs[0].assignments)
        assert np.array_equal(r.centroids, runs[0].centroids)
        assert r.l2_loss == runs[0].l2_loss
    want = O.kmeans_run(osp.encode(idx), 9, 5, restarts=1, impl="ref")
    assert np.array_equal(runs[0].assignments, want["assignments"])
    assert np.array_equal(runs[0].centroids, want["centroids"])
    assert runs[0].l2_loss == want["loss"]


@pytest.mark.parametrize("name,k", [("alexnet_c3_u16", 40), ("resnet_c2", 8)])
def test_kmeans_run_device_points_equal_host(O, ctx, name, k):
    """kmeans_run over a device-resident candidate set (the forced sweep's input): the same
    centroids, assignments, loss and per-iteration losses as the host-array call."""
    import torch
    from paper_2001_08743_b200.sampling import kmeans_run
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    cidx, cids, _ = candidate_set(O, osp, 30_000, 3)
    ds = _space(ctx, sp)
    host = kmeans_run(ds, cidx, k, 77)
    didx = torch.from_numpy(np.ascontiguousarray(cidx, dtype=ds.idx_dtype)).cuda()
    dev = kmeans_run(ds, didx, k, 77)
    assert torch.is_tensor(dev.centroids) and dev.centroids.is_cuda
    assert np.array_equal(dev.centroids.cpu().numpy(), host.centroids)
    assert np.array_equal(dev.assignments.cpu().numpy(), host.assignments)
    assert dev.l2_loss == host.l2_loss and dev.iteration_losses == host.iteration_losses


def test_kmeans_run_device_points_dtype_checked(ctx):
    """Device points in the wrong index width are rejected, not reinterpreted."""
    import torch
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.errors import ConfigError
    from paper_2001_08743_b200.sampling import kmeans_run
    ds = _space(ctx, S.synthetic_space(0, 4))
    with pytest.raises(ConfigError, match="device points"):
        kmeans_run(ds, torch.zeros((100, 4), dtype=torch.int64, device="cuda"), 2, 0)


def test_kmeans_c4_scale_matches_reference(O, ctx):
    """SURVEY C4 scale in the driver-run suite: kmeans_run over ~1M distinct AlexNet-conv2 candidates
    (uint16 indices), k = 8, 3 restarts, equal to the REFERENCE's own kmeans_run (oracle/_ref:
    assignments, centroids and loss bit for bit), from host arrays and from device-resident points;
    and the whole adaptive sweep + snap equal to the reference's own adaptive_sample."""
    import torch
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.sampling import kmeans_run
    from workloads.tasks import random_configs
    sp = S.alexnet_tasks()[1]
    ds = _space(ctx, sp)
    idx = random_configs(sp, 1 << 20, 123)
    ids = ds.id_of(idx)
    _, first = np.unique(ids, return_index=True)
    idx = idx[np.sort(first)]
    want = O.kmeans_run(O.OSpace(sp).encode(idx), 8, 11, restarts=3, impl="ref")
    got = kmeans_run(ds, idx, 8, 11, restarts=3)
    assert np.array_equal(got.assignments, want["assignments"])
    assert np.array_equal(got.centroids, want["centroids"])
    assert got.l2_loss == want["loss"]
    dev = kmeans_run(ds, torch.from_numpy(np.ascontiguousarray(idx, dtype=ds.idx_dtype)).cuda(), 8, 11, restarts=3)
    assert np.array_equal(dev.assignments.cpu().numpy(), want["assignments"])
    assert dev.l2_loss == want["loss"]
    from paper_2001_08743_b200.sampling import CandidateSet, SamplingParams, adaptive_sweep
    ids = ds.id_of(idx)
    pred = np.zeros(len(idx))
    res = adaptive_sweep(ds, CandidateSet(idx, ids, pred), SamplingParams(), rng_seed=5)
    ref = O.ref_adaptive_sample(O.OSpace(sp), idx, ids, pred, [], rng_seed=5)
    assert res.k == len(ref["configs"])
    assert np.allclose(res.k_losses, ref["k_losses"], rtol=1e-12, atol=0)
    assert np.array_equal(res.snapped, ref["configs"])
