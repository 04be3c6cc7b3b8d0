"""make_candidate_set on the GPU vs the reference build's
make_candidate_set (sampling.cpp:16-31): dedup keeps the first occurrence, rank
by (predicted desc, id asc)."""
import numpy as np
import pytest

from helpers import SPACES

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,n,seed", [("resnet_c2", 20000, 0), ("synthetic8", 50000, 1),
                                         ("resnet_dense_u16", 3000, 2),
                                         # radix-sort edges: one row, one tile exactly, tile + 1,
                                         # several tiles, 64-bit ids (synthetic16 > 2^32 configs)
                                         ("resnet_c2", 1, 3), ("resnet_c2", 2048, 4), ("synthetic8", 2049, 5),
                                         ("synthetic16", 300_001, 6), ("vgg_c4", 1_000_003, 7)])
def test_candidates_from_rows_matches_reference(O, ctx, ref_ok, name, n, seed):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.sampling import candidates_from_rows
    sp = SPACES[name]()
    osp = O.OSpace(sp)
    g = np.random.default_rng(seed)
    base = np.stack([g.integers(0, c, max(1, n // 3)) for c in sp.cards], 1).astype(np.int32)
    idx = base[g.integers(0, len(base), n)]          # many duplicates
    ids = osp.ids(idx)
    pred_of = {i: v for i, v in zip(np.unique(ids), np.round(g.random(len(np.unique(ids))), 2))}
    pred = np.array([pred_of[i] for i in ids])        # same id => same prediction; many ties
    want = O.make_candidate_set(sp.num_knobs, idx, ids, pred, "ref")
    got = candidates_from_rows(Space(sp, ctx), idx.astype(np.uint16), pred)
    assert np.array_equal(got.ids, ids[want])
    assert np.array_equal(got.idx, idx[want])
    assert np.array_equal(got.predicted, pred[want])


def test_rollout_to_candidates_on_device(O, ctx):
    """Trajectory -> candidate set without leaving the device."""
    import torch
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.sampling import candidates_from_rows, make_candidate_set
    from helpers import fitted
    sp = SPACES["resnet_c2"]()
    osp, og, pm = fitted(O, sp, seed=4)
    ds = Space(sp, ctx)
    agent = ActorCritic(8, 128, 64, seed=3, ctx=ctx)
    init = torch.from_numpy(np.ones((256, 8), np.uint16)).cuda()  # every card >= 2
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    out = run_episodes_batch([RolloutTask(ds, agent, DeviceGbt(pm, ds), init, 0, 1)], 40, ctx)[0]
    rows, ids = candidates_from_rows(ds, out["idx"].reshape(-1, 8), out["score"].reshape(-1))
    torch.cuda.synchronize()
    ctx.set_stream(None)
    host = make_candidate_set(ds, out["idx"].cpu().numpy().reshape(-1, 8).astype(np.int32),
                              out["score"].cpu().numpy().reshape(-1))
    assert np.array_equal(ids.cpu().numpy(), host.ids)


@pytest.mark.parametrize("name,n", [("alexnet_c3_u16", 50000), ("synthetic16", 30000), ("resnet_c2", 1)])
def test_knob_histogram_matches_counts(ctx, name, n):
    """knob_options' counting pass (sampling.cpp:249-256) on the device."""
    import ctypes as C
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.context import Space
    sp = SPACES[name]()
    ds = Space(sp, ctx)
    g = np.random.default_rng(n)
    idx = np.stack([g.integers(0, c, n) for c in sp.cards], 1).astype(ds.idx_dtype)
    counts = np.zeros(sum(sp.cards), np.uint64)
    ctx.check(L.lib().ktune_knob_histogram(ctx.h, ds.h, idx.ctypes.data_as(C.c_void_p), ds.index_bytes, n,
                                           counts.ctypes.data_as(C.c_void_p), 0))
    off = 0
    for d, c in enumerate(sp.cards):
        assert np.array_equal(counts[off:off + c], np.bincount(idx[:, d].astype(np.int64), minlength=c)), d
        off += c
