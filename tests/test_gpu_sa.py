"""K7 sa_search on the GPU vs the oracle restatement
(builder-pinned semantics): chain states, predicted fitness and
acceptance flags bit-exact; SPEC examples as properties."""
import numpy as np
import pytest

from helpers import SPACES, fitted

pytestmark = pytest.mark.gpu


def _setup(O, ctx, name, seed):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    sp = SPACES[name]()
    osp, og, pm = fitted(O, sp, seed=seed)
    ds = Space(sp, ctx)
    return sp, osp, og, ds, DeviceGbt(pm, ds)


@pytest.mark.parametrize("name,E,T", [("resnet_c2", 128, 60), ("synthetic16", 300, 40), ("resnet_dense_u16", 7, 90)])
def test_sa_matches_oracle(O, ctx, name, E, T):
    from paper_2001_08743_b200.exploration import SaParams, sa_search
    from paper_2001_08743_b200.spaces import stream_seed
    sp, osp, og, ds, dg = _setup(O, ctx, name, E)
    seeds = osp.random_valid(E, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
    p = SaParams(num_chains=E, max_steps=T, initial_temperature=0.02, cooling_rate=0.97)
    cands, tr = sa_search(ds, dg, seeds, p, rng_seed=9)
    want = O.sa_search(osp, og, seeds, T, 0, stream_seed(9, "sa"), 0.02, 0.97)
    assert np.array_equal(tr["idx"].astype(np.int32), want["idx"])
    assert np.array_equal(tr["score"], want["score"])
    assert np.array_equal(tr["accepted"], want["accepted"])
    assert 0 < tr["accepted"].mean() < 1  # a non-degenerate schedule
    # CandidateSet: deduplicated, ranked by predicted fitness (desc)
    assert len(np.unique(cands.ids)) == len(cands.ids)
    assert np.all(np.diff(cands.predicted) <= 0)


def test_sa_spec_examples(O, ctx):
    """T -> 0: only improvements are accepted, so every chain's fitness is
    non-decreasing (SPEC.md:235 hill-climb limit); a Δ = 0 proposal is always
    accepted (exp(0) = 1)."""
    from paper_2001_08743_b200.exploration import SaParams, sa_search
    sp, osp, og, ds, dg = _setup(O, ctx, "resnet_c2", 3)
    _, tr = sa_search(ds, dg, np.zeros((0, sp.num_knobs)), SaParams(64, 80, 1e-300, 0.5), rng_seed=1)
    assert np.all(np.diff(tr["score"], axis=1) >= 0)
    assert tr["score"][:, -1].min() >= tr["score"][:, 0].min()
    same = np.diff(tr["score"], axis=1) == 0
    moved = np.any(tr["idx"][:, 1:] != tr["idx"][:, :-1], axis=2)
    assert np.all(tr["accepted"][same & moved] == 1)  # equal fitness moves were taken


def test_sa_chain_sharding_invariance(O, ctx):
    """Chains keyed by global id: a shard with chain_offset reproduces the full run."""
    from paper_2001_08743_b200.exploration import SaParams, sa_search
    sp, osp, og, ds, dg = _setup(O, ctx, "synthetic8", 5)
    seeds = np.random.default_rng(0).integers(0, 2, (100, sp.num_knobs))
    p = SaParams(100, 30, 0.05, 0.95)
    _, full = sa_search(ds, dg, seeds, p, rng_seed=4)
    _, part = sa_search(ds, dg, seeds[60:], SaParams(40, 30, 0.05, 0.95), rng_seed=4, chain_offset=60)
    assert np.array_equal(full["idx"][60:], part["idx"])
    assert np.array_equal(full["score"][60:], part["score"])


def test_sa_grouped_launch_equals_single_calls(O, ctx):
    """sa_search_batch: several spaces in one launch = one call per task; the
    device-resident variant returns the same trajectory."""
    import torch
    from paper_2001_08743_b200.exploration import SaParams, SaTask, sa_search, sa_search_batch, sa_seeds
    p = SaParams(96, 25, 0.05, 0.95)
    tasks, singles = [], []
    for k, name in enumerate(["resnet_c2", "synthetic16", "resnet_dense_u16"]):
        sp, osp, og, ds, dg = _setup(O, ctx, name, 11 + k)
        init = sa_seeds(ds, np.zeros((0, sp.num_knobs)), p.num_chains, rng_seed=k)
        tasks.append(SaTask(ds, dg, init, 0, k))
        singles.append(sa_search(ds, dg, init, p, rng_seed=k)[1])
    grouped = sa_search_batch(tasks, p)
    dev_tasks = [SaTask(t.space, t.cost_model, torch.from_numpy(t.init_idx.view(np.int16)).cuda(), 0, t.rng_seed)
                 for t in tasks]
    on_dev = sa_search_batch(dev_tasks, p, device_out=True)
    ctx.synchronize()  # device-pointer calls are stream-ordered on the context's stream
    for g, s1, d in zip(grouped, singles, on_dev):
        for key in ("idx", "score", "accepted"):
            assert np.array_equal(g[key], s1[key])
        assert np.array_equal(d["idx"].view(torch.int16).cpu().numpy().view(np.uint16), g["idx"])
        assert np.array_equal(d["score"].cpu().numpy(), g["score"])
        assert np.array_equal(d["accepted"].cpu().numpy(), g["accepted"])


@pytest.mark.parametrize("depth,ntrees", [(2, 13), (6, 9), (1, 20)])
def test_sa_every_tree_depth(O, ctx, depth, ntrees):
    """K7's walk is compiled per tree depth and interleaves trees 8 at a time
    (remainder trees walked singly): bit-exact with the oracle at other depths
    and tree counts."""
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt, GbtModel
    from paper_2001_08743_b200.exploration import SaParams, sa_search
    from paper_2001_08743_b200.spaces import stream_seed
    sp = SPACES["synthetic16"]()
    osp = O.OSpace(sp)
    g = O.fitted_model(osp, seed=depth, n_train=800, num_trees=ntrees, max_depth=depth)
    pm = GbtModel(g.base, g.lr, g.num_features, g.offsets, g.feature, g.left, g.right, g.threshold, g.value)
    ds = Space(sp, ctx)
    E, T = 70, 30
    seeds = osp.random_valid(3, E)
    p = SaParams(num_chains=E, max_steps=T, initial_temperature=0.05, cooling_rate=0.95)
    _, tr = sa_search(ds, DeviceGbt(pm, ds), seeds, p, rng_seed=depth)
    want = O.sa_search(osp, g, seeds, T, 0, stream_seed(depth, "sa"), 0.05, 0.95)
    assert np.array_equal(tr["idx"].astype(np.int32), want["idx"])
    assert np.array_equal(tr["score"], want["score"])
    assert np.array_equal(tr["accepted"], want["accepted"])
