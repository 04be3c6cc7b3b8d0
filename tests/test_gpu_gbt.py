"""K1 GBT scoring on the GPU through the C-ABI: bit-exact with the oracle
(restatement of cost_model.cpp:117-124,179-199) and the reference build."""
import numpy as np
import pytest

from helpers import SPACES, fitted, random_idx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", list(SPACES))
def test_predict_idx_bit_exact(O, ctx, name):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    sp = SPACES[name]()
    osp, g, pm = fitted(O, sp, seed=3)
    dspace = Space(sp, ctx)
    dg = DeviceGbt(pm, dspace)
    idx = random_idx(sp, 50_000, 11)
    got = dg.predict_idx(idx.astype(dspace.idx_dtype))
    want = O.port_predict_idx(g, osp, idx)
    assert np.array_equal(got, want)
    # generic fp64 feature seam (CostModel::predict(MatrixXd))
    assert np.array_equal(dg.predict_features(osp.encode(idx[:5000])), want[:5000])


def test_predict_matches_reference_build(O, ctx, ref_ok):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt, fit_gbt
    sp = SPACES["synthetic16"]()
    osp = O.OSpace(sp)
    tr = osp.random_valid(5, 1000)
    y = np.nan_to_num(O.synthetic_fitness(osp, tr, seed=5))
    X = osp.encode(tr)
    pm = fit_gbt(X, y, seed=5)  # product host fit
    q = random_idx(sp, 20_000, 6)
    want = O.ref_fit_predict(X, y, osp.encode(q), seed=5)  # the reference's own predict_batch
    dg = DeviceGbt(pm, Space(sp, ctx))
    assert np.array_equal(dg.predict_idx(q.astype(np.uint8)), want)


def test_predict_edge_cases(O, ctx):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import CostModel, DeviceGbt, GbtModel
    from paper_2001_08743_b200.errors import ConfigError
    sp = SPACES["synthetic8"]()
    osp, g, pm = fitted(O, sp, seed=1)
    dg = DeviceGbt(pm, Space(sp, ctx))
    assert len(dg.predict_idx(np.zeros((0, sp.num_knobs), np.uint8))) == 0
    with pytest.raises(ConfigError):
        dg.predict_features(np.zeros((3, sp.num_knobs + 1)))
    with pytest.raises(ConfigError):
        CostModel(ctx=ctx).predict(np.zeros((2, 2)))
    # single-leaf trees (constant model) and extreme indices
    const = GbtModel(2.5, 0.3, sp.num_knobs, np.arange(4, dtype=np.int32), np.full(3, -1, np.int32),
                     np.full(3, -1, np.int32), np.full(3, -1, np.int32), np.zeros(3), np.array([1.0, -2.0, 0.5]))
    dc = DeviceGbt(const, Space(sp, ctx))
    top = np.array([[c - 1 for c in sp.cards]], np.uint8)
    assert dc.predict_idx(top)[0] == 2.5 + 0.3 * ((1.0 + -2.0) + 0.5)


def test_predict_1m_device_resident(O, ctx):
    import torch
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    sp = SPACES["synthetic16"]()
    osp, g, pm = fitted(O, sp, seed=2)
    dspace = Space(sp, ctx)
    dg = DeviceGbt(pm, dspace)
    idx = random_idx(sp, 1 << 20, 3)
    t = torch.from_numpy(idx.astype(np.uint8)).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    out = dg.predict_idx(t)
    torch.cuda.synchronize()
    ctx.set_stream(None)
    sel = np.random.default_rng(0).choice(len(idx), 20_000, replace=False)
    assert np.array_equal(out.cpu().numpy()[sel], O.port_predict_idx(g, osp, idx[sel]))


def _host_predict(pm, X):
    """Plain restatement of predict_one (cost_model.cpp:117-124,179-187): sequential fp64."""
    out = np.empty(len(X))
    for r, x in enumerate(X):
        s = 0.0
        for t in range(pm.num_trees):
            nd = int(pm.offsets[t])
            while pm.feature[nd] >= 0:
                nd = int(pm.offsets[t] + (pm.left[nd] if x[pm.feature[nd]] <= pm.threshold[nd] else pm.right[nd]))
            s = s + float(pm.value[nd])
        out[r] = pm.base_prediction + pm.learning_rate * s
    return out


@pytest.mark.parametrize("depth", [1, 2, 3, 5, 8])
def test_predict_idx_every_tree_depth(O, ctx, depth):
    """K1 is compiled per complete-tree depth (levels 0-1 from one broadcast load
    when depth >= 2): every depth agrees bit-for-bit with a host restatement."""
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt, GbtParams, fit_gbt
    sp = SPACES["synthetic16"]()
    osp = O.OSpace(sp)
    tr = osp.random_valid(7, 1500)
    y = np.nan_to_num(O.synthetic_fitness(osp, tr, seed=7))
    pm = fit_gbt(osp.encode(tr), y, GbtParams(num_trees=12, max_depth=depth, min_samples_leaf=1), seed=7)
    dg = DeviceGbt(pm, Space(sp, ctx))
    q = random_idx(sp, 3000, 8)
    want = _host_predict(pm, osp.encode(q))
    assert np.array_equal(dg.predict_idx(q.astype(np.uint8)), want)
