"""Pins the oracle restatement (oracle/ktune_oracle.c) against the reference's own
sources compiled in place (oracle/_ref) on seeded inputs. CPU only."""
import numpy as np
import pytest

from paper_2001_08743_b200 import spaces as S

pytestmark = pytest.mark.usefixtures("ref_ok")


def test_rng_primitives(O):
    R, Pt = O.ref(), O.port()
    for z in [0, 1, 2**63, 2**64 - 1, 0x1234567890ABCDEF]:
        assert R.ref_mix64(z) == Pt.ko_mix64(z) == S.mix64(z)
        assert R.ref_seed_combine(z, 7) == Pt.ko_seed_combine(z, 7) == S.seed_combine(z, 7)
        for name in [b"explore", b"synthesis", b"", b"landscape-peaks"]:
            assert R.ref_stream_seed(z, name) == Pt.ko_stream_seed(z, name) == S.stream_seed(z, name.decode())
        for c in [0, 1, 99, 2**40]:
            assert R.ref_hash01(z, c) == Pt.ko_hash01(z, c)


def test_rng_draws_below_rejection(O):
    out = np.zeros(1000, np.uint64)
    O.ref().ref_rng_draws(5, 2, 3, 1000, out)
    assert set(np.unique(out)) <= {0, 1, 2}


@pytest.mark.parametrize("seed", range(4))
def test_space_ops_and_validity(O, seed):
    sp = S.conv_space("t", 64, 128, 28, 28, 3, 3)
    osp = O.OSpace(sp)
    g = np.random.default_rng(seed)
    idx = np.stack([g.integers(0, c, 500) for c in sp.cards], 1).astype(np.int32)
    ref_valid = np.zeros(500, np.uint8)
    O.ref().ref_validate(osp.ref, idx, 500, ref_valid)
    assert np.array_equal(osp.validate(idx), ref_valid)
    assert 0 < ref_valid.mean() < 1
    enc = np.zeros((500, sp.num_knobs))
    O.ref().ref_encode_batch(osp.ref, idx, 500, enc)
    assert np.array_equal(osp.encode(idx), enc)
    ids = osp.ids(idx)
    out = np.zeros(sp.num_knobs, np.int32)
    for i in range(20):
        O.ref().ref_config_at(osp.ref, int(ids[i]), out)
        assert np.array_equal(out, idx[i])


@pytest.mark.parametrize("space_fn,seed", [(lambda: S.synthetic_space(0, 16), 1),
                                           (lambda: S.conv_space("r", 64, 64, 56, 56, 3, 3), 2),
                                           (lambda: S.synthetic_space(3, 8), 3)])
def test_gbt_predict_matches_reference(O, space_fn, seed):
    osp = O.OSpace(space_fn())
    idx = osp.random_valid(seed, 1000)
    y = O.synthetic_fitness(osp, idx, seed=seed)
    y = np.where(np.isnan(y), 0.0, y)
    X = osp.encode(idx)
    g = O.ref_fit_gbt(X, y, seed=seed)
    q = osp.encode(osp.random_valid(seed + 100, 2000))
    assert np.array_equal(O.port_predict_features(g, q), O.ref_fit_predict(X, y, q, seed=seed))


@pytest.mark.parametrize("n,d,k,seed", [(300, 8, 1, 0), (500, 8, 8, 1), (2000, 16, 9, 2), (700, 3, 5, 3),
                                        (64, 16, 63, 4), (1500, 16, 20, 5)])
def test_kmeans_matches_reference(O, n, d, k, seed):
    sp = S.synthetic_space(seed, d)
    osp = O.OSpace(sp)
    P = osp.encode(osp.random_valid(seed, n))
    a = O.kmeans_run(P, k, seed * 7 + 1, impl="port")
    b = O.kmeans_run(P, k, seed * 7 + 1, impl="ref")
    assert np.array_equal(a["assignments"], b["assignments"])
    assert np.array_equal(a["centroids"], b["centroids"])
    assert a["loss"] == b["loss"]
    assert np.array_equal(a["iteration_losses"], b["iteration_losses"])


@pytest.mark.parametrize("seed", range(3))
def test_adaptive_sweep_matches_reference(O, seed):
    sp = S.synthetic_space(seed + 10, 8)
    osp = O.OSpace(sp)
    idx = osp.random_valid(seed, 3000)
    ids = osp.ids(idx)
    rows = O.make_candidate_set(sp.num_knobs, idx, ids, np.zeros(len(ids)), "ref")
    cidx, cids = idx[rows], ids[rows]
    P = osp.encode(cidx)
    sw = O.adaptive_sweep(P, rng_seed=seed)
    r = O.ref_adaptive_sample(osp, cidx, cids, np.zeros(len(cids)), [], rng_seed=seed)
    assert sw["k"] == len(r["configs"])
    assert np.array_equal(sw["k_losses"], r["k_losses"])
    snapped = np.stack([O.snap_centroid(osp, c, cidx, cids) for c in sw["centroids"]])
    assert np.array_equal(snapped, r["configs"])


@pytest.mark.parametrize("seed", range(6))
def test_snap_with_rule_fallback(O, seed):
    rule = "k0 * k1 + k2 <= 30"
    sp = S.synthetic_space(seed, 6, rule=rule)
    osp = O.OSpace(sp)
    g = np.random.default_rng(seed)
    idx = np.stack([g.integers(0, c, 400) for c in sp.cards], 1).astype(np.int32)
    ids = osp.ids(idx)
    rows = O.make_candidate_set(sp.num_knobs, idx, ids, g.random(400), "ref")
    cidx, cids = idx[rows], ids[rows]
    for t in range(25):
        c = g.random(sp.num_knobs)
        assert np.array_equal(O.snap_centroid(osp, c, cidx, cids), O.snap_centroid(osp, c, cidx, cids, impl="ref"))


def test_make_candidate_set_dedup_and_ties(O):
    g = np.random.default_rng(0)
    ids = g.integers(0, 50, 400).astype(np.uint64)
    pred = np.round(g.random(400), 1)  # many ties -> id ascending
    pred = np.array([pred[np.argmax(ids == i)] if True else 0 for i in ids])  # same id => same pred
    idx = np.zeros((400, 2), np.int32)
    a = O.make_candidate_set(2, idx, ids, pred, "port")
    b = O.make_candidate_set(2, idx, ids, pred, "ref")
    assert np.array_equal(a, b)
    assert len(a) == len(np.unique(ids))
