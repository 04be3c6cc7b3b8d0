"""SPEC.md known-answer examples for the hot path, against the oracle (and the
reference build where reference code exists). CPU only."""
import math

import numpy as np
import pytest

from paper_2001_08743_b200 import spaces as S


def small(cards, rule=None):
    return S.DesignSpace("kat", [S.Knob(n, v) for n, v in cards], rule)


def test_design_space_kats(O):
    # SPEC.md:70-72 config_at / :80-82 id_of / :110-112 encode_features
    sp = small([("a", [1, 2]), ("b", [4, 8, 16])])
    assert sp.size == 6
    osp = O.OSpace(sp)
    out = np.zeros(2, np.int32)
    O.port().ko_config_at(osp.ko, 0, out)
    assert list(out) == [0, 0]
    O.port().ko_config_at(osp.ko, 4, out)
    assert list(out) == [1, 1]
    assert list(osp.ids([[0, 0], [1, 1], [1, 2]])) == [0, 4, 5]
    assert np.array_equal(osp.encode([[1, 1], [0, 0]]), [[1.0, 0.5], [0.0, 0.0]])
    single = O.OSpace(small([("a", [7]), ("b", [1, 2, 3])]))
    assert single.encode([[0, 2]])[0, 0] == 0.0


def test_design_space_errors():
    from paper_2001_08743_b200.errors import ConfigError
    with pytest.raises(ConfigError, match="duplicate value"):
        small([("a", [4, 4, 8])])
    with pytest.raises(ConfigError):
        small([("a", [8, 4])])
    with pytest.raises(ConfigError, match="duplicate knob"):
        small([("a", [1]), ("a", [2])])
    with pytest.raises(ConfigError, match="overflows"):
        S.DesignSpace("big", [S.Knob(f"k{i}", list(range(300))) for i in range(9)])


def test_validate_kats(O, ref_ok):
    # "tile_y * tile_x <= 64"
    sp = small([("tile_y", [1, 2, 4, 8, 16]), ("tile_x", [1, 2, 4, 8])], "tile_y * tile_x <= 64")
    osp = O.OSpace(sp)
    assert list(osp.validate([[3, 3], [4, 3]])) == [1, 0]
    ref = np.zeros(2, np.uint8)
    O.ref().ref_validate(osp.ref, np.array([[3, 3], [4, 3]], np.int32), 2, ref)
    assert list(ref) == [1, 0]
    norule = O.OSpace(small([("a", [1, 2])]))
    assert list(norule.validate([[0], [1]])) == [1, 1]


def test_neighbor_kats(O, ref_ok):
    # saturating neighbor
    osp = O.OSpace(small([("a", [1, 2, 3, 4, 5])]))
    out = np.zeros(1, np.int32)
    for start, d, want in [(2, 1, 3), (0, -1, 0), (4, 1, 4), (3, 0, 3)]:
        O.ref().ref_neighbor(osp.ref, np.array([start], np.int32), 0, d, out)
        assert out[0] == want


def test_gbt_kats(O, ref_ok):
    # SPEC.md:164-166 single example -> constant; depth-1 stump; constant dataset
    g = O.ref_fit_gbt(np.array([[0.3, 0.7]]), np.array([7.0]), seed=0)
    assert np.all(O.port_predict_features(g, np.random.default_rng(0).random((5, 2))) == 7.0)
    X = np.array([[0.0], [1.0]])
    g = O.ref_fit_gbt(X, np.array([0.0, 10.0]), num_trees=1, max_depth=1, lr=1.0, min_leaf=1)
    assert list(O.port_predict_features(g, X)) == [0.0, 10.0]
    Xc = np.random.default_rng(1).random((20, 3))
    g = O.ref_fit_gbt(Xc, np.full(20, 3.5), seed=1)
    assert np.all(O.port_predict_features(g, Xc) == 3.5)
    assert len(O.port_predict_features(g, np.zeros((0, 3)))) == 0
    # monotone training loss
    Xr = np.random.default_rng(2).random((200, 4))
    yr = np.random.default_rng(3).random(200)
    g = O.ref_fit_gbt(Xr, yr, seed=2)
    assert np.all(np.diff(g.training_sse) <= 1e-12)


def test_kmeans_kats(O):
    # SPEC.md:343-345
    P = np.array([[0.0], [0.0], [10.0], [10.0]])
    r = O.kmeans_run(P, 2, 1)
    assert sorted(r["centroids"][:, 0]) == [0.0, 10.0] and r["loss"] == 0.0
    Q = np.random.default_rng(0).random((12, 3))
    assert O.kmeans_run(Q, 12, 3)["loss"] == 0.0
    r = O.kmeans_run(Q, 1, 3)
    assert np.allclose(r["centroids"][0], Q.mean(0), rtol=0, atol=1e-15)
    assert math.isclose(r["loss"], ((Q - Q.mean(0)) ** 2).sum(), rel_tol=1e-12)
    # Lloyd loss non-increasing
    for s in range(5):
        R = np.random.default_rng(s).random((300, 4))
        il = O.kmeans_run(R, 7, s)["iteration_losses"]
        assert np.all(np.diff(il) <= 1e-9)


def test_snap_kat(O):
    # centroid [0.49] on a 3-valued knob -> index 1
    osp = O.OSpace(small([("a", [1, 2, 3])]))
    out = O.snap_centroid(osp, [0.49], np.zeros((0, 1), np.int32), np.zeros(0, np.uint64))
    assert out[0] == 1


def test_policy_value_forward_kats(O):
    # zero output layers -> uniform 1/3 per action, value 0;
    # triples sum to 1 (+-1e-9); batched is order-preserving.
    n, h, g = 4, 8, 6
    p = O.ac_init(n, h, g, 1)
    z = p.copy()
    off_wp2 = h * n + h + g * h + g
    z[off_wp2:off_wp2 + 3 * n * g] = 0.0
    off_wv2 = off_wp2 + 3 * n * g + 3 * n + g * h + g
    z[off_wv2:off_wv2 + g] = 0.0
    S_ = np.random.default_rng(0).random((5, n))
    out = O.ac_forward(n, h, g, z, S_)
    assert np.allclose(out["probs"], 1 / 3, rtol=0, atol=1e-15)
    assert np.all(out["values"] == 0.0)
    out = O.ac_forward(n, h, g, p, S_)
    assert np.all(np.abs(out["probs"].reshape(5, n, 3).sum(-1) - 1) <= 1e-9)
    one = O.ac_forward(n, h, g, p, S_[2:3])
    assert np.array_equal(one["log_probs"][0], out["log_probs"][2])


def test_sample_actions_kats(O):
    # uniform over 3 actions -> joint logp = -k ln3; degenerate
    # (1,0,0) -> all-decrement with logp 0; fixed seed reproducible.
    n, h, g = 5, 8, 4
    p = O.ac_init(n, h, g, 3)
    off_wp2 = h * n + h + g * h + g
    off_bp2 = off_wp2 + 3 * n * g
    z = p.copy()
    z[off_wp2:off_bp2] = 0.0
    sp = O.OSpace(S.small_space([4] * n))
    init = np.full((3, n), 2, np.int32)
    r = O.run_episodes(sp, None, h, g, z, init, T=4, episode_offset=0, explore_seed=11)
    assert np.allclose(r["logp"], -n * math.log(3), rtol=0, atol=1e-12)
    d = z.copy()
    d[off_bp2:off_bp2 + 3 * n] = np.tile([0.0, -800.0, -800.0], n)  # p = (1, 0, 0) exactly
    r = O.run_episodes(sp, None, h, g, d, init, T=3, episode_offset=0, explore_seed=11)
    assert np.all(r["actions"] == -1) and np.all(r["logp"] == 0.0)
    assert np.all(r["idx"][:, -1] == 0)
    a = O.run_episodes(sp, None, h, g, p, init, T=6, episode_offset=0, explore_seed=5)
    b = O.run_episodes(sp, None, h, g, p, init, T=6, episode_offset=0, explore_seed=5)
    assert np.array_equal(a["actions"], b["actions"])


def test_run_episodes_kats(O, ref_ok):
    # constant cost model -> all rewards 0; episodes x T shape
    n = 4
    sp = O.OSpace(S.small_space([5] * n))
    g = O.ref_fit_gbt(np.random.default_rng(0).random((10, n)), np.full(10, 2.0))
    p = O.ac_init(n, 16, 8, 0)
    init = np.zeros((6, n), np.int32)
    r = O.run_episodes(sp, g, 16, 8, p, init, T=7, episode_offset=0, explore_seed=1)
    assert r["idx"].shape == (6, 8, n) and np.all(np.diff(r["score"], axis=1) == 0.0)


def test_episode_sharding_invariance(O):
    # the RNG is keyed by the global episode id: a sharded run equals the full run
    n = 6
    sp = O.OSpace(S.synthetic_space(2, n))
    p = O.ac_init(n, 32, 16, 4)
    init = sp.random_valid(1, 10) if O.ref_available() else np.zeros((10, n), np.int32)
    full = O.run_episodes(sp, None, 32, 16, p, init, T=9, episode_offset=0, explore_seed=3)
    a = O.run_episodes(sp, None, 32, 16, p, init[:4], T=9, episode_offset=0, explore_seed=3)
    b = O.run_episodes(sp, None, 32, 16, p, init[4:], T=9, episode_offset=4, explore_seed=3, threads=3)
    assert np.array_equal(np.concatenate([a["idx"], b["idx"]]), full["idx"])
    assert np.array_equal(np.concatenate([a["logp"], b["logp"]]), full["logp"])


def test_portable_math_faithful(O):
    L = O.port()
    g = np.random.default_rng(0)
    xs = np.concatenate([g.normal(0, 3, 5000), g.uniform(-0.7, 0.7, 2000), [0.625, -0.625, 1e-300, 40.0]])
    for x in xs:
        assert abs(L.ko_tanh(x) - math.tanh(x)) <= 4e-16 * max(1.0, abs(math.tanh(x)))
        assert abs(L.ko_exp(x) - math.exp(x)) <= 4e-16 * math.exp(x)
        if x > 0:
            assert abs(L.ko_log(x) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))


def test_sa_search_oracle_spec_examples(O):
    """sa_search on the oracle: T -> 0 is a hill climb
    (fitness non-decreasing); Δ = 0 proposals are accepted
    (exp(0) = 1); deterministic from the seed."""
    from helpers import SPACES, fitted
    sp = SPACES["synthetic8"]()
    osp, og, _ = fitted(O, sp, seed=2)
    init = np.zeros((16, sp.num_knobs), np.int32)
    r = O.sa_search(osp, og, init, 60, 0, 77, 1e-300, 0.5)
    assert np.all(np.diff(r["score"], axis=1) >= 0)
    same = np.diff(r["score"], axis=1) == 0
    moved = np.any(r["idx"][:, 1:] != r["idx"][:, :-1], axis=2)
    assert np.all(r["accepted"][same & moved] == 1)
    r2 = O.sa_search(osp, og, init, 60, 0, 77, 1e-300, 0.5)
    assert np.array_equal(r["idx"], r2["idx"])
    hot = O.sa_search(osp, og, init, 60, 0, 77, 1.0, 0.99)  # T = 1: nearly every move accepted
    assert hot["accepted"].mean() > 0.9
