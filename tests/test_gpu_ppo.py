"""PPO training step on the device (csrc/ppo.cu) bit-exact against the oracle restatement
(ko_ac_forward/ko_ac_backward/ko_adam_step/ko_compute_gae/ko_ppo_update):
the Forward caches, the backward pass, Adam, GAE and whole ppo_update calls on a real
rollout trajectory (two consecutive updates: the Adam state carries over)."""
import numpy as np
import pytest

from helpers import SPACES, fitted

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["synthetic16", "resnet_c2"])
def test_forward_cache_and_backward_bit_exact(O, ctx, name):
    from paper_2001_08743_b200.exploration import ActorCritic
    sp = SPACES[name]()
    n = sp.num_knobs
    agent = ActorCritic(n, 128, 64, seed=3, ctx=ctx)
    g = np.random.default_rng(2)
    S = g.random((203, n))
    got = agent.forward_cache(S)
    want = O.ac_forward(n, 128, 64, agent.params, S)
    for k in ("h0", "hp", "hv", "logits", "log_probs", "probs", "values"):
        assert np.array_equal(got[k], want[k]), k
    dl, dv = g.normal(size=(203, 3 * n)), g.normal(size=203)
    assert np.array_equal(agent.backward(got, dl, dv), O.ac_backward(n, 128, 64, agent.params, got, dl, dv))


def test_adam_and_gae_bit_exact(O, ctx):
    from paper_2001_08743_b200.exploration import Adam, compute_gae
    g = np.random.default_rng(5)
    P = 21873
    p_dev, p_ref = g.normal(size=P), None
    p_ref = p_dev.copy()
    m, v = np.zeros(P), np.zeros(P)
    opt = Adam(P, 1e-3, ctx=ctx)
    for t in range(1, 4):
        gr = g.normal(size=P) * 10.0 ** g.integers(-6, 3)
        opt.step(p_dev, gr)
        O.adam_step(p_ref, gr, m, v, t)
    dm, dv, dt = opt.state()
    assert np.array_equal(p_dev, p_ref) and np.array_equal(dm, m) and np.array_equal(dv, v) and dt == 3
    r, val, tv = g.normal(size=(37, 50)), g.normal(size=(37, 50)), g.normal(size=37)
    a1, r1 = compute_gae(r, val, tv, 0.9, 0.99, ctx=ctx)
    a2, r2 = O.compute_gae(r, val, tv, 0.9, 0.99)
    assert np.array_equal(a1, a2) and np.array_equal(r1, r2)
    a1, _ = compute_gae([1.0, 1.0], [0.5, 0.5], [0.0], ctx=ctx)
    assert np.allclose(a1, [1.3955, 0.5], rtol=0, atol=1e-12)


def test_ppo_update_on_a_rollout_bit_exact(O, ctx):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import (ActorCritic, Adam, PpoParams, RolloutTask, compute_gae,
                                                   ppo_update, run_episodes_batch)
    sp = SPACES["resnet_c2"]()
    osp, og, pm = fitted(O, sp, seed=7)
    ds = Space(sp, ctx)
    agent = ActorCritic(sp.num_knobs, 128, 64, seed=11, ctx=ctx)
    n = sp.num_knobs
    E, T = 40, 30
    init = osp.random_valid(3, E) if O.ref_available() else np.zeros((E, n), np.int32)
    params = PpoParams(minibatch_size=256)
    opt = Adam(agent.num_parameters, params.adam_step_size, ctx=ctx)
    p_ref = agent.params.copy()
    m, v, t = np.zeros_like(p_ref), np.zeros_like(p_ref), 0
    for it in range(2):
        tr = run_episodes_batch([RolloutTask(ds, agent, DeviceGbt(pm, ds), init, 0, 5 + it)], T, exact=True)[0]
        X = osp.encode(tr["idx"].reshape(-1, n).astype(np.int32)).reshape(E, T + 1, n)
        term = agent.forward_cache(X[:, T])["values"]
        rew = tr["score"][:, 1:] - tr["score"][:, :-1]
        adv, ret = compute_gae(rew, tr["value"], term, params.discount_gamma, params.gae_lambda, ctx=ctx)
        a_ref, r_ref = O.compute_gae(rew, tr["value"], term, params.discount_gamma, params.gae_lambda)
        assert np.array_equal(adv, a_ref) and np.array_equal(ret, r_ref)
        S = X[:, :T].reshape(-1, n)
        st = ppo_update(agent, opt, S, tr["actions"].reshape(-1, n), tr["logp"].reshape(-1), adv.reshape(-1),
                        ret.reshape(-1), params, seed=100 + it)
        t, st_ref = O.ppo_update(n, 128, 64, p_ref, m, v, t, S, tr["actions"].reshape(-1, n), tr["logp"].reshape(-1),
                                 adv.reshape(-1), ret.reshape(-1), params.num_epochs, params.minibatch_size,
                                 params.adam_step_size, params.clip_epsilon, params.value_coef,
                                 params.entropy_coef, 100 + it)
        assert np.array_equal(agent.params, p_ref), f"update {it}: parameters differ"
        dm, dv, dt = opt.state()
        assert np.array_equal(dm, m) and np.array_equal(dv, v) and dt == t
        assert [st["policy_loss"], st["value_loss"], st["entropy"]] == list(st_ref)
        agent.set_parameters(agent.params)  # the rollout's TC path re-derives its scales from the host copy
