"""SPEC known answers and properties of the PPO training step on the
oracle restatement (oracle/ktune_oracle.c) the device path is checked
against: the GAE examples and the direct-sum identity, the finite-difference gradient
check of the full loss (relative error <= 1e-4), zero-advantage and
on-policy identities."""
import numpy as np
import pytest


def test_gae_known_answers(O):
    adv, ret = O.compute_gae([1.0, 1.0], [0.5, 0.5], [0.0], 0.9, 0.99)
    assert np.allclose(adv, [1.3955, 0.5], rtol=0, atol=1e-12)
    assert np.allclose(ret, [1.8955, 1.0], rtol=0, atol=1e-12)
    adv, _ = O.compute_gae(np.zeros(7), np.zeros(7), [0.0])
    assert np.array_equal(adv, np.zeros(7))
    adv, _ = O.compute_gae([0.7], [0.2], [1.5], 1.0, 1.0)  # A_0 = r_0 + terminal - v_0
    assert adv[0] == 0.7 + 1.5 - 0.2


def test_gae_matches_direct_sum(O):
    g = np.random.default_rng(3)
    E, T, gam, lam = 5, 40, 0.9, 0.99
    r, v, tv = g.normal(size=(E, T)), g.normal(size=(E, T)), g.normal(size=E)
    adv, ret = O.compute_gae(r, v, tv, gam, lam)
    vn = np.concatenate([v[:, 1:], tv[:, None]], 1)
    delta = r + gam * vn - v
    for t in range(T):
        direct = sum((gam * lam) ** k * delta[:, t + k] for k in range(T - t))
        assert np.allclose(adv[:, t], direct, rtol=1e-10, atol=1e-10)
    assert np.allclose(ret, adv + v, rtol=0, atol=0)


def _loss(O, n, h, g, p, S, A, old, adv, ret, ce=0.1, cv=1.0, eps=0.3):
    f = O.ac_forward(n, h, g, p, S)
    B = len(S)
    lp = np.array([sum(f["log_probs"][b, 3 * d + A[b, d] + 1] for d in range(n)) for b in range(B)])
    rho = np.exp(lp - old)
    s = np.minimum(rho * adv, np.clip(rho, 1 - eps, 1 + eps) * adv)
    H = -(f["probs"] * f["log_probs"]).sum(1)
    return -s.mean() + cv * ((f["values"] - ret) ** 2).mean() - ce * H.mean(), f


def test_finite_difference_gradient(O):
    """analytic gradient of the total loss vs central differences on a 2-knob,
    hidden_dim = 4 net, step 1e-5, relative error <= 1e-4."""
    n, h, g = 2, 4, 4
    p = O.ac_init(n, h, g, 5) * 1.7
    rng = np.random.default_rng(0)
    B = 6
    S = rng.random((B, n))
    A = rng.integers(-1, 2, (B, n)).astype(np.int8)
    f0 = O.ac_forward(n, h, g, p, S)
    old = np.array([sum(f0["log_probs"][b, 3 * d + A[b, d] + 1] for d in range(n)) for b in range(B)])
    adv, ret = rng.normal(size=B), rng.normal(size=B)
    _, f = _loss(O, n, h, g, p, S, A, old, adv, ret)
    dl, dv, _ = O.ppo_loss_grad(n, f, A, old, adv, ret)
    grad = O.ac_backward(n, h, g, p, dict(states=S, h0=f["h0"], hp=f["hp"], hv=f["hv"]), dl, dv)
    fd = np.zeros_like(p)
    for i in range(len(p)):
        q = p.copy()
        q[i] += 1e-5
        lp_, _ = _loss(O, n, h, g, q, S, A, old, adv, ret)
        q[i] -= 2e-5
        lm_, _ = _loss(O, n, h, g, q, S, A, old, adv, ret)
        fd[i] = (lp_ - lm_) / 2e-5
    rel = np.abs(grad - fd) / np.maximum(np.abs(fd), 1e-3)
    assert rel.max() <= 1e-4, rel.max()


def test_zero_advantage_and_on_policy_identities(O):
    n, h, g = 3, 8, 5
    p = O.ac_init(n, h, g, 9)
    rng = np.random.default_rng(1)
    B = 10
    S = rng.random((B, n))
    A = rng.integers(-1, 2, (B, n)).astype(np.int8)
    f = O.ac_forward(n, h, g, p, S)
    lp = np.array([sum(f["log_probs"][b, 3 * d + A[b, d] + 1] for d in range(n)) for b in range(B)])
    # zero advantages, no value/entropy terms: no gradient reaches the logits
    dl, dv, sums = O.ppo_loss_grad(n, f, A, lp, np.zeros(B), f["values"], 0.3, 0.0, 0.0)
    assert np.array_equal(dl, np.zeros_like(dl)) and np.array_equal(dv, np.zeros(B)) and sums[0] == 0.0
    # rho = 1 on-policy: clipped and unclipped surrogates agree
    adv = rng.normal(size=B)
    _, _, s1 = O.ppo_loss_grad(n, f, A, lp, adv, f["values"], 0.3, 1.0, 0.1)
    _, _, s2 = O.ppo_loss_grad(n, f, A, lp, adv, f["values"], 1e-9, 1.0, 0.1)
    assert np.isclose(s1[0], adv.sum(), rtol=1e-12) and np.isclose(s2[0], adv.sum(), rtol=1e-12)


def test_ppo_update_reduces_the_loss(O):
    n, h, g = 2, 16, 8
    p = O.ac_init(n, h, g, 2)
    rng = np.random.default_rng(4)
    N = 300
    S = rng.random((N, n))
    f = O.ac_forward(n, h, g, p, S)
    A = rng.integers(-1, 2, (N, n)).astype(np.int8)
    old = np.array([sum(f["log_probs"][b, 3 * d + A[b, d] + 1] for d in range(n)) for b in range(N)])
    adv = (A[:, 0] == 1).astype(float) - 0.5  # reward "increment knob 0"
    ret = np.zeros(N)
    m, v = np.zeros_like(p), np.zeros_like(p)
    q = p.copy()
    t, st = O.ppo_update(n, h, g, q, m, v, 0, S, A, old, adv, ret, num_epochs=3, mb=64, lr=1e-2)
    assert t == 3 * 5 and np.all(np.isfinite(st))
    f2 = O.ac_forward(n, h, g, q, S)
    assert f2["probs"][:, 2].mean() > f["probs"][:, 2].mean()  # P(increment knob 0) went up
