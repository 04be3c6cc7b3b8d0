"""K2 persistent rollout + K1 scoring through the C-ABI, bit-exact with the
oracle's run_episodes restatement."""
import numpy as np
import pytest

from helpers import SPACES, fitted

pytestmark = pytest.mark.gpu


def _setup(O, ctx, name, seed=0, h=128, g=64):
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import ActorCritic
    sp = SPACES[name]()
    osp, og, pm = fitted(O, sp, seed=seed)
    dspace = Space(sp, ctx)
    agent = ActorCritic(sp.num_knobs, h, g, seed=seed + 1, ctx=ctx)
    return sp, osp, og, dspace, DeviceGbt(pm, dspace), agent


def test_debug_math_bitwise(O, ctx):
    import ctypes as C
    from paper_2001_08743_b200 import _lib as L
    g = np.random.default_rng(0)
    xs = np.concatenate([g.normal(0, 4, 200_000), g.uniform(-0.7, 0.7, 100_000), g.uniform(0, 3, 100_000),
                         [0.0, -0.0, 0.625, -0.625, 1e-300, 709.0, -745.0, 800.0, 2 ** -30, 22.0, 400.0]])
    for op, fn in [(0, O.port().ko_exp), (1, O.port().ko_log), (2, O.port().ko_tanh)]:
        x = np.abs(xs) + 1e-300 if op == 1 else xs
        out = np.zeros_like(x)
        ctx.check(L.lib().ktune_debug_math(ctx.h, op, x.ctypes.data_as(C.c_void_p), len(x),
                                           out.ctypes.data_as(C.c_void_p)))
        want = np.array([fn(float(v)) for v in x])
        assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), op


@pytest.mark.parametrize("name", ["synthetic8", "synthetic16", "resnet_c2"])
def test_ac_forward_bit_exact(O, ctx, name):
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, name)
    S_ = np.random.default_rng(1).random((77, sp.num_knobs))
    got = agent.forward(S_)
    want = O.ac_forward(sp.num_knobs, 128, 64, agent.params, S_)
    for k in ["log_probs", "probs", "values"]:
        assert np.array_equal(got[k], want[k]), k


@pytest.mark.parametrize("name,E,T", [("resnet_c2", 37, 25), ("synthetic16", 33, 20),
                                      ("resnet_dense_u16", 5, 40), ("vgg_c4", 64, 12)])
def test_rollout_bit_exact(O, ctx, name, E, T):
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=E)
    init = osp.random_valid(E, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
    out = run_episodes_batch([RolloutTask(dspace, agent, dg, init, episode_offset=5, root_seed=17)], T,
                             exact=True)[0]
    from paper_2001_08743_b200.spaces import stream_seed
    want = O.run_episodes(osp, og, 128, 64, agent.params, init, T, 5, stream_seed(17, "explore"))
    assert np.array_equal(out["idx"].astype(np.int32), want["idx"])
    assert np.array_equal(out["actions"], want["actions"])
    assert np.array_equal(out["logp"], want["logp"])
    assert np.array_equal(out["value"], want["value"])
    assert np.array_equal(out["score"], want["score"])


def test_grouped_launch_matches_per_task(O, ctx):
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    tasks, wants = [], []
    for i, name in enumerate(["resnet_c2", "synthetic8", "resnet_dense_u16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=i)
        init = osp.random_valid(i, 40) if O.ref_available() else np.zeros((40, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=100 * i, root_seed=i))
        wants.append(O.run_episodes(osp, og, 128, 64, agent.params, init, 15, 100 * i, stream_seed(i, "explore")))
    outs = run_episodes_batch(tasks, 15, exact=True)
    for o, w in zip(outs, wants):
        assert np.array_equal(o["idx"].astype(np.int32), w["idx"])
        assert np.array_equal(o["score"], w["score"])
        assert np.array_equal(o["logp"], w["logp"])


def test_rollout_large_spot_replay(O, ctx):
    """4096 episodes on the GPU; 24 random episodes replayed individually on the
    oracle (counter-based RNG keyed by the global episode id)."""
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "resnet_c2", seed=9)
    E, T = 4096, 60
    init = osp.random_valid(9, E) if O.ref_available() else np.zeros((E, 8), np.int32)
    out = run_episodes_batch([RolloutTask(dspace, agent, dg, init, episode_offset=0, root_seed=3)], T)[0]
    for e in np.random.default_rng(0).choice(E, 24, replace=False):
        w = O.run_episodes(osp, og, 128, 64, agent.params, init[e:e + 1], T, int(e), stream_seed(3, "explore"))
        assert np.array_equal(out["idx"][e].astype(np.int32), w["idx"][0])
        assert np.array_equal(out["score"][e], w["score"][0])
    # properties at scale: saturating moves stay in range and move by at most 1 per knob
    idx = out["idx"].astype(np.int64)
    assert np.all(idx.max(axis=(0, 1)) < np.array(sp.cards))
    assert np.all(np.abs(np.diff(idx, axis=1)) <= 1)
    # every move is the saturating application of the recorded action (design_space.cpp:175-187)
    cards = np.array(sp.cards)
    assert np.array_equal(np.diff(idx, axis=1), np.clip(idx[:, :-1] + out["actions"], 0, cards - 1) - idx[:, :-1])


# ---------------------------------------------------------------- tcgen05 path
# Tolerances of the fast path (north star): configurations, actions and scores
# bit-exact; log-probabilities and values within 1e-5 relative (fp32-accurate;
# an absolute floor of 1e-5 covers values near zero).
def _close(a, b, tol=1e-5):
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("name,E,T", [("resnet_c2", 37, 25), ("synthetic16", 200, 30),
                                      ("resnet_dense_u16", 5, 40), ("vgg_c4", 300, 12),
                                      ("synthetic8", 129, 17)])
def test_rollout_tc_matches_oracle(O, ctx, name, E, T):
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=E)
    init = osp.random_valid(E, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
    out = run_episodes_batch([RolloutTask(dspace, agent, dg, init, episode_offset=5, root_seed=17)], T)[0]
    want = O.run_episodes(osp, og, 128, 64, agent.params, init, T, 5, stream_seed(17, "explore"))
    assert np.array_equal(out["idx"].astype(np.int32), want["idx"])
    assert np.array_equal(out["actions"], want["actions"])
    assert np.array_equal(out["score"], want["score"])
    assert _close(out["logp"], want["logp"]), np.abs(out["logp"] - want["logp"]).max()
    assert _close(out["value"], want["value"]), np.abs(out["value"] - want["value"]).max()


def test_rollout_tc_equals_exact_kernel_at_scale(O, ctx):
    """Grouped 12-task launch (the bench's shape, shorter episodes): the tcgen05
    path and the exact fp64 kernel visit identical configurations."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    names = ["resnet_c2", "vgg_c4", "synthetic8", "synthetic16"]
    tasks = []
    for i in range(12):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, names[i % 4], seed=i)
        init = osp.random_valid(i, 1024) if O.ref_available() else np.zeros((1024, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=1024 * i, root_seed=i))
    ctx.set_option(L.OPT_ROLLOUT_CHECK, 0)
    ctx.reset_stats()
    fast = run_episodes_batch(tasks, 64)
    nfb = ctx.stat(L.STAT_ROLLOUT_FALLBACKS)
    exact = run_episodes_batch(tasks, 64, exact=True)
    for f, x in zip(fast, exact):
        assert np.array_equal(f["idx"], x["idx"])
        assert np.array_equal(f["actions"], x["actions"])
        assert np.array_equal(f["score"], x["score"])
        assert _close(f["logp"], x["logp"]) and _close(f["value"], x["value"])
    steps = 12 * 1024 * 64
    print(f"fallback knob decisions: {nfb} / {steps * 8}+")
    assert nfb < 0.01 * steps


@pytest.mark.parametrize("E,T", [(60_001, 6), (2 * 56_832 + 97, 6), (60_001, 130)])
def test_rollout_more_episodes_than_one_wave(O, ctx, E, T):
    """A workload larger than one resident wave (12 warps on every SM) runs as full
    waves plus a thin remainder over every SM: the same trajectories as the exact
    kernel, episodes keyed by their global id across the wave boundary."""
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "synthetic8", seed=4)
    init = np.random.default_rng(E).integers(0, 2, (E, sp.num_knobs))
    task = RolloutTask(dspace, agent, dg, init, episode_offset=5, root_seed=4)
    fast = run_episodes_batch([task], T)[0]  # T >= 128: the segmented host path, every segment in waves
    exact = run_episodes_batch([task], T, exact=True)[0]
    assert np.array_equal(fast["idx"], exact["idx"])
    assert np.array_equal(fast["actions"], exact["actions"])
    assert np.array_equal(fast["score"], exact["score"])
    assert _close(fast["logp"], exact["logp"]) and _close(fast["value"], exact["value"])


def test_rollout_tc_certificate_check_mode(O, ctx):
    """Check mode re-decides every knob exactly: certified fast decisions never
    disagree, and the fast probabilities stay well inside the margin."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    tasks = []
    for i, name in enumerate(["resnet_c2", "synthetic16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=40 + i)
        init = osp.random_valid(i, 256) if O.ref_available() else np.zeros((256, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=0, root_seed=i))
    ctx.reset_stats()
    ctx.set_option(L.OPT_ROLLOUT_CHECK, 1)
    try:
        out = run_episodes_batch(tasks, 20)
    finally:
        ctx.set_option(L.OPT_ROLLOUT_CHECK, 0)
    checked = ctx.stat(L.STAT_ROLLOUT_CHECKED)
    assert checked == 256 * 20 * (8 + 16)
    assert ctx.stat(L.STAT_ROLLOUT_MISMATCH) == 0
    maxerr = ctx.stat(L.STAT_ROLLOUT_MAXERR) * 1e-12
    print(f"max |p_fast - p_exact| = {maxerr:.3e}")
    assert maxerr < 2 ** -18
    ref = run_episodes_batch(tasks, 20, exact=True)
    for o, r in zip(out, ref):
        assert np.array_equal(o["idx"], r["idx"])


def test_rollout_tc_fused_scores_equal_unfused(O, ctx):
    """GBT walk fused into the rollout epilogue vs the separate K1 launch: identical scores."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    tasks = []
    for i, name in enumerate(["resnet_c2", "synthetic16", "resnet_dense_u16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=60 + i)
        init = osp.random_valid(i, 300) if O.ref_available() else np.zeros((300, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=7, root_seed=i))
    sep = run_episodes_batch(tasks, 33)
    ctx.set_option(L.OPT_ROLLOUT_FUSE_GBT, 1)
    try:
        fused = run_episodes_batch(tasks, 33)
    finally:
        ctx.set_option(L.OPT_ROLLOUT_FUSE_GBT, 0)
    for f, s_ in zip(fused, sep):
        assert np.array_equal(f["idx"], s_["idx"])
        assert np.array_equal(f["score"], s_["score"])


def test_rollout_tc_segmented_host_path(O, ctx):
    """Host buffers with T >= 128: the rollout runs in step segments whose
    scoring and D2H copies overlap the next segment; results equal the
    device-buffer (single launch) path and the oracle."""
    import torch
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    tasks, dtasks, inits = [], [], []
    for i, name in enumerate(["resnet_c2", "synthetic16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=80 + i)
        init = osp.random_valid(i, 70) if O.ref_available() else np.zeros((70, sp.num_knobs), np.int32)
        inits.append((osp, og, agent, init))
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=3, root_seed=i))
        dtasks.append(RolloutTask(dspace, agent, dg, torch.from_numpy(init.astype(np.int32)).cuda(),
                                  episode_offset=3, root_seed=i))
    T = 333
    host = run_episodes_batch(tasks, T)
    devo = run_episodes_batch(dtasks, T)
    torch.cuda.synchronize()
    for h, d in zip(host, devo):
        for k in ["idx", "actions", "score", "logp", "value"]:
            diff = h[k] != d[k].cpu().numpy()
            where = np.nonzero(diff.any(-1) if diff.ndim == 3 else diff)
            assert not diff.any(), (k, int(diff.sum()), sorted(set(where[0].tolist()))[:8],
                                    sorted(set(where[1].tolist()))[:40])
    osp, og, agent, init = inits[0]
    want = O.run_episodes(osp, og, 128, 64, agent.params, init[:6], T, 3, stream_seed(0, "explore"))
    assert np.array_equal(host[0]["idx"][:6].astype(np.int32), want["idx"])
    assert np.array_equal(host[0]["score"][:6], want["score"])


@pytest.mark.parametrize("cards,E,T", [((5,), 1, 7), ((1, 3, 1, 9), 33, 12), ((2,) * 21, 40, 6), ((7, 4, 2), 65, 0),
                                       ((3, 17, 2, 5, 11), 97, 1)])
def test_rollout_tc_edge_shapes(O, ctx, cards, E, T):
    """Edge shapes on the tcgen05 path: one knob, cardinality-1 knobs, 21 knobs (the
    largest N3 <= 64), T = 0 / 1, episode counts that leave partial warps and tiles."""
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    sp = S.small_space(list(cards))
    osp, og, pm = fitted(O, sp, seed=E + T)
    ds = Space(sp, ctx)
    agent = ActorCritic(sp.num_knobs, 128, 64, seed=E, ctx=ctx)
    g = np.random.default_rng(E)
    init = np.stack([g.integers(0, c, E) for c in cards], 1).astype(np.int32)
    out = run_episodes_batch([RolloutTask(ds, agent, DeviceGbt(pm, ds), init, 11, 5)], T)[0]
    want = O.run_episodes(osp, og, 128, 64, agent.params, init, T, 11, stream_seed(5, "explore"))
    assert np.array_equal(out["idx"].astype(np.int32), want["idx"])
    assert np.array_equal(out["score"], want["score"])
    if T:
        assert np.array_equal(out["actions"], want["actions"])
        assert _close(out["logp"], want["logp"]) and _close(out["value"], want["value"])


@pytest.mark.parametrize("exact", [False, True])
def test_rollout_fp32_outputs(O, ctx, exact):
    """logp_f32 / value_f32 are the fp32 roundings of the fp64 outputs (host path, segmented)."""
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "resnet_c2", seed=91)
    E, T = 50, 140
    init = osp.random_valid(91, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
    mk = lambda: dict(idx=np.zeros((E, T + 1, sp.num_knobs), np.uint16), score=np.zeros((E, T + 1)),
                      actions=np.zeros((E, T, sp.num_knobs), np.int8), logp=np.zeros((E, T)),
                      value=np.zeros((E, T)), logp32=np.zeros((E, T), np.float32),
                      value32=np.zeros((E, T), np.float32))
    o = mk()
    o["idx8"] = np.zeros((E, T + 1, sp.num_knobs), np.uint8)
    o["score32"] = np.zeros((E, T + 1), np.float32)
    run_episodes_batch([RolloutTask(dspace, agent, dg, init, 0, 3)], T, host_out=[o], exact=exact)
    assert np.array_equal(o["score32"], o["score"].astype(np.float32))
    assert np.array_equal(o["logp32"], o["logp"].astype(np.float32))
    assert np.array_equal(o["value32"], o["value"].astype(np.float32))
    assert np.array_equal(o["idx8"], o["idx"].astype(np.uint8)) and o["idx"].max() < 256
    o2 = mk()
    o2["idx"] = None
    o2["idx8"] = np.zeros((E, T + 1, sp.num_knobs), np.uint8)
    o2["actions"] = None
    o2["actions2"] = np.zeros((E, T, (sp.num_knobs + 3) // 4), np.uint8)
    o2["score"] = None
    o2["score32"] = np.zeros((E, T + 1), np.float32)
    run_episodes_batch([RolloutTask(dspace, agent, dg, init, 0, 3)], T, host_out=[o2], exact=exact)
    assert np.array_equal(o2["idx8"], o["idx8"]) and np.array_equal(o2["score32"], o["score32"])
    from paper_2001_08743_b200.exploration import unpack_actions
    assert np.array_equal(unpack_actions(o2["actions2"], sp.num_knobs), o["actions"])


def test_rollout_tc_planted_draws(O, ctx):
    """Check mode 5: every draw is PLANTED 2 delta below or above a fast CDF value (where
    the certificate's margin is tightest) and every knob is then re-decided exactly with
    the same draw: the fast decisions never disagree."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    tasks = []
    for i, name in enumerate(["resnet_c2", "synthetic16", "vgg_c4"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=140 + i)
        init = osp.random_valid(i, 512) if O.ref_available() else np.zeros((512, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=0, root_seed=i))
    ctx.reset_stats()
    ctx.set_option(L.OPT_ROLLOUT_CHECK, 5)
    try:
        run_episodes_batch(tasks, 24)
    finally:
        ctx.set_option(L.OPT_ROLLOUT_CHECK, 0)
    assert ctx.stat(L.STAT_ROLLOUT_CHECKED) == 512 * 24 * (8 + 16 + 8)
    assert ctx.stat(L.STAT_ROLLOUT_MISMATCH) == 0
    print(f"planted: max |p0_fast - p0_exact| = {ctx.stat(L.STAT_ROLLOUT_MAXERR) * 1e-12:.3e}")


def test_rollout_tc_check_mode_c2_shape(O, ctx):
    """The bench's FULL shape (BASELINE configs[1]: 12 ResNet-18 tasks x 4096 episodes x T = 500,
    one grouped launch) in check mode: all 196.6M knob decisions re-decided exactly, 0
    disagreements, the fast probabilities well inside the margin; the trajectories (device
    buffers, step-major) equal the normal run's and the exact fp64 kernel's, spot episodes
    replay on the oracle, and the bench's end-to-end host call (streamed, configuration ids,
    compact and full-precision encodings) returns the same trajectories."""
    import torch
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import ActorCritic, RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    E, T = 4096, 500
    tasks, orc = [], []
    for i, sp in enumerate(S.resnet18_tasks()):
        osp, og, pm = fitted(O, sp, seed=200 + i)
        ds = Space(sp, ctx)
        agent = ActorCritic(sp.num_knobs, 128, 64, seed=200 + i, ctx=ctx)
        init = osp.random_valid(i, E) if O.ref_available() else np.zeros((E, sp.num_knobs), np.int32)
        tasks.append(RolloutTask(ds, agent, DeviceGbt(pm, ds), torch.from_numpy(init).cuda(), episode_offset=0,
                                 root_seed=i))
        orc.append((osp, og, agent, init))
    ctx.reset_stats()
    ctx.set_option(L.OPT_ROLLOUT_CHECK, 1)
    try:
        chk = run_episodes_batch(tasks, T, step_major=True)
        torch.cuda.synchronize()
    finally:
        ctx.set_option(L.OPT_ROLLOUT_CHECK, 0)
    assert ctx.stat(L.STAT_ROLLOUT_CHECKED) == 12 * E * T * 8
    assert ctx.stat(L.STAT_ROLLOUT_MISMATCH) == 0
    maxerr = ctx.stat(L.STAT_ROLLOUT_MAXERR) * 1e-12
    print(f"C2 shape: max |p_fast - p_exact| = {maxerr:.3e} over {12 * E * T * 8} decisions")
    assert maxerr < 2 ** -18
    ctx.reset_stats()
    fast = run_episodes_batch(tasks, T, step_major=True)
    exact = run_episodes_batch(tasks, T, exact=True, step_major=True)
    torch.cuda.synchronize()
    close = lambda a, b: bool(((a - b).abs() <= 1e-5 * b.abs().clamp_min(1.0)).all())
    for f, c, x in zip(fast, chk, exact):
        for k in ("idx", "actions", "score"):
            assert torch.equal(f[k], x[k]) and torch.equal(c[k], x[k]), k
        assert close(f["logp"], x["logp"]) and close(f["value"], x["value"])
    # the live margin monitor of the normal run: every fallback re-decision inside the margin
    assert ctx.stat(L.STAT_ROLLOUT_FALLBACKS) > 0 and ctx.stat(L.STAT_ROLLOUT_MAXERR) * 1e-12 < 2 ** -18
    g = np.random.default_rng(5)
    for i in g.choice(12, 3, replace=False):
        osp, og, agent, init = orc[i]
        for e in g.choice(E, 2, replace=False):
            w = O.run_episodes(osp, og, 128, 64, agent.params, init[e:e + 1], T, int(e), stream_seed(int(i), "explore"))
            assert np.array_equal(fast[i]["idx"][:, e].cpu().numpy().astype(np.int32), w["idx"][0])
            assert np.array_equal(fast[i]["actions"][:, e].cpu().numpy(), w["actions"][0])
            assert np.array_equal(fast[i]["score"][:, e].cpu().numpy(), w["score"][0])
    # the bench's end-to-end call at the same shape: host buffers, the streamed path, grouped
    # step-major compact outputs (configuration ids, 2-bit actions, fp32 / fp64 values)
    from paper_2001_08743_b200.context import host_empty
    from paper_2001_08743_b200.exploration import compact_grouped_outputs, unpack_actions
    htasks = [RolloutTask(t.space, t.agent, t.cost_model, o[3], episode_offset=0, root_seed=i)
              for i, (t, o) in enumerate(zip(tasks, orc))]
    for full in (False, True):
        outs = compact_grouped_outputs(htasks, T, lambda shape, dt: host_empty(shape, dt), score64=full,
                                       logp64=full, ids=True)
        run_episodes_batch(htasks, T, host_out=outs, grouped=True)
        for t, f, o in zip(tasks, fast, outs):
            ids = torch.zeros(f["idx"].shape[:-1], dtype=torch.int64, device="cuda")
            for d, c in enumerate(t.space.card):
                ids = ids * int(c) + f["idx"][..., d].to(torch.int64)
            assert np.array_equal(o["ids32"].astype(np.int64), ids.cpu().numpy())
            assert np.array_equal(unpack_actions(o["actions2"], t.space.D), f["actions"].cpu().numpy())
            sc, lp, va = (f[k].cpu().numpy() for k in ("score", "logp", "value"))
            if full:
                assert np.array_equal(o["score"], sc) and np.array_equal(o["logp"], lp) and np.array_equal(o["value"], va)
            else:  # the fp32 values the kernel computed (the device path widens the same fp32 values)
                assert np.array_equal(o["score32"], sc.astype(np.float32))
                assert np.array_equal(o["logp32"], lp.astype(np.float32)) and np.array_equal(o["value32"], va.astype(np.float32))
        del outs
    del chk, fast, exact
    torch.cuda.empty_cache()


@pytest.mark.parametrize("exact", [False, True])
def test_rollout_step_major_layout(O, ctx, exact):
    """KTUNE_F_STEP_MAJOR: the same trajectories transposed to [T+1][E] / [T][E] on every path -
    device buffers (one launch), host buffers (segmented, 1-D copies per segment), the compact
    outputs (idx_u8, actions_u2, score_f32, fp32 logp/value) and the exact fp64 kernel; equal to
    the episode-major call bit for bit and to the oracle."""
    import torch
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch, unpack_actions
    from paper_2001_08743_b200.spaces import stream_seed
    tasks, dtasks, inits = [], [], []
    for i, name in enumerate(["resnet_c2", "synthetic16", "synthetic8"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=120 + i)
        E = [70, 33, 129][i]
        init = np.random.default_rng(i).integers(0, 2, (E, sp.num_knobs)).astype(np.int32)
        inits.append((osp, og, agent, init))
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=7, root_seed=i))
        dtasks.append(RolloutTask(dspace, agent, dg, torch.from_numpy(init).cuda(), episode_offset=7, root_seed=i))
    T = 260
    em = run_episodes_batch(tasks, T, exact=exact)
    sm = run_episodes_batch(tasks, T, exact=exact, step_major=True)
    dv = run_episodes_batch(dtasks, T, exact=exact, step_major=True)
    torch.cuda.synchronize()
    for a, b, d in zip(em, sm, dv):
        for k in ["idx", "actions", "score", "logp", "value"]:
            assert b[k].shape[:2] == (a[k].shape[1], a[k].shape[0]), k
            assert np.array_equal(np.swapaxes(a[k], 0, 1), b[k]), k
            assert np.array_equal(d[k].cpu().numpy(), b[k]), k
    osp, og, agent, init = inits[0]
    want = O.run_episodes(osp, og, 128, 64, agent.params, init[:5], T, 7, stream_seed(0, "explore"))
    assert np.array_equal(np.swapaxes(sm[0]["idx"][:, :5], 0, 1).astype(np.int32), want["idx"])
    assert np.array_equal(np.swapaxes(sm[0]["score"][:, :5], 0, 1), want["score"])
    # compact outputs, step-major, on the resnet task (every cardinality <= 256)
    E, D = len(inits[0][3]), tasks[0].space.D
    o = dict(idx=None, idx8=np.zeros((T + 1, E, D), np.uint8), actions=None,
             actions2=np.zeros((T, E, (D + 3) // 4), np.uint8), score=None, score32=np.zeros((T + 1, E), np.float32),
             logp=None, value=None, logp32=np.zeros((T, E), np.float32), value32=np.zeros((T, E), np.float32))
    run_episodes_batch(tasks[:1], T, host_out=[o], exact=exact, step_major=True)
    assert np.array_equal(o["idx8"], sm[0]["idx"].astype(np.uint8))
    assert np.array_equal(unpack_actions(o["actions2"], D), sm[0]["actions"])
    assert np.array_equal(o["score32"], sm[0]["score"].astype(np.float32))
    assert np.array_equal(o["logp32"], sm[0]["logp"].astype(np.float32))
    assert np.array_equal(o["value32"], sm[0]["value"].astype(np.float32))


def test_rollout_step_major_multi_wave(O, ctx):
    """Step-major with more episodes than one resident wave (full waves + the spread remainder
    advance the trajectory pointers by episode, i.e. by one row within every step block)."""
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "synthetic8", seed=9)
    E, T = 60_001, 5
    init = np.random.default_rng(E).integers(0, 2, (E, sp.num_knobs))
    task = RolloutTask(dspace, agent, dg, init, episode_offset=2, root_seed=9)
    a = run_episodes_batch([task], T)[0]
    b = run_episodes_batch([task], T, step_major=True)[0]
    for k in ["idx", "actions", "score", "logp", "value"]:
        assert np.array_equal(np.swapaxes(a[k], 0, 1), b[k]), k


def test_rollout_step_major_grouped(O, ctx):
    """KTUNE_F_STEP_MAJOR_GROUPED: all tasks' episodes side by side in one step-major array per
    output (one PCIe copy per output per segment); every task's column block equals its own
    step-major call, on the host (segmented) and device paths and for the compact outputs."""
    import torch
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, grouped_outputs, run_episodes_batch, unpack_actions
    from paper_2001_08743_b200.errors import ConfigError
    tasks, dtasks = [], []
    for i, name in enumerate(["resnet_c2", "vgg_c4", "synthetic8"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=160 + i)
        E = [70, 129, 33][i]
        init = np.random.default_rng(i).integers(0, 2, (E, sp.num_knobs)).astype(np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=3 * i, root_seed=i))
        dtasks.append(RolloutTask(dspace, agent, dg, torch.from_numpy(init).cuda(), episode_offset=3 * i, root_seed=i))
    T = 260
    ref = run_episodes_batch(tasks, T, step_major=True)
    grp = run_episodes_batch(tasks, T, grouped=True)
    dgp = run_episodes_batch(dtasks, T, grouped=True)
    torch.cuda.synchronize()
    for a, b, d in zip(ref, grp, dgp):
        for k in ["idx", "actions", "score", "logp", "value"]:
            assert np.array_equal(a[k], b[k]), k
            assert np.array_equal(a[k], d[k].cpu().numpy()), k
    D = tasks[0].space.D
    fields = {"idx8": (T + 1, D), "actions2": (T, (D + 3) // 4), "score32": (T + 1, None), "logp32": (T, None),
              "value32": (T, None)}
    dts = {"idx8": np.uint8, "actions2": np.uint8, "score32": np.float32, "logp32": np.float32, "value32": np.float32}
    outs = grouped_outputs(tasks, T, lambda shape, name: np.zeros(shape, dts[name]), fields)
    for o in outs:
        o.update(idx=None, actions=None, score=None, logp=None, value=None)
    run_episodes_batch(tasks, T, host_out=outs, grouped=True)
    for a, o in zip(ref, outs):
        assert np.array_equal(o["idx8"], a["idx"].astype(np.uint8))
        assert np.array_equal(unpack_actions(o["actions2"], D), a["actions"])
        assert np.array_equal(o["score32"], a["score"].astype(np.float32))
        assert np.array_equal(o["logp32"], a["logp"].astype(np.float32))
    # the bench's shape: a task whose cardinalities exceed 256 ships uint16 idx while the others ship
    # idx_u8; each output's run of tasks is its own W-wide array (2-D copies out of the Etot-wide rows)
    from paper_2001_08743_b200 import spaces as S
    from paper_2001_08743_b200.context import Space
    from paper_2001_08743_b200.cost_model import DeviceGbt
    from paper_2001_08743_b200.exploration import ActorCritic
    sp = SPACES["resnet_dense_u16"]()
    osp, og, pm = fitted(O, sp, seed=7)
    ds = Space(sp, ctx)
    wide = RolloutTask(ds, ActorCritic(sp.num_knobs, 128, 64, seed=7, ctx=ctx), DeviceGbt(pm, ds),
                       np.zeros((45, sp.num_knobs), np.int32), 0, 7)
    mixed = tasks[:2] + [wide]
    refm = run_episodes_batch(mixed, T, step_major=True)
    f8 = {"idx8": (T + 1, D), "score32": (T + 1, None)}
    o8 = grouped_outputs(mixed[:2], T, lambda shape, name: np.zeros(shape, np.uint8 if name == "idx8" else np.float32), f8)
    o16 = grouped_outputs(mixed[2:], T, lambda shape, name: np.zeros(shape, np.uint16 if name == "idx" else np.float32),
                          {"idx": (T + 1, D), "score32": (T + 1, None)})
    sc = np.zeros((T + 1, sum(len(t.init_idx) for t in mixed)), np.float32)  # one score32 array over all three
    offs = np.cumsum([0] + [len(t.init_idx) for t in mixed])
    outs_m = []
    for i, o in enumerate(o8 + o16):
        o = dict(o)
        o["score32"] = sc[:, offs[i]:offs[i + 1]]
        o.setdefault("idx", None)
        o.setdefault("idx8", None)
        o.update(actions=None, score=None, logp=None, value=None)
        outs_m.append(o)
    run_episodes_batch(mixed, T, host_out=outs_m, grouped=True)
    for a, o in zip(refm, outs_m):
        got = o["idx8"] if o["idx8"] is not None else o["idx"]
        assert np.array_equal(got.astype(np.int64), a["idx"].astype(np.int64))
        assert np.array_equal(o["score32"], a["score"].astype(np.float32))
    # misplaced task pointers are rejected
    bad = grouped_outputs(tasks[:2], T, lambda shape, name: np.zeros(shape, np.float64 if name != "idx" else np.uint16),
                          {"idx": (T + 1, D), "score": (T + 1, None)})
    bad[1]["idx"] = np.zeros((T + 1, 129, D), np.uint16)
    for o in bad:
        o.update(actions=None, logp=None, value=None)
    with pytest.raises(ConfigError):
        run_episodes_batch(tasks[:2], T, host_out=bad, grouped=True)


def test_rollout_ids_u32(O, ctx):
    """ids_u32: one id_of(Θ_t) per visited configuration (design_space.cpp:158-167) instead of D
    knob indices - equal to the mixed-radix id of the idx trajectory on every layout (grouped over
    tasks of different radices incl. a uint16 space, step-major, episode-major segmented host path,
    device pointers); configs_from_ids inverts it; spaces over 2^32 configurations are rejected."""
    import torch
    from paper_2001_08743_b200.errors import ConfigError
    from paper_2001_08743_b200.exploration import (RolloutTask, compact_grouped_outputs, configs_from_ids,
                                                   run_episodes_batch)

    def id_of(idx, cards):
        r = np.zeros(idx.shape[:-1], np.uint64)
        for d, c in enumerate(cards):
            r = r * np.uint64(c) + idx[..., d].astype(np.uint64)
        return r

    tasks, dtasks = [], []
    for i, name in enumerate(["resnet_c2", "vgg_c4", "resnet_dense_u16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=170 + i)
        E = [70, 129, 45][i]
        init = np.random.default_rng(i).integers(0, np.asarray(sp.cards), (E, sp.num_knobs)).astype(np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=5 * i, root_seed=i))
        dtasks.append(RolloutTask(dspace, agent, dg, torch.from_numpy(init).cuda(), episode_offset=5 * i, root_seed=i))
    T = 260
    cards = [t.space.card for t in tasks]
    ref = run_episodes_batch(tasks, T, step_major=True)
    # grouped compact outputs with ids: no idx array at all crosses PCIe
    outs = compact_grouped_outputs(tasks, T, lambda shape, dt: np.zeros(shape, dt), ids=True)
    run_episodes_batch(tasks, T, host_out=outs, grouped=True)
    for a, o, c in zip(ref, outs, cards):
        assert o["idx"] is None and o["idx8"] is None
        assert np.array_equal(o["ids32"].astype(np.uint64), id_of(a["idx"], c))
        assert np.array_equal(configs_from_ids(o["ids32"], c), a["idx"])
        assert np.array_equal(o["score32"], a["score"].astype(np.float32))
    # step-major and episode-major (segmented) host calls, per task buffers
    for sm in (True, False):
        hs = []
        for t in tasks:
            E = len(t.init_idx)
            hs.append(dict(idx=None, score=np.zeros((T + 1, E) if sm else (E, T + 1)), actions=None, logp=None,
                           value=None, ids32=np.zeros((T + 1, E) if sm else (E, T + 1), np.uint32)))
        run_episodes_batch(tasks, T, host_out=hs, step_major=sm)
        for a, o, c in zip(ref, hs, cards):
            want = id_of(a["idx"], c) if sm else id_of(a["idx"], c).T
            assert np.array_equal(o["ids32"].astype(np.uint64), want), sm
            assert np.array_equal(o["score"], a["score"] if sm else a["score"].T), sm
    # device pointers (idx alongside, as every device call needs)
    dref = run_episodes_batch(dtasks, T, device_out=True, step_major=True)
    douts = []
    for t, o in zip(dtasks, dref):
        o = dict(o)
        o["ids32"] = torch.zeros((T + 1, len(t.init_idx)), dtype=torch.int32, device="cuda")
        douts.append(o)
    run_episodes_batch(dtasks, T, host_out=douts, step_major=True)
    torch.cuda.synchronize()
    for a, o, c in zip(ref, douts, cards):
        got = o["ids32"].cpu().numpy().view(np.uint32).astype(np.uint64)
        assert np.array_equal(got, id_of(a["idx"], c))
    # > 2^32 configurations: rejected
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "synthetic8", seed=3)
    big = RolloutTask(dspace, agent, dg, np.zeros((4, sp.num_knobs), np.int32))
    with pytest.raises(ConfigError):
        run_episodes_batch([big], 8, host_out=[dict(idx=None, score=None, actions=None, logp=None, value=None,
                                                    ids32=np.zeros((4, 9), np.uint32))])


def test_rollout_streamed_host_path_repeated(O, ctx):
    """The streamed host-buffer path (one rollout launch; the copy stream waits on the kernel's
    per-segment progress counter) against the per-segment launches and the device path, over
    repeated calls and several shapes (segment counts, one and several launches, every
    encoding): the copies never read a row before it is written."""
    import torch
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, compact_grouped_outputs, run_episodes_batch
    tasks = []
    for i, name in enumerate(["resnet_c2", "vgg_c4", "alexnet_c3_u16"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=190 + i)
        E = [600, 257, 1000][i]
        init = np.random.default_rng(i).integers(0, np.asarray(sp.cards), (E, sp.num_knobs)).astype(np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=11 * i, root_seed=i))
    for T, segs in [(200, 0), (333, 0), (128, 2), (260, 32)]:
        dref = run_episodes_batch([RolloutTask(t.space, t.agent, t.cost_model, torch.from_numpy(t.init_idx).cuda(),
                                               t.episode_offset, t.root_seed) for t in tasks], T, step_major=True)
        torch.cuda.synchronize()
        ref = [{k: v.cpu().numpy() for k, v in o.items()} for o in dref]
        ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, segs)
        try:
            for rep in range(3):
                hs = run_episodes_batch(tasks, T, step_major=True)
                for a, h in zip(ref, hs):
                    for k in ["idx", "actions", "score", "logp", "value"]:
                        assert np.array_equal(a[k], h[k]), (T, segs, rep, k)
                outs = compact_grouped_outputs(tasks, T, lambda shape, dt: np.zeros(shape, dt), ids=(rep % 2 == 0))
                run_episodes_batch(tasks, T, host_out=outs, grouped=True)
                for a, o, t in zip(ref, outs, tasks):
                    if o["ids32"] is not None:
                        r = np.zeros(a["idx"].shape[:-1], np.uint64)
                        for d, c in enumerate(t.space.card):
                            r = r * np.uint64(c) + a["idx"][..., d].astype(np.uint64)
                        assert np.array_equal(o["ids32"].astype(np.uint64), r), (T, segs, rep)
                    else:
                        got = o["idx8"] if o["idx8"] is not None else o["idx"]
                        assert np.array_equal(got.astype(np.int64), a["idx"].astype(np.int64)), (T, segs, rep)
                    assert np.array_equal(o["score32"], a["score"].astype(np.float32)), (T, segs, rep)
                    assert np.array_equal(o["logp32"], a["logp"].astype(np.float32)), (T, segs, rep)
        finally:
            ctx.set_option(L.OPT_ROLLOUT_SEGMENTS, 0)


def test_rollout_streamed_more_tasks_than_one_launch(O, ctx):
    """More tasks than one tcgen05 launch holds (several launches in stream order, every slot of
    every launch counted per segment), host buffers: equal to the device path."""
    import torch
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    names = ["resnet_c2", "vgg_c4", "synthetic8", "alexnet_c3_u16"]
    tasks, dtasks = [], []
    for i in range(20):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, names[i % 4], seed=300 + i)
        E = 33 + 7 * i
        init = np.random.default_rng(i).integers(0, np.asarray(sp.cards), (E, sp.num_knobs)).astype(np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=i, root_seed=i))
        dtasks.append(RolloutTask(dspace, agent, dg, torch.from_numpy(init).cuda(), episode_offset=i, root_seed=i))
    T = 150
    host = run_episodes_batch(tasks, T)
    dev = run_episodes_batch(dtasks, T)
    torch.cuda.synchronize()
    for h, d in zip(host, dev):
        for k in ["idx", "actions", "score", "logp", "value"]:
            assert np.array_equal(h[k], d[k].cpu().numpy()), k


def test_rollout_c5_shape_equals_exact_kernel(O, ctx):
    """SURVEY C5's shape in the driver-run suite (synthetic 16-knob space, 2^20 episodes: ~18
    resident waves of the tcgen05 kernel), T = 48: visited configurations, actions and scores equal
    to the exact fp64 kernel's, logp/value within 1e-5; spot episodes replay on the oracle."""
    import torch
    from paper_2001_08743_b200.exploration import RolloutTask, run_episodes_batch
    from paper_2001_08743_b200.spaces import stream_seed
    sp, osp, og, dspace, dg, agent = _setup(O, ctx, "synthetic16", seed=500)
    E, T = 1 << 20, 48
    init = torch.zeros((E, sp.num_knobs), dtype=torch.uint16, device="cuda")
    task = RolloutTask(dspace, agent, dg, init, episode_offset=0, root_seed=9)
    fast = run_episodes_batch([task], T, step_major=True)[0]
    exact = run_episodes_batch([task], T, exact=True, step_major=True)[0]
    torch.cuda.synchronize()
    for k in ("idx", "actions", "score"):
        assert torch.equal(fast[k], exact[k]), k
    for k in ("logp", "value"):
        assert bool(((fast[k] - exact[k]).abs() <= 1e-5 * exact[k].abs().clamp_min(1.0)).all()), k
    for e in (0, 123_457, E - 1):
        w = O.run_episodes(osp, og, 128, 64, agent.params, np.zeros((1, sp.num_knobs), np.int32), T, e,
                           stream_seed(9, "explore"))
        assert np.array_equal(fast["idx"][:, e].cpu().numpy().astype(np.int32), w["idx"][0])
    del fast, exact
    torch.cuda.empty_cache()


def test_rollout_segmented_fallback_path(O, ctx):
    """KTUNE_OPT_ROLLOUT_STREAMED = 1 (one launch per segment: the path taken when the driver has
    no stream memory operations) gives the same trajectories as the streamed default."""
    from paper_2001_08743_b200 import _lib as L
    from paper_2001_08743_b200.exploration import RolloutTask, compact_grouped_outputs, run_episodes_batch
    tasks = []
    for i, name in enumerate(["resnet_c2", "vgg_c4"]):
        sp, osp, og, dspace, dg, agent = _setup(O, ctx, name, seed=400 + i)
        E = [300, 170][i]
        init = np.random.default_rng(i).integers(0, np.asarray(sp.cards), (E, sp.num_knobs)).astype(np.int32)
        tasks.append(RolloutTask(dspace, agent, dg, init, episode_offset=i, root_seed=i))
    T = 210
    res = {}
    for mode in (0, 1):
        ctx.set_option(L.OPT_ROLLOUT_STREAMED, mode)
        try:
            plain = run_episodes_batch(tasks, T)
            comp = compact_grouped_outputs(tasks, T, lambda shape, dt: np.zeros(shape, dt), ids=True)
            run_episodes_batch(tasks, T, host_out=comp, grouped=True)
        finally:
            ctx.set_option(L.OPT_ROLLOUT_STREAMED, 0)
        res[mode] = (plain, comp)
    for a, b in zip(res[0][0], res[1][0]):
        for k in ["idx", "actions", "score", "logp", "value"]:
            assert np.array_equal(a[k], b[k]), k
    for a, b in zip(res[0][1], res[1][1]):
        for k in ["ids32", "actions2", "score32", "logp32", "value32"]:
            assert np.array_equal(a[k], b[k]), k
