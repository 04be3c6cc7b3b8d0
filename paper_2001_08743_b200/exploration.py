"""Adaptive Exploration on the GPU: ActorCritic (actor_critic.hpp:18-64) and
run_episodes through the persistent rollout kernel (K2).

Builder-pinned details (no reference code exists for this module):
DESIGN.md §5 — flat parameter layout of actor_critic.hpp:52-53 with
column-major matrices, seeded init, fp64 forward with the portable
tanh/exp/log, counter-based RNG u(e,t,d) = hash01(stream_seed(root,"explore"),
(e*T+t)*D+d) keyed by the GLOBAL episode id e, inverse-CDF sampling,
saturating apply, every episode runs exactly T steps.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _lib as L
from .context import Context, Space, default_context, host_empty, ptr_of
from .cost_model import DeviceGbt
from .errors import ConfigError
from .spaces import mix64, stream_seed


def num_parameters(n: int, h: int = 128, g: int = 64) -> int:
    return int(L.lib().ktune_ac_num_params(n, h, g))


def init_parameters(n: int, h: int = 128, g: int = 64, seed: int = 0) -> np.ndarray:
    p = np.zeros(num_parameters(n, h, g), np.float64)
    L.check(L.lib().ktune_ac_init_params(n, h, g, seed, p.ctypes.data_as(C.c_void_p)))
    return p


class ActorCritic:
    """ktune::ActorCritic (actor_critic.hpp:18-64); forward runs on the GPU."""

    def __init__(self, num_knobs: int, hidden_dim: int = 128, head_hidden: int = 64, seed: int = 0,
                 params: Optional[np.ndarray] = None, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.n, self.h, self.g = num_knobs, hidden_dim, head_hidden
        self.params = (np.ascontiguousarray(params, np.float64).copy() if params is not None
                       else init_parameters(num_knobs, hidden_dim, head_hidden, seed))
        if len(self.params) != num_parameters(num_knobs, hidden_dim, head_hidden):
            raise ConfigError("actor-critic: parameter vector has the wrong length")
        self.h_dev = None
        self._upload()

    def _upload(self):
        if self.h_dev is not None:
            L.lib().ktune_ac_destroy(self.h_dev)
        h = C.c_void_p()
        self.ctx.check(L.lib().ktune_ac_create(self.ctx.h, self.n, self.h, self.g,
                                               self.params.ctypes.data_as(C.c_void_p), C.byref(h)))
        self.h_dev = h

    def set_parameters(self, params: np.ndarray) -> None:
        self.params = np.ascontiguousarray(params, np.float64).copy()
        self._upload()

    @property
    def num_parameters(self) -> int:
        return len(self.params)

    def forward(self, states):
        """Returns dict(log_probs B x 3n, probs B x 3n, values B) (actor_critic.hpp:30-43)."""
        S = np.ascontiguousarray(states, np.float64).reshape(-1, self.n)
        B = len(S)
        lp = np.zeros((B, 3 * self.n))
        pr = np.zeros((B, 3 * self.n))
        v = np.zeros(B)
        if B:
            self.ctx.check(L.lib().ktune_ac_forward(self.ctx.h, self.h_dev, S.ctypes.data_as(C.c_void_p), B,
                                                    lp.ctypes.data_as(C.c_void_p), pr.ctypes.data_as(C.c_void_p),
                                                    v.ctypes.data_as(C.c_void_p), 0))
        return dict(log_probs=lp, probs=pr, values=v)

    def forward_cache(self, states):
        """ActorCritic::forward with the full Forward cache (actor_critic.hpp:31-43): dict(states,
        h0, hp, hv, logits, log_probs, probs, values), exact fp64 (bit-exact with the oracle)."""
        S = np.ascontiguousarray(states, np.float64).reshape(-1, self.n)
        B = len(S)
        out = dict(states=S, h0=np.zeros((B, self.h)), hp=np.zeros((B, self.g)), hv=np.zeros((B, self.g)),
                   logits=np.zeros((B, 3 * self.n)), log_probs=np.zeros((B, 3 * self.n)),
                   probs=np.zeros((B, 3 * self.n)), values=np.zeros(B))
        if B:
            p = lambda k: out[k].ctypes.data_as(C.c_void_p)
            self.ctx.check(L.lib().ktune_ac_forward_cache(self.ctx.h, self.h_dev, p("states"), B, p("h0"), p("hp"),
                                                          p("hv"), p("logits"), p("log_probs"), p("probs"),
                                                          p("values"), 0))
        return out

    def backward(self, cache, d_logits, d_values) -> np.ndarray:
        """ActorCritic::backward (actor_critic.hpp:45-49) -> flat parameter gradient."""
        B = len(cache["states"])
        dl = np.ascontiguousarray(d_logits, np.float64).reshape(B, 3 * self.n)
        dv = np.ascontiguousarray(d_values, np.float64).reshape(B)
        grad = np.zeros(self.num_parameters)
        c = {k: np.ascontiguousarray(cache[k], np.float64) for k in ("states", "h0", "hp", "hv")}
        p = lambda a: a.ctypes.data_as(C.c_void_p)
        self.ctx.check(L.lib().ktune_ac_backward(self.ctx.h, self.h_dev, p(c["states"]), p(c["h0"]), p(c["hp"]),
                                                 p(c["hv"]), B, p(dl), p(dv), p(grad), 0))
        return grad

    def sync_parameters(self) -> np.ndarray:
        """Refresh the host copy after device-side training (ppo_update)."""
        self.ctx.check(L.lib().ktune_ac_get_params(self.ctx.h, self.h_dev, self.params.ctypes.data_as(C.c_void_p)))
        return self.params

    def __del__(self):
        try:
            if self.h_dev is not None:
                L.lib().ktune_ac_destroy(self.h_dev)
        except Exception:
            pass


class Adam:
    """ktune::AdamOptimizer (actor_critic.hpp:66-79); moments live on the device."""

    def __init__(self, dim: int, step_size: float = 1e-3, beta1: float = 0.9, beta2: float = 0.999,
                 epsilon: float = 1e-8, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.dim = dim
        h = C.c_void_p()
        self.ctx.check(L.lib().ktune_adam_create(self.ctx.h, dim, step_size, beta1, beta2, epsilon, C.byref(h)))
        self.h = h

    def step(self, params: np.ndarray, grad) -> None:
        """AdamOptimizer::step: params updated in place (host array)."""
        g = np.ascontiguousarray(grad, np.float64)
        self.ctx.check(L.lib().ktune_adam_step(self.ctx.h, self.h, params.ctypes.data_as(C.c_void_p),
                                               g.ctypes.data_as(C.c_void_p), 0))

    def state(self):
        m, v, t = np.zeros(self.dim), np.zeros(self.dim), C.c_int64()
        self.ctx.check(L.lib().ktune_adam_state(self.ctx.h, self.h, m.ctypes.data_as(C.c_void_p),
                                                v.ctypes.data_as(C.c_void_p), C.byref(t)))
        return m, v, t.value

    def __del__(self):
        try:
            L.lib().ktune_adam_destroy(self.h)
        except Exception:
            pass


@dataclass
class PpoParams:  # SPEC.md PpoParams (:209-216)
    adam_step_size: float = 1e-3
    discount_gamma: float = 0.9
    gae_lambda: float = 0.99
    num_epochs: int = 3
    clip_epsilon: float = 0.3
    value_coef: float = 1.0
    entropy_coef: float = 0.1
    minibatch_size: int = 256


def compute_gae(rewards, values, terminal_values, gamma: float = 0.9, lam: float = 0.99,
                ctx: Optional[Context] = None):
    """compute_gae over E episodes x T steps on the GPU -> (advantages, returns)."""
    ctx = ctx or default_context()
    r = np.ascontiguousarray(rewards, np.float64)
    r2 = r.reshape(-1, r.shape[-1]) if r.ndim > 1 else r.reshape(1, -1)
    E, T = r2.shape
    v = np.ascontiguousarray(values, np.float64).reshape(E, T)
    if v.shape != r2.shape:
        raise ConfigError("compute_gae: length mismatch")
    tv = np.ascontiguousarray(terminal_values, np.float64).reshape(E)
    adv, ret = np.zeros((E, T)), np.zeros((E, T))
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    ctx.check(L.lib().ktune_compute_gae(ctx.h, E, T, p(r2), p(v), p(tv), gamma, lam, p(adv), p(ret), 0))
    return adv.reshape(r.shape), ret.reshape(r.shape)


def ppo_update(agent: ActorCritic, adam: Adam, states, actions, old_logp, advantages, returns,
               params: PpoParams = PpoParams(), seed: int = 0) -> dict:
    """ppo_update on the GPU; the agent's parameters are updated in place
    (device and host copies). Returns the training statistics."""
    n = agent.n
    S = np.ascontiguousarray(states, np.float64).reshape(-1, n)
    N = len(S)
    A = np.ascontiguousarray(actions, np.int8).reshape(N, n)
    arr = [np.ascontiguousarray(x, np.float64).reshape(N) for x in (old_logp, advantages, returns)]
    st = np.zeros(3)
    pc = L.PpoParamsC(params.clip_epsilon, params.value_coef, params.entropy_coef, params.num_epochs, 0,
                      params.minibatch_size)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    agent.ctx.check(L.lib().ktune_ppo_update(agent.ctx.h, agent.h_dev, adam.h, C.byref(pc), N, p(S), p(A),
                                             p(arr[0]), p(arr[1]), p(arr[2]), seed, p(st), 0))
    agent.sync_parameters()
    return dict(policy_loss=st[0], value_loss=st[1], entropy=st[2])


@dataclass
class RolloutTask:
    """One workload of a grouped rollout launch."""
    space: Space
    agent: ActorCritic
    cost_model: Optional[DeviceGbt]
    init_idx: object          # E x D (numpy int / CUDA uint16 tensor)
    episode_offset: int = 0   # global id of the first episode (RNG key; sharding)
    root_seed: int = 0        # explore seed = stream_seed(root_seed, "explore")
    want_trajectory: bool = True


def grouped_outputs(tasks: Sequence[RolloutTask], T: int, alloc, fields=None) -> list:
    """Per-task output dicts for the GROUPED step-major layout (KTUNE_F_STEP_MAJOR_GROUPED): one
    (rows, sum E_k[, D]) array per output, task k's entries are the column views [off_k, off_k + E_k).
    alloc(shape, name) -> array (numpy, pinned numpy or torch); fields: name -> (rows, last-dim or
    None), default the full-precision set."""
    D = tasks[0].space.D
    if any(t.space.D != D for t in tasks):
        raise ConfigError("rollout: grouped layout needs the same knob count in every task")
    Es = [len(t.init_idx) for t in tasks]
    Et = sum(Es)
    fields = fields or {"idx": (T + 1, D), "score": (T + 1, None), "actions": (T, D), "logp": (T, None),
                        "value": (T, None)}
    big = {name: alloc((rows,) + ((Et,) if last is None else (Et, last)), name) for name, (rows, last) in fields.items()}
    outs, off = [], 0
    for E in Es:
        outs.append({name: a[:, off:off + E] for name, a in big.items()})
        off += E
    return outs


def compact_grouped_outputs(tasks: Sequence[RolloutTask], T: int, alloc, score64: bool = False,
                            logp64: bool = False, ids: bool = False) -> list:
    """Grouped step-major outputs in the compact encoding (what crosses PCIe): visited
    configurations as uint8 for every run of consecutive tasks whose cardinalities fit (uint16
    for the others) - or, with ids=True, as one uint32 configuration id per visited
    configuration (`ids32`, id_of: design_space.cpp:158-167; `configs_from_ids` inverts it) -
    directions as 2-bit codes, scores fp32 (fp64 with score64) and log-probs / values fp32 (fp64
    with logp64; the tcgen05 path computes them in fp32). alloc(shape, dtype) -> array. Every
    output but idx spans all tasks; idx is one array per run."""
    D = tasks[0].space.D
    Es = [len(t.init_idx) for t in tasks]
    offs = np.cumsum([0] + Es)
    Et = int(offs[-1])
    big = {"actions2": alloc((T, Et, (D + 3) // 4), np.uint8),
           ("score" if score64 else "score32"): alloc((T + 1, Et), np.float64 if score64 else np.float32),
           ("logp" if logp64 else "logp32"): alloc((T, Et), np.float64 if logp64 else np.float32),
           ("value" if logp64 else "value32"): alloc((T, Et), np.float64 if logp64 else np.float32)}
    if ids:
        big["ids32"] = alloc((T + 1, Et), np.uint32)
    outs = [{k: a[:, offs[i]:offs[i + 1]] for k, a in big.items()} for i in range(len(tasks))]
    small = [max(t.space.card) <= 256 for t in tasks]
    i = 0
    while i < len(tasks) and not ids:  # runs of consecutive tasks with the same idx width
        j = i
        while j < len(tasks) and small[j] == small[i]:
            j += 1
        name, dt = ("idx8", np.uint8) if small[i] else ("idx", np.uint16)
        a = alloc((T + 1, int(offs[j] - offs[i]), D), dt)
        for q in range(i, j):
            outs[q][name] = a[:, offs[q] - offs[i]:offs[q + 1] - offs[i]]
        i = j
    for o in outs:
        for k in ("idx", "idx8", "ids32", "score", "score32", "actions", "logp", "value", "logp32", "value32"):
            o.setdefault(k, None)
    return outs


def configs_from_ids(ids, cards: Sequence[int]) -> np.ndarray:
    """config_at (design_space.cpp:141-156) of the `ids_u32` output: ... -> ... x D uint16 knob
    indices (mixed radix, last knob fastest)."""
    r = np.asarray(ids).astype(np.uint64)
    out = np.empty(r.shape + (len(cards),), np.uint16)
    for d in range(len(cards) - 1, -1, -1):
        out[..., d] = (r % np.uint64(cards[d])).astype(np.uint16)
        r = r // np.uint64(cards[d])
    return out


def run_episodes_batch(tasks: Sequence[RolloutTask], T: int, ctx: Optional[Context] = None,
                       device_out: bool = False, host_out: Optional[list] = None, exact: bool = False,
                       step_major: bool = False, grouped: bool = False):
    """Grouped run_episodes over several workloads in ONE persistent-kernel launch.

    Host arrays in/out by default; with CUDA-tensor init_idx and device_out=True
    everything stays on the device (torch tensors) and the call is stream-ordered.
    Returns per task dict(idx E x (T+1) x D uint16, score E x (T+1), actions
    E x T x D int8, logp E x T, value E x T).

    Default: the tcgen05 rollout with certified sampling (configurations,
    actions and scores bit-exact; logp/value fp32-accurate). exact=True runs
    the fp64 forward on every config-step (logp/value bit-exact as well).
    step_major=True (KTUNE_F_STEP_MAJOR) lays the trajectories out step-major:
    idx (T+1) x E x D, score (T+1) x E, actions T x E x D, logp/value T x E -
    the same values transposed; each step is one contiguous block on the device
    and each segment of a host-buffer call one contiguous PCIe copy. grouped=True
    (KTUNE_F_STEP_MAJOR_GROUPED) lays ALL tasks' episodes side by side in one
    step-major array per output (see grouped_outputs; host_out must come from it,
    or is allocated that way): one copy per output per segment for every task.
    """
    if grouped:
        step_major = True
        if host_out is None:
            dev0 = hasattr(tasks[0].init_idx, "is_cuda") and tasks[0].init_idx.is_cuda
            want = {"idx": (T + 1, tasks[0].space.D)}
            if tasks[0].cost_model is not None:
                want["score"] = (T + 1, None)
            if tasks[0].want_trajectory:
                want.update({"actions": (T, tasks[0].space.D), "logp": (T, None), "value": (T, None)})
            dt = {"idx": np.uint16, "score": np.float64, "actions": np.int8, "logp": np.float64, "value": np.float64}
            if dev0:
                import torch
                tdt = {np.uint16: torch.uint16, np.float64: torch.float64, np.int8: torch.int8}
                alloc = lambda shape, name: torch.empty(shape, dtype=tdt[dt[name]], device=tasks[0].init_idx.device)
            else:
                alloc = lambda shape, name: host_empty(shape, dt[name])
            host_out = grouped_outputs(tasks, T, alloc, want)
            for o in host_out:
                for k in ("idx", "score", "actions", "logp", "value"):
                    o.setdefault(k, None)
    ctx = ctx or tasks[0].space.ctx
    arr = (L.RolloutTaskC * len(tasks))()
    outs = []
    keep = []
    dev = False
    for i, t in enumerate(tasks):
        D = t.space.D
        if t.agent.n != D:
            raise ConfigError("rollout: agent/space knob count mismatch")
        dev = hasattr(t.init_idx, "is_cuda") and t.init_idx.is_cuda
        if dev:
            import torch
            init = t.init_idx.to(torch.uint16).contiguous() if t.init_idx.dtype != torch.uint16 else t.init_idx.contiguous()
            E = init.shape[0]
            if host_out is not None:  # caller-provided persistent device buffers
                o = host_out[i]
            else:
                mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=init.device)
                o = dict(idx=mk(_shape(E, T + 1, step_major, D), torch.uint16),
                         score=mk(_shape(E, T + 1, step_major), torch.float64) if t.cost_model is not None else None,
                         actions=mk(_shape(E, T, step_major, D), torch.int8) if t.want_trajectory else None,
                         logp=mk(_shape(E, T, step_major), torch.float64) if t.want_trajectory else None,
                         value=mk(_shape(E, T, step_major), torch.float64) if t.want_trajectory else None)
            pp = lambda a: None if a is None else C.c_void_p(a.data_ptr())
            init_p = C.c_void_p(init.data_ptr())
            keep.append(init)
        else:
            init = np.ascontiguousarray(t.init_idx, np.uint16).reshape(-1, D)
            E = len(init)
            if host_out is not None:  # caller-provided (e.g. pinned) host buffers
                o = host_out[i]
            else:
                o = dict(idx=host_empty(_shape(E, T + 1, step_major, D), np.uint16),
                         score=host_empty(_shape(E, T + 1, step_major), np.float64) if t.cost_model is not None else None,
                         actions=host_empty(_shape(E, T, step_major, D), np.int8) if t.want_trajectory else None,
                         logp=host_empty(_shape(E, T, step_major), np.float64) if t.want_trajectory else None,
                         value=host_empty(_shape(E, T, step_major), np.float64) if t.want_trajectory else None)
            pp = lambda a: None if a is None else a.__array_interface__["data"][0]  # int address: no ctypes objects
            init_p = init.ctypes.data_as(C.c_void_p)
            keep.append(init)
        a = arr[i]
        a.space = t.space.h
        a.ac = t.agent.h_dev
        a.gbt = t.cost_model.h if t.cost_model is not None else None
        a.num_episodes = E
        a.episode_offset = t.episode_offset
        a.explore_seed = stream_seed(t.root_seed, "explore")
        a.init_idx = init_p
        a.idx = pp(o["idx"])
        a.score = pp(o["score"])
        a.actions = pp(o["actions"])
        a.logp = pp(o["logp"])
        a.value = pp(o["value"])
        a.logp_f32 = pp(o.get("logp32"))
        a.value_f32 = pp(o.get("value32"))
        a.idx_u8 = pp(o.get("idx8"))
        a.actions_u2 = pp(o.get("actions2"))
        a.score_f32 = pp(o.get("score32"))
        a.ids_u32 = pp(o.get("ids32"))
        outs.append(o)
    ctx.check(L.lib().ktune_rollout(ctx.h, len(tasks), arr, T,
                                    (L.F_DEVICE if dev else 0) | (L.F_EXACT_ROLLOUT if exact else 0) |
                                    (L.F_STEP_MAJOR if step_major else 0) |
                                    (L.F_STEP_MAJOR_GROUPED if grouped else 0)))
    return outs


def _shape(E: int, rows: int, step_major: bool, D: Optional[int] = None) -> tuple:
    s = (rows, E) if step_major else (E, rows)
    return s + ((D,) if D is not None else ())


def unpack_actions(packed, D: int) -> np.ndarray:
    """Directions from the 2-bit `actions_u2` output: ... x ceil(D/4) bytes -> ... x D int8."""
    p = np.asarray(packed, np.uint8)
    codes = (p[..., :, None] >> (2 * np.arange(4, dtype=np.uint8))) & 3
    return (codes.reshape(*p.shape[:-1], -1)[..., :D].astype(np.int8) - 1)


def run_episodes(space: Space, cost_model: Optional[DeviceGbt], agent: ActorCritic, init_idx, T: int,
                 root_seed: int = 0, episode_offset: int = 0, exact: bool = False):
    """run_episodes(space, cost_model, net, params, initial_configs, rng).

    Returns (candidates, trajectory): candidates is a CandidateSet over every
    visited configuration Θ_0..Θ_T of every episode with its predicted
    fitness; trajectory holds actions, log-probabilities, values and the
    per-step rewards r_t = pred(Θ_{t+1}) - pred(Θ_t).
    """
    from .sampling import candidates_from_rows
    o = run_episodes_batch([RolloutTask(space, agent, cost_model, init_idx, episode_offset, root_seed)], T,
                           exact=exact)[0]
    flat = o["idx"].reshape(-1, space.D)
    score = o["score"].reshape(-1) if o["score"] is not None else np.zeros(len(flat))
    cands = candidates_from_rows(space, flat, score)  # make_candidate_set on the device
    traj = dict(o)
    if o["score"] is not None:
        traj["reward"] = o["score"][:, 1:] - o["score"][:, :-1]
    return cands, traj


@dataclass
class SaParams:  # SPEC.md SaParams (the temperature schedule is SPEC-invented)
    num_chains: int = 128
    max_steps: int = 500
    initial_temperature: float = 1.0
    cooling_rate: float = 0.99


@dataclass
class SaTask:
    """One workload of a grouped sa_search launch (chains = rows of init_idx)."""
    space: Space
    cost_model: DeviceGbt
    init_idx: object          # E x D knob indices (numpy / CUDA uint16 tensor); see sa_seeds
    chain_offset: int = 0     # global id of the first chain (RNG key; sharding)
    rng_seed: int = 0         # SA stream = stream_seed(rng_seed, "sa")


def sa_seeds(space: Space, seeds, num_chains: int, rng_seed: int = 0) -> np.ndarray:
    """The chains' start states: the given seeds, padded with uniformly random
    configurations from stream_seed(rng_seed, "sa-pad")."""
    D = space.D
    seeds = np.asarray(seeds, np.int64).reshape(-1, D) if len(seeds) else np.zeros((0, D), np.int64)
    if len(seeds) < num_chains:
        st = stream_seed(rng_seed, "sa-pad")
        pad = np.zeros((num_chains - len(seeds), D), np.int64)
        for i in range(len(pad)):
            for d, c in enumerate(space.card):
                pad[i, d] = mix64((st + i * D + d + 1) & 0xFFFFFFFFFFFFFFFF) % int(c)
        seeds = np.concatenate([seeds, pad])
    return np.ascontiguousarray(seeds[:num_chains], np.uint16)


def sa_search_batch(tasks: Sequence[SaTask], params: SaParams, ctx: Optional[Context] = None,
                    device_out: bool = False, host_out: Optional[list] = None, want_accepted: bool = True):
    """Grouped sa_search over several workloads in ONE kernel launch (K7).

    Host arrays by default (pass pinned `host_out` buffers for full PCIe speed);
    with CUDA-tensor init_idx and device_out=True the trajectory stays on the
    device and the call is stream-ordered. Returns per task dict(idx E x (T+1)
    x D uint16, score E x (T+1), accepted E x T uint8)."""
    ctx = ctx or tasks[0].space.ctx
    T = params.max_steps
    arr = (L.SaTaskC * len(tasks))()
    outs, keep = [], []
    dev = False
    for i, t in enumerate(tasks):
        D = t.space.D
        dev = hasattr(t.init_idx, "is_cuda") and t.init_idx.is_cuda
        if dev:
            import torch
            init = t.init_idx.to(torch.uint16).contiguous()
            E = init.shape[0]
            mk = lambda shape, dt: torch.empty(shape, dtype=dt, device=init.device)
            pp = lambda a: None if a is None else C.c_void_p(a.data_ptr())
            if not device_out:
                raise ConfigError("sa_search_batch: device inputs need device_out=True")
        else:
            init = np.ascontiguousarray(t.init_idx, np.uint16).reshape(-1, D)
            E = len(init)
            mk = lambda shape, dt: host_empty(shape, {"u16": np.uint16, "f64": np.float64, "u8": np.uint8}[dt])
            pp = lambda a: None if a is None else a.__array_interface__["data"][0]  # int address: no ctypes objects
        if host_out is not None:
            o = host_out[i]
        elif dev:
            import torch
            o = dict(idx=mk((E, T + 1, D), torch.uint16), score=mk((E, T + 1), torch.float64),
                     accepted=mk((E, T), torch.uint8) if want_accepted else None)
        else:
            o = dict(idx=mk((E, T + 1, D), "u16"), score=mk((E, T + 1), "f64"),
                     accepted=mk((E, T), "u8") if want_accepted else None)
        keep.append(init)
        a = arr[i]
        a.space = t.space.h
        a.gbt = t.cost_model.h
        a.num_chains = E
        a.chain_offset = t.chain_offset
        a.sa_seed = stream_seed(t.rng_seed, "sa")
        a.init_idx = pp(init)
        a.idx = pp(o["idx"])
        a.score = pp(o["score"])
        a.accepted = pp(o.get("accepted"))
        outs.append(o)
    p = L.SaParamsC(params.initial_temperature, params.cooling_rate)
    ctx.check(L.lib().ktune_sa_search(ctx.h, len(tasks), arr, T, C.byref(p), L.F_DEVICE if dev else 0))
    return outs


def sa_search(space: Space, cost_model: DeviceGbt, seeds, params: SaParams = SaParams(), rng_seed: int = 0,
              chain_offset: int = 0, ctx: Optional[Context] = None):
    """sa_search(space, cost_model, seeds, params, rng_seed) -> CandidateSet.

    The AutoTVM parallel simulated-annealing baseline on the GPU (K7, sa.cu):
    `num_chains` chains of `max_steps` Metropolis steps on the cost model,
    builder-pinned semantics. Seeds are padded with uniformly
    random configurations (stream_seed(rng_seed, "sa-pad")) when fewer than
    num_chains are given. Returns (CandidateSet over every chain state ranked by
    predicted fitness and deduplicated, trajectory dict(idx, score, accepted)).
    """
    from .sampling import candidates_from_rows
    init = sa_seeds(space, seeds, params.num_chains, rng_seed)
    o = sa_search_batch([SaTask(space, cost_model, init, chain_offset, rng_seed)], params, ctx)[0]
    cands = candidates_from_rows(space, o["idx"].reshape(-1, space.D), o["score"].reshape(-1))  # on the device
    return cands, o
