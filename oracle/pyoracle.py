"""ctypes wrappers for the oracle libraries — TEST INFRASTRUCTURE ONLY.

  ref  : oracle/_ref/libktune_ref.so  — the reference's own sources (unmodified)
         built with the Eigen shim; the ground truth where reference code exists.
  port : oracle/libktune_oracle.so    — the plain-C restatement (incl. the
         rollout, which has no reference code).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libktune_ref.so")
PORT_SO = os.path.join(HERE, "libktune_oracle.so")

_port = None
_ref = None


def build() -> None:
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), "all"], check=True)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        _port = C.CDLL(PORT_SO)
        _setup_port(_port)
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        _ref = C.CDLL(REF_SO)
        _setup_ref(_ref)
    return _ref


P = C.c_void_p
i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
i8p = np.ctypeslib.ndpointer(np.int8, flags="C")


class KoRuleOp(C.Structure):
    _fields_ = [("code", C.c_int32), ("pad", C.c_int32), ("arg", C.c_int64)]


class KoSpace(C.Structure):
    _fields_ = [("D", C.c_int32), ("card", C.POINTER(C.c_int32)), ("values", C.POINTER(C.c_int64)),
                ("value_offsets", C.POINTER(C.c_int64)), ("ops", C.POINTER(KoRuleOp)),
                ("nops", C.c_int32)]


class KoGbt(C.Structure):
    _fields_ = [("num_trees", C.c_int32), ("num_features", C.c_int32), ("base", C.c_double),
                ("lr", C.c_double), ("offsets", C.POINTER(C.c_int32)),
                ("feature", C.POINTER(C.c_int32)), ("left", C.POINTER(C.c_int32)),
                ("right", C.POINTER(C.c_int32)), ("threshold", C.POINTER(C.c_double)),
                ("value", C.POINTER(C.c_double))]


def _setup_port(L):
    L.ko_mix64.restype = C.c_uint64
    L.ko_mix64.argtypes = [C.c_uint64]
    L.ko_seed_combine.restype = C.c_uint64
    L.ko_seed_combine.argtypes = [C.c_uint64, C.c_uint64]
    L.ko_stream_seed.restype = C.c_uint64
    L.ko_stream_seed.argtypes = [C.c_uint64, C.c_char_p]
    L.ko_hash01.restype = C.c_double
    L.ko_hash01.argtypes = [C.c_uint64, C.c_uint64]
    for f in ("ko_exp", "ko_log", "ko_tanh"):
        getattr(L, f).restype = C.c_double
        getattr(L, f).argtypes = [C.c_double]
    L.ko_validate_batch.argtypes = [C.POINTER(KoSpace), i32p, C.c_int64, u8p]
    L.ko_encode_batch.argtypes = [C.POINTER(KoSpace), i32p, C.c_int64, f64p]
    L.ko_id_of.restype = C.c_uint64
    L.ko_id_of.argtypes = [C.POINTER(KoSpace), i32p]
    L.ko_config_at.argtypes = [C.POINTER(KoSpace), C.c_uint64, i32p]
    L.ko_gbt_predict_features.argtypes = [C.POINTER(KoGbt), f64p, C.c_int64, f64p]
    L.ko_gbt_predict_idx.argtypes = [C.POINTER(KoGbt), C.POINTER(KoSpace), i32p, C.c_int64, f64p]
    L.ko_ac_num_params.restype = C.c_int64
    L.ko_ac_num_params.argtypes = [C.c_int, C.c_int, C.c_int]
    L.ko_ac_init.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, f64p]
    L.ko_ac_forward.argtypes = [C.c_int, C.c_int, C.c_int, f64p, f64p, C.c_int64] + [P] * 7
    L.ko_run_episodes.argtypes = [C.POINTER(KoSpace), C.POINTER(KoGbt), C.c_int, C.c_int, f64p,
                                  C.c_int64, C.c_int32, C.c_int64, C.c_uint64, i32p, i32p, P, P,
                                  P, P, C.c_int]
    L.ko_sa_search.argtypes = [C.POINTER(KoSpace), C.POINTER(KoGbt), C.c_int64, C.c_int32, C.c_int64,
                               C.c_uint64, C.c_double, C.c_double, i32p, i32p, f64p, P, C.c_int]
    L.ko_make_candidate_set.restype = C.c_int64
    L.ko_make_candidate_set.argtypes = [C.c_int, i32p, u64p, f64p, C.c_int64, i64p]
    L.ko_kmeans_run.argtypes = [f64p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                f64p, i32p, P, f64p, P]
    L.ko_adaptive_sweep.argtypes = [f64p, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_uint64, P, f64p, i32p, P, f64p, P]
    L.ko_snap_centroid.argtypes = [C.POINTER(KoSpace), f64p, i32p, u64p, C.c_int64, i32p]


def _setup_ref(L):
    L.ref_last_error.restype = C.c_char_p
    L.ref_mix64.restype = C.c_uint64
    L.ref_mix64.argtypes = [C.c_uint64]
    L.ref_seed_combine.restype = C.c_uint64
    L.ref_seed_combine.argtypes = [C.c_uint64, C.c_uint64]
    L.ref_stream_seed.restype = C.c_uint64
    L.ref_stream_seed.argtypes = [C.c_uint64, C.c_char_p]
    L.ref_hash01.restype = C.c_double
    L.ref_hash01.argtypes = [C.c_uint64, C.c_uint64]
    L.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int64, u64p]
    L.ref_space_new.restype = P
    L.ref_space_new.argtypes = [C.c_char_p]
    L.ref_space_free.argtypes = [P]
    L.ref_config_at.argtypes = [P, C.c_uint64, i32p]
    L.ref_id_of.argtypes = [P, i32p, C.POINTER(C.c_uint64)]
    L.ref_validate.argtypes = [P, i32p, C.c_int64, u8p]
    L.ref_neighbor.argtypes = [P, i32p, C.c_int, C.c_int, i32p]
    L.ref_encode_batch.argtypes = [P, i32p, C.c_int64, f64p]
    L.ref_random_valid_configs.argtypes = [P, C.c_uint64, C.c_int64, i32p]
    L.ref_synthetic_fitness.argtypes = [P, C.c_char_p, C.c_uint64, C.c_int, C.c_double,
                                        C.c_double, i32p, C.c_int64, f64p]
    L.ref_gbt_fit.restype = P
    L.ref_gbt_fit.argtypes = [f64p, f64p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                              C.c_int, C.c_uint64]
    L.ref_gbt_free.argtypes = [P]
    L.ref_gbt_shape.restype = C.c_int64
    L.ref_gbt_shape.argtypes = [P, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.ref_gbt_export.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_double), i32p, i32p,
                                 i32p, i32p, f64p, f64p, f64p]
    L.ref_gbt_predict.argtypes = [P, f64p, C.c_int64, C.c_int, f64p]
    L.ref_make_candidate_set.restype = C.c_int64
    L.ref_make_candidate_set.argtypes = [C.c_int, i32p, u64p, f64p, C.c_int64, i64p]
    L.ref_kmeans_run.argtypes = [f64p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int,
                                 f64p, i32p, P, f64p, P]
    L.ref_snap_centroid.argtypes = [P, f64p, i32p, u64p, f64p, C.c_int64, i32p]
    L.ref_adaptive_sample.argtypes = [P, i32p, u64p, f64p, C.c_int64, u64p, C.c_int64, C.c_double,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, i32p, P, P, P]
    L.ref_synthesize_sample.argtypes = [P, i32p, u64p, f64p, C.c_int64, u64p, C.c_int64,
                                        C.c_uint64, i32p]
    L.ref_greedy_select.argtypes = [P, i32p, u64p, f64p, C.c_int64, C.c_int, i32p]


def ref_error() -> str:
    return ref().ref_last_error().decode()


# ---------------------------------------------------------------------------
# validity rule: restatement of validity.cpp:19-212 (tokenizer + parser)
# ---------------------------------------------------------------------------
PUSH_CONST, PUSH_KNOB, ADD, MUL, LE, LT, EQ = range(7)


def compile_rule(source: Optional[str], names: List[str]) -> List[tuple]:
    if not source:
        return []
    toks = []
    i = 0
    while i < len(source):
        c = source[i]
        if c.isspace():
            i += 1
        elif c.isdigit():
            j = i
            while j < len(source) and source[j].isdigit():
                j += 1
            toks.append(("num", int(source[i:j])))
            i = j
        elif c.isalpha() or c == "_":
            m = re.match(r"[A-Za-z_][A-Za-z0-9_]*", source[i:])
            toks.append(("name", m.group(0)))
            i += len(m.group(0))
        elif c in "+*()":
            toks.append((c, None))
            i += 1
        elif c == "<":
            if source[i + 1:i + 2] == "=":
                toks.append(("<=", None))
                i += 2
            else:
                toks.append(("<", None))
                i += 1
        elif c == "=" and source[i + 1:i + 2] == "=":
            toks.append(("==", None))
            i += 2
        else:
            raise ValueError(f"unexpected character {c!r}")
    toks.append(("end", None))
    ops: List[tuple] = []
    pos = [0]

    def adv():
        t = toks[pos[0]]
        pos[0] += 1
        return t

    def atom():
        t = adv()
        if t[0] == "num":
            ops.append((PUSH_CONST, t[1]))
        elif t[0] == "name":
            if t[1] not in names:
                raise ValueError(f"unknown knob {t[1]}")
            ops.append((PUSH_KNOB, names.index(t[1])))
        elif t[0] == "(":
            sum_()
            if adv()[0] != ")":
                raise ValueError("missing )")
        else:
            raise ValueError("expected value")

    def prod():
        atom()
        while toks[pos[0]][0] == "*":
            adv()
            atom()
            ops.append((MUL, 0))

    def sum_():
        prod()
        while toks[pos[0]][0] == "+":
            adv()
            prod()
            ops.append((ADD, 0))

    sum_()
    cmp = adv()[0]
    code = {"<=": LE, "<": LT, "==": EQ}.get(cmp)
    if code is None:
        raise ValueError("expected comparison")
    sum_()
    ops.append((code, 0))
    if toks[pos[0]][0] != "end":
        raise ValueError("trailing input")
    return ops


# ---------------------------------------------------------------------------
# Wrappers
# ---------------------------------------------------------------------------
class OSpace:
    """A design space seen by both oracles (keeps ctypes buffers alive)."""

    def __init__(self, space):
        self.space = space
        self.D = space.num_knobs
        self.card = np.array(space.cards, np.int32)
        vals = []
        offs = [0]
        for k in space.knobs:
            vals.extend(k.values)
            offs.append(len(vals))
        self.values = np.array(vals, np.int64)
        self.offsets = np.array(offs, np.int64)
        ops = compile_rule(space.validity_rule, space.names)
        self.ops = (KoRuleOp * max(1, len(ops)))()
        for i, (c, a) in enumerate(ops):
            self.ops[i].code = c
            self.ops[i].arg = a
        self.nops = len(ops)
        self.ko = KoSpace(self.D, self.card.ctypes.data_as(C.POINTER(C.c_int32)),
                          self.values.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.offsets.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.ops if self.nops else None, self.nops)
        self._ref = None

    @property
    def ref(self):
        if self._ref is None:
            h = ref().ref_space_new(self.space.to_json().encode())
            if not h:
                raise ValueError(ref_error())
            self._ref = h
        return self._ref

    def __del__(self):
        if self._ref is not None and _ref is not None:
            _ref.ref_space_free(self._ref)

    # -- port (C restatement)
    def validate(self, idx):
        idx = np.ascontiguousarray(idx, np.int32).reshape(-1, self.D)
        out = np.zeros(len(idx), np.uint8)
        port().ko_validate_batch(C.byref(self.ko), idx, len(idx), out)
        return out

    def encode(self, idx):
        idx = np.ascontiguousarray(idx, np.int32).reshape(-1, self.D)
        out = np.zeros((len(idx), self.D), np.float64)
        port().ko_encode_batch(C.byref(self.ko), idx, len(idx), out)
        return out

    def ids(self, idx):
        idx = np.asarray(idx, np.int64).reshape(-1, self.D)
        ids = np.zeros(len(idx), np.uint64)
        acc = np.zeros(len(idx), np.uint64)
        for d in range(self.D):
            acc = acc * np.uint64(self.card[d]) + idx[:, d].astype(np.uint64)
        ids[:] = acc
        return ids

    def random_valid(self, seed, n):
        out = np.zeros((n, self.D), np.int32)
        rc = ref().ref_random_valid_configs(self.ref, seed, n, out)
        assert rc == 0, ref_error()
        return out


@dataclass
class Gbt:
    base: float
    lr: float
    num_features: int
    offsets: np.ndarray
    feature: np.ndarray
    left: np.ndarray
    right: np.ndarray
    threshold: np.ndarray
    value: np.ndarray
    training_sse: np.ndarray

    @property
    def num_trees(self):
        return len(self.offsets) - 1

    def ko(self):
        I = C.POINTER(C.c_int32)
        D_ = C.POINTER(C.c_double)
        self._keep = KoGbt(self.num_trees, self.num_features, self.base, self.lr,
                           self.offsets.ctypes.data_as(I), self.feature.ctypes.data_as(I),
                           self.left.ctypes.data_as(I), self.right.ctypes.data_as(I),
                           self.threshold.ctypes.data_as(D_), self.value.ctypes.data_as(D_))
        return self._keep


def ref_fit_gbt(X, y, num_trees=50, max_depth=4, lr=0.3, min_leaf=2, seed=0) -> Gbt:
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    L = ref()
    h = L.ref_gbt_fit(X, y, X.shape[0], X.shape[1], num_trees, max_depth, lr, min_leaf, seed)
    if not h:
        raise ValueError(ref_error())
    nt, nf = C.c_int(), C.c_int()
    total = L.ref_gbt_shape(h, C.byref(nt), C.byref(nf))
    base, lrv = C.c_double(), C.c_double()
    offs = np.zeros(nt.value + 1, np.int32)
    feat = np.zeros(total, np.int32)
    left = np.zeros(total, np.int32)
    right = np.zeros(total, np.int32)
    thr = np.zeros(total, np.float64)
    val = np.zeros(total, np.float64)
    sse = np.zeros(nt.value, np.float64)
    L.ref_gbt_export(h, C.byref(base), C.byref(lrv), offs, feat, left, right, thr, val, sse)
    L.ref_gbt_free(h)
    return Gbt(base.value, lrv.value, nf.value, offs, feat, left, right, thr, val, sse)


def ref_gbt_predict(g: Gbt, X) -> np.ndarray:
    """Reference predict_batch on a model re-fitted? No: rebuild via the port layout.
    (The reference GbtModel is opaque after export; the port's predict is checked
    against ref_fit_predict in tests instead.)"""
    raise NotImplementedError


def ref_fit_predict(X, y, Xq, **kw) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    Xq = np.ascontiguousarray(Xq, np.float64)
    L = ref()
    h = L.ref_gbt_fit(X, y, X.shape[0], X.shape[1], kw.get("num_trees", 50), kw.get("max_depth", 4),
                      kw.get("lr", 0.3), kw.get("min_leaf", 2), kw.get("seed", 0))
    if not h:
        raise ValueError(ref_error())
    out = np.zeros(len(Xq), np.float64)
    rc = L.ref_gbt_predict(h, Xq, len(Xq), Xq.shape[1], out)
    L.ref_gbt_free(h)
    assert rc == 0, ref_error()
    return out


def port_predict_features(g: Gbt, X) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    out = np.zeros(len(X), np.float64)
    port().ko_gbt_predict_features(C.byref(g.ko()), X, len(X), out)
    return out


def port_predict_idx(g: Gbt, sp: OSpace, idx) -> np.ndarray:
    idx = np.ascontiguousarray(idx, np.int32).reshape(-1, sp.D)
    out = np.zeros(len(idx), np.float64)
    port().ko_gbt_predict_idx(C.byref(g.ko()), C.byref(sp.ko), idx, len(idx), out)
    return out


def synthetic_fitness(sp: OSpace, idx, seed=0, num_peaks=8, sharpness=8.0, noise=0.03,
                      invalid_rule="") -> np.ndarray:
    idx = np.ascontiguousarray(idx, np.int32).reshape(-1, sp.D)
    out = np.zeros(len(idx), np.float64)
    rc = ref().ref_synthetic_fitness(sp.ref, invalid_rule.encode(), seed, num_peaks, sharpness,
                                     noise, idx, len(idx), out)
    assert rc == 0, ref_error()
    return out


def fitted_model(sp: OSpace, seed=0, n_train=1000, **kw) -> Gbt:
    """GBT fitted on n_train uniform configs measured by the reference SyntheticBackend."""
    idx = sp.random_valid(seed, n_train)
    y = synthetic_fitness(sp, idx, seed=seed)
    y = np.where(np.isnan(y), 0.0, y)
    return ref_fit_gbt(sp.encode(idx), y, seed=seed, **kw)


def ac_init(n, h, g, seed) -> np.ndarray:
    p = np.zeros(port().ko_ac_num_params(n, h, g), np.float64)
    port().ko_ac_init(n, h, g, seed, p)
    return p


def ac_forward(n, h, g, params, states):
    states = np.ascontiguousarray(states, np.float64).reshape(-1, n)
    B = len(states)
    outs = dict(h0=np.zeros((B, h)), hp=np.zeros((B, g)), hv=np.zeros((B, g)),
                logits=np.zeros((B, 3 * n)), log_probs=np.zeros((B, 3 * n)),
                probs=np.zeros((B, 3 * n)), values=np.zeros(B))
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    port().ko_ac_forward(n, h, g, np.ascontiguousarray(params, np.float64), states, B,
                         ptr(outs["h0"]), ptr(outs["hp"]), ptr(outs["hv"]), ptr(outs["logits"]),
                         ptr(outs["log_probs"]), ptr(outs["probs"]), ptr(outs["values"]))
    return outs


def run_episodes(sp: OSpace, g: Optional[Gbt], h, gh, params, init_idx, T, episode_offset,
                 explore_seed, threads=1, want_traj=True):
    init_idx = np.ascontiguousarray(init_idx, np.int32).reshape(-1, sp.D)
    E = len(init_idx)
    idx = np.zeros((E, T + 1, sp.D), np.int32)
    score = np.zeros((E, T + 1), np.float64)
    acts = np.zeros((E, T, sp.D), np.int8) if want_traj else None
    logp = np.zeros((E, T), np.float64) if want_traj else None
    val = np.zeros((E, T), np.float64) if want_traj else None
    ptr = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)
    gk = C.byref(g.ko()) if g is not None else None
    port().ko_run_episodes(C.byref(sp.ko), gk, h, gh, np.ascontiguousarray(params, np.float64),
                           E, T, episode_offset, explore_seed, init_idx, idx, ptr(score),
                           ptr(acts), ptr(logp), ptr(val), threads)
    return dict(idx=idx, score=score, actions=acts, logp=logp, value=val)


def sa_search(sp: OSpace, g: Gbt, init_idx, T, chain_offset, sa_seed, t0=1.0, rate=0.99, threads=1):
    """sa_search, builder-pinned: chain states, their
    predicted fitness and the acceptance flags."""
    init_idx = np.ascontiguousarray(init_idx, np.int32).reshape(-1, sp.D)
    E = len(init_idx)
    idx = np.zeros((E, T + 1, sp.D), np.int32)
    score = np.zeros((E, T + 1), np.float64)
    acc = np.zeros((E, T), np.uint8)
    port().ko_sa_search(C.byref(sp.ko), C.byref(g.ko()), E, T, chain_offset, sa_seed, t0, rate, init_idx, idx,
                        score, acc.ctypes.data_as(C.c_void_p), threads)
    return dict(idx=idx, score=score, accepted=acc)


def make_candidate_set(D, idx, ids, pred, impl="port"):
    idx = np.ascontiguousarray(idx, np.int32).reshape(-1, D)
    ids = np.ascontiguousarray(ids, np.uint64)
    pred = np.ascontiguousarray(pred, np.float64)
    rows = np.zeros(len(ids), np.int64)
    fn = port().ko_make_candidate_set if impl == "port" else ref().ref_make_candidate_set
    m = fn(D, idx, ids, pred, len(ids), rows)
    return rows[:m]


def kmeans_run(points, k, seed, max_iters=100, restarts=3, impl="port"):
    points = np.ascontiguousarray(points, np.float64)
    N, D = points.shape
    cen = np.zeros((k, D), np.float64)
    asg = np.zeros(N, np.int32)
    loss = C.c_double()
    il = np.zeros(max_iters + 1, np.float64)
    nl = C.c_int32()
    fn = port().ko_kmeans_run if impl == "port" else ref().ref_kmeans_run
    rc = fn(points, N, D, k, seed, max_iters, restarts, cen, asg, C.cast(C.pointer(loss), C.c_void_p),
            il, C.cast(C.pointer(nl), C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"kmeans rc={rc}" + (": " + ref_error() if impl == "ref" else ""))
    return dict(centroids=cen, assignments=asg, loss=loss.value, iteration_losses=il[:nl.value])


def adaptive_sweep(points, threshold=2.5, k_min=8, k_max_exclusive=64, max_iters=100, restarts=3,
                   rng_seed=0):
    points = np.ascontiguousarray(points, np.float64)
    N, D = points.shape
    kc = C.c_int32()
    cen = np.zeros((64, D), np.float64)
    asg = np.zeros(N, np.int32)
    loss = C.c_double()
    kl = np.zeros(64, np.float64)
    nk = C.c_int32()
    rc = port().ko_adaptive_sweep(points, N, D, threshold, k_min, k_max_exclusive, max_iters,
                                  restarts, rng_seed, C.cast(C.pointer(kc), C.c_void_p), cen, asg,
                                  C.cast(C.pointer(loss), C.c_void_p), kl,
                                  C.cast(C.pointer(nk), C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"sweep rc={rc}")
    return dict(k=kc.value, centroids=cen[:kc.value], assignments=asg, loss=loss.value,
                k_losses=kl[:nk.value])


def snap_centroid(sp: OSpace, centroid, cand_idx, cand_ids, cand_pred=None, impl="port"):
    cand_idx = np.ascontiguousarray(cand_idx, np.int32).reshape(-1, sp.D)
    cand_ids = np.ascontiguousarray(cand_ids, np.uint64)
    centroid = np.ascontiguousarray(centroid, np.float64)
    out = np.zeros(sp.D, np.int32)
    if impl == "port":
        port().ko_snap_centroid(C.byref(sp.ko), centroid, cand_idx, cand_ids, len(cand_ids), out)
    else:
        pred = np.zeros(len(cand_ids)) if cand_pred is None else np.ascontiguousarray(cand_pred, np.float64)
        rc = ref().ref_snap_centroid(sp.ref, centroid, cand_idx, cand_ids, pred, len(cand_ids), out)
        assert rc == 0, ref_error()
    return out


def ref_adaptive_sample(sp: OSpace, cand_idx, cand_ids, cand_pred, visited, threshold=2.5,
                        k_min=8, k_max_exclusive=64, max_iters=100, restarts=3, rng_seed=0):
    cand_idx = np.ascontiguousarray(cand_idx, np.int32).reshape(-1, sp.D)
    out = np.zeros((64, sp.D), np.int32)
    cnt = C.c_int32()
    kl = np.zeros(64, np.float64)
    kc = C.c_int32()
    visited = np.ascontiguousarray(visited, np.uint64)
    rc = ref().ref_adaptive_sample(sp.ref, cand_idx, np.ascontiguousarray(cand_ids, np.uint64),
                                   np.ascontiguousarray(cand_pred, np.float64), len(cand_ids),
                                   visited, len(visited), threshold, k_min, k_max_exclusive,
                                   max_iters, restarts, rng_seed, out,
                                   C.cast(C.pointer(cnt), C.c_void_p), kl.ctypes.data_as(C.c_void_p),
                                   C.cast(C.pointer(kc), C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"adaptive_sample rc={rc}: {ref_error()}")
    return dict(configs=out[:cnt.value], k_losses=kl[:kc.value])


# ---------------------------------------------------------------- PPO
def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def ac_backward(n, h, g, params, cache, d_logits, d_values):
    P = port()
    B = len(cache["states"])
    grad = np.zeros(P.ko_ac_num_params(n, h, g))
    c = {k: np.ascontiguousarray(cache[k], np.float64) for k in ("states", "h0", "hp", "hv")}
    dl = np.ascontiguousarray(d_logits, np.float64)
    dv = np.ascontiguousarray(d_values, np.float64)
    P.ko_ac_backward(n, h, g, _p(np.ascontiguousarray(params, np.float64)), _p(c["states"]), _p(c["h0"]),
                     _p(c["hp"]), _p(c["hv"]), C.c_int64(B), _p(dl), _p(dv), _p(grad))
    return grad


def adam_step(params, grad, m, v, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """One AdamOptimizer::step at step number t (1-based); arrays updated in place."""
    P = port()
    bc1, bc2 = C.c_double(), C.c_double()
    P.ko_adam_bias(C.c_double(b1), C.c_double(b2), C.c_int64(t), C.byref(bc1), C.byref(bc2))
    P.ko_adam_step(C.c_int64(len(params)), _p(params), _p(np.ascontiguousarray(grad, np.float64)), _p(m), _p(v),
                   C.c_double(lr), C.c_double(b1), C.c_double(b2), C.c_double(eps), bc1, bc2)


def compute_gae(rewards, values, terminal_values, gamma=0.9, lam=0.99):
    r = np.ascontiguousarray(rewards, np.float64)
    r2 = r.reshape(-1, r.shape[-1]) if r.ndim > 1 else r.reshape(1, -1)
    E, T = r2.shape
    v = np.ascontiguousarray(values, np.float64).reshape(E, T)
    tv = np.ascontiguousarray(terminal_values, np.float64).reshape(E)
    adv, ret = np.zeros((E, T)), np.zeros((E, T))
    port().ko_compute_gae(C.c_int64(E), C.c_int32(T), _p(r2), _p(v), _p(tv), C.c_double(gamma), C.c_double(lam),
                          _p(adv), _p(ret))
    return adv.reshape(r.shape), ret.reshape(r.shape)


def ppo_loss_grad(n, fwd, actions, old_logp, adv, ret, clip_eps=0.3, c_v=1.0, c_e=0.1):
    B = len(fwd["values"])
    dl, dv, sums = np.zeros((B, 3 * n)), np.zeros(B), np.zeros(3)
    a = np.ascontiguousarray(actions, np.int8)
    f = {k: np.ascontiguousarray(fwd[k], np.float64) for k in ("log_probs", "probs", "values")}
    port().ko_ppo_loss_grad(n, C.c_int64(B), _p(f["log_probs"]), _p(f["probs"]), _p(f["values"]), _p(a),
                            _p(np.ascontiguousarray(old_logp, np.float64)), _p(np.ascontiguousarray(adv, np.float64)),
                            _p(np.ascontiguousarray(ret, np.float64)), C.c_double(clip_eps), C.c_double(c_v),
                            C.c_double(c_e), _p(dl), _p(dv), _p(sums))
    return dl, dv, sums


def ppo_update(n, h, g, params, adam_m, adam_v, adam_t, states, actions, old_logp, adv, ret, num_epochs=3, mb=256,
               lr=1e-3, clip_eps=0.3, c_v=1.0, c_e=0.1, seed=0):
    """ko_ppo_update: params / adam_m / adam_v updated in place; returns (adam_t, stats)."""
    t = C.c_int64(adam_t)
    st = np.zeros(3)
    S = np.ascontiguousarray(states, np.float64)
    N = len(S)
    rc = port().ko_ppo_update(n, h, g, _p(params), _p(adam_m), _p(adam_v), C.byref(t), C.c_int64(N), _p(S),
                              _p(np.ascontiguousarray(actions, np.int8)), _p(np.ascontiguousarray(old_logp, np.float64)),
                              _p(np.ascontiguousarray(adv, np.float64)), _p(np.ascontiguousarray(ret, np.float64)),
                              num_epochs, C.c_int64(mb), C.c_double(lr), C.c_double(clip_eps), C.c_double(c_v),
                              C.c_double(c_e), C.c_uint64(seed), _p(st))
    assert rc == 0
    return t.value, st
