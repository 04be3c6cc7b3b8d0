"""Synthetic workloads for bench.py (builder-defined).

Each task = one design space + a GBT cost model fitted on 1000 configurations
measured by the seeded multi-peak landscape of SyntheticBackend
(measurement.cpp:88-151: 8 peaks, sharpness 8, noise 0.03; restated here as a
bench fixture — measurement is out of the hot path) + a seeded actor-critic +
E initial configurations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List

import numpy as np

from .spaces import MASK64, mix64, stream_seed


class Rng:
    """splitmix64 generator (rng.hpp:50-69)."""

    def __init__(self, seed: int):
        self.s = seed & MASK64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        return mix64(self.s)

    def below(self, n: int) -> int:
        """Unbiased integer in [0, n) by rejection (rng.hpp:63-69)."""
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= threshold:
                return r % n

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def hash01(seed: int, counter: int) -> float:
    u = mix64((seed ^ mix64((counter + 0x9E3779B97F4A7C15) & MASK64)) & MASK64)
    return (u >> 11) * 2.0 ** -53


def synthetic_fitness(space, idx: np.ndarray, seed: int, num_peaks: int = 8,
                      sharpness: float = 8.0, noise: float = 0.03) -> np.ndarray:
    """SyntheticBackend::evaluate (measurement.cpp:143-151), no invalid region."""
    D = space.num_knobs
    rng = Rng(stream_seed(seed, "landscape-peaks"))
    centers = np.zeros((num_peaks, D))
    amps = np.zeros(num_peaks)
    for p in range(num_peaks):
        for d in range(D):
            centers[p, d] = rng.uniform01()
        amps[p] = 0.5 + 0.5 * rng.uniform01()
    cards = space.cards
    out = np.zeros(len(idx))
    for r, row in enumerate(np.asarray(idx)):
        x = [row[d] / (cards[d] - 1) if cards[d] > 1 else 0.0 for d in range(D)]
        s = 0.0
        for p in range(num_peaks):
            d2 = (x[0] - centers[p, 0]) ** 2
            for d in range(1, D):
                d2 = d2 + (x[d] - centers[p, d]) ** 2
            s += amps[p] * math.exp(-sharpness * d2)
        cid = 0
        for d in range(D):
            cid = cid * cards[d] + int(row[d])
        out[r] = s + noise * hash01(seed, cid)
    return out


def encode(space, idx: np.ndarray) -> np.ndarray:
    c = np.array(space.cards, np.float64)
    den = np.where(c > 1, c - 1, 1.0)
    return np.where(c > 1, np.asarray(idx, np.float64) / den, 0.0)


def _rule_fn(space):
    """The space's validity rule (validity.hpp:10-19 grammar: + * ( ) integers, knob names,
    one <=/</== comparison) as a Python predicate on knob VALUES (exact integers)."""
    rule = getattr(space, "validity_rule", None)
    if not rule:
        return None
    import re
    names = [k.name for k in space.knobs]
    expr = re.sub(r"[A-Za-z_][A-Za-z0-9_]*", lambda m: f"v[{names.index(m.group(0))}]", rule)
    code = compile(expr, "<rule>", "eval")
    return lambda v: bool(eval(code, {}, {"v": v}))


def random_valid_configs(space, n: int, seed: int, max_attempts: int = 256) -> np.ndarray:
    """n draws of random_valid_configuration (design_space.cpp:211-228, default 256 attempts,
    design_space.hpp:95-96) from ONE Rng(stream_seed(seed, "init")): per
    knob Rng::below(card) (rejection sampling, rng.hpp:63-69), redrawn while invalid."""
    rng = Rng(stream_seed(seed, "init"))
    cards = space.cards
    vals = [k.values for k in space.knobs]
    ok = _rule_fn(space)
    out = np.zeros((n, len(cards)), np.int32)
    for r in range(n):
        cfg = [rng.below(c) for c in cards]
        a = 0
        while ok is not None and a < max_attempts and not ok([vals[d][i] for d, i in enumerate(cfg)]):
            cfg = [rng.below(c) for c in cards]
            a += 1
        out[r] = cfg
    return out


def random_configs(space, n: int, seed: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, c, n) for c in space.cards], 1).astype(np.int32)


@dataclass
class TaskSpec:
    space: object
    seed: int
    train_idx: np.ndarray
    train_y: np.ndarray
    init_idx: np.ndarray


def make_tasks(spaces: list, episodes: int, seed: int = 0, n_train: int = 1000) -> List[TaskSpec]:
    out = []
    for i, sp in enumerate(spaces):
        s = seed * 1000 + i
        tr = random_configs(sp, n_train, s)
        y = synthetic_fitness(sp, tr, s)
        init = random_valid_configs(sp, episodes, s)
        out.append(TaskSpec(sp, s, tr, y, init))
    return out
