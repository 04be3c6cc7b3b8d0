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

from .spaces import DesignSpace, MASK64, mix64, stream_seed


class Rng:
    """splitmix64 generator (rng.hpp:50-69)."""

    def __init__(self, seed: int):
        self.s = seed & MASK64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK64
        return mix64(self.s)

    def uniform01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53


def hash01(seed: int, counter: int) -> float:
    u = mix64((seed ^ mix64((counter + 0x9E3779B97F4A7C15) & MASK64)) & MASK64)
    return (u >> 11) * 2.0 ** -53


def synthetic_fitness(space: DesignSpace, idx: np.ndarray, seed: int, num_peaks: int = 8,
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


def encode(space: DesignSpace, idx: np.ndarray) -> np.ndarray:
    c = np.array(space.cards, np.float64)
    den = np.where(c > 1, c - 1, 1.0)
    return np.where(c > 1, np.asarray(idx, np.float64) / den, 0.0)


def random_configs(space: DesignSpace, n: int, seed: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, c, n) for c in space.cards], 1).astype(np.int32)


@dataclass
class TaskSpec:
    space: DesignSpace
    seed: int
    train_idx: np.ndarray
    train_y: np.ndarray
    init_idx: np.ndarray


def make_tasks(spaces: List[DesignSpace], episodes: int, seed: int = 0, n_train: int = 1000) -> List[TaskSpec]:
    out = []
    for i, sp in enumerate(spaces):
        s = seed * 1000 + i
        tr = random_configs(sp, n_train, s)
        y = synthetic_fitness(sp, tr, s)
        init = random_configs(sp, episodes, s + 500)
        out.append(TaskSpec(sp, s, tr, y, init))
    return out
