"""Builder-defined design-space catalogue (the reference ships no examples/).

Pure Python, no dependency on the product package, so the bench's reference arm
can build the same workloads without importing paper_2001_08743_b200.

* `conv_space`: one conv2d task with the 8 Table-1 knobs.
  Split knobs use AutoTVM's ordered factorisations (4-way for f/y/x, 2-way for
  rc/ry/rx); a split knob's integer value is the lexicographic code of its
  factor tuple (strictly increasing in enumeration order). The validity rule
  "auto_unroll_max_step * unroll_explicit <= 512" marks explicit unrolling at
  step 1500 invalid (1/6 of every space).
* `resnet18_tasks` (12), `vgg16_tasks` (9), `alexnet_tasks` (5): PAPER.md:610-612.
* `synthetic_space`: D knobs of cardinality 2 + mix64(seed + d) % 31 (2..32),
  values 1..card, optional rule.

Every constructor takes `make(workload, knobs, rule)`; the default builds a
`SpaceSpec`, a plain value with the attributes of the reference's DesignSpace
(design_space.hpp:18-60) that the oracle wrappers and the product read.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from functools import lru_cache
from typing import List, Optional, Sequence

MASK64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 finalizer (rng.hpp:16-23)."""
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


def seed_combine(a: int, b: int) -> int:
    """rng.hpp:26-28."""
    return mix64((a + 0x9E3779B97F4A7C15 + mix64(b)) & MASK64)


def stream_seed(root: int, name: str) -> int:
    """FNV-1a named stream (rng.hpp:33-40)."""
    h = 0xCBF29CE484222325
    for c in name.encode():
        h ^= c
        h = (h * 0x100000001B3) & MASK64
    return seed_combine(root, h)


@dataclass
class KnobSpec:
    name: str
    values: List[int]

    @property
    def cardinality(self) -> int:
        return len(self.values)


@dataclass
class SpaceSpec:
    workload: str
    knobs: List[KnobSpec]
    validity_rule: Optional[str] = None
    size: int = field(init=False, default=0)

    def __post_init__(self) -> None:
        size = 1
        for k in self.knobs:
            size *= k.cardinality
        self.size = size

    @property
    def num_knobs(self) -> int:
        return len(self.knobs)

    @property
    def cards(self) -> List[int]:
        return [k.cardinality for k in self.knobs]

    @property
    def names(self) -> List[str]:
        return [k.name for k in self.knobs]

    @property
    def max_card(self) -> int:
        return max(self.cards)

    @property
    def index_bytes(self) -> int:
        return 1 if self.max_card <= 256 else 2

    def to_json(self) -> str:
        doc = {"workload": self.workload,
               "knobs": [{"name": k.name, "values": list(k.values)} for k in self.knobs]}
        if self.validity_rule:
            doc["validity_rule"] = self.validity_rule
        return json.dumps(doc)


def _spec(workload, knobs, rule):
    return SpaceSpec(workload, [KnobSpec(n, list(v)) for n, v in knobs], rule)


# ---------------------------------------------------------------------------
# AutoTVM-style conv2d spaces
# ---------------------------------------------------------------------------

@lru_cache(maxsize=None)
def ordered_factorizations(n: int, parts: int) -> tuple:
    """All ordered tuples of `parts` positive integers whose product is n, lexicographic."""
    if parts == 1:
        return ((n,),)
    out = []
    for f in range(1, n + 1):
        if n % f == 0:
            for rest in ordered_factorizations(n // f, parts - 1):
                out.append((f,) + rest)
    return tuple(out)


def _split_knob(name: str, n: int, parts: int) -> tuple:
    base = n + 1
    vals = []
    for tup in ordered_factorizations(n, parts):
        code = 0
        for f in tup:
            code = code * base + f
        vals.append(code)
    return (name, vals)


CONV_RULE = "auto_unroll_max_step * unroll_explicit <= 512"


def conv_space(workload: str, c_in: int, c_out: int, h_out: int, w_out: int, kh: int, kw: int,
               rule: Optional[str] = CONV_RULE, make=_spec):
    knobs = [
        _split_knob("tile_f", c_out, 4),
        _split_knob("tile_y", h_out, 4),
        _split_knob("tile_x", w_out, 4),
        _split_knob("tile_rc", c_in, 2),
        _split_knob("tile_ry", kh, 2),
        _split_knob("tile_rx", kw, 2),
        ("auto_unroll_max_step", [0, 512, 1500]),
        ("unroll_explicit", [0, 1]),
    ]
    return make(workload, knobs, rule)


def resnet18_tasks(make=_spec) -> list:
    """The 12 tuning tasks of ResNet-18: its 11 distinct conv2d
    workloads plus the final 512->1000 dense layer expressed as a 1x1 conv on a
    1x1 map (single-valued tile_y/tile_x knobs, tile_f cardinality 400)."""
    L = [("resnet18.c1", 3, 64, 112, 112, 7, 7), ("resnet18.c2", 64, 64, 56, 56, 3, 3),
         ("resnet18.c3", 64, 128, 28, 28, 3, 3), ("resnet18.c4", 64, 128, 28, 28, 1, 1),
         ("resnet18.c5", 128, 128, 28, 28, 3, 3), ("resnet18.c6", 128, 256, 14, 14, 3, 3),
         ("resnet18.c7", 128, 256, 14, 14, 1, 1), ("resnet18.c8", 256, 256, 14, 14, 3, 3),
         ("resnet18.c9", 256, 512, 7, 7, 3, 3), ("resnet18.c10", 256, 512, 7, 7, 1, 1),
         ("resnet18.c11", 512, 512, 7, 7, 3, 3), ("resnet18.dense", 512, 1000, 1, 1, 1, 1)]
    return [conv_space(*a, make=make) for a in L]


def vgg16_tasks(make=_spec) -> list:
    """The 9 distinct conv2d workloads of VGG-16."""
    L = [("vgg16.c1", 3, 64, 224, 224, 3, 3), ("vgg16.c2", 64, 64, 224, 224, 3, 3),
         ("vgg16.c3", 64, 128, 112, 112, 3, 3), ("vgg16.c4", 128, 128, 112, 112, 3, 3),
         ("vgg16.c5", 128, 256, 56, 56, 3, 3), ("vgg16.c6", 256, 256, 56, 56, 3, 3),
         ("vgg16.c7", 256, 512, 28, 28, 3, 3), ("vgg16.c8", 512, 512, 28, 28, 3, 3),
         ("vgg16.c9", 512, 512, 14, 14, 3, 3)]
    return [conv_space(*a, make=make) for a in L]


def alexnet_tasks(make=_spec) -> list:
    """The 5 conv2d workloads of AlexNet."""
    L = [("alexnet.c1", 3, 64, 55, 55, 11, 11), ("alexnet.c2", 64, 192, 27, 27, 5, 5),
         ("alexnet.c3", 192, 384, 13, 13, 3, 3), ("alexnet.c4", 384, 256, 13, 13, 3, 3),
         ("alexnet.c5", 256, 256, 13, 13, 3, 3)]
    return [conv_space(*a, make=make) for a in L]


def synthetic_space(seed: int = 0, num_knobs: int = 16, rule: Optional[str] = None,
                    workload: str = "synthetic", make=_spec):
    knobs = []
    for d in range(num_knobs):
        card = 2 + mix64((seed + d) & MASK64) % 31
        knobs.append((f"k{d}", list(range(1, card + 1))))
    return make(f"{workload}{num_knobs}", knobs, rule)


def small_space(cards: Sequence[int], rule: Optional[str] = None, workload: str = "small", make=_spec):
    return make(workload, [(f"k{i}", list(range(1, c + 1))) for i, c in enumerate(cards)], rule)
