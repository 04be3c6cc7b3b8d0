"""Design spaces (design_space.hpp:18-60).

`DesignSpace` mirrors the reference's value type: ordered knobs with strictly
increasing integer values, an optional validity rule in the validity.hpp:10-19
grammar, mixed-radix size (design_space.cpp:13-58). It validates exactly the
way the reference constructor does and raises `ConfigError` on the same
conditions.

The synthetic workload catalogue (AutoTVM-style conv spaces, the synthetic
16-knob space) lives in the top-level `workloads` package (bench/test
fixtures); the wrappers below build product `DesignSpace`s from it.
"""
from __future__ import annotations

import functools
import json
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from .errors import ConfigError

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


@functools.lru_cache(maxsize=4096)
def stream_seed(root: int, name: str) -> int:
    """FNV-1a named stream (rng.hpp:33-40)."""
    h = 0xCBF29CE484222325
    for c in name.encode():
        h ^= c
        h = (h * 0x100000001B3) & MASK64
    return seed_combine(root, h)


@dataclass
class Knob:
    name: str
    values: List[int]

    @property
    def cardinality(self) -> int:
        return len(self.values)


@dataclass
class DesignSpace:
    workload: str
    knobs: List[Knob]
    validity_rule: Optional[str] = None
    size: int = field(init=False, default=0)

    def __post_init__(self) -> None:  # design_space.cpp:13-58
        if not self.knobs:
            raise ConfigError(f"design space '{self.workload}': needs at least one knob")
        seen = set()
        for k in self.knobs:
            if not k.name:
                raise ConfigError(f"design space '{self.workload}': knob with empty name")
            if k.name in seen:
                raise ConfigError(f"design space '{self.workload}': duplicate knob name '{k.name}'")
            seen.add(k.name)
            if not k.values:
                raise ConfigError(f"knob '{k.name}': values must be non-empty")
            for i in range(1, len(k.values)):
                if k.values[i] == k.values[i - 1]:
                    raise ConfigError(f"knob '{k.name}': duplicate value {k.values[i]}")
                if k.values[i] < k.values[i - 1]:
                    raise ConfigError(
                        f"knob '{k.name}': values not strictly increasing at position {i}")
        size = 1
        for k in self.knobs:
            size *= k.cardinality
            if size > MASK64:
                raise ConfigError(
                    f"design space '{self.workload}': size overflows 64 bits at knob '{k.name}'")
        self.size = size
        if self.validity_rule == "":
            self.validity_rule = None

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
        """Device index width: uint8 when every cardinality <= 256, else uint16."""
        return 1 if self.max_card <= 256 else 2

    def to_json(self) -> str:
        doc = {"workload": self.workload,
               "knobs": [{"name": k.name, "values": list(k.values)} for k in self.knobs]}
        if self.validity_rule:
            doc["validity_rule"] = self.validity_rule
        return json.dumps(doc)

    @staticmethod
    def from_json_text(text: str) -> "DesignSpace":  # design_space.cpp:60-107
        try:
            doc = json.loads(text)
        except json.JSONDecodeError as e:
            raise ConfigError(f"design space: JSON parse error: {e}") from e
        if not isinstance(doc, dict) or "workload" not in doc or "knobs" not in doc:
            raise ConfigError("design space: document must be an object with 'workload' and 'knobs'")
        if not isinstance(doc["workload"], str):
            raise ConfigError("design space: 'workload' must be a string")
        if not isinstance(doc["knobs"], list):
            raise ConfigError("design space: 'knobs' must be an array")
        knobs = []
        for pos, item in enumerate(doc["knobs"]):
            if (not isinstance(item, dict) or not isinstance(item.get("name"), str)
                    or not isinstance(item.get("values"), list)):
                raise ConfigError(f"design space: knob #{pos} must be an object with 'name' and integer 'values'")
            vals = []
            for v in item["values"]:
                if isinstance(v, bool) or not isinstance(v, int):
                    raise ConfigError(f"knob '{item['name']}': non-integer value")
                vals.append(v)
            knobs.append(Knob(item["name"], vals))
        rule = doc.get("validity_rule")
        if rule is not None and not isinstance(rule, str):
            raise ConfigError("design space: 'validity_rule' must be a string")
        return DesignSpace(doc["workload"], knobs, rule)


# ---------------------------------------------------------------------------
# The builder-defined catalogue (workloads/spaces.py) as product DesignSpaces
# ---------------------------------------------------------------------------

def _make(workload, knobs, rule):
    return DesignSpace(workload, [Knob(n, list(v)) for n, v in knobs], rule)


def conv_space(*a, **k) -> DesignSpace:
    from workloads import spaces as W
    return W.conv_space(*a, make=_make, **k)


def resnet18_tasks() -> List[DesignSpace]:
    from workloads import spaces as W
    return W.resnet18_tasks(make=_make)


def vgg16_tasks() -> List[DesignSpace]:
    from workloads import spaces as W
    return W.vgg16_tasks(make=_make)


def alexnet_tasks() -> List[DesignSpace]:
    from workloads import spaces as W
    return W.alexnet_tasks(make=_make)


def synthetic_space(seed: int = 0, num_knobs: int = 16, rule: Optional[str] = None,
                    workload: str = "synthetic") -> DesignSpace:
    from workloads import spaces as W
    return W.synthetic_space(seed, num_knobs, rule, workload, make=_make)


def small_space(cards: Sequence[int], rule: Optional[str] = None, workload: str = "small") -> DesignSpace:
    from workloads import spaces as W
    return W.small_space(cards, rule, workload, make=_make)
