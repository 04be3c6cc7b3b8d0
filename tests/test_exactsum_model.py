"""CPU model of the exact parallel sequential-sum algorithm used by the k-means
kernels (paper_2001_08743_b200/csrc/exactsum.cuh): segment maps composed in
order must reproduce left-to-right fp64 summation bit-for-bit."""
import random

import pytest

from xsum_model import exact, seq


@pytest.mark.parametrize("kind", range(4))
def test_segment_maps_reproduce_sequential_sum(kind):
    rnd = random.Random(kind)
    for trial in range(60):
        n = rnd.randint(1, 5000)
        if kind == 0:
            xs = [rnd.random() for _ in range(n)]
        elif kind == 1:
            card = rnd.choice([2, 3, 5, 7, 12, 31, 224, 336])
            xs = [rnd.randrange(card) / (card - 1) for _ in range(n)]
        elif kind == 2:
            xs = [rnd.random() ** 8 * 16 for _ in range(n)]
        else:
            xs = [rnd.choice([0.0, 0.5, 0.25, 1.0, 3.0, 1e-20]) for _ in range(n)]
        got, _ = exact(xs)
        assert got == seq(xs)
