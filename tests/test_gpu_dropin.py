"""The reference's own adaptive_sample / kmeans_run / predict_batch (compiled
from /root/reference/proj/src) with the GPU plugged into its seams via
include/ktune_gpu.hpp (the Clusterer hook, sampling.hpp:44-46): results must be
bit-identical to the all-CPU reference."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


def test_reference_adaptive_sample_with_gpu_clusterer(ctx):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_test not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith(")") and r.stdout.startswith("OK")
