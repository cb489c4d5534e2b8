"""Randomized determinism stress (scripts/stress.py) for a few seconds: random
configs, pair ranges and three concurrent streams must reproduce a cold
single-stream run bit for bit."""

import os
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_random_configs_streams_and_shards_bit_identical():
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import stress

    assert stress.run_stress(8.0, seed=1) > 0
