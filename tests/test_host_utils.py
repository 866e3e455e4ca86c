"""Host utilities of §5.1 and the conclusion, and the
input generator's determinism."""
import json
import os

import numpy as np

import oracle
from holo_synth import WORKLOADS, Region, blobs_target, splitmix64_stream, target_for

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_primes_and_limits():
    g = GOLD["next_prime_above_10000"]
    assert oracle.next_prime_above(g["n"]) == g["expect"]
    assert not oracle.is_prime(256) and oracle.is_prime(2) and oracle.is_prime(10007)
    assert oracle.next_prime_above(0) == 2
    for key in ("hard_limits_256_256_24", "hard_limits_64_128_8"):
        g = GOLD[key]
        assert list(oracle.hard_limits(*g["args"])) == g["expect"]


def test_input_stream_matches_published_splitmix():
    assert int(splitmix64_stream(0, 1)[0]) == 0xE220A8397B1DCDAF
    assert int(splitmix64_stream(0, 1, start=2)[0]) == 0x06C45D188009454F


def test_blob_target_recipe():
    w = WORKLOADS["C1"]
    T = target_for(w)
    assert T.dtype == np.float32 and T.shape == (64, 64)
    assert T.max() == 1.0 and T.min() >= 0
    assert np.all(T[0] == 0) and np.all(T[32:] == 0)       # zero outside Ω (R-13)
    assert np.array_equal(T, target_for(w))                 # deterministic
    T2 = blobs_target(2, 64, 4, 4.0, 10.0, Region.full(64))
    assert not np.array_equal(T, T2)
