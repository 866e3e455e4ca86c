"""Pins of the oracle's GS path (Fig. 2 left; steps g0-g6)."""
import json
import os

import numpy as np
import pytest

import oracle
from holo_synth import Region, blobs_target

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _constrain(h, levels):
    """One-pixel projection through gs_step on a 1x1 field (F = identity at N = 1)."""
    out = oracle.gs_step(np.array([[h]], complex), np.ones((1, 1), np.float32), levels, (0, 1, 0, 1))
    return out["holo"][0, 0], int(out["levels"][0, 0])


def test_constraint_examples():
    h, _ = _constrain(3 + 4j, 0)
    assert abs(h - (0.6 + 0.8j)) < 1e-15
    h, _ = _constrain(0j, 0)        # a zero pixel maps to +1
    assert h == 1
    # Q = 4 levels {1, i, -1, -i}: nearest angle, wrap at 2 pi (R-15)
    for z, j in [(1 + 0.9j, 0), (1 + 1.1j, 1), (-1 - 0.01j, 2), (0.2 - 1j, 3),
                 (np.exp(1j * np.deg2rad(350)), 0)]:
        h, lev = _constrain(z, 4)
        assert lev == j and abs(h - 1j ** j) < 1e-15


def test_fixed_point():
    """if T is the replay amplitude of a phase-only hologram h0, one step
    from R = F{h0} recovers h0 and amplitude replacement keeps the phase."""
    n = 32
    rng = np.random.default_rng(8)
    h0 = np.exp(2j * np.pi * rng.random((n, n)))
    R = oracle.fft2(h0)
    T = np.abs(R).astype(np.float32)
    out = oracle.gs_step(R, T, 0, (0, n, 0, n))
    assert np.max(np.abs(out["holo"] - h0)) <= 1e-10
    assert np.max(np.abs(np.angle(out["R"] / R))) <= 1e-10
    assert np.array_equal(np.abs(out["R"]).astype(np.float32), T)
    assert abs(out["E"] - np.sum((np.abs(R) - T.astype(np.float64)) ** 2)) <= 1e-12


@pytest.mark.parametrize("levels", [0, 2, 256])
def test_error_reduction_monotone(levels):
    """GS error reduction (Fienup 1982): E_k = sum (|R'_k| - T)^2 is
    non-increasing for continuous and level-quantised in-loop projection (R-14)."""
    n = 64
    T = blobs_target(2, n, 4, 4.0, 10.0, Region.full(n))
    out = oracle.gs(T, 20, oracle.lut_build(2004, 4096), 0, levels, (0, n, 0, n))
    E = out["E"]
    assert np.all(E[1:] <= E[:-1] * (1 + 1e-12))
    assert E[-1] < E[0]


def test_energy_and_scale():
    n = 32
    T = blobs_target(5, n, 3, 3.0, 6.0, Region.full(n))
    out = oracle.gs(T, 3, oracle.lut_build(2004, 97), 0, 0, (0, n, 0, n))
    assert abs(out["I"].sum() - n * n) <= 1e-9 * n * n        # unit-modulus hologram
    assert np.max(np.abs(np.abs(out["holo"]) - 1)) <= 1e-12


def test_gs_equals_chain_of_steps():
    n, iters, Q = 32, 4, 256
    T = blobs_target(6, n, 3, 3.0, 6.0, Region.full(n))
    lut = oracle.lut_build(2004, 4096)
    full = oracle.gs(T, iters, lut, 17, Q, (0, n, 0, n))
    R = oracle.apply_phase(T, lut, 17)
    for k in range(iters):
        st = oracle.gs_step(R, T, Q, (0, n, 0, n))
        assert st["mse"] == full["mse"][k] and st["E"] == full["E"][k]
        R = st["R"]
    assert np.array_equal(st["levels"], full["levels"])
    assert np.array_equal(st["I"], full["I"])
