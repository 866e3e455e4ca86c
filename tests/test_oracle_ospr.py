"""Pins of the oracle's OSPR path (Fig. 2 right; steps a1-a7) and metrics.

Each pin is fixed by the paper, the spec or the mathematics, not by the
oracle itself: worked examples, Parseval energy, conjugate
symmetry of a real hologram's replay, the DC closed form, the L | N^2
degeneracy, sub-frame averaging and the resolution spike.
"""
import json
import os

import numpy as np
import pytest

import oracle
from holo_synth import Region, WORKLOADS, blobs_target, target_for

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _unpack(bits, n):
    return np.unpackbits(np.asarray(bits, np.uint8).reshape(-1, n, n // 8), axis=2)


def _mirror(a):
    return np.roll(np.flip(a, (-2, -1)), 1, axis=(-2, -1))


def test_quantise_examples():
    for re, _im, expect in GOLD["quantise_binary"]["cases"]:
        assert oracle.quantise_binary(re) == expect


def test_pack_examples():
    for key in ("pack_8x1_all_plus", "pack_8x1_all_minus", "pack_4x1_alternating"):
        g = GOLD[key]
        out = oracle.pack_bits(np.array([g["pm"]], np.uint8))
        assert list(out.ravel()) == g["expect"]


@pytest.fixture(scope="module")
def c1():
    w = WORKLOADS["C1"]
    T = target_for(w)
    return w, T


def test_replay_energy_symmetry_and_dc(c1):
    """Parseval with |h'| = 1: sum I_s = N^2 exactly; real h' => I[k] = I[-k];
    DC = (2 popcount - N^2)^2 / N^2 (Eq. (1) at u = v = 0)."""
    w, T = c1
    n, P = w.n, w.n * w.n
    lut = oracle.lut_build(2004, 1021)
    for s in range(3):
        bits, h, Iv = oracle.ospr_subframe(T, lut, cursor=s * P)
        assert abs(Iv.sum() - P) <= 1e-9 * P
        assert np.max(np.abs(Iv - _mirror(Iv))) <= 1e-12 * Iv.max()
        pop = int(_unpack(bits, n).sum())
        assert abs(Iv[0, 0] - (2 * pop - P) ** 2 / P) <= 1e-9 * max(1.0, Iv[0, 0])
        # bits are the sign of Re H (R-7)
        assert np.array_equal(_unpack(bits, n)[0], (h >= 0).astype(np.uint8))


def test_all_plus_hologram_is_dc_spike():
    """a single all-(+1) frame replays to a DC spike of height N^2."""
    n = 32
    I = oracle.replay_from_bits(np.full((1, n, n // 8), 255, np.uint8), n)
    assert abs(I[0, 0] - n * n) < 1e-9
    I[0, 0] = 0
    assert np.max(np.abs(I)) < 1e-9


def test_flat_source_identical_subframes(c1):
    """with no randomisation all sub-frames are identical; mean = single."""
    w, T = c1
    bits, I, _ = oracle.ospr(T, 4, None, 0, Region.upper_half(w.n).as_tuple())
    assert all(np.array_equal(bits[0, 0], bits[0, s]) for s in range(4))
    _, _, I1 = oracle.ospr_subframe(T, None, 0)
    assert np.max(np.abs(I[0] - I1)) <= 1e-12 * I1.max()


def test_lut_dividing_frame_size_degenerates(c1):
    """Pin c3 #13: if N_LUT divides N^2 every sub-frame draws the same phases (the
    BASELINE lengths all do), so the bits are identical; a non-dividing length differs."""
    w, T = c1
    region = Region.upper_half(w.n).as_tuple()
    bits, _, _ = oracle.ospr(T, 4, oracle.lut_build(2004, 256), 0, region)
    assert all(np.array_equal(bits[0, 0], bits[0, s]) for s in range(4))
    bits, _, _ = oracle.ospr(T, 4, oracle.lut_build(2004, 257), 0, region)
    assert not np.array_equal(bits[0, 0], bits[0, 1])


def test_prefix_property_subframe0(c1):
    """Pin c3 #14: for L >= N^2, sub-frame 0 uses lut[0:N^2] whatever L is."""
    w, T = c1
    P = w.n * w.n
    b = [oracle.ospr_subframe(T, oracle.lut_build(2004, L), 0, False, False)[0] for L in (P, P + 1, 3 * P)]
    assert np.array_equal(b[0], b[1]) and np.array_equal(b[0], b[2])


def test_continuing_cursor(c1):
    """sub-frames continue where the previous left off: a 6-sub-frame run equals
    a 3-sub-frame run followed by one starting 3 N^2 draws later."""
    w, T = c1
    P = w.n * w.n
    lut = oracle.lut_build(2004, 10007)
    region = Region.upper_half(w.n).as_tuple()
    b6, _, _ = oracle.ospr(T, 6, lut, 0, region)
    b3, _, _ = oracle.ospr(T, 3, lut, 3 * P, region)
    assert np.array_equal(b6[0, 3:], b3[0])
    # and two frames of 3 sub-frames equal one frame of 6 (frames continue too)
    b2, _, _ = oracle.ospr(np.stack([T, T]), 3, lut, 0, region)
    assert np.array_equal(b2.reshape(6, w.n, w.n // 8), b6[0])


def test_full_length_lut_equals_independent_phases(c1):
    """a LUT of length N^2 N_SF filled from the PRNG stream
    gives bit-identical sub-frames to drawing independent phases on the fly."""
    w, T = c1
    n, P, K = w.n, w.n * w.n, 4
    bits, _, _ = oracle.ospr(T, K, oracle.lut_build(2004, K * P), 0, Region.upper_half(n).as_tuple())
    for s in range(K):
        H = oracle.fft2(oracle.apply_phase_prng(T, 2004, s * P), inverse=True)
        expect = oracle.pack_bits((H.real >= 0).astype(np.uint8))
        assert np.array_equal(bits[0, s], expect)


def test_replay_from_bits_consistent(c1):
    w, T = c1
    bits, I, _ = oracle.ospr(T, 3, oracle.lut_build(2004, 257), 0, Region.upper_half(w.n).as_tuple())
    assert np.max(np.abs(oracle.replay_from_bits(bits[0], w.n) - I[0])) <= 1e-12 * I.max()


def test_mse_m1_hand_example_and_invariances():
    g = GOLD["mse_m1_2x2"]
    T = np.array(g["T"], np.float32)
    I = np.array(g["I"], np.float64)
    assert abs(oracle.mse_m1(I, T, (0, 2, 0, 2)) - g["expect"]) < 1e-15
    rng = np.random.default_rng(3)
    T = rng.random((16, 16)).astype(np.float32)
    I = rng.random((16, 16)) * 7
    reg = (1, 8, 0, 16)
    m = oracle.mse_m1(I, T, reg)
    assert m >= 0
    assert abs(oracle.mse_m1(I * 123.25, T, reg) - m) <= 1e-12 * m          # S:338 scale invariance
    assert oracle.mse_m1(5.0 * T.astype(np.float64) ** 2, T, reg) <= 1e-30  # 0 iff a I = T^2
    t = T[1:8].astype(np.float64)
    assert abs(oracle.mse_m1(np.zeros((16, 16)), T, reg) - np.mean(t ** 4)) <= 1e-15  # I = 0


def test_mse_alpha_closed_form_is_minimum():
    """the closed-form alpha attains the minimum of a brute-force alpha scan."""
    rng = np.random.default_rng(4)
    T = rng.random((16, 16)).astype(np.float32)
    I = rng.random((16, 16)) * 3
    reg = (0, 16, 0, 16)
    m = oracle.mse_alpha(I, T, reg)
    A = np.sqrt(I)
    grid = np.linspace(0, 2, 10001)
    scan = [np.mean((a * A - T) ** 2) for a in grid]
    assert m <= min(scan) + 1e-12
    assert abs(m - min(scan)) <= 1e-6


def test_time_averaging_reduces_mse_like_one_over_k():
    """P:64 'Time averaging then ensures a reduction in MSE'; BASELINE north_star 'MSE
    falling roughly as 1/N_sub': independent sub-frames at 128^2, MSE(K) strictly
    decreasing over K in {1,2,4,8,16,24}, A/K + B fit R^2 >= 0.999, MSE(24)/MSE(1) < 0.2.
    The target fills Ω like the paper's natural images (16 blobs, sigma scaled N/64 as
    in reading R-20); with a sparse target the K-independent floor B dominates."""
    n, Kmax = 128, 24
    region = Region.upper_half(n)
    Ks = [1, 2, 4, 8, 16, 24]
    curves = []
    for seed in (11, 12, 13):
        T = blobs_target(seed, n, 16, 8.0, 20.0, region)
        lut = oracle.lut_build(2004 + seed, n * n * Kmax)  # full length: independent
        Is = [oracle.ospr_subframe(T, lut, s * n * n, False, True)[2] for s in range(Kmax)]
        cum = np.cumsum(Is, axis=0)
        curves.append([oracle.mse_m1(cum[K - 1] / K, T, region.as_tuple()) for K in Ks])
    m = np.mean(curves, axis=0)
    assert np.all(np.diff(m) < 0)
    X = np.stack([1.0 / np.array(Ks), np.ones(len(Ks))], 1)
    coef, *_ = np.linalg.lstsq(X, m, rcond=None)
    r2 = 1 - np.sum((X @ coef - m) ** 2) / np.sum((m - m.mean()) ** 2)
    assert r2 >= 0.999
    assert m[-1] / m[0] < 0.2


def test_resolution_spike():
    """N_LUT = 256 at 256x256 gives a sharp increase in error (every image row
    has the same phase behaviour) versus the neighbouring prime 257."""
    g = GOLD["resolution_spike"]
    n, K = g["n"], g["n_sub"]
    region = Region.upper_half(n).as_tuple()
    T = blobs_target(21, n, 16, 16.0, 40.0, Region.upper_half(n))  # fills Ω (R-20 scaling)
    _, _, m_spike = oracle.ospr(T, K, oracle.lut_build(2004, g["spike_len"]), 0, region)
    _, _, m_prime = oracle.ospr(T, K, oracle.lut_build(2004, g["prime_len"]), 0, region)
    assert m_spike[0] > 1.3 * m_prime[0]


def test_flat_phase_edge_enhancement():
    """without randomisation energy concentrates on the edges of a filled
    rectangle; with independent phases the edge/interior ratio is lower."""
    n, K = 64, 8
    T = np.zeros((n, n), np.float32)
    T[8:24, 20:44] = 1.0
    edge = np.zeros((n, n), bool)
    edge[8:24, 20:44] = True
    inner = np.zeros((n, n), bool)
    inner[10:22, 22:42] = True
    edge &= ~inner
    region = (1, n // 2, 0, n)

    def ratio(lut):
        _, I, _ = oracle.ospr(T, K, lut, 0, region)
        return I[0][edge].mean() / I[0][inner].mean()

    flat = ratio(None)
    indep = ratio(oracle.lut_build(2004, K * n * n))
    assert flat > 1.5 * indep


def test_speckle_independence():
    """P:64 / S:275: independent sub-frames carry independent speckle.  The fluctuations
    d_s = I_s - mean_t I_t over Ω of K independent sub-frames have pairwise correlation
    -1/(K-1) in expectation (the sample mean is removed); a LUT that divides N^2 makes
    every sub-frame identical (d_s = 0)."""
    n, K = 128, 24
    reg = Region.upper_half(n)
    T = blobs_target(31, n, 16, 8.0, 20.0, reg)

    def fluct(lut):
        Is = np.array([oracle.ospr_subframe(T, lut, s * n * n, False, True)[2][reg.row0:reg.row1].ravel()
                       for s in range(K)])
        return Is - Is.mean(0)

    d = fluct(oracle.lut_build(2004, K * n * n))
    c = np.corrcoef(d)
    off = c[~np.eye(K, dtype=bool)]
    assert abs(off.mean() + 1.0 / (K - 1)) < 0.01
    assert np.max(np.abs(off + 1.0 / (K - 1))) < 0.05
    assert np.max(np.abs(fluct(oracle.lut_build(2004, 256)))) <= 1e-12  # mean-removal rounding only
