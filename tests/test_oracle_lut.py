"""Pins of the oracle's phase pool (step a0) and cyclic consumption (a1, a2).

P:68 "Random numbers can be generated at compile time to fill the LUT which
then acts as a pool of random numbers for algorithms to sequentially draw
from"; "The pool ... is cycled through sequentially with successive
frames and sub-frames continuing from where the previous left off".
"""
import json
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))


def test_splitmix64_published_vector():
    for line in open(os.path.join(HERE, "golden", "splitmix64.txt")):
        if line.startswith("#") or not line.strip():
            continue
        seed, k, hexv = line.split()
        assert oracle.splitmix64(int(seed), int(k)) == int(hexv, 16)


def test_angle_code_is_high_word():
    for k in range(5):
        assert oracle.angle_code(2004, k) == oracle.splitmix64(2004, k) >> 32


def _f32(x):
    return float(np.float32(x))


def test_recipe_closed_forms():
    """R-5 at angles with closed-form cos/sin: every octant boundary plus pi/8 and 3pi/8."""
    r2 = np.sqrt(0.5)
    c8, s8 = np.sqrt(2 + np.sqrt(2)) / 2, np.sqrt(2 - np.sqrt(2)) / 2
    cases = {
        0: (1, 0), 1 << 29: (r2, r2), 1 << 30: (0, 1), 3 << 29: (-r2, r2), 1 << 31: (-1, 0),
        5 << 29: (-r2, -r2), 3 << 30: (0, -1), 7 << 29: (r2, -r2),
        1 << 28: (c8, s8), 3 << 28: (s8, c8), 5 << 28: (-s8, c8), 15 << 28: (c8, -s8),
    }
    u = np.array(list(cases), dtype=np.uint32)
    got = oracle.phase_f64(u)
    for (uu, (c, s)), (gc, gs) in zip(cases.items(), got):
        assert abs(gc - c) <= 2e-16 and abs(gs - s) <= 2e-16, uu
    # the fp32 pool value (R-5 step 5) is the correct rounding of the closed form
    for (uu, (c, s)), (gc, gs) in zip(cases.items(), got):
        assert np.float32(gc) == np.float32(c) and np.float32(gs) == np.float32(s)


def test_recipe_matches_libm():
    u = np.random.default_rng(1).integers(0, 2 ** 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    got = oracle.phase_f64(u)
    ang = 2 * np.pi * (u.astype(np.float64) / 2.0 ** 32)
    assert np.max(np.abs(got[:, 0] - np.cos(ang))) <= 2e-15
    assert np.max(np.abs(got[:, 1] - np.sin(ang))) <= 2e-15


def test_lut_entries_unit_modulus_no_negative_zero():
    lut = oracle.lut_build(2004, 100_000).astype(np.float64)
    assert np.max(np.abs(np.hypot(lut[:, 0], lut[:, 1]) - 1)) <= 1e-7
    z = lut == 0
    assert not np.any(np.signbit(lut[z]))


def test_lut_uniformity_chi2_and_mean():
    """S:129 mean modulus of 10007 entries <= 0.05; S:179 16-bin chi-square at p=0.001."""
    lut = oracle.lut_build(2004, 1_000_000).astype(np.float64)
    phi = np.mod(np.arctan2(lut[:, 1], lut[:, 0]), 2 * np.pi)
    counts = np.histogram(phi, bins=16, range=(0, 2 * np.pi))[0]
    e = len(phi) / 16
    chi2 = np.sum((counts - e) ** 2 / e)
    assert chi2 < 37.70  # chi-square(15) upper 0.001 quantile
    small = oracle.lut_build(2004, 10007).astype(np.float64)
    assert abs(np.mean(small[:, 0] + 1j * small[:, 1])) <= 0.05


def test_prefix_property():
    """R-4: counter-based generation makes LUT(seed, L1) a prefix of LUT(seed, L2)."""
    a = oracle.lut_build(7, 1000)
    b = oracle.lut_build(7, 4099)
    assert np.array_equal(a, b[:1000])


def _index_probe(n_lut):
    """A LUT whose entry k encodes k (probe only; the recipe is tested above)."""
    return np.stack([np.arange(n_lut, dtype=np.float32) + 1, np.zeros(n_lut, np.float32)], 1)


def test_cursor_examples():
    g = GOLD["cursor_len5_9draws"]
    assert [oracle.lut_index(d, g["n_lut"]) for d in range(g["draws"])] == g["expect"]
    g = GOLD["cursor_2x2_two_subframes"]
    lut = _index_probe(g["n_lut"])
    T = np.ones((g["n"], g["n"]), np.float32)
    P = g["n"] ** 2
    for s, expect in enumerate(g["expect"]):
        R = oracle.apply_phase(T, lut, cursor=s * P)
        assert list(np.rint(R.real).astype(int).ravel() - 1) == expect


def test_apply_phase_examples():
    g = GOLD["apply_phase_1x1"]
    cs = oracle.phase_f64(np.array([g["u"]], np.uint32))[0]
    lut = np.array([[np.float32(cs[0]) if cs[0] != 0 else 0.0, np.float32(cs[1])]], np.float32)
    R = oracle.apply_phase(np.full((1, 1), g["T"], np.float32), lut, 0)
    assert R[0, 0] == complex(*g["expect"])
    # |R| = T for unit-modulus entries and zero image -> zero field
    lut = oracle.lut_build(3, 257)
    T = np.random.default_rng(0).random((16, 16)).astype(np.float32)
    R = oracle.apply_phase(T, lut, 12345)
    assert np.max(np.abs(np.abs(R) - T)) <= 1e-7
    assert np.all(oracle.apply_phase(np.zeros((16, 16), np.float32), lut, 5) == 0)


def test_lut_length_one_and_flat():
    lut = oracle.lut_build(9, 1)
    T = np.random.default_rng(1).random((8, 8)).astype(np.float32)
    R = oracle.apply_phase(T, lut, 77)
    c = complex(float(lut[0, 0]), float(lut[0, 1]))
    assert np.all(R == T.astype(np.float64) * c)
    flat = oracle.apply_phase(T, None, 5)       # N_LUT = 0 -> 1 + 0i (R-6)
    assert np.all(flat == T.astype(np.float64))


def test_period_is_exactly_n_lut():
    """the cyclic stream is periodic with period N_LUT."""
    L = 13
    lut = oracle.lut_build(5, L)
    T = np.ones((8, 8), np.float32)
    r = oracle.apply_phase(T, lut, 0).ravel()
    assert np.array_equal(r[:L], r[L:2 * L])
    assert not np.array_equal(r[:L], r[1:L + 1])


def test_full_length_lut_equals_prng_stream():
    """P:68/P:120 (pin c3 #15): a LUT at least as long as all draws is the PRNG source."""
    n, draws = 16, 16 * 16 * 3
    lut = oracle.lut_build(2004, draws)
    T = np.random.default_rng(2).random((n, n)).astype(np.float32)
    for s in range(3):
        assert np.array_equal(oracle.apply_phase(T, lut, s * n * n),
                              oracle.apply_phase_prng(T, 2004, s * n * n))


# ---- P:170 / R-25: PRNG + a 2^q-entry sin/cos table ----------------------------------------------

def _codes(seed, cursor, m):
    return np.array([oracle.angle_code(seed, cursor + k) for k in range(m)], dtype=np.uint64)


def test_prng_table_q2_is_quarter_turns_exactly():
    """q = 2: the phase is i^(u >> 30) exactly (cos, sin in {0, +-1}), so R = T * i^k with no
    rounding at all -- a closed form that a wrong shift, mask or octant would break."""
    n, seed, cur = 16, 2004, 12345
    T = np.linspace(0.1, 1.0, n * n, dtype=np.float32).reshape(n, n)
    R = oracle.apply_phase_prng_q(T, seed, cur, 2)
    k = (_codes(seed, cur, n * n) >> 30).astype(np.int64).reshape(n, n)
    assert np.array_equal(R, T.astype(np.float64) * (1j ** k))


def test_prng_table_q3_eighth_turns_and_q32_is_the_prng_source():
    n, seed, cur = 16, 7, 99
    T = np.ones((n, n), np.float32)
    R = oracle.apply_phase_prng_q(T, seed, cur, 3)
    k = (_codes(seed, cur, n * n) >> 29).astype(np.float64).reshape(n, n)
    assert np.max(np.abs(R - np.exp(2j * np.pi * k / 8))) <= 2.0 ** -24
    # no truncation: the full-precision on-the-fly source
    assert np.array_equal(oracle.apply_phase_prng_q(T, seed, cur, 32), oracle.apply_phase_prng(T, seed, cur))


@pytest.mark.parametrize("q", [5, 8, 12, 16])
def test_prng_table_levels(q):
    """The phase of draw g is the angle of the top q bits of its code, 2 pi (u >> (32-q)) / 2^q,
    at unit modulus (fp32 rounding of the recipe: 1e-7)."""
    n, seed, cur = 32, 11, 5
    T = np.ones((n, n), np.float32)
    R = oracle.apply_phase_prng_q(T, seed, cur, q)
    k = (_codes(seed, cur, n * n) >> (32 - q)).astype(np.float64).reshape(n, n)
    assert np.max(np.abs(R - np.exp(2j * np.pi * k / 2 ** q))) <= 1e-7
    assert np.max(np.abs(np.abs(R) - 1)) <= 1e-7


def test_prng_table_levels_uniform_chi2():
    """S:179's uniformity check on the quantised source: the 256 levels of q = 8 over 2^16
    draws pass a chi^2 test at p = 0.001 (critical value of chi^2 with 255 dof: 330.5)."""
    n, seed = 256, 2004
    R = oracle.apply_phase_prng_q(np.ones((n, n), np.float32), seed, 0, 8)
    lev = np.rint(np.mod(np.angle(R), 2 * np.pi) * 256 / (2 * np.pi)).astype(np.int64) % 256
    cnt = np.bincount(lev.ravel(), minlength=256)
    exp = n * n / 256
    assert ((cnt - exp) ** 2 / exp).sum() < 330.5
