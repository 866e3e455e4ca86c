"""Pins of the oracle's unitary DFT pair (Eqs. (1)-(2); P:43 FFT).

The oracle FFT is checked against things other than itself: the O(N^4)
direct sum of Eq. (1)/(2), an O(N^3) separable direct sum, the closed-form
delta/constant pairs of S:48-58, Parseval, the round trip, Hermitian
symmetry of a real input, and numpy's pocketfft (a library routine that the
unitary DFT reduces to with norm="ortho").
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _rand_field(n, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal((n, n)) + 1j * r.standard_normal((n, n))


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft_matches_direct_sum(n, inverse):
    f = _rand_field(n, n + 7 * inverse)
    direct = oracle.dft2_direct(f, inverse)
    fast = oracle.fft2(f, inverse)
    assert np.max(np.abs(direct - fast)) <= 1e-9 * max(1.0, np.max(np.abs(direct)))


@pytest.mark.parametrize("n", [32, 64])
def test_fft_matches_separable_direct(n):
    f = _rand_field(n, 3)
    for inv in (False, True):
        d = oracle.dft2_separable(f, inv)
        assert np.max(np.abs(d - oracle.fft2(f, inv))) <= 1e-9 * np.max(np.abs(d))


def test_direct_sums_agree_with_each_other():
    f = _rand_field(8, 11)
    assert np.max(np.abs(oracle.dft2_direct(f) - oracle.dft2_separable(f))) <= 1e-12


def test_delta_and_constant_examples():
    g = GOLD["dft_delta_4x4"]
    d = np.zeros((4, 4), complex)
    d[0, 0] = 1
    F = oracle.fft2(d)
    assert np.allclose(F, g["expect_constant"], atol=1e-15)
    g = GOLD["dft_ones_2x2"]
    F = oracle.fft2(np.ones((2, 2), complex))
    expect = np.zeros((2, 2))
    expect[0, 0] = g["expect_dc"]
    assert np.allclose(F, expect, atol=1e-15)
    g = GOLD["idft_delta_4x4"]
    assert np.allclose(oracle.fft2(d, inverse=True), g["expect_constant"], atol=1e-15)


def test_sign_convention_single_frequency():
    """Eq. (1): a plane wave exp(+2 pi i (u0 x / N)) transforms to a delta at u0 (forward
    uses exp(-2 pi i ...)); a transposed index or a flipped sign moves the peak."""
    n = 16
    x = np.arange(n)
    u0, v0 = 3, 5
    f = np.exp(2j * np.pi * (u0 * x[None, :] + v0 * x[:, None]) / n)
    F = oracle.fft2(f)
    peak = np.unravel_index(np.argmax(np.abs(F)), F.shape)
    assert peak == (v0, u0)              # data[y][x]: row index is v (y-frequency)
    assert abs(F[v0, u0] - n) < 1e-9     # 1/sqrt(N^2) * N^2


@pytest.mark.parametrize("n", [64, 256, 1024])
def test_roundtrip_and_parseval(n):
    f = _rand_field(n, n)
    F = oracle.fft2(f)
    e0, e1 = np.sum(np.abs(f) ** 2), np.sum(np.abs(F) ** 2)
    assert abs(e1 - e0) <= 1e-10 * e0
    back = oracle.fft2(F, inverse=True)
    assert np.max(np.abs(back - f)) <= 1e-10 * np.max(np.abs(f))


def test_hermitian_symmetry_of_real_input():
    n = 64
    f = np.random.default_rng(5).standard_normal((n, n)).astype(complex)
    F = oracle.fft2(f)
    mirror = np.roll(np.flip(F, (0, 1)), 1, axis=(0, 1))  # F[(-v) mod N][(-u) mod N]
    assert np.max(np.abs(F - np.conj(mirror))) <= 1e-12 * np.max(np.abs(F))


@pytest.mark.parametrize("n", [128, 1024])
def test_matches_pocketfft_ortho(n):
    f = _rand_field(n, 99)
    assert np.max(np.abs(oracle.fft2(f) - np.fft.fft2(f, norm="ortho"))) <= 1e-12 * np.sqrt(n * n)
    assert np.max(np.abs(oracle.fft2(f, True) - np.fft.ifft2(f, norm="ortho"))) <= 1e-12 * np.sqrt(n * n)


def test_rejects_non_power_of_two():
    with pytest.raises(ValueError):
        oracle.fft2(np.ones((12, 12), complex))
