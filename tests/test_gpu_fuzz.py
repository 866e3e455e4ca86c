"""Seeded randomised parity sweep over the OSPR and GS plan space (GPU vs the fp64 oracle).

The fixed tests pin the BASELINE configurations and the P-9 lengths; this sweep draws
(N, N_SF, N_LUT, phase offset, frames, sub-frame shard, region, GS levels) at random so
that the rarely taken paths -- LUT modes wrap / power-of-two / Lemire below N, odd pair
tails inside shards, several frames per call, GS constraints -- are exercised together.
Protocol and tolerances as in test_gpu_ospr.py / test_gpu_gs.py.
"""
import numpy as np
import pytest

import oracle
from holo_synth import LUT_SEED, Region, blobs_target, splitmix64_stream
from parity import REL_TOL, check_bits, check_intensity, cuda_target, lut_pair, rel, to_np

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")


def draw(seed, k):
    """k uniform integers from the seeded stream (the test's own RNG, no method arithmetic)."""
    return splitmix64_stream(seed, k)


@pytest.mark.parametrize("case", range(40))
def test_ospr_random_plans(case):
    u = draw(9000 + case, 8)
    n = [16, 32, 64, 128, 256][int(u[0] % 5)]
    S = 1 + int(u[1] % 9)
    L = [0, 1, 3, 7, n - 1, n, n + 3, 2 * n, 1021, 4096, 10007][int(u[2] % 11)]
    offset = int(u[3] % (1 << 40))
    F = 1 + int(u[4] % 2)
    b = int(u[5] % S)
    e = b + 1 + int(u[6] % (S - b))
    Ts = np.stack([blobs_target(100 * case + f, n, 4, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
                   for f in range(F)])
    lg, lo = lut_pair(LUT_SEED + case, L)
    om = Region.upper_half(n).as_tuple()
    res = hb.ospr_generate(cuda_target(Ts), S, lg, phase_offset=offset, sf_range=(b, e), omega=om)
    bits, I = to_np(res.bits), to_np(res.intensity)
    P = n * n
    for f in range(F):
        for j, s in enumerate(range(b, e)):
            _, h_re, _ = oracle.ospr_subframe(Ts[f], lo, offset + (f * S + s) * P, want_h=True, want_intensity=False)
            check_bits(bits[f, j], h_re, n)
        # the full range returns the mean; a shard the partial SUM of its sub-frames (R-18)
        full = (b, e) == (0, S)
        check_intensity(I[f] if full else I[f] / (e - b), oracle.replay_from_bits(bits[f], n))
    if (b, e) == (0, S):
        _, _, mse_ref = oracle.ospr(Ts, S, lo, offset, om)
        mse = to_np(res.mse)
        for f in range(F):
            assert rel(mse[f], mse_ref[f]) <= REL_TOL


@pytest.mark.parametrize("case", range(16))
def test_gs_random_plans(case):
    """Iteration 1 against the oracle (continuous: MSE and h; Q levels: MSE, levels outside the
    decision band) for random N, batch, LUT length, offset and Q."""
    u = draw(9500 + case, 6)
    n = [16, 32, 64, 128, 256][int(u[0] % 5)]
    B = 1 + int(u[1] % 3)
    L = [0, 5, n, 1021, 4096][int(u[2] % 5)]
    offset = int(u[3] % (1 << 36))
    Q = [0, 0, 2, 7, 256][int(u[4] % 5)]
    Ts = np.stack([blobs_target(300 * case + f, n, 4, max(1.0, n / 16), max(2.0, n / 6), Region.full(n))
                   for f in range(B)])
    lg, lo = lut_pair(LUT_SEED, L)
    res = hb.gs_generate(cuda_target(Ts), 1, lg, phase_offset=offset, levels=Q)
    mse = to_np(res.mse)
    for f in range(B):
        ref = oracle.gs(Ts[f], 1, lo, offset + f * n * n, Q, (0, n, 0, n))
        assert rel(mse[f, 0], ref["mse"][0]) <= REL_TOL, (case, f, mse[f, 0], ref["mse"][0])
