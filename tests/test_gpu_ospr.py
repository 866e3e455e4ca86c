"""GPU parity of the OSPR path (steps a0-a7) against the fp64 oracle.

Protocol: P-1 LUT bit-exact; P-2 randomisation bit-exact; P-3
bits exact outside the |Re H| < 1e-5 max band; P-4 intensity conditional on
the GPU's bits, rel 1e-4; P-5 MSE unconditional, rel 1e-4; P-8 shards
reproduce the single call; P-9 LUT lengths beyond the BASELINE ones.
All calls go through the C ABI (paper_2004_04049_b200 -> libholo.so).
"""
import numpy as np
import pytest
import torch

import oracle
from holo_synth import LUT_SEED, WORKLOADS, Region, blobs_target, p9_lengths, target_for
from parity import (REL_TOL, check_bits, check_intensity, cuda_target, lut_pair, rel, to_np, unpack)

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")


# ---- P-1 / P-2 ----------------------------------------------------------------------------------

@pytest.mark.parametrize("L", [1, 5, 256, 4096, 10007, 1 << 16, 1 << 20, 1024 * 1024 * 24])
def test_lut_bit_exact(L):
    g = to_np(torch.view_as_real(hb.lut_generate(LUT_SEED, L)).contiguous())
    o = oracle.lut_build(LUT_SEED, L)
    assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_lut_other_seeds_and_prefix():
    for seed in (0, 1, 2 ** 63 + 17):
        g = to_np(torch.view_as_real(hb.lut_generate(seed, 3001)).contiguous())
        assert np.array_equal(g.view(np.uint32), oracle.lut_build(seed, 3001).view(np.uint32))
    a = hb.lut_generate(9, 1000)
    b = hb.lut_generate(9, 70001)
    assert torch.equal(a, b[:1000])


@pytest.mark.parametrize("L", [0, 1, 5, 13, 256, 257, 1021, 10007, 65, 4097])
@pytest.mark.parametrize("offset", [0, 12345, (1 << 33) + 7])
def test_randomise_bit_exact(L, offset):
    n = 64
    T = target_for(WORKLOADS["C1"])
    lg, lo = lut_pair(LUT_SEED, L)
    R = to_np(hb.debug_randomise(cuda_target(T), lg, offset))
    ref = oracle.apply_phase(T, lo, offset).astype(np.complex64)
    assert np.array_equal(R.view(np.uint32), ref.view(np.uint32))


# ---- pass A's production producer (a1, a2 + Hermitian pairing) ----------------------------------------

def _mirror(R):
    """R(-p): (y, x) -> ((-y) mod N, (-x) mod N)."""
    return np.roll(np.flip(R, (0, 1)), 1, (0, 1))


@pytest.mark.parametrize("n,S,L,offset,rng", [
    (64, 5, 4096, 0, (0, 5)),              # LUT_WRAP fast path (no wrap), odd tail
    (64, 4, 1021, 77, (1, 4)),             # LUT_GENERAL, shard with an odd last pair
    (128, 3, 1 << 12, 3 * 128 + 5, (0, 3)),   # LUT_POW2 (L a power of two), unaligned offset
    (128, 2, 0, 0, (0, 2)),                # L = 0: the flat pool
    (256, 2, 100003, (1 << 33) + 9, (0, 2)),  # offset beyond 2^32
    (1024, 3, 65536, 0, (0, 3)),           # the C3 pool (rows_a2 kernel)
    (1024, 2, 1009, 12345, (0, 2)),        # rows_a2, LUT_GENERAL
    (2048, 1, 7, 3, (0, 1)),               # rows_a2, tiny LUT, unpaired
    (4096, 3, 10007, 5, (0, 3)),           # rows_a4 (two warps per row, R-26), unpaired tail
    (4096, 2, 1 << 16, 0, (0, 2)),         # rows_a4, LUT_POW2
])
def test_pass_a_pairs_match_oracle(n, S, L, offset, rng):
    """The randomisation pass A feeds the row IFFT: conj(Z) with Z = H_a + i H_b,
    H_s = R_s + conj(R_s(-p)) and R_s = oracle.apply_phase at cursor offset + s N^2 (R-7,
    DESIGN.md §5). fp32: each component is a sum of two products |t c| <= 1, so every
    element is within 2 ulp(4)."""
    T = blobs_target(41 + n + S, n, 6, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
    lg, lo = lut_pair(LUT_SEED + 3, L)
    b, e = rng
    Z = to_np(hb.debug_ospr_pairs(cuda_target(T), S, lg, offset, (b, e)))
    P = n * n
    for j, s in enumerate(range(b, e, 2)):
        Ra = oracle.apply_phase(T, lo, offset + s * P)
        Rb = oracle.apply_phase(T, lo, offset + (s + 1) * P) if s + 1 < e else np.zeros_like(Ra)
        ref = np.conj((Ra + np.conj(_mirror(Ra))) + 1j * (Rb + np.conj(_mirror(Rb))))
        assert np.max(np.abs(Z[j] - ref)) <= 2.0 ** -20, (n, s)


@pytest.mark.parametrize("n,offset", [(64, 0), (1024, (1 << 35) + 17), (2048, 11), (4096, 3)])
def test_pass_a_pairs_prng_match_oracle(n, offset):
    """The same with the on-the-fly source (R-5 phases of SplitMix64 draws; recipe
    computed in fp64 on both sides, so R matches apply_phase_prng to fp32 rounding)."""
    T = blobs_target(77 + n, n, 6, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
    S, seed = 3, 2004
    Z = to_np(hb.debug_ospr_pairs(cuda_target(T), S, None, offset, (0, S), prng_seed=seed))
    P = n * n
    for j, s in enumerate(range(0, S, 2)):
        Ra = oracle.apply_phase_prng(T, seed, offset + s * P)
        Rb = oracle.apply_phase_prng(T, seed, offset + (s + 1) * P) if s + 1 < S else np.zeros_like(Ra)
        ref = np.conj((Ra + np.conj(_mirror(Ra))) + 1j * (Rb + np.conj(_mirror(Rb))))
        assert np.max(np.abs(Z[j] - ref)) <= 2.0 ** -20, (n, s)


@pytest.mark.parametrize("q", [1, 2, 8, 12, 16])
def test_phase_table_matches_recipe(q):
    """holo_phase_table: entry k is recipe R-5 at the code k << (32 - q), rounded to fp32 with
    -0 -> +0 (R-5 steps 5-6), bit for bit against the oracle's recipe."""
    tbl = to_np(hb.phase_table(q))
    codes = (np.arange(1 << q, dtype=np.uint64) << np.uint64(32 - q)).astype(np.uint32)
    ref = oracle.phase_f64(codes).astype(np.float32)
    ref[ref == 0] = 0.0                                   # -0 -> +0
    assert np.array_equal(tbl.real.view(np.uint32), ref[:, 0].view(np.uint32))
    assert np.array_equal(tbl.imag.view(np.uint32), ref[:, 1].view(np.uint32))


@pytest.mark.parametrize("n,q,offset", [(64, 8, 0), (64, 2, 977), (256, 12, 3 << 33), (1024, 16, 5), (2048, 8, 7)])
def test_pass_a_pairs_prng_table_match_oracle(n, q, offset):
    """P:170 / R-25: pass A with the PRNG + 2^q sin/cos table source equals the oracle's
    quantised source (apply_phase_prng_q) to fp32 rounding."""
    T = blobs_target(91 + n, n, 6, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
    S, seed = 3, 2004
    Z = to_np(hb.debug_ospr_pairs(cuda_target(T), S, None, offset, (0, S), prng_seed=seed, phase_bits=q))
    P = n * n
    for j, s in enumerate(range(0, S, 2)):
        Ra = oracle.apply_phase_prng_q(T, seed, offset + s * P, q)
        Rb = oracle.apply_phase_prng_q(T, seed, offset + (s + 1) * P, q) if s + 1 < S else np.zeros_like(Ra)
        ref = np.conj((Ra + np.conj(_mirror(Ra))) + 1j * (Rb + np.conj(_mirror(Rb))))
        assert np.max(np.abs(Z[j] - ref)) <= 2.0 ** -20, (n, q, s)


@pytest.mark.parametrize("n,S,q", [(64, 5, 8), (256, 4, 12), (1024, 6, 16), (2048, 3, 8)])
def test_ospr_prng_table_against_oracle(n, S, q):
    """The whole OSPR path with the table source: bits against the oracle's fp64 IDFT of its
    quantised-source randomisation (P-3 band), intensity conditional on the GPU bits (P-4),
    MSE against the oracle's own bits (P-5)."""
    T = blobs_target(17, n, 6, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
    seed, off = 2004, 4242
    res = hb.ospr_generate(cuda_target(T), S, prng_seed=seed, phase_bits=q, phase_offset=off)
    bits = to_np(res.bits)[0]
    ref_bits = []
    for s in range(S):
        h_re = oracle.fft2(oracle.apply_phase_prng_q(T, seed, off + s * n * n, q), True).real
        check_bits(bits[s], h_re, n)
        ref_bits.append(oracle.pack_bits((h_re >= 0).astype(np.uint8)))
    check_intensity(to_np(res.intensity)[0], oracle.replay_from_bits(bits, n))
    I_ref = oracle.replay_from_bits(np.stack(ref_bits), n)
    m_ref = oracle.mse_m1(I_ref, T, Region.upper_half(n).as_tuple())
    assert rel(to_np(res.mse)[0], m_ref) <= REL_TOL


# ---- unitary DFT hook ------------------------------------------------------------------------------

@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 512, 1024, 2048, 4096])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft2_matches_oracle(n, inverse):
    rng = np.random.default_rng(n)
    x = (rng.standard_normal((2, n, n)) + 1j * rng.standard_normal((2, n, n))).astype(np.complex64)
    y = to_np(hb.fft2(torch.from_numpy(x).cuda(), inverse=inverse))
    for b in range(2):
        ref = oracle.fft2(x[b].astype(np.complex128), inverse)
        d = y[b] - ref
        assert np.linalg.norm(d) / np.linalg.norm(ref) <= 1e-6
        assert np.max(np.abs(d)) <= 1e-5 * np.max(np.abs(ref))


# ---- OSPR end to end -----------------------------------------------------------------------------------

def ospr_parity(T, n_sub, L, offset=0, region=None, frames_T=None):
    """Run GPU OSPR and check P-3/P-4/P-5 for every sub-frame of every frame."""
    Ts = np.stack(frames_T) if frames_T is not None else T[None]
    F, n, _ = Ts.shape
    region = region or Region.upper_half(n).as_tuple()
    lg, lo = lut_pair(LUT_SEED, L)
    res = hb.ospr_generate(cuda_target(Ts), n_sub, lg, phase_offset=offset, omega=region)
    bits, I, mse = to_np(res.bits), to_np(res.intensity), to_np(res.mse)
    P = n * n
    flips = exempt = 0
    for f in range(F):
        for s in range(n_sub):
            _, h_re, _ = oracle.ospr_subframe(Ts[f], lo, offset + (f * n_sub + s) * P, want_h=True,
                                              want_intensity=False)
            e, fl = check_bits(bits[f, s], h_re, n)
            exempt += e
            flips += fl
        I_cond = oracle.replay_from_bits(bits[f], n)              # P-4: oracle propagates GPU bits
        check_intensity(I[f], I_cond)
    _, I_ref, mse_ref = oracle.ospr(Ts, n_sub, lo, offset, region)
    for f in range(F):
        assert rel(mse[f], mse_ref[f]) <= REL_TOL, (f, mse[f], mse_ref[f])   # P-5
    return res, flips, exempt


@pytest.mark.parametrize("L", [256] + list(p9_lengths(64)))
def test_ospr_c1_all_lengths(L):
    """BASELINE configs[0] (64x64, N_SF = 8, L = 256) plus the P-9 lengths."""
    w = WORKLOADS["C1"]
    ospr_parity(target_for(w), w.n_sub, L)


@pytest.mark.parametrize("offset", [1, 777, (1 << 35) + 3])
def test_ospr_phase_offset(offset):
    ospr_parity(target_for(WORKLOADS["C1"]), 8, 1021, offset=offset)


def test_ospr_odd_subframes_multi_frame():
    """Odd N_SF leaves an unpaired sub-frame; frames continue the cursor."""
    n = 64
    Ts = [blobs_target(40 + f, n, 4, 4.0, 10.0, Region.upper_half(n)) for f in range(3)]
    ospr_parity(None, 5, 1021, offset=99, frames_T=Ts)


@pytest.mark.parametrize("n", [16, 32, 128, 256, 512])
def test_ospr_sizes(n):
    T = blobs_target(7, n, 4, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n))
    ospr_parity(T, 3, 10007)


def test_ospr_single_subframe_and_flat():
    T = target_for(WORKLOADS["C1"])
    ospr_parity(T, 1, 257)
    res, _, _ = ospr_parity(T, 4, 0)           # flat: all sub-frames identical
    b = to_np(res.bits)[0]
    assert all(np.array_equal(b[0], b[s]) for s in range(4))


@pytest.mark.parametrize("n", [1024, 2048])
def test_ospr_single_subframe_fused_a7(n):
    """N_SF = 1 at the sizes with a7 fused into pass C: one unpaired sub-frame (h'_b = 0), the
    mirrored row-pair epilogue and its ticket on a single pair (P-3/P-4/P-5)."""
    T = blobs_target(21 + n, n, 16, n / 16, n / 6.4, Region.upper_half(n))
    ospr_parity(T, 1, 10007, offset=31)


def test_ospr_shards_reproduce_single_call():
    """P-8 on one GPU: shard ranges with global draw indices give bit-identical
    holograms, and finalize(sum of partial sums) matches the single call."""
    n, S = 64, 7
    T = target_for(WORKLOADS["C1"])
    tg = cuda_target(T)
    lut = hb.lut_generate(LUT_SEED, 1021)
    full = hb.ospr_generate(tg, S, lut, phase_offset=5)
    parts = [(0, 3), (3, 4), (4, 7)]
    acc = torch.zeros_like(full.intensity)
    for b, e in parts:
        r = hb.ospr_generate(tg, S, lut, phase_offset=5, sf_range=(b, e))
        assert r.mse is None
        assert torch.equal(r.bits, full.bits[:, b:e])
        acc += r.intensity
    mean, mse = hb.ospr_finalize(tg, acc, S)
    d = (mean - full.intensity).abs().max().item() / full.intensity.abs().max().item()
    assert d <= 1e-6
    assert rel(mse.item(), full.mse.item()) <= 1e-5


@pytest.mark.parametrize("chunk_pairs", [0, 2])
def test_ospr_fused_a7_shards_chunks_frames(monkeypatch, chunk_pairs):
    """The fused pass C + a7 of N >= 1024 in every mode it has: whole range with MSE, shards
    (partial sums, no MSE, odd boundaries), several frames per call (the ticket re-armed by each
    frame's pass A) and, with 2-pair chunks, the accumulator carried into the last chunk.  The
    shards' finalize(sum) must match the single call (P-8), and frame f must equal a single-frame
    call at cursor f N_SF N^2 (R-2), bit for bit."""
    if chunk_pairs:
        monkeypatch.setenv("HOLO_OSPR_CHUNK_BYTES", str(chunk_pairs * 1024 * 1024 * 8))
    n, S, off = 1024, 7, 321
    Ts = np.stack([blobs_target(80 + f, n, 16, 64.0, 160.0, Region.upper_half(n)) for f in range(2)])
    tg = cuda_target(Ts)
    lut = hb.lut_generate(LUT_SEED, 10007)
    full = hb.ospr_generate(tg, S, lut, phase_offset=off)
    for f in range(2):
        one = hb.ospr_generate(cuda_target(Ts[f]), S, lut, phase_offset=off + f * S * n * n)
        assert torch.equal(one.bits[0], full.bits[f]) and torch.equal(one.intensity[0], full.intensity[f])
        assert torch.equal(one.mse[0], full.mse[f])
    acc = torch.zeros_like(full.intensity)
    for b, e in [(0, 3), (3, 4), (4, 7)]:
        r = hb.ospr_generate(tg, S, lut, phase_offset=off, sf_range=(b, e))
        assert r.mse is None
        assert torch.equal(r.bits, full.bits[:, b:e])
        acc += r.intensity
    mean, mse = hb.ospr_finalize(tg, acc, S)
    d = (mean - full.intensity).abs().max().item() / full.intensity.abs().max().item()
    assert d <= 1e-6
    for f in range(2):
        assert rel(mse[f].item(), full.mse[f].item()) <= 1e-5
    # and the whole-range result against the oracle (frame 1, two sub-frames' bits, the MSE)
    lo = oracle.lut_build(LUT_SEED, 10007)
    bits = to_np(full.bits)
    for s_ in (0, 6):
        _, h_re, _ = oracle.ospr_subframe(Ts[1], lo, off + (S + s_) * n * n, want_h=True, want_intensity=False)
        check_bits(bits[1, s_], h_re, n)
    check_intensity(to_np(full.intensity)[1], oracle.replay_from_bits(bits[1], n))


def test_ospr_deterministic():
    T = cuda_target(target_for(WORKLOADS["C1"]))
    lut = hb.lut_generate(LUT_SEED, 257)
    a = hb.ospr_generate(T, 8, lut)
    b = hb.ospr_generate(T, 8, lut)
    assert torch.equal(a.bits, b.bits) and torch.equal(a.intensity, b.intensity) and torch.equal(a.mse, b.mse)


def test_ospr_properties():
    """Energy (Parseval, sum I = N^2), conjugate symmetry and the DC closed form on the
    GPU output alone."""
    n, S = 128, 6
    T = blobs_target(3, n, 8, 4.0, 12.0, Region.upper_half(n))
    res = hb.ospr_generate(cuda_target(T), S, hb.lut_generate(LUT_SEED, 10007))
    I = to_np(res.intensity)[0].astype(np.float64)
    assert abs(I.sum() - n * n) <= 1e-5 * n * n
    mirror = np.roll(np.flip(I, (0, 1)), 1, axis=(0, 1))
    assert np.max(np.abs(I - mirror)) <= 1e-6 * I.max()
    pops = unpack(to_np(res.bits)[0], n).reshape(S, -1).sum(1).astype(np.float64)
    dc = np.mean((2 * pops - n * n) ** 2 / (n * n))
    assert abs(I[0, 0] - dc) <= 1e-5 * max(dc, 1.0)


# ---- BASELINE full-size configurations ------------------------------------------------------------------

@pytest.mark.parametrize("L", [1 << 16, 1024 * 1024 * 24])
def test_ospr_c3_full_parity(L):
    """BASELINE configs[2] at full size (1024^2, N_SF = 24) in the bench's launch
    configuration: every sub-frame's bits, conditional intensity and MSE."""
    w = WORKLOADS["C3"]
    _, flips, exempt = ospr_parity(target_for(w), w.n_sub, L)
    assert flips <= exempt


@pytest.mark.parametrize("L,offset,S", [(1021, 0, 5), (509, (1 << 33) + 12345, 5), (1023, 777, 5), (65537, 1 << 40, 5),
                                        (1021, 3, 1), (1021, 3, 2)])   # one unpaired sub-frame; one pair
def test_ospr_1024_non_degenerate_lengths(L, offset, S):
    """Non-degenerate pool lengths at 1024^2 (L does not divide N^2, so every sub-frame draws
    different phases), in the index modes the BASELINE lengths never reach at this size:
    Lemire fast-mod below N (1021, 509, 1023) and a single wrap above it (65537), with
    cursors beyond 2^32: every sub-frame's bits, conditional intensity and MSE."""
    T = target_for(WORKLOADS["C3"])
    _, flips, exempt = ospr_parity(T, S, L, offset=offset)
    assert flips <= exempt


@pytest.mark.parametrize("L", [1 << 8, 1 << 12, 1 << 20])
def test_ospr_c3_sampled_and_degenerate(L):
    """The other C3 lengths all divide N^2 (pin c3 #13), so every sub-frame draws the
    same phases and the oracle's sub-frames are identical: each GPU sub-frame is checked
    against the oracle's sub-frame 0 (the GPU computes the two sub-frames of a pair as
    Re and Im of one transform, so they may differ from each other inside the band);
    the MSE of the mean equals the oracle's single-sub-frame MSE."""
    w = WORKLOADS["C3"]
    T = target_for(w)
    lg, lo = lut_pair(LUT_SEED, L)
    res = hb.ospr_generate(cuda_target(T), w.n_sub, lg)
    bits = to_np(res.bits)[0]
    _, h_re, I1 = oracle.ospr_subframe(T, lo, 0, want_h=True, want_intensity=True)
    for s in range(w.n_sub):
        check_bits(bits[s], h_re, w.n)
    check_intensity(to_np(res.intensity)[0], oracle.replay_from_bits(bits, w.n))
    m_ref = oracle.mse_m1(I1, T, w.omega().as_tuple())
    assert rel(to_np(res.mse)[0], m_ref) <= REL_TOL


def test_ospr_c5_sampled():
    """BASELINE configs[4] shape (2048^2, N_SF = 32, L = 2^16), two frames.  L divides
    N^2 (pin c3 #13), so all oracle sub-frames of a frame are identical: all 32 GPU
    sub-frames of both frames (frame 1 starts at cursor N_SF N^2; the GPU computes each
    pair as the Re and Im parts of one transform) are checked against the oracle's, the
    intensity conditionally on all 32 GPU sub-frames, and each frame's MSE against the
    oracle's single-sub-frame MSE (equal by the degeneracy)."""
    w = WORKLOADS["C5"]
    Ts = np.stack([target_for(w, f) for f in range(2)])
    lg, lo = lut_pair(LUT_SEED, 1 << 16)
    res = hb.ospr_generate(cuda_target(Ts), w.n_sub, lg)
    bits, I, mse = to_np(res.bits), to_np(res.intensity), to_np(res.mse)
    n, P = w.n, w.n * w.n
    for f in range(2):
        _, h_re, I1 = oracle.ospr_subframe(Ts[f], lo, f * w.n_sub * P, want_h=True, want_intensity=True)
        for s in range(w.n_sub):
            check_bits(bits[f, s], h_re, n)
        assert rel(mse[f], oracle.mse_m1(I1, Ts[f], w.omega().as_tuple())) <= REL_TOL
        check_intensity(I[f], oracle.replay_from_bits(bits[f], n))


def test_ospr_2048_prime_lut_all_subframes():
    """N = 2048 (nibble-staged column tiles) with a prime LUT length, so every
    sub-frame draws different phases (no L | N^2 degeneracy) and an unpaired tail: all bits
    against the oracle (P-3), the intensity conditionally (P-4) and the MSE (P-5)."""
    n, S, L, off = 2048, 3, 10007, 987654321
    T = blobs_target(11, n, 16, n / 16, n / 6.4, Region.upper_half(n))
    lg, lo = lut_pair(LUT_SEED, L)
    om = Region.upper_half(n).as_tuple()
    res = hb.ospr_generate(cuda_target(T), S, lg, phase_offset=off, omega=om)
    bits, I = to_np(res.bits)[0], to_np(res.intensity)[0]
    for s in range(S):
        _, h_re, _ = oracle.ospr_subframe(T, lo, off + s * n * n, want_h=True, want_intensity=False)
        check_bits(bits[s], h_re, n)
    check_intensity(I, oracle.replay_from_bits(bits, n))
    _, _, mse_ref = oracle.ospr(T[None], S, lo, off, om)
    assert rel(to_np(res.mse)[0], mse_ref[0]) <= REL_TOL


@pytest.mark.parametrize("S,L,off,chunk_pairs", [(3, 10007, 987654321, 0), (4, 1 << 16, 0, 1)])
def test_ospr_4096_all_subframes(S, L, off, chunk_pairs, monkeypatch):
    """N = 4096, the top of the supported range (R-26: two-warp row passes, single-stage
    4-column tiles): every sub-frame's bits against the oracle (P-3), the intensity
    conditionally (P-4) and the MSE (P-5); a prime LUT with an unpaired tail, and a
    power-of-two LUT run one pair per chunk (accumulation across chunks)."""
    if chunk_pairs:
        monkeypatch.setenv("HOLO_OSPR_CHUNK_BYTES", str(chunk_pairs * 4096 * 4096 * 8))
    n = 4096
    T = blobs_target(12, n, 16, n / 16, n / 6.4, Region.upper_half(n))
    lg, lo = lut_pair(LUT_SEED, L)
    om = Region.upper_half(n).as_tuple()
    res = hb.ospr_generate(cuda_target(T), S, lg, phase_offset=off, omega=om)
    bits, I = to_np(res.bits)[0], to_np(res.intensity)[0]
    for s in range(S):
        _, h_re, _ = oracle.ospr_subframe(T, lo, off + s * n * n, want_h=True, want_intensity=False)
        check_bits(bits[s], h_re, n)
    check_intensity(I, oracle.replay_from_bits(bits, n))
    _, _, mse_ref = oracle.ospr(T[None], S, lo, off, om)
    assert rel(to_np(res.mse)[0], mse_ref[0]) <= REL_TOL


def test_ospr_chunked_equals_single_chunk(monkeypatch):
    """Several chunks of pairs (a ragged last one, the odd unpaired tail, accumulation
    across chunks) give the same holograms as one chunk, and the same intensity up to
    fp32 summation order; the plan query reports the chunk size used."""
    n, S = 256, 11
    T = cuda_target(blobs_target(4, n, 6, 4.0, 10.0, Region.upper_half(n)))
    lut = hb.lut_generate(LUT_SEED, 10007)
    one = hb.ospr_generate(T, S, lut, phase_offset=77)
    assert hb.ospr_chunk_pairs(n, S) == (S + 1) // 2
    monkeypatch.setenv("HOLO_OSPR_CHUNK_BYTES", str(2 * n * n * 8))       # 2 pairs per chunk
    assert hb.ospr_chunk_pairs(n, S) == 2
    many = hb.ospr_generate(T, S, lut, phase_offset=77)
    assert torch.equal(one.bits, many.bits)
    d = (one.intensity - many.intensity).abs().max().item() / one.intensity.abs().max().item()
    assert d <= 1e-6
    assert rel(one.mse.item(), many.mse.item()) <= 1e-6


def test_ospr_graph_replay_bit_identical():
    """The step captured into a CUDA graph (as bench.py times it) replays to exactly the
    eager result."""
    n, S = 128, 6
    T = cuda_target(blobs_target(5, n, 6, 4.0, 10.0, Region.upper_half(n)))
    lut = hb.lut_generate(LUT_SEED, 4099)
    ws = torch.empty(hb.ospr_workspace_bytes(n, 1, S), dtype=torch.uint8, device="cuda")
    eager = hb.ospr_generate(T, S, lut, workspace=ws)
    out = hb.OsprResult(bits=torch.empty_like(eager.bits), intensity=torch.empty_like(eager.intensity),
                        mse=torch.empty_like(eager.mse))
    hb.ospr_generate(T, S, lut, workspace=ws, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        hb.ospr_generate(T, S, lut, workspace=ws, out=out)
    out.bits.zero_()
    out.intensity.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.bits, eager.bits) and torch.equal(out.intensity, eager.intensity)
    assert torch.equal(out.mse, eager.mse)


@pytest.mark.parametrize("n,S,offset", [(64, 8, 0), (128, 5, 12345), (256, 6, (1 << 33) + 7), (2048, 3, 5),
                                        (4096, 3, 0)])
def test_ospr_prng_source_equals_full_length_lut(n, S, offset):
    """phases drawn on the fly (SplitMix64 + R-5 in pass A) give
    bit-identical holograms, intensity and MSE to a pool from the same seed that is longer
    than every draw index -- here the pool covers [0, offset + S N^2)."""
    T = cuda_target(blobs_target(7, n, 6, 4.0, 10.0, Region.upper_half(n)))
    seed = 2004
    ref = None
    if offset + S * n * n < (1 << 31):
        ref = hb.ospr_generate(T, S, hb.lut_generate(seed, offset + S * n * n), phase_offset=offset)
    got = hb.ospr_generate(T, S, prng_seed=seed, phase_offset=offset)
    if ref is not None:
        assert torch.equal(got.bits, ref.bits) and torch.equal(got.intensity, ref.intensity)
        assert torch.equal(got.mse, ref.mse)
    else:
        # beyond any pool: the oracle's own PRNG source (apply_phase_prng) + fp64 IDFT, P-3 band
        Tn = to_np(T)
        bits = to_np(got.bits)[0]
        for s in range(S):
            h_re = oracle.fft2(oracle.apply_phase_prng(Tn, seed, offset + s * n * n), True).real
            check_bits(bits[s], h_re, n)


def test_ospr_prng_c3_matches_full_length_pool():
    """C3 size, full N_SF = 24: on-the-fly phases == the 25,165,824-entry pool (BASELINE
    configs[2]'s full-frame PRNG baseline)."""
    w = WORKLOADS["C3"]
    T = cuda_target(target_for(w))
    lut = hb.lut_generate(LUT_SEED, w.n * w.n * w.n_sub)
    ref = hb.ospr_generate(T, w.n_sub, lut)
    got = hb.ospr_generate(T, w.n_sub, prng_seed=LUT_SEED)
    assert torch.equal(got.bits, ref.bits) and torch.equal(got.intensity, ref.intensity)
    assert torch.equal(got.mse, ref.mse)


def test_f1_lut_sweep_shape_and_oracle_point():
    """SURVEY.md §8(f) f1 at a small scale: the GPU Monte-Carlo LUT sweep (tools/lut_sweep.py)
    shows the paper's qualitative results: error highest at N_LUT = 0, the
    resolution spike at N_LUT = N above N + 1, and at 64x64 a prime LUT of 10007 within 5 %
    of independent phases ("less than 5% additional error"; SURVEY probe A.7 reproduces
    it at 64^2).  One entry is re-derived by the fp64 oracle."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "lut_sweep", os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools", "lut_sweep.py"))
    ls = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ls)
    n, runs = 64, 6
    keys, mse, _ = ls.run(n, runs, lmax=12000)
    nm = mse.mean(axis=(1, 2))
    at = {k: nm[j] for j, k in enumerate(keys)}
    assert at[("lut", 0)] > 3 * at[("lut", 10007)]
    assert at[("lut", n)] > at[("lut", n + 1)]
    assert abs(at[("lut", 10007)] / at[("prng", -1)] - 1.0) < 0.05
    # oracle: run 0 of L = 13, all six targets as frames, phase offset 0
    T = ls.targets(n)
    j = keys.index(("lut", 13))
    _, _, mse_ref = oracle.ospr(T, ls.N_SF, oracle.lut_build(7000, 13), 0, Region.upper_half(n).as_tuple())
    assert np.all(np.abs(mse[j, 0] - mse_ref) <= 1e-4 * np.abs(mse_ref))


@pytest.mark.parametrize("n", [1024, 2048])
def test_ospr_repeat_bit_identical_multichunk(n, monkeypatch):
    """Repeated calls are bit-identical at the large sizes too, with several chunks (the pass-C
    accumulator round trip and its TMA slot refills): guards the cross-proxy WAR ordering of
    the single-slot row pipeline (a missing proxy fence made N = 2048 intensities vary)."""
    monkeypatch.setenv("HOLO_OSPR_CHUNK_BYTES", str(2 * n * n * 8))      # 2 pairs per chunk
    T = cuda_target(blobs_target(11, n, 8, n / 16, n / 6, Region.upper_half(n)))
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    runs = [hb.ospr_generate(T, 7, lut) for _ in range(3)]
    for r in runs[1:]:
        assert torch.equal(r.bits, runs[0].bits) and torch.equal(r.intensity, runs[0].intensity)
        assert torch.equal(r.mse, runs[0].mse)


def test_grouped_column_pipeline_equals_plain():
    """N = 2048 runs the column pass on the grouped pipeline (two consumer groups share one
    TMA ring).  With the same transform code it must reproduce the plain
    pipeline (HOLO_COL_G1=1, one group) bit for bit: holograms, intensity and MSE.  The plain
    run happens in a subprocess because the variant is chosen once per process."""
    import os
    import subprocess
    import sys
    import tempfile
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2004_04049_b200 as hb
from holo_synth import LUT_SEED, Region, blobs_target
n, S = 2048, 5
T = torch.from_numpy(blobs_target(21, n, 16, 128.0, 320.0, Region.upper_half(n))).cuda()
lut = hb.lut_generate(LUT_SEED, 10007)
r = hb.ospr_generate(T, S, lut, phase_offset=77)
torch.cuda.synchronize()
np.savez(sys.argv[1], bits=r.bits.cpu().numpy(), inten=r.intensity.cpu().numpy(), mse=r.mse.cpu().numpy())
""" % ROOT
    out = []
    with tempfile.TemporaryDirectory() as d:
        for plain in (False, True):
            env = dict(os.environ)
            env.pop("HOLO_COL_G1", None)
            if plain:
                env["HOLO_COL_G1"] = "1"
            f = os.path.join(d, f"r{int(plain)}.npz")
            subprocess.run([sys.executable, "-c", code, f], check=True, env=env, timeout=300)
            out.append(np.load(f))
    g, p = out
    assert np.array_equal(g["bits"], p["bits"])
    assert np.array_equal(g["inten"], p["inten"])
    assert np.array_equal(g["mse"], p["mse"])


def test_binding_rejects_mismatched_outputs():
    """The ABI writes through raw device pointers, so the binding checks caller-supplied
    outputs and workspaces (dtype, shape, device) before the call."""
    n, S = 64, 4
    T = cuda_target(blobs_target(3, n, 4, 4.0, 10.0, Region.upper_half(n)))
    lut = hb.lut_generate(LUT_SEED, 256)
    good = hb.ospr_generate(T, S, lut)
    bad_bits = hb.OsprResult(bits=torch.empty((1, S, n, n // 16), dtype=torch.uint8, device=T.device),
                             intensity=good.intensity, mse=good.mse)
    with pytest.raises(ValueError):
        hb.ospr_generate(T, S, lut, out=bad_bits)
    bad_int = hb.OsprResult(bits=good.bits, intensity=torch.empty((1, n, n), dtype=torch.float64, device=T.device),
                            mse=good.mse)
    with pytest.raises(TypeError):
        hb.ospr_generate(T, S, lut, out=bad_int)
    with pytest.raises(TypeError):
        hb.ospr_generate(T, S, lut, workspace=torch.empty(1 << 24, dtype=torch.float32, device=T.device))
    with pytest.raises(ValueError):
        hb.gs_generate(T, 2, lut, out=hb.GsResult(holo=None, levels=None, intensity=None,
                                                   mse=torch.empty((1, 3), dtype=torch.float64, device=T.device),
                                                   err_e=None))
    with pytest.raises(ValueError):
        hb.lut_generate(LUT_SEED, 256, out=torch.empty(128, dtype=torch.complex64, device=T.device))
    with pytest.raises(ValueError):
        hb.fft2(torch.zeros((1, n, n), dtype=torch.complex64, device=T.device),
                out=torch.empty((1, n, n // 2), dtype=torch.complex64, device=T.device))
