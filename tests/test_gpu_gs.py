"""GPU parity of the GS path (steps g0-g6) against the fp64 oracle.

P-6 (continuous): per-iteration MSE along the whole trajectory, rel 1e-4.
P-7 (Q levels, chaotic under fp32 perturbation): one-step parity -- the oracle
runs iteration k from the GPU's own R_{k-1}; levels exact except near a
decision boundary or where |H| is tiny; MSE rel 1e-4; intensity conditional
on the GPU hologram.  gs_generate must be bit-identical to the chain of
gs_step calls it is made of.
"""
import numpy as np
import pytest
import torch

import oracle
from holo_synth import LUT_SEED, WORKLOADS, Region, blobs_target, target_for
from parity import REL_TOL, check_intensity, cuda_target, lut_pair, rel, to_np

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")


def level_band_ok(lev_gpu, lev_ref, H_ref, Q, step_band=1e-3, mag_band=1e-2):
    """Levels must agree except within step_band of a decision boundary, or where
    |H_ref| < mag_band * rms|H_ref| (phase ill-conditioned)."""
    th = np.mod(np.angle(H_ref), 2 * np.pi) * Q / (2 * np.pi) + 0.5
    near = np.abs(th - np.rint(th)) < step_band
    small = np.abs(H_ref) < mag_band * np.sqrt(np.mean(np.abs(H_ref) ** 2))
    bad = (lev_gpu != lev_ref) & ~near & ~small
    assert not bad.any(), f"{int(bad.sum())} level mismatches outside the band"
    return int((lev_gpu != lev_ref).sum())


def one_step_chain(T, iters, L, Q, offset=0):
    """Run gs_step on the GPU from the GPU's own state and compare each step with the
    oracle started from the same (GPU) R_{k-1}."""
    n = T.shape[0]
    lg, lo = lut_pair(LUT_SEED, L)
    tg = cuda_target(T)
    r = hb.debug_randomise(tg, lg, offset).unsqueeze(0)
    region = (0, n, 0, n)
    mses, Es = [], []
    for k in range(iters):
        r_prev = to_np(r[0]).astype(np.complex128)
        r, res = hb.gs_step(r, tg, levels=Q)
        ref = oracle.gs_step(r_prev, T, Q, region)
        if Q:
            H_ref = oracle.fft2(r_prev, inverse=True)
            level_band_ok(to_np(res.levels)[0], ref["levels"], H_ref, Q)
        else:
            H_ref = oracle.fft2(r_prev, inverse=True)
            ok = np.abs(H_ref) > 1e-3 * np.sqrt(np.mean(np.abs(H_ref) ** 2))
            assert np.max(np.abs(to_np(res.holo)[0][ok] - ref["holo"][ok])) <= 1e-3
        m = to_np(res.mse)[0, 0]
        assert rel(m, ref["mse"]) <= REL_TOL, (k, m, ref["mse"])
        I_cond = np.abs(oracle.fft2(to_np(res.holo)[0].astype(np.complex128))) ** 2
        check_intensity(to_np(res.intensity)[0], I_cond)
        mses.append(m)
        Es.append(to_np(res.err_e)[0, 0])
    return np.array(mses), np.array(Es), r


def test_gs_c2_one_step_parity_and_fused_equals_steps():
    """BASELINE configs[1]: 256x256, 20 iterations, LUT 4096, 256 levels."""
    w = WORKLOADS["C2"]
    T = target_for(w)
    mses, Es, r_last = one_step_chain(T, w.iters, 4096, w.levels)
    lg, lo = lut_pair(LUT_SEED, 4096)
    full = hb.gs_generate(cuda_target(T), w.iters, lg, levels=w.levels, want_levels=True)
    # the fused loop is the same arithmetic as the chain of steps: bit-identical
    assert np.array_equal(to_np(full.mse)[0], mses)
    assert np.array_equal(to_np(full.err_e)[0], Es)
    # whole-trajectory sanity vs the oracle (chaotic under fp32: 2% bound, SURVEY P-7)
    ref = oracle.gs(T, w.iters, lo, 0, w.levels, (0, w.n, 0, w.n))
    assert rel(to_np(full.mse)[0, -1], ref["mse"][-1]) <= 0.02
    # GS error reduction holds on the GPU trajectory (fp32 slack)
    assert np.all(Es[1:] <= Es[:-1] * (1 + 1e-5))


@pytest.mark.parametrize("Q", [0, 2, 16])
def test_gs_one_step_other_levels(Q):
    n = 64
    T = blobs_target(5, n, 4, 4.0, 10.0, Region.full(n))
    one_step_chain(T, 6, 1021, Q, offset=31)


def test_gs_continuous_trajectory_parity():
    """P-6: continuous phase-only GS is not chaotic; the whole trajectory's MSE matches."""
    n, B, iters = 256, 3, 20
    Ts = np.stack([blobs_target(1000 + b, n, 16, 16.0, 40.0, Region.full(n)) for b in range(B)])
    lg, lo = lut_pair(LUT_SEED, 1 << 16)
    res = hb.gs_generate(cuda_target(Ts), iters, lg, phase_offset=3, levels=0)
    mse, E, I = to_np(res.mse), to_np(res.err_e), to_np(res.intensity)
    for b in range(B):
        ref = oracle.gs(Ts[b], iters, lo, 3 + b * n * n, 0, (0, n, 0, n))
        for k in range(iters):
            assert rel(mse[b, k], ref["mse"][k]) <= REL_TOL, (b, k)
        assert np.all(E[b, 1:] <= E[b, :-1] * (1 + 1e-5))
        assert abs(I[b].astype(np.float64).sum() - n * n) <= 1e-4 * n * n
        assert np.max(np.abs(np.abs(to_np(res.holo)[b]) - 1)) <= 1e-5


@pytest.mark.parametrize("Q", [0, 16])
def test_gs_partial_region_metrics(Q):
    """R-12 over a region that is not the full plane: the metric prior a0 = sum T^2 / |Omega|
    is then not R-12's a, and the correction terms (a - a0) S_dI, (a - a0)^2 S_II carry the
    difference (gs_frame_metrics).  One-step MSE against the oracle, and the fused loop equals
    the step chain bit for bit, with an odd-shaped Omega."""
    n = 128
    region = (3, 101, 7, 122)
    T = blobs_target(77, n, 6, 6.0, 14.0, Region.full(n))
    lg, lo = lut_pair(LUT_SEED, 1021)
    tg = cuda_target(T)
    full = hb.gs_generate(tg, 4, lg, phase_offset=5, levels=Q, omega=region)
    r = hb.debug_randomise(tg, lg, 5).unsqueeze(0)
    for k in range(4):
        r_prev = to_np(r[0]).astype(np.complex128)
        r, st = hb.gs_step(r, tg, levels=Q, omega=region)
        one = oracle.gs_step(r_prev, T, Q, region)
        assert rel(to_np(st.mse)[0, 0], one["mse"]) <= REL_TOL, (Q, k)
        assert to_np(st.mse)[0, 0] == to_np(full.mse)[0, k]
    ref = oracle.gs(T, 1, lo, 5, Q, region)
    assert rel(to_np(full.mse)[0, 0], ref["mse"][0]) <= REL_TOL


def test_gs_levels_output_and_holo_consistent():
    n, Q = 64, 8
    T = blobs_target(9, n, 4, 4.0, 10.0, Region.full(n))
    res = hb.gs_generate(cuda_target(T), 3, hb.lut_generate(LUT_SEED, 97), levels=Q, want_levels=True)
    lev = to_np(res.levels)[0].astype(np.float64)
    h = to_np(res.holo)[0]
    assert np.max(np.abs(h - np.exp(2j * np.pi * lev / Q))) <= 1e-6
    assert lev.max() < Q


def test_gs_flat_and_deterministic():
    n = 64
    T = cuda_target(blobs_target(9, n, 4, 4.0, 10.0, Region.full(n)))
    a = hb.gs_generate(T, 4, None)
    b = hb.gs_generate(T, 4, None)
    assert torch.equal(a.mse, b.mse) and torch.equal(a.holo, b.holo)
    ref = oracle.gs(to_np(T), 4, None, 0, 0, (0, n, 0, n))
    assert rel(to_np(a.mse)[0, 0], ref["mse"][0]) <= REL_TOL


def test_gs_c4_full_size_trajectory():
    """BASELINE configs[3] at full size (1024^2, batch 64, 50 iterations, LUT 2^16,
    continuous) in the bench's launch configuration.  Every frame: energy and error
    reduction.  Frames 0, 31 and 63 (SURVEY.md §8(d) parity subset): P-6 -- the whole
    50-iteration MSE trajectory matches the oracle's within rel 1e-4 (north_star); the
    fused trajectory equals a chain of gs_step calls bit for bit; and at EVERY iteration
    the oracle's step from the GPU's own R_{k-1} matches (one-step, rel 1e-4).  Measured
    margins (profiles/r02_gs_drift.json): trajectory <= 5.0e-5, one-step <= 9e-8, against
    2.1e-4 for a plain numpy complex64 GS on the same inputs (R-22)."""
    from concurrent.futures import ThreadPoolExecutor
    w = WORKLOADS["C4"]
    Ts = np.stack([target_for(w, b) for b in range(w.frames)])
    lg, lo = lut_pair(LUT_SEED, 1 << 16)
    res = hb.gs_generate(cuda_target(Ts), w.iters, lg, levels=0, want_holo=False)
    mse, E, I = to_np(res.mse), to_np(res.err_e), to_np(res.intensity)
    P = w.n * w.n
    assert np.all(np.abs(I.reshape(w.frames, -1).astype(np.float64).sum(1) - P) <= 1e-4 * P)
    assert np.all(E[:, 1:] <= E[:, :-1] * (1 + 1e-5))
    region = (0, w.n, 0, w.n)
    with ThreadPoolExecutor(max_workers=16) as ex:
        for b in (0, 31, 63):
            tg = cuda_target(Ts[b])
            fut_ref = ex.submit(oracle.gs, Ts[b], w.iters, lo, b * P, 0, region)
            r = hb.debug_randomise(tg, lg, b * P).unsqueeze(0)
            steps = []
            for k in range(w.iters):
                r_prev = to_np(r[0]).astype(np.complex128)
                r, st = hb.gs_step(r, tg, levels=0)
                assert to_np(st.mse)[0, 0] == mse[b, k], (b, k)         # fused == chain of steps
                steps.append(ex.submit(oracle.gs_step, r_prev, Ts[b], 0, region))
            for k, f in enumerate(steps):
                assert rel(mse[b, k], f.result()["mse"]) <= REL_TOL, ("one-step", b, k)
            ref = fut_ref.result()
            for k in range(w.iters):
                assert rel(mse[b, k], ref["mse"][k]) <= REL_TOL, ("trajectory", b, k, rel(mse[b, k], ref["mse"][k]))


def test_gs_groups_bit_identical(monkeypatch):
    """Frames are independent: splitting the batch into launch groups (a ragged last
    group) changes no bit of any output; the plan query reports the group size."""
    n, B, iters = 128, 5, 4
    T = cuda_target(np.stack([blobs_target(100 + b, n, 4, 4.0, 10.0, Region.full(n)) for b in range(B)]))
    lut = hb.lut_generate(LUT_SEED, 4096)
    a = hb.gs_generate(T, iters, lut, levels=0)
    monkeypatch.setenv("HOLO_GS_GROUP_BYTES", str(2 * n * n * 8))        # 2 frames per group
    assert hb.gs_group_frames(n, B) == 2
    b = hb.gs_generate(T, iters, lut, levels=0)
    assert torch.equal(a.mse, b.mse) and torch.equal(a.holo, b.holo) and torch.equal(a.intensity, b.intensity)


@pytest.mark.parametrize("n", [512, 2048, 4096])
def test_gs_large_sizes_one_iteration(n):
    """GS at the sizes the fixed configurations skip (512: two-pass rows with E = 16 values;
    2048: the single-stage column pipeline and E = 64; 4096: two-warp row passes and
    4-column tiles, R-26): MSE and E_k against the oracle, continuous (three iterations, so
    iterations 1 and 2 go through the column pass's prologue reduction of the previous row
    pass's partials) and 8-level (first iteration: later ones may take fp32-vs-fp64 level
    decisions differently, R-22) constraints."""
    T = blobs_target(4242 + n, n, 8, n / 32, n / 8, Region.full(n))
    lg, lo = lut_pair(LUT_SEED, 4099)
    for Q, iters in ((0, 3), (8, 1)):
        res = hb.gs_generate(cuda_target(T[None]), iters, lg, phase_offset=77, levels=Q)
        ref = oracle.gs(T, iters, lo, 77, Q, (0, n, 0, n))
        for k in range(iters):
            assert rel(to_np(res.mse)[0, k], ref["mse"][k]) <= REL_TOL, (n, Q, k)
            assert rel(to_np(res.err_e)[0, k], ref["E"][k]) <= REL_TOL, (n, Q, k)
