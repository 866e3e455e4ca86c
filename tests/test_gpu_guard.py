"""Out-of-bounds and unwritten-output checks of every libholo entry point (compute-sanitizer is
not available on this GPU pool, so the checks are our own):

* every caller buffer the ABI writes through a raw pointer -- outputs and the workspace -- is a
  view into a larger allocation whose guard bands on both sides hold a sentinel; after the call
  the guards must be intact (no write outside the buffer);
* every output element must be written: float outputs are pre-filled with NaN and must come
  back finite; byte outputs are computed twice, pre-filled with 0x00 and with 0xFF, and must
  agree (a byte the kernels skip would keep its fill);
* sizes span the row-pass families (64, 256: several rows per warp; 1024, 2048: one row per
  warp; 2048: the grouped column pipeline), odd sub-frame counts, partial ranges and several
  chunks of pairs.
"""
import numpy as np
import pytest
import torch

from holo_synth import LUT_SEED, Region, blobs_target

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")

GUARD = 4096          # elements of guard band on each side


class Guarded:
    """A tensor of `shape` inside a larger allocation with guard bands filled with `fill`."""

    def __init__(self, shape, dtype, fill):
        numel = int(np.prod(shape))
        self.base = torch.empty(numel + 2 * GUARD, dtype=dtype, device="cuda")
        self.fill_value = fill
        self.base.fill_(fill)
        self.t = self.base[GUARD:GUARD + numel].view(shape)
        self.numel = numel

    def guards_intact(self):
        g = torch.cat([self.base[:GUARD], self.base[GUARD + self.numel:]])
        if g.is_complex():
            return bool(torch.isnan(torch.view_as_real(g)).all())
        if g.dtype.is_floating_point and np.isnan(self.fill_value):
            return bool(torch.isnan(g).all())
        return bool((g == self.fill_value).all())


def _target(n, F=1, seed=5):
    Ts = np.stack([blobs_target(seed + f, n, 6, n / 16, n / 6, Region.upper_half(n)) for f in range(F)])
    return torch.from_numpy(Ts).cuda()


def _ospr_once(T, S, lut, sf, bits_fill, ws_fill=0x5A, prng=False):
    F, n, _ = T.shape
    b, e = sf
    full = (b, e) == (0, S)
    bits = Guarded((F, e - b, n, n // 8), torch.uint8, bits_fill)
    inten = Guarded((F, n, n), torch.float32, float("nan"))
    mse = Guarded((F,), torch.float64, float("nan")) if full else None
    need = hb.ospr_workspace_bytes(n, F, S)
    ws = Guarded((need,), torch.uint8, ws_fill)
    out = hb.OsprResult(bits=bits.t, intensity=inten.t, mse=mse.t if mse else None)
    if prng:
        hb.ospr_generate(T, S, prng_seed=LUT_SEED, phase_offset=9, sf_range=sf, workspace=ws.t, out=out)
    else:
        hb.ospr_generate(T, S, lut, phase_offset=9, sf_range=sf, workspace=ws.t, out=out)
    torch.cuda.synchronize()
    for g in (bits, inten, ws) + ((mse,) if mse else ()):
        assert g.guards_intact(), "write outside a caller buffer"
    assert torch.isfinite(inten.t).all(), "unwritten intensity"
    if mse:
        assert torch.isfinite(mse.t).all(), "unwritten MSE"
    return bits.t.clone(), inten.t.clone()


@pytest.mark.parametrize("n,F,S,L,sf,chunk_pairs", [
    (64, 2, 5, 1021, None, None), (64, 1, 5, 0, (1, 4), None), (256, 2, 4, 4096, None, 1),
    (256, 1, 7, 257, (2, 7), None), (1024, 1, 5, 1 << 16, None, 2), (1024, 1, 3, 1021, (0, 2), None),
    (2048, 1, 3, 10007, None, None), (2048, 1, 4, 1 << 16, (2, 4), None), (4096, 1, 3, 10007, None, None)])
def test_ospr_outputs_guarded_and_complete(n, F, S, L, sf, chunk_pairs, monkeypatch):
    if chunk_pairs:
        monkeypatch.setenv("HOLO_OSPR_CHUNK_BYTES", str(chunk_pairs * n * n * 8))
    T = _target(n, F)
    lut = hb.lut_generate(LUT_SEED, L) if L else None
    sf = sf or (0, S)
    b0, i0 = _ospr_once(T, S, lut, sf, 0x00)
    b1, i1 = _ospr_once(T, S, lut, sf, 0xFF, ws_fill=0xA5)
    assert torch.equal(b0, b1), "unwritten hologram bytes (they kept their fill)"
    assert torch.equal(i0, i1)


@pytest.mark.parametrize("n", [256, 1024])
def test_ospr_prng_outputs_guarded_and_complete(n):
    T = _target(n)
    b0, i0 = _ospr_once(T, 5, None, (0, 5), 0x00, prng=True)
    b1, i1 = _ospr_once(T, 5, None, (0, 5), 0xFF, prng=True)
    assert torch.equal(b0, b1) and torch.equal(i0, i1)


@pytest.mark.parametrize("n", [64, 1024, 2048])
def test_finalize_paths_guarded(n):
    T = _target(n)
    S = 4
    part = hb.ospr_generate(T, S, hb.lut_generate(LUT_SEED, 1021), sf_range=(0, 2), want_mse=False)
    need = int(hb.lib().holo_ospr_finalize_workspace_size())
    ws = Guarded((need,), torch.uint8, 0x33)
    mean = Guarded((1, n, n), torch.float32, float("nan"))
    mse = Guarded((1,), torch.float64, float("nan"))
    hb.ospr_finalize(T, part.intensity, S, out=mean.t, mse_out=mse.t, workspace=ws.t)
    rows = Guarded((n // 4, n), torch.float32, float("nan"))
    sums = Guarded((5,), torch.float64, float("nan"))
    hb.ospr_finalize_rows(T[0], part.intensity[0, n // 4: n // 2].contiguous(), n // 4, S, out=rows.t,
                          sums_out=sums.t, workspace=ws.t)
    mse2 = Guarded((1,), torch.float64, float("nan"))
    hb.ospr_mse_from_sums(sums.t.view(1, 5), hb.default_omega(n, "ospr"), out=mse2.t)
    torch.cuda.synchronize()
    for g in (ws, mean, mse, rows, sums, mse2):
        assert g.guards_intact()
    for g in (mean, mse, rows, sums, mse2):
        assert torch.isfinite(g.t).all()


@pytest.mark.parametrize("n,B,levels", [(64, 3, 0), (256, 2, 16), (1024, 2, 0), (2048, 1, 8), (4096, 1, 8)])
def test_gs_outputs_guarded_and_complete(n, B, levels):
    T = torch.from_numpy(np.stack([blobs_target(30 + b, n, 6, n / 16, n / 6, Region.full(n))
                                   for b in range(B)])).cuda()
    lut = hb.lut_generate(LUT_SEED, 4099)
    iters = 3
    res = []
    for fill in (0x00, 0xFF):
        holo = Guarded((B, n, n), torch.complex64, complex("nan+nanj"))
        lev = Guarded((B, n, n), torch.uint8, fill) if levels else None
        inten = Guarded((B, n, n), torch.float32, float("nan"))
        mse = Guarded((B, iters), torch.float64, float("nan"))
        err = Guarded((B, iters), torch.float64, float("nan"))
        ws = Guarded((hb.gs_workspace_bytes(n, B, iters),), torch.uint8, fill ^ 0x5A)
        out = hb.GsResult(holo=holo.t, levels=lev.t if lev else None, intensity=inten.t, mse=mse.t, err_e=err.t)
        hb.gs_generate(T, iters, lut, phase_offset=3, levels=levels, workspace=ws.t, out=out)
        torch.cuda.synchronize()
        guards = (holo, inten, mse, err, ws) + ((lev,) if lev else ())
        assert all(g.guards_intact() for g in guards), "write outside a caller buffer"
        assert torch.isfinite(torch.view_as_real(holo.t)).all() and torch.isfinite(inten.t).all()
        assert torch.isfinite(mse.t).all() and torch.isfinite(err.t).all()
        res.append((lev.t.clone() if lev else None, mse.t.clone()))
    if levels:
        assert torch.equal(res[0][0], res[1][0]), "unwritten level bytes"
    assert torch.equal(res[0][1], res[1][1])


@pytest.mark.parametrize("n", [16, 128, 1024, 2048, 4096])
def test_fft2_and_lut_guarded(n):
    x = torch.randn(2, n, n, dtype=torch.complex64, device="cuda")
    for inv in (False, True):
        out = Guarded((2, n, n), torch.complex64, complex("nan+nanj"))
        hb.fft2(x, inverse=inv, out=out.t)
        torch.cuda.synchronize()
        assert out.guards_intact() and torch.isfinite(torch.view_as_real(out.t)).all()
    for L in (1, 5, 257, 65536):
        lut = Guarded((L,), torch.complex64, complex("nan+nanj"))
        hb.lut_generate(LUT_SEED, L, out=lut.t)
        torch.cuda.synchronize()
        assert lut.guards_intact() and torch.isfinite(torch.view_as_real(lut.t)).all()


def test_concurrent_streams_match_serial():
    """Two independent calls on two streams at once (each with its own workspace) give the
    results of the same calls made one after the other: no hidden shared state on the device
    (the twiddle pool is read-only; tickets and partial sums live in the caller's workspace)."""
    n, S = 1024, 6
    T1, T2 = _target(n, seed=11), _target(n, seed=12)
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    ref1 = hb.ospr_generate(T1, S, lut)
    ref2 = hb.gs_generate(T2, 4, lut)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for _ in range(3):
        with torch.cuda.stream(s1):
            a = hb.ospr_generate(T1, S, lut)
        with torch.cuda.stream(s2):
            b = hb.gs_generate(T2, 4, lut)
        torch.cuda.synchronize()
        outs.append((a, b))
    for a, b in outs:
        assert torch.equal(a.bits, ref1.bits) and torch.equal(a.intensity, ref1.intensity)
        assert torch.equal(a.mse, ref1.mse)
        assert torch.equal(b.mse, ref2.mse) and torch.equal(b.holo, ref2.holo)
