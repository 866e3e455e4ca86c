"""Python binding of libholo with the C ABI's names (include/holo.h).

Argument marshalling only: tensors are passed by ``data_ptr()`` together with
the current CUDA stream; every step of the hot path runs in the library's
sm_100a kernels.  torch supplies device memory and streams, nothing else.

Conventions (see include/holo.h): targets are float32 CUDA tensors
[frames][N][N]; complex fields and the LUT are complex64 (interleaved fp32
re, im); OSPR holograms are packed bits uint8 [frames][sub-frames][N][N/8].
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import torch

from ._lib import HoloRegion, check, lib

__all__ = [
    "lut_generate", "phase_table", "ospr_workspace_bytes", "ospr_chunk_pairs", "gs_group_frames", "ospr_generate", "ospr_finalize",
    "ospr_finalize_rows", "ospr_mse_from_sums", "gs_workspace_bytes",
    "gs_generate", "gs_step", "fft2", "debug_randomise", "debug_ospr_pairs", "launch_count", "profile_enable", "profile_read",
    "kernel_names", "version", "default_omega", "OsprResult", "GsResult",
]


def version() -> str:
    return lib().holo_version().decode()


def _stream(dev: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _need_out(t: Optional[torch.Tensor], dtype: torch.dtype, shape: Tuple[int, ...], dev: torch.device,
              name: str) -> Optional[torch.Tensor]:
    """A caller-supplied output must match what the ABI will write through its raw pointer
    (dtype, exact shape, device, contiguity): the library cannot check a device buffer's size."""
    if t is None:
        return None
    _need(t, dtype, name)
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if t.device != dev:
        raise ValueError(f"{name} must be on {dev}, got {t.device}")
    return t


def _workspace(ws: Optional[torch.Tensor], need: int, dev: torch.device) -> torch.Tensor:
    if ws is None or ws.numel() < need:
        return torch.empty(need, dtype=torch.uint8, device=dev)
    _need(ws, torch.uint8, "workspace")
    if ws.device != dev:
        raise ValueError(f"workspace must be on {dev}, got {ws.device}")
    return ws


def default_omega(n: int, algo: str) -> Tuple[int, int, int, int]:
    """R-13: OSPR measures rows [1, N/2) x all columns; GS the full plane."""
    return (1, n // 2, 0, n) if algo == "ospr" else (0, n, 0, n)


def _region(om: Sequence[int]) -> HoloRegion:
    return HoloRegion(*[int(v) for v in om])


def _lut_args(lut: Optional[torch.Tensor]):
    if lut is None or lut.numel() == 0:
        return None, 0
    _need(lut, torch.complex64, "lut")
    return lut.data_ptr(), lut.numel()


# ---- a0 --------------------------------------------------------------------------------------

def lut_generate(seed: int, n_lut: int, device=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The phase pool: complex64 [n_lut] = (cos, sin) of 2 pi u_k / 2^32 (R-3..R-5)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty(n_lut, dtype=torch.complex64, device=dev)
    _need(out, torch.complex64, "out")
    if out.numel() != n_lut:
        raise ValueError(f"out must hold n_lut = {n_lut} entries, got {out.numel()}")
    check(lib().holo_lut_generate(seed & 0xFFFFFFFFFFFFFFFF, n_lut, out.data_ptr(), _stream(out.device)))
    return out


def phase_table(phase_bits: int, device=None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The sin/cos table of the quantised PRNG source (R-25): complex64 [2^phase_bits],
    entry k = (cos, sin)(2 pi k / 2^phase_bits) by recipe R-5."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    m = 1 << phase_bits
    if out is None:
        out = torch.empty(m, dtype=torch.complex64, device=dev)
    _need_out(out, torch.complex64, (m,), out.device, "out")
    check(lib().holo_phase_table(phase_bits, out.data_ptr(), _stream(out.device)))
    return out


# ---- OSPR --------------------------------------------------------------------------------------

@dataclass
class OsprResult:
    bits: Optional[torch.Tensor]        # uint8 [F][S][N][N/8] (S = shard size)
    intensity: torch.Tensor             # float32 [F][N][N] (mean, or partial sum for a shard)
    mse: Optional[torch.Tensor]         # float64 [F]


def ospr_workspace_bytes(n: int, n_frames: int, n_sub: int) -> int:
    return int(lib().holo_ospr_workspace_size(n, n_frames, n_sub))


def ospr_chunk_pairs(n: int, n_sub: int) -> int:
    """Sub-frame pairs per chunk of the OSPR plan (instrumentation)."""
    return int(lib().holo_ospr_chunk_pairs(n, n_sub))


def gs_group_frames(n: int, batch: int) -> int:
    """Frames per launch group of the GS plan (instrumentation)."""
    return int(lib().holo_gs_group_frames(n, batch))


def ospr_generate(target: torch.Tensor, n_sub: int, lut: Optional[torch.Tensor] = None, phase_offset: int = 0,
                  sf_range: Optional[Tuple[int, int]] = None, want_bits: bool = True, want_mse: bool = True,
                  omega: Optional[Sequence[int]] = None, workspace: Optional[torch.Tensor] = None,
                  out: Optional[OsprResult] = None, prng_seed: Optional[int] = None,
                  phase_bits: Optional[int] = None, table: Optional[torch.Tensor] = None) -> OsprResult:
    """OSPR over target [F][N][N] (or [N][N]); see holo_ospr_generate.  With prng_seed the
    phases are drawn on the fly (holo_ospr_generate_prng) and `lut` must be None; with
    prng_seed and phase_bits = q the draws index a 2^q sin/cos table instead of running the
    recipe (holo_ospr_generate_prng_table; `table` from phase_table(q), built if None)."""
    _need(target, torch.float32, "target")
    t3 = target if target.dim() == 3 else target.unsqueeze(0)
    F, n, _ = t3.shape
    b, e = sf_range if sf_range is not None else (0, n_sub)
    full = (b == 0 and e == n_sub)
    om = omega if omega is not None else default_omega(n, "ospr")
    dev = t3.device
    if out is None:
        out = OsprResult(
            bits=torch.empty((F, e - b, n, n // 8), dtype=torch.uint8, device=dev) if want_bits else None,
            intensity=torch.empty((F, n, n), dtype=torch.float32, device=dev),
            mse=torch.empty(F, dtype=torch.float64, device=dev) if (want_mse and full) else None)
    else:
        _need_out(out.bits, torch.uint8, (F, e - b, n, n // 8), dev, "out.bits")
        if out.intensity is None:
            raise ValueError("out.intensity is required")
        _need_out(out.intensity, torch.float32, (F, n, n), dev, "out.intensity")
        _need_out(out.mse, torch.float64, (F,), dev, "out.mse")
    workspace = _workspace(workspace, ospr_workspace_bytes(n, F, n_sub), dev)
    if prng_seed is not None and phase_bits is not None:
        if lut is not None:
            raise ValueError("pass either lut or prng_seed, not both")
        tbl = table if table is not None else phase_table(phase_bits, device=dev)
        _need_out(tbl, torch.complex64, (1 << phase_bits,), dev, "table")
        check(lib().holo_ospr_generate_prng_table(t3.data_ptr(), n, F, n_sub, prng_seed & 0xFFFFFFFFFFFFFFFF,
                                                  tbl.data_ptr(), phase_bits, phase_offset, b, e, _ptr(out.bits),
                                                  out.intensity.data_ptr(), _ptr(out.mse), _region(om),
                                                  workspace.data_ptr(), workspace.numel(), _stream(dev)))
        return out
    if prng_seed is not None:
        if lut is not None:
            raise ValueError("pass either lut or prng_seed, not both")
        check(lib().holo_ospr_generate_prng(t3.data_ptr(), n, F, n_sub, prng_seed & 0xFFFFFFFFFFFFFFFF, phase_offset,
                                            b, e, _ptr(out.bits), out.intensity.data_ptr(), _ptr(out.mse),
                                            _region(om), workspace.data_ptr(), workspace.numel(), _stream(dev)))
        return out
    lp, L = _lut_args(lut)
    check(lib().holo_ospr_generate(t3.data_ptr(), n, F, n_sub, lp, L, phase_offset, b, e, _ptr(out.bits),
                                   out.intensity.data_ptr(), _ptr(out.mse), _region(om), workspace.data_ptr(),
                                   workspace.numel(), _stream(dev)))
    return out


def ospr_finalize(target: torch.Tensor, intensity_sum: torch.Tensor, n_sub: int,
                  omega: Optional[Sequence[int]] = None, want_mse: bool = True,
                  out: Optional[torch.Tensor] = None, mse_out: Optional[torch.Tensor] = None,
                  workspace: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, Optional[torch.Tensor]]:
    """Mean intensity (= sum / n_sub; in place if out is intensity_sum) and MSE.  Passing
    mse_out and workspace makes the call allocation-free (CUDA-graph capturable)."""
    _need(target, torch.float32, "target")
    _need(intensity_sum, torch.float32, "intensity_sum")
    t3 = target if target.dim() == 3 else target.unsqueeze(0)
    F, n, _ = t3.shape
    om = omega if omega is not None else default_omega(n, "ospr")
    _need_out(intensity_sum, torch.float32, (F, n, n), t3.device, "intensity_sum")
    out = torch.empty_like(intensity_sum) if out is None else _need_out(out, torch.float32, (F, n, n), t3.device, "out")
    mse = (_need_out(mse_out, torch.float64, (F,), t3.device, "mse_out") if mse_out is not None
           else torch.empty(F, dtype=torch.float64, device=t3.device)) if want_mse else None
    ws = _workspace(workspace, int(lib().holo_ospr_finalize_workspace_size()), t3.device)
    check(lib().holo_ospr_finalize(t3.data_ptr(), intensity_sum.data_ptr(), n, F, n_sub, _region(om),
                                   out.data_ptr(), _ptr(mse), ws.data_ptr(), ws.numel(), _stream(t3.device)))
    return out, mse


def ospr_finalize_rows(target: torch.Tensor, intensity_sum_rows: torch.Tensor, row0: int, n_sub: int,
                       omega: Optional[Sequence[int]] = None, out: Optional[torch.Tensor] = None,
                       sums_out: Optional[torch.Tensor] = None,
                       workspace: Optional[torch.Tensor] = None) -> Tuple[torch.Tensor, torch.Tensor]:
    """Step a7 on rows [row0, row0 + rows) of one frame (the slice a rank owns after the
    reduce-scatter C-1): the mean (in place if out is intensity_sum_rows) and the five fp64
    partial sums of R-12 over omega within the slice, to be all-reduced (C-2) before
    ospr_mse_from_sums.  target: the whole frame [N][N]; intensity_sum_rows: [rows][N]."""
    _need(target, torch.float32, "target")
    _need(intensity_sum_rows, torch.float32, "intensity_sum_rows")
    n = target.shape[-1]
    t2 = target.reshape(n, n) if target.numel() == n * n else None
    if t2 is None:
        raise ValueError("target must be one [N][N] frame")
    rows = intensity_sum_rows.numel() // n
    if intensity_sum_rows.numel() != rows * n or rows < 1:
        raise ValueError("intensity_sum_rows must hold whole rows of N")
    om = omega if omega is not None else default_omega(n, "ospr")
    dev = target.device
    out = torch.empty_like(intensity_sum_rows) if out is None else \
        _need_out(out, torch.float32, tuple(intensity_sum_rows.shape), dev, "out")
    sums = torch.empty(5, dtype=torch.float64, device=dev) if sums_out is None else \
        _need_out(sums_out, torch.float64, (5,), dev, "sums_out")
    ws = _workspace(workspace, int(lib().holo_ospr_finalize_workspace_size()), dev)
    check(lib().holo_ospr_finalize_rows(t2.data_ptr(), intensity_sum_rows.data_ptr(), n, row0, row0 + rows, n_sub,
                                        _region(om), out.data_ptr(), sums.data_ptr(), ws.data_ptr(), ws.numel(),
                                        _stream(dev)))
    return out, sums


def ospr_mse_from_sums(sums: torch.Tensor, omega: Sequence[int], out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """R-12 from reduced sums [F][5] (float64, device) -> mse [F]."""
    _need(sums, torch.float64, "sums")
    F = sums.numel() // 5
    if sums.numel() != 5 * F or F < 1:
        raise ValueError("sums must be [F][5]")
    out = torch.empty(F, dtype=torch.float64, device=sums.device) if out is None else \
        _need_out(out, torch.float64, (F,), sums.device, "out")
    check(lib().holo_ospr_mse_from_sums(sums.data_ptr(), F, _region(omega), out.data_ptr(), _stream(sums.device)))
    return out


# ---- GS ------------------------------------------------------------------------------------------

@dataclass
class GsResult:
    holo: Optional[torch.Tensor]        # complex64 [B][N][N]
    levels: Optional[torch.Tensor]      # uint8 [B][N][N]
    intensity: Optional[torch.Tensor]   # float32 [B][N][N]
    mse: Optional[torch.Tensor]         # float64 [B][iters]
    err_e: Optional[torch.Tensor]       # float64 [B][iters]


def gs_workspace_bytes(n: int, batch: int, iters: int) -> int:
    return int(lib().holo_gs_workspace_size(n, batch, iters))


def gs_generate(target: torch.Tensor, iters: int, lut: Optional[torch.Tensor] = None, phase_offset: int = 0,
                levels: int = 0, want_holo: bool = True, want_levels: bool = False, want_intensity: bool = True,
                want_mse: bool = True, want_err: bool = True, omega: Optional[Sequence[int]] = None,
                workspace: Optional[torch.Tensor] = None, out: Optional[GsResult] = None) -> GsResult:
    """GS over target [B][N][N] (or [N][N]); see holo_gs_generate."""
    _need(target, torch.float32, "target")
    t3 = target if target.dim() == 3 else target.unsqueeze(0)
    B, n, _ = t3.shape
    om = omega if omega is not None else default_omega(n, "gs")
    dev = t3.device
    if out is None:
        out = GsResult(
            holo=torch.empty((B, n, n), dtype=torch.complex64, device=dev) if want_holo else None,
            levels=torch.empty((B, n, n), dtype=torch.uint8, device=dev) if want_levels else None,
            intensity=torch.empty((B, n, n), dtype=torch.float32, device=dev) if want_intensity else None,
            mse=torch.empty((B, iters), dtype=torch.float64, device=dev) if want_mse else None,
            err_e=torch.empty((B, iters), dtype=torch.float64, device=dev) if want_err else None)
    else:
        _need_out(out.holo, torch.complex64, (B, n, n), dev, "out.holo")
        _need_out(out.levels, torch.uint8, (B, n, n), dev, "out.levels")
        _need_out(out.intensity, torch.float32, (B, n, n), dev, "out.intensity")
        _need_out(out.mse, torch.float64, (B, iters), dev, "out.mse")
        _need_out(out.err_e, torch.float64, (B, iters), dev, "out.err_e")
    workspace = _workspace(workspace, gs_workspace_bytes(n, B, iters), dev)
    lp, L = _lut_args(lut)
    check(lib().holo_gs_generate(t3.data_ptr(), n, B, iters, lp, L, phase_offset, levels, _ptr(out.holo),
                                 _ptr(out.levels), _ptr(out.intensity), _ptr(out.mse), _ptr(out.err_e),
                                 _region(om), workspace.data_ptr(), workspace.numel(), _stream(dev)))
    return out


def gs_step(r_in: torch.Tensor, target: torch.Tensor, levels: int = 0, omega: Optional[Sequence[int]] = None):
    """One GS iteration from R_{k-1} (complex64 [B][N][N]); returns (R_k, GsResult)."""
    _need(r_in, torch.complex64, "r_in")
    _need(target, torch.float32, "target")
    t3 = target if target.dim() == 3 else target.unsqueeze(0)
    r3 = r_in if r_in.dim() == 3 else r_in.unsqueeze(0)
    B, n, _ = t3.shape
    om = omega if omega is not None else default_omega(n, "gs")
    dev = t3.device
    r_out = torch.empty_like(r3)
    res = GsResult(holo=torch.empty_like(r3),
                   levels=torch.empty((B, n, n), dtype=torch.uint8, device=dev) if 2 <= levels <= 256 else None,
                   intensity=torch.empty((B, n, n), dtype=torch.float32, device=dev),
                   mse=torch.empty((B, 1), dtype=torch.float64, device=dev),
                   err_e=torch.empty((B, 1), dtype=torch.float64, device=dev))
    need = gs_workspace_bytes(n, B, 1)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    check(lib().holo_gs_step(r3.data_ptr(), t3.data_ptr(), n, B, levels, r_out.data_ptr(), res.holo.data_ptr(),
                             _ptr(res.levels), res.intensity.data_ptr(), res.mse.data_ptr(), res.err_e.data_ptr(),
                             _region(om), ws.data_ptr(), ws.numel(), _stream(dev)))
    return r_out, res


# ---- hooks -------------------------------------------------------------------------------------------

def fft2(x: torch.Tensor, inverse: bool = False, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Unitary 2D DFT (Eq. (1)) or IDFT (Eq. (2)) of complex64 [B][N][N] / [N][N]."""
    _need(x, torch.complex64, "x")
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    B, n, _ = x3.shape
    out = torch.empty_like(x3) if out is None else _need_out(out, torch.complex64, tuple(x3.shape), x3.device, "out")
    check(lib().holo_fft2(x3.data_ptr(), out.data_ptr(), n, B, int(inverse), _stream(x3.device)))
    return out if x.dim() == 3 else out[0]


def debug_randomise(target: torch.Tensor, lut: Optional[torch.Tensor], offset: int) -> torch.Tensor:
    """Step a2 alone: R = T * lut[(offset + p) mod N_LUT] (flat if lut is None)."""
    _need(target, torch.float32, "target")
    n = target.shape[-1]
    out = torch.empty((n, n), dtype=torch.complex64, device=target.device)
    lp, L = _lut_args(lut)
    check(lib().holo_debug_randomise(target.data_ptr(), n, lp, L, offset, out.data_ptr(), _stream(target.device)))
    return out


# ---- instrumentation -------------------------------------------------------------------------------------

def debug_ospr_pairs(target: torch.Tensor, n_sub: int, lut: Optional[torch.Tensor], offset: int = 0,
                     sf_range: Optional[Tuple[int, int]] = None, prng_seed: Optional[int] = None,
                     phase_bits: Optional[int] = None) -> torch.Tensor:
    """Test hook: pass A's randomisation (conj of the Hermitian-paired Z) for frame 0's
    sub-frame pairs in sf_range; complex64 [pairs][N][N].  prng_seed: the on-the-fly source;
    with phase_bits = q also the 2^q sin/cos table source."""
    _need(target, torch.float32, "target")
    n = target.shape[-1]
    b, e = sf_range if sf_range is not None else (0, n_sub)
    out = torch.empty(((e - b + 1) // 2, n, n), dtype=torch.complex64, device=target.device)
    lp, L = _lut_args(lut)
    use_prng = 0 if prng_seed is None else (1 if phase_bits is None else 2)
    if use_prng == 2:
        tbl = phase_table(phase_bits, device=target.device)
        lp, L = tbl.data_ptr(), phase_bits
    check(lib().holo_debug_ospr_pairs(target.data_ptr(), n, n_sub, lp, L, use_prng, prng_seed or 0, offset, b, e,
                                      out.data_ptr(),
                                      _stream(target.device)))
    return out


def launch_count() -> int:
    return int(lib().holo_launch_count())


def profile_enable(on: bool) -> None:
    check(lib().holo_profile_enable(int(on)))


def profile_read(name: str) -> Tuple[int, float]:
    n = C.c_uint64(0)
    ms = C.c_double(0.0)
    check(lib().holo_profile_read(name.encode(), C.byref(n), C.byref(ms)))
    return int(n.value), float(ms.value)


def kernel_names():
    return lib().holo_kernel_names().decode().split(",")
