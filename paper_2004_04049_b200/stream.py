"""Pipelined OSPR frame stream: SURVEY.md §8(f) f3, the "packed-frame output stream for a binary
display at video rate" (the 1024x1024 ferroelectric SLM demonstration).

A display shows frame set f as N_SF binary sub-frames (Fig. 2 right); frame set f + 1 uses
the continuing phase cursor, off0 + (f + 1) N_SF N^2 (reading R-2).  The stream takes each
frame set's target amplitude from pinned host memory and returns its packed sub-frame holograms
(R-8 layout, [N_SF][N][N/8] bytes) and its MSE (R-12) to pinned host memory.  Three CUDA streams
overlap the steps of consecutive frame sets:

    h2d  : target f + 1  host -> device            (copy engine)
    comp : [a0,] ospr_generate of frame set f        (libholo kernels)
    d2h  : holograms + MSE of f - 1  device -> host  (copy engine)

with `depth` device slots for the per-frame buffers (targets and outputs) and one workspace (the
compute steps of consecutive frame sets run in order on `comp`).  Cross-stream order comes from
CUDA events only; the host never blocks in submit().  The sequencing is native
(holo_ospr_stream_*: one C call per frame set enqueues the copies, a0 when `lut_seed` is given,
and the passes); this module allocates the buffers.  A Python `before_each` hook (any work to
enqueue on the compute stream ahead of each frame set) selects an equivalent Python sequencer.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Optional, Sequence, Tuple

import torch

from . import api
from ._lib import check, lib
from .api import OsprResult, default_omega, ospr_workspace_bytes


class OsprStream:
    """Frame-set pipeline over one GPU.

    submit(target_host) enqueues frame set f (returns f); result(f) waits for its outputs and
    returns host views (bits [N_SF][N][N/8] uint8, mse float64 [1], intensity [N][N] float32 or
    None) that stay valid until frame set f + depth is submitted.  The caller keeps target_host
    unchanged until done(f) (or any later result) reports the frame set's copy complete.
    """

    def __init__(self, n: int, n_sub: int, lut: Optional[torch.Tensor] = None, *, depth: int = 3,
                 phase_offset: int = 0, advance: bool = True, frame_stride: int = 1,
                 omega: Optional[Sequence[int]] = None,
                 want_intensity: bool = False, before_each: Optional[Callable[[], None]] = None,
                 lut_seed: Optional[int] = None, device: Optional[torch.device] = None):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.n, self.n_sub, self.lut, self.depth = n, n_sub, lut, depth
        self.off0, self.advance, self.frame_stride = phase_offset, advance, frame_stride
        self.omega = tuple(omega) if omega is not None else default_omega(n, "ospr")
        self.before_each = before_each
        self.dev = dev
        self.h2d = torch.cuda.Stream(dev)
        self.comp = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ws = torch.empty(ospr_workspace_bytes(n, 1, n_sub), dtype=torch.uint8, device=dev)
        f32, u8, f64 = torch.float32, torch.uint8, torch.float64
        self.t_dev = [torch.empty((1, n, n), dtype=f32, device=dev) for _ in range(depth)]
        self.out = [OsprResult(bits=torch.empty((1, n_sub, n, n // 8), dtype=u8, device=dev),
                               intensity=torch.empty((1, n, n), dtype=f32, device=dev),
                               mse=torch.empty(1, dtype=f64, device=dev)) for _ in range(depth)]
        self.bits_host = [torch.empty((n_sub, n, n // 8), dtype=u8).pin_memory() for _ in range(depth)]
        self.mse_host = [torch.empty(1, dtype=f64).pin_memory() for _ in range(depth)]
        self.inten_host = [torch.empty((n, n), dtype=f32).pin_memory() for _ in range(depth)] \
            if want_intensity else None
        ev = lambda: [torch.cuda.Event() for _ in range(depth)]   # noqa: E731
        self.h2d_done, self.comp_done, self.d2h_done = ev(), ev(), ev()
        self.used = [False] * depth
        self.f = 0
        # per-submit host work kept small (the host must stay ahead of ~0.1 ms frame sets): views
        # and the holo_ospr_generate arguments are prepared once per slot; only the cursor varies
        self.t_view = [t[0] for t in self.t_dev]
        self.bits_view = [o.bits[0] for o in self.out]
        self.inten_view = [o.intensity[0] for o in self.out]
        lp, L = api._lut_args(lut)
        self._gen = lib().holo_ospr_generate
        self._args = [(t.data_ptr(), n, 1, n_sub, lp, L) for t in self.t_dev]
        self._tail = [(0, n_sub, o.bits.data_ptr(), o.intensity.data_ptr(), o.mse.data_ptr(), api._region(self.omega),
                       self.ws.data_ptr(), self.ws.numel(), self.comp.cuda_stream) for o in self.out]
        if lut_seed is not None and before_each is not None:
            raise ValueError("lut_seed (native a0) and before_each are exclusive")
        if lut_seed is not None and lut is None:
            raise ValueError("lut_seed needs the pool tensor `lut` to regenerate")
        self._native = None
        self._closed = False
        if before_each is None:          # the native sequencer (one C call per frame set)
            slots = []
            for d in range(depth):
                o = self.out[d]
                slots += [self.t_dev[d].data_ptr(), o.bits.data_ptr(), o.intensity.data_ptr(), o.mse.data_ptr(),
                          self.bits_host[d].data_ptr(), self.mse_host[d].data_ptr(),
                          self.inten_host[d].data_ptr() if self.inten_host is not None else 0]
            self._slots = (C.c_void_p * len(slots))(*[C.c_void_p(p) if p else None for p in slots])
            h = C.c_void_p()
            with torch.cuda.device(dev):
                check(lib().holo_ospr_stream_create(n, n_sub, depth, lp, L, 1 if lut_seed is not None else 0,
                                                    (lut_seed or 0) & 0xFFFFFFFFFFFFFFFF, phase_offset,
                                                    frame_stride, 1 if advance else 0, api._region(self.omega),
                                                    self._slots, self.ws.data_ptr(), self.ws.numel(), C.byref(h)))
            self._native = h
            self._frame = C.c_int64()
            hs = [C.c_void_p() for _ in range(3)]
            check(lib().holo_ospr_stream_handles(h, *[C.byref(x) for x in hs]))
            # the native streams, wrapped so that callers can record events on them (timing)
            self.h2d, self.comp, self.d2h = [torch.cuda.ExternalStream(x.value, device=dev) for x in hs]

    def frame_offset(self, f: int) -> int:
        """Phase cursor of this stream's frame set f: off0 + f * frame_stride * N_SF N^2 when
        advancing (R-2).  frame_stride = k with off0 = r N_SF N^2 gives stream r of k the global
        frame sets r, r + k, r + 2k, ... (one stream per GPU)."""
        return self.off0 + (f * self.frame_stride * self.n_sub * self.n * self.n if self.advance else 0)

    def submit(self, target_host: torch.Tensor) -> int:
        if target_host.dtype != torch.float32 or tuple(target_host.shape[-2:]) != (self.n, self.n):
            raise ValueError(f"target_host must be float32 [{self.n}][{self.n}]")
        if self._closed:
            raise RuntimeError("the stream is closed")
        if self._native is not None:
            if target_host.is_cuda or not target_host.is_contiguous():
                raise ValueError("target_host must be a contiguous host tensor")
            check(lib().holo_ospr_stream_submit(self._native, target_host.data_ptr(), C.byref(self._frame)))
            self.f = self._frame.value + 1
            return self._frame.value
        f = self.f
        s = f % self.depth
        if self.used[s]:
            # slot reuse: the previous frame set of this slot must have read its target (comp)
            # and shipped its outputs (d2h) before they are overwritten
            self.h2d.wait_event(self.comp_done[s])
            self.comp.wait_event(self.d2h_done[s])
        with torch.cuda.stream(self.h2d):
            self.t_view[s].copy_(target_host, non_blocking=True)
            self.h2d_done[s].record(self.h2d)
        self.comp.wait_event(self.h2d_done[s])
        if self.before_each is not None:
            with torch.cuda.stream(self.comp):
                self.before_each()
        check(self._gen(*self._args[s], self.frame_offset(f), *self._tail[s]))   # ospr_generate on comp
        self.comp_done[s].record(self.comp)
        self.d2h.wait_event(self.comp_done[s])
        with torch.cuda.stream(self.d2h):
            self.bits_host[s].copy_(self.bits_view[s], non_blocking=True)
            self.mse_host[s].copy_(self.out[s].mse, non_blocking=True)
            if self.inten_host is not None:
                self.inten_host[s].copy_(self.inten_view[s], non_blocking=True)
            self.d2h_done[s].record(self.d2h)
        self.used[s] = True
        self.f = f + 1
        return f

    def _slot(self, f: int) -> int:
        if self._closed:
            raise RuntimeError("the stream is closed")
        if not (self.f - self.depth <= f < self.f):
            raise ValueError(f"frame set {f} is not among the last {self.depth} submitted")
        return f % self.depth

    def done(self, f: int) -> bool:
        """True once frame set f's outputs are in host memory (its target copy is complete too)."""
        s = self._slot(f)
        if self._native is not None:
            r = lib().holo_ospr_stream_done(self._native, f)
            if r < 0:
                raise RuntimeError(lib().holo_last_error().decode())
            return r == 1
        return self.d2h_done[s].query()

    def result(self, f: int) -> Tuple[torch.Tensor, torch.Tensor, Optional[torch.Tensor]]:
        s = self._slot(f)
        if self._native is not None:
            check(lib().holo_ospr_stream_wait(self._native, f))
        else:
            self.d2h_done[s].synchronize()
        return self.bits_host[s], self.mse_host[s], (self.inten_host[s] if self.inten_host is not None else None)

    def drain(self) -> None:
        """Block until every submitted frame set is complete."""
        if self._closed:
            return
        if self._native is not None:
            check(lib().holo_ospr_stream_drain(self._native))
        else:
            self.d2h.synchronize()

    def close(self) -> None:
        """Drain and release the native sequencer's streams and events (also done on deletion)."""
        if getattr(self, "_native", None) is not None:
            lib().holo_ospr_stream_destroy(self._native)
            self._native = None
            self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
