"""Multi-GPU partitioning of the hot path.

One process per GPU (torch.distributed over NCCL).  The units of the method are
independent, so the partition is a plain shard of them:

* OSPR: the N_SF sub-frames of every frame are split into contiguous ranges
  of whole Hermitian pairs, one per rank (``subframe_range``).  Draw indices stay global (frame f, sub-frame s starts at
  phase_offset + (f N_SF + s) N^2), so every rank produces exactly the
  holograms the single-GPU call would.  The one real exchange step of the path
  is the time average: the per-rank partial intensity sums are added by
  a reduce-scatter (collective C-1; each rank owns N/world rows), step a7 runs
  on the owned rows, and only after an all-reduce of five doubles per frame
  (C-2) is the MSE computed (it is nonlinear in I).
* OSPR video (BASELINE configs[4], ``SubframeShardPipeline``): per frame, the
  sub-frame shards are finished by a reduce-scatter of the partial intensity
  (C-1: each rank owns N/world rows of the frame), step a7 on the owned rows
  (mean and the five fp64 sums of R-12, ``ospr_finalize_rows``), an all-reduce
  of the five sums (C-2, 40 bytes) and the MSE (``ospr_mse_from_sums``), all on
  a side stream, so that frame f's collectives overlap frame f+1's passes.
* GS: frames are independent replicas; frame b of the batch draws its initial
  phases from phase_offset + b N^2, so a rank owning frames [fb, fe) passes
  phase_offset + fb N^2.  No collective is needed on the data path; metrics can
  be gathered for reporting.

The compute and collective callables are injectable so that the host logic can
be exercised on CPU with the gloo backend (tests/test_parallel.py); the
defaults are the libholo binding and torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import torch

from . import api
from ._lib import check


def shard_range(n_units: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [begin, end) of n_units for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (n_units * rank) // world, (n_units * (rank + 1)) // world


def subframe_range(n_sub: int, world: int, rank: int) -> Tuple[int, int]:
    """The OSPR sub-frames [begin, end) of `rank`: whole Hermitian pairs (2s, 2s+1) are dealt
    out (shard_range over the ceil(n_sub/2) pairs), so every rank transforms exactly the pairs
    the single-GPU call does -- its holograms are bit-identical to that call's (P-8) -- and an
    odd n_sub leaves its unpaired tail on the last rank holding pairs, as the single call does.
    A rank's pass cost is its pair count, so this is never more unbalanced than splitting the
    sub-frames themselves (3 sub-frames cost 2 pair transforms, as 4 do)."""
    pb, pe = shard_range((n_sub + 1) // 2, world, rank)
    return min(2 * pb, n_sub), min(2 * pe, n_sub)


def _default_all_reduce(t: torch.Tensor) -> None:
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM)


def _default_reduce_scatter(out: torch.Tensor, inp: torch.Tensor) -> None:
    import torch.distributed as dist
    dist.reduce_scatter_tensor(out, inp, op=dist.ReduceOp.SUM)


@dataclass
class ShardedOsprResult:
    sf_range: Tuple[int, int]          # this rank's sub-frames
    bits: Optional[torch.Tensor]       # [F][sf_end - sf_begin][N][N/8] (this rank's holograms)
    intensity: torch.Tensor            # mean over ALL sub-frames of this rank's owned rows [F][rows][N]
    mse: Optional[torch.Tensor]        # [F] (every rank, after C-2)
    rows: Tuple[int, int]              # the owned rows [row0, row1) (world = 1: all of them)


class ShardedOspr:
    """OSPR with sub-frames sharded across `world` ranks.  The exchange is C-1, a reduce-scatter
    of the fp32 partial intensity sums (rank r owns rows [r N/world, (r+1) N/world) of every
    frame), then a7 on the owned rows (mean + five fp64 sums), C-2 (an all-reduce of the five
    sums per frame) and the MSE (nonlinear in I, so only after C-2)."""

    def __init__(self, world: int, rank: int,
                 generate: Callable = api.ospr_generate,
                 finalize_rows: Callable = api.ospr_finalize_rows,
                 mse_from_sums: Callable = api.ospr_mse_from_sums,
                 reduce_scatter: Callable = _default_reduce_scatter,
                 all_reduce: Callable[[torch.Tensor], None] = _default_all_reduce):
        self.world, self.rank = world, rank
        self.generate, self.finalize_rows, self.mse_from_sums = generate, finalize_rows, mse_from_sums
        self.reduce_scatter, self.all_reduce = reduce_scatter, all_reduce

    def rows(self, n: int) -> Tuple[int, int]:
        if n % self.world:
            raise ValueError(f"n = {n} must divide among {self.world} ranks (owned row slices)")
        return self.rank * n // self.world, (self.rank + 1) * n // self.world

    def exchange(self, target: torch.Tensor, part: torch.Tensor, n_sub: int, mean: torch.Tensor,
                 sums: torch.Tensor, mse: Optional[torch.Tensor], omega, fin_workspace=None) -> None:
        """C-1, a7 on the owned rows, C-2 and the MSE, into caller buffers: part [F][N][N] (the
        partial sums, consumed), mean [F][rows][N], sums [F][5] fp64, mse [F] or None."""
        t3 = target if target.dim() == 3 else target.unsqueeze(0)
        F, n, _ = t3.shape
        r0, _ = self.rows(n)
        omega = omega if omega is not None else api.default_omega(n, "ospr")
        for f in range(F):
            self.reduce_scatter(mean[f].reshape(-1), part[f].reshape(-1))                       # C-1
            self.finalize_rows(t3[f], mean[f], r0, n_sub, omega=omega, out=mean[f], sums_out=sums[f],
                               workspace=fin_workspace)                                          # a7
        self.all_reduce(sums)                                                                    # C-2
        if mse is not None:
            self.mse_from_sums(sums, omega, out=mse)

    def run(self, target: torch.Tensor, n_sub: int, lut: Optional[torch.Tensor], phase_offset: int = 0,
            want_bits: bool = True, want_mse: bool = True, omega=None, workspace=None) -> ShardedOsprResult:
        t3 = target if target.dim() == 3 else target.unsqueeze(0)
        F, n, _ = t3.shape
        om = omega if omega is not None else api.default_omega(n, "ospr")
        b, e = subframe_range(n_sub, self.world, self.rank)
        if self.world == 1:
            r = self.generate(target, n_sub, lut, phase_offset=phase_offset, want_bits=want_bits,
                              want_mse=want_mse, omega=om, workspace=workspace)
            return ShardedOsprResult((0, n_sub), r.bits, r.intensity, r.mse, (0, n))
        if b == e:                       # more ranks than sub-frames: a zero partial sum
            part_i, bits = torch.zeros_like(t3), None
        else:
            part = self.generate(target, n_sub, lut, phase_offset=phase_offset, sf_range=(b, e),
                                 want_bits=want_bits, want_mse=False, omega=om, workspace=workspace)
            part_i, bits = part.intensity, part.bits
        r0, r1 = self.rows(n)
        mean = torch.empty((F, r1 - r0, n), dtype=part_i.dtype, device=part_i.device)
        sums = torch.zeros((F, 5), dtype=torch.float64, device=part_i.device)
        mse = torch.empty(F, dtype=torch.float64, device=part_i.device) if want_mse else None
        self.exchange(target, part_i, n_sub, mean, sums, mse, om)
        return ShardedOsprResult((b, e), bits, mean, mse, (r0, r1))


class ShardedGs:
    """GS with frames sharded across ranks (no data-path collective)."""

    def __init__(self, world: int, rank: int, generate: Callable = api.gs_generate):
        self.world, self.rank, self.generate = world, rank, generate

    def frame_range(self, batch: int) -> Tuple[int, int]:
        return shard_range(batch, self.world, self.rank)

    def run(self, targets: torch.Tensor, iters: int, lut: Optional[torch.Tensor], phase_offset: int = 0,
            levels: int = 0, **kw):
        """targets: the FULL batch [B][N][N] (only this rank's frames are used)."""
        B, n, _ = targets.shape
        fb, fe = self.frame_range(B)
        if fb == fe:
            return (fb, fe), None
        res = self.generate(targets[fb:fe].contiguous(), iters, lut, phase_offset=phase_offset + fb * n * n,
                            levels=levels, **kw)
        return (fb, fe), res


class SubframeShardPipeline:
    """OSPR over a stream of video frames with each frame's n_sub sub-frames sharded across
    `world` ranks (BASELINE configs[4]).  Per frame f (slot f mod depth):

      compute stream: [before_each (e.g. a0)] + this rank's shard of the frame (a1-a6; draw
                      indices global: cursor phase_offset + f n_sub N^2) -> the partial
                      intensity sum and this shard's packed holograms;
      side stream:    C-1 reduce-scatter of the partial sums (rank r owns rows
                      [r N/world, (r+1) N/world)); a7 on the owned rows (mean + five fp64
                      sums); C-2 all-reduce of the five sums; MSE from the sums.

    The side stream of frame f runs while the compute stream runs frame f+1; a slot is reused
    only after its side-stream work is done (CUDA events).  world = 1 runs the whole range with
    the fused a7 on the compute stream.  The collectives and library calls are injectable, so
    the host logic also runs on CPU tensors (no streams) under gloo (tests/test_parallel.py)."""

    def __init__(self, n: int, n_sub: int, world: int, rank: int, lut: Optional[torch.Tensor],
                 device=None, depth: int = 2, omega=None, phase_offset: int = 0, before_each=None,
                 lut_seed: Optional[int] = None,
                 generate: Callable = api.ospr_generate, finalize_rows: Callable = api.ospr_finalize_rows,
                 mse_from_sums: Callable = api.ospr_mse_from_sums,
                 reduce_scatter: Callable = _default_reduce_scatter,
                 all_reduce: Callable[[torch.Tensor], None] = _default_all_reduce):
        if n % world:
            raise ValueError(f"n = {n} must divide among {world} ranks (owned row slices)")
        self.n, self.n_sub, self.world, self.rank, self.lut = n, n_sub, world, rank, lut
        self.dev = torch.device(device) if device is not None else \
            (lut.device if lut is not None else torch.device("cuda", torch.cuda.current_device()))
        self.cuda = self.dev.type == "cuda"
        self.depth, self.phase_offset, self.before_each = depth, phase_offset, before_each
        self.omega = omega if omega is not None else api.default_omega(n, "ospr")
        self.generate = generate
        self.sh = ShardedOspr(world, rank, generate=generate, finalize_rows=finalize_rows,
                              mse_from_sums=mse_from_sums, reduce_scatter=reduce_scatter, all_reduce=all_reduce)
        self.sf = subframe_range(n_sub, world, rank)     # empty if more ranks than pairs (zeros)
        self.rows = self.sh.rows(n)
        nb, nr = self.sf[1] - self.sf[0], n // world
        d, f32, f64 = self.dev, torch.float32, torch.float64
        self.bits = [torch.empty((1, nb, n, n // 8), dtype=torch.uint8, device=d) for _ in range(depth)]
        self.isum = [torch.empty((1, n, n), dtype=f32, device=d) for _ in range(depth)]
        self.mean_rows = [torch.empty((1, nr, n), dtype=f32, device=d) for _ in range(depth)]
        self.sums = [torch.zeros((1, 5), dtype=f64, device=d) for _ in range(depth)]
        self.mse = [torch.zeros(1, dtype=f64, device=d) for _ in range(depth)]
        self.targets = [None] * depth
        self.ws = self.ws_side = None
        if self.cuda:
            self.ws = torch.empty(api.ospr_workspace_bytes(n, 1, n_sub), dtype=torch.uint8, device=d)
            # a7's partial sums and ticket on the side stream: its own buffer (the compute stream's
            # workspace is in use by the next frame's passes meanwhile)
            self.ws_side = torch.empty(int(api.lib().holo_ospr_finalize_workspace_size()), dtype=torch.uint8,
                                       device=d)
            self.compute = torch.cuda.current_stream(d)
            self.side = torch.cuda.Stream(d)
            self.gen_done = [torch.cuda.Event() for _ in range(depth)]
            self.slot_free = [torch.cuda.Event() for _ in range(depth)]
        self.f = 0
        # the library calls with the default bindings go straight to the C ABI with arguments
        # prepared once (the host must keep ahead of ~0.1 ms shards at 8 GPUs); the collectives
        # stay torch.distributed (or the injected stand-ins)
        self._fast = (self.cuda and generate is api.ospr_generate and finalize_rows is api.ospr_finalize_rows
                      and mse_from_sums is api.ospr_mse_from_sums)
        if self._fast:
            lp, L = api._lut_args(lut)
            self._lib, self._lutp, self._L = api.lib(), lp, L
            self._reg = api._region(self.omega)
            self._cs, self._ss = self.compute.cuda_stream, self.side.cuda_stream
        if lut_seed is not None:         # a0 before each frame: the pool regenerated on the compute stream
            if before_each is not None or lut is None or not self.cuda:
                raise ValueError("lut_seed needs a CUDA pool `lut` and no before_each")
            fn, ptr, n_lut, cs = api.lib().holo_lut_generate, lut.data_ptr(), lut.numel(), self.compute.cuda_stream
            self.before_each = lambda: check(fn(lut_seed & 0xFFFFFFFFFFFFFFFF, n_lut, ptr, cs))

    def _local(self, f: int, s: int):
        if self._fast and self.sf[0] != self.sf[1]:
            t = self.targets[s]
            off = self.phase_offset + f * self.n_sub * self.n * self.n
            b, e = (0, self.n_sub) if self.world == 1 else self.sf
            check(self._lib.holo_ospr_generate(t.data_ptr(), self.n, 1, self.n_sub, self._lutp, self._L, off, b, e,
                                               self.bits[s].data_ptr(), self.isum[s].data_ptr(),
                                               self.mse[s].data_ptr() if self.world == 1 else None, self._reg,
                                               self.ws.data_ptr(), self.ws.numel(), self._cs))
            return
        out = api.OsprResult(bits=self.bits[s], intensity=self.isum[s],
                             mse=self.mse[s] if self.world == 1 else None)
        if self.sf[0] == self.sf[1]:     # no pair for this rank: a zero partial sum
            self.isum[s].zero_()
        elif self.world == 1:
            self.generate(self.targets[s], self.n_sub, self.lut, phase_offset=self.phase_offset + f * self.n_sub *
                          self.n * self.n, omega=self.omega, workspace=self.ws, out=out)
        else:
            self.generate(self.targets[s], self.n_sub, self.lut, phase_offset=self.phase_offset + f * self.n_sub *
                          self.n * self.n, sf_range=self.sf, want_mse=False, omega=self.omega, workspace=self.ws,
                          out=out)

    def _exchange(self, s: int):          # C-1, a7 on the owned rows, C-2, MSE
        if self._fast:                    # (on the side stream: the caller's context)
            r0, r1 = self.rows
            mr, sm = self.mean_rows[s], self.sums[s]
            self.sh.reduce_scatter(mr.view(-1), self.isum[s].view(-1))                                  # C-1
            check(self._lib.holo_ospr_finalize_rows(self.targets[s].data_ptr(), mr.data_ptr(), self.n, r0, r1,
                                                    self.n_sub, self._reg, mr.data_ptr(), sm.data_ptr(),
                                                    self.ws_side.data_ptr(), self.ws_side.numel(), self._ss))  # a7
            self.sh.all_reduce(sm)                                                                        # C-2
            check(self._lib.holo_ospr_mse_from_sums(sm.data_ptr(), 1, self._reg, self.mse[s].data_ptr(), self._ss))
            return
        self.sh.exchange(self.targets[s], self.isum[s], self.n_sub, self.mean_rows[s], self.sums[s], self.mse[s],
                         self.omega, fin_workspace=self.ws_side)

    def submit(self, target: torch.Tensor) -> int:
        """Queue frame self.f (target [N][N] on this rank's device); returns its index."""
        if self._fast and (target.dtype != torch.float32 or not target.is_cuda or not target.is_contiguous()
                           or target.numel() != self.n * self.n or target.device != self.dev):
            raise ValueError(f"target must be a contiguous float32 [{self.n}][{self.n}] tensor on {self.dev}")
        f, s = self.f, self.f % self.depth
        self.targets[s] = target
        if not self.cuda:
            if self.before_each is not None:
                self.before_each()
            self._local(f, s)
            if self.world > 1:
                self._exchange(s)
            self.f += 1
            return f
        if f >= self.depth:
            self.compute.wait_event(self.slot_free[s])       # frame f - depth's exchange is done
        if self.before_each is not None:
            self.before_each()
        self._local(f, s)
        if self.world > 1:
            self.gen_done[s].record(self.compute)
            self.side.wait_event(self.gen_done[s])
            with torch.cuda.stream(self.side):
                self._exchange(s)
            self.slot_free[s].record(self.side)
        else:
            self.slot_free[s].record(self.compute)
        self.f += 1
        return f

    def drain(self) -> None:
        if self.cuda:
            for e in self.slot_free:
                e.synchronize()

    def result(self, f: int):
        """(this rank's packed holograms [1][shard][N][N/8], the mean intensity of its owned
        rows [1][N/world][N] (world = 1: the whole frame [1][N][N]), mse [1]) of frame f; valid
        after drain() and until frame f + depth is submitted."""
        if f < self.f - self.depth or f >= self.f:
            raise ValueError(f"frame {f} is not in the pipeline's window")
        s = f % self.depth
        if self.cuda:
            self.slot_free[s].synchronize()
        mean = self.isum[s] if self.world == 1 else self.mean_rows[s]
        return self.bits[s], mean, self.mse[s]
