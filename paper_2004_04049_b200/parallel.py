"""Multi-GPU partitioning of the hot path.

One process per GPU (torch.distributed over NCCL).  The units of the method are
independent, so the partition is a plain shard of them:

* OSPR: the N_SF sub-frames of every frame are split into contiguous ranges,
  one per rank.  Draw indices stay global (frame f, sub-frame s starts at
  phase_offset + (f N_SF + s) N^2), so every rank produces exactly the
  holograms the single-GPU call would.  The one real exchange step of the path
  is the time average: the per-rank partial intensity sums are added
  with an all-reduce (collective C-1) and only then is the MSE computed (it is
  nonlinear in I) by ``ospr_finalize``.
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


def shard_range(n_units: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced [begin, end) of n_units for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (n_units * rank) // world, (n_units * (rank + 1)) // world


def _default_all_reduce(t: torch.Tensor) -> None:
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM)


@dataclass
class ShardedOsprResult:
    sf_range: Tuple[int, int]          # this rank's sub-frames
    bits: Optional[torch.Tensor]       # [F][sf_end - sf_begin][N][N/8] (this rank's holograms)
    intensity: torch.Tensor            # [F][N][N] mean over ALL sub-frames (after the all-reduce)
    mse: Optional[torch.Tensor]        # [F]


class ShardedOspr:
    """OSPR with sub-frames sharded across `world` ranks (collective C-1)."""

    def __init__(self, world: int, rank: int,
                 generate: Callable = api.ospr_generate,
                 finalize: Callable = api.ospr_finalize,
                 all_reduce: Callable[[torch.Tensor], None] = _default_all_reduce):
        self.world, self.rank = world, rank
        self.generate, self.finalize, self.all_reduce = generate, finalize, all_reduce

    def stages(self, target: torch.Tensor, n_sub: int, lut: Optional[torch.Tensor], workspace: torch.Tensor,
               out, mse_out: Optional[torch.Tensor], phase_offset: int = 0, omega=None):
        """The step split around its one collective, for CUDA-graph capture of the two local
        parts: (pre, collective, post).  pre: this rank's shard into out (bits and the partial
        intensity sum); collective: C-1 on out.intensity; post: mean and MSE in place (a
        single rank skips the collective).  All buffers are caller-owned, so pre and post
        allocate nothing."""
        b, e = shard_range(n_sub, self.world, self.rank)
        if b == e:
            raise ValueError("more ranks than sub-frames: use run()")
        if self.world == 1:                          # the whole range: mean and MSE in one call
            def whole():
                out.mse = mse_out
                self.generate(target, n_sub, lut, phase_offset=phase_offset, omega=omega, workspace=workspace,
                              out=out)
            def no_exchange():
                pass
            no_exchange.local = True                 # marks a collective with nothing to exchange
            return whole, no_exchange, (lambda: None)

        def pre():
            self.generate(target, n_sub, lut, phase_offset=phase_offset, sf_range=(b, e), want_mse=False,
                          omega=omega, workspace=workspace, out=out)

        def collective():
            if self.world > 1:
                self.all_reduce(out.intensity)
        collective.local = False

        def post():
            self.finalize(target, out.intensity, n_sub, omega=omega, out=out.intensity, mse_out=mse_out,
                          workspace=workspace)
        return pre, collective, post

    def run(self, target: torch.Tensor, n_sub: int, lut: Optional[torch.Tensor], phase_offset: int = 0,
            want_bits: bool = True, want_mse: bool = True, omega=None, workspace=None) -> ShardedOsprResult:
        b, e = shard_range(n_sub, self.world, self.rank)
        if self.world == 1:
            r = self.generate(target, n_sub, lut, phase_offset=phase_offset, want_bits=want_bits,
                              want_mse=want_mse, omega=omega, workspace=workspace)
            return ShardedOsprResult((0, n_sub), r.bits, r.intensity, r.mse)
        if b == e:
            # more ranks than sub-frames: contribute a zero partial sum
            t3 = target if target.dim() == 3 else target.unsqueeze(0)
            part_i = torch.zeros_like(t3)
            bits = None
        else:
            part = self.generate(target, n_sub, lut, phase_offset=phase_offset, sf_range=(b, e),
                                 want_bits=want_bits, want_mse=False, omega=omega, workspace=workspace)
            part_i, bits = part.intensity, part.bits
        self.all_reduce(part_i)                                  # C-1: sum of partial intensities
        mean, mse = self.finalize(target, part_i, n_sub, omega=omega, want_mse=want_mse, out=part_i)
        return ShardedOsprResult((b, e), bits, mean, mse)


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
