"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no phase randomisation, no DFT,
no quantisation, no metric).  It only produces the *inputs* of the hot path:

* ``blobs_target`` -- the synthetic target amplitude image T (DESIGN.md
  "Input recipe"; SURVEY.md §8(d) "Synthetic inputs", reading R-20).  It stands
  in for the six USC-SIPI test images of PAPER.md Fig. 4, which are
  not available; no item of that suite is reproduced.
* ``WORKLOADS`` -- the five configurations of BASELINE.json ``configs`` as
  plain data (resolution, sub-frame / iteration counts, LUT lengths, seeds,
  measurement region Ω).

The random stream used here is SplitMix64 (Steele, Lea & Flood 2014) in
counter form: output k = mix64(seed + (k+1)*0x9E3779B97F4A7C15).  The oracle
and the CUDA library each implement their own copy of the same published
generator for the phase LUT (step a0); this module is not imported by either
for that purpose.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "splitmix64_stream",
    "uniform01",
    "blobs_target",
    "Region",
    "Workload",
    "WORKLOADS",
    "LUT_SEED",
    "target_for",
]

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

#: LUT seed used by every configuration ("LUT seed = 2004").
LUT_SEED = 2004


def splitmix64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs ``start .. start+count-1`` of SplitMix64 seeded with ``seed``."""
    k = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (k + np.uint64(1)) * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Uniform doubles on [0, 1) from the top 53 bits of the stream."""
    return (splitmix64_stream(seed, count, start) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclass(frozen=True)
class Region:
    """Half-open measurement / placement region Ω in unshifted replay coordinates."""

    row0: int
    row1: int
    col0: int
    col1: int

    def as_tuple(self) -> Tuple[int, int, int, int]:
        return (self.row0, self.row1, self.col0, self.col1)

    @staticmethod
    def upper_half(n: int) -> "Region":
        """OSPR Ω: rows [1, N/2) x all columns (reading R-13: excludes the
        self-conjugate rows 0 and N/2, hence DC, and the twin image)."""
        return Region(1, n // 2, 0, n)

    @staticmethod
    def full(n: int) -> "Region":
        return Region(0, n, 0, n)


def blobs_target(seed: int, n: int, n_blobs: int, sigma_lo: float, sigma_hi: float,
                 region: Region, noise: float = 0.05) -> np.ndarray:
    """Target amplitude T (float32, [n][n], max 1) = sum of Gaussian blobs + noise.

    Recipe:
      1. draws 3b, 3b+1, 3b+2 of the stream give blob b's centre row
         U[row0, row1), centre column U[0, n) and width sigma U[sigma_lo, sigma_hi];
      2. T = sum_b exp(-(y-cy)^2/2s^2) * exp(-(x-cx)^2/2s^2) (non-periodic, peak 1
         per blob), evaluated in double;
      3. draws 3*n_blobs + i add U[0, noise) to the i-th pixel of Ω (row-major);
      4. T = 0 outside Ω; T /= max T; rounded to float32.
    """
    u = uniform01(seed, 3 * n_blobs)
    rows = region.row1 - region.row0
    cy = region.row0 + u[0::3] * rows
    cx = u[1::3] * n
    sig = sigma_lo + u[2::3] * (sigma_hi - sigma_lo)
    yy = np.arange(n, dtype=np.float64)
    gy = np.exp(-((yy[None, :] - cy[:, None]) ** 2) / (2.0 * sig[:, None] ** 2))  # [b][y]
    gx = np.exp(-((yy[None, :] - cx[:, None]) ** 2) / (2.0 * sig[:, None] ** 2))  # [b][x]
    t = gy.T @ gx
    out = np.zeros((n, n), dtype=np.float64)
    r0, r1, c0, c1 = region.as_tuple()
    npix = (r1 - r0) * (c1 - c0)
    nz = uniform01(seed, npix, start=3 * n_blobs).reshape(r1 - r0, c1 - c0) * noise
    out[r0:r1, c0:c1] = t[r0:r1, c0:c1] + nz
    m = out.max()
    if m > 0:
        out /= m
    return out.astype(np.float32)


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration as plain data."""

    name: str
    algo: str                 # "ospr" | "gs"
    n: int
    frames: int               # OSPR frames or GS batch
    n_sub: int                # OSPR sub-frames per frame (0 for GS)
    iters: int                # GS iterations (0 for OSPR)
    lut_lens: Tuple[int, ...]
    levels: int               # GS: 0 = continuous phase-only, Q > 0 = Q levels; OSPR: 2 (binary)
    target_seed0: int
    n_blobs: int
    sigma: Tuple[float, float]
    region: str               # "upper" | "full"
    baseline_index: int       # index into BASELINE.json configs

    def omega(self) -> Region:
        return Region.upper_half(self.n) if self.region == "upper" else Region.full(self.n)


#: SURVEY.md §8(d) table; BASELINE.json configs[0..4].
WORKLOADS = {
    "C1": Workload("C1", "ospr", 64, 1, 8, 0, (256,), 2, 1, 4, (4.0, 10.0), "upper", 0),
    "C2": Workload("C2", "gs", 256, 1, 0, 20, (4096,), 256, 2, 4, (4.0, 10.0), "full", 1),
    "C3": Workload("C3", "ospr", 1024, 1, 24, 0, (1 << 8, 1 << 12, 1 << 16, 1 << 20, 1024 * 1024 * 24),
                   2, 3, 16, (64.0, 160.0), "upper", 2),
    "C4": Workload("C4", "gs", 1024, 64, 0, 50, (1 << 16,), 0, 1000, 16, (64.0, 160.0), "full", 3),
    "C5": Workload("C5", "ospr", 2048, 60, 32, 0, (1 << 16,), 2, 2000, 16, (128.0, 320.0), "upper", 4),
}

#: Extra LUT lengths of the parity protocol P-9 (the BASELINE lengths all divide N^2).
def p9_lengths(n: int) -> Tuple[int, ...]:
    return (0, 1, 5, 13, 257, 1021, 10007, n + 1, n * n + 1)


def target_for(w: Workload, index: int = 0) -> np.ndarray:
    """Target of frame ``index`` of workload ``w`` (C1-C3 use one seed; C4/C5 use seed0 + index)."""
    seed = w.target_seed0 + (index if w.frames > 1 else 0)
    return blobs_target(seed, w.n, w.n_blobs, w.sigma[0], w.sigma[1], w.omega())
