"""Shared helpers of the GPU parity tests (protocol P-1..P-9).

The oracle (fp64 CPU, oracle/) and the CUDA path (paper_2004_04049_b200) are
run on the same seeded inputs (holo_synth); these helpers compare them with
the tolerances BASELINE.json's north_star states.
"""
import numpy as np
import torch

import oracle

#: north_star: "binary hologram pixels bit-exact except where |Re H| < 1e-5 max|H|"
BIT_BAND = 1e-5
#: north_star: "replay intensity and MSE within a relative 1e-4"
REL_TOL = 1e-4


def lut_pair(seed, L):
    """(GPU LUT complex64 or None, oracle-side float32 [L][2] or None) -- each side builds its own."""
    import paper_2004_04049_b200 as hb
    if L == 0:
        return None, None
    return hb.lut_generate(seed, L), oracle.lut_build(seed, L)


def unpack(bits, n):
    return np.unpackbits(np.asarray(bits, np.uint8).reshape(-1, n, n // 8), axis=-1).reshape(-1, n, n)


def check_bits(gpu_bits, h_re_ref, n, band=BIT_BAND):
    """P-3: every mismatch must lie where |Re H_ref| < band * max|Re H_ref| (max over the
    real part, a conservative stand-in for max|H|).  Returns (exempt, flips)."""
    g = unpack(gpu_bits, n)[0].astype(bool)
    o = h_re_ref >= 0
    thr = band * np.max(np.abs(h_re_ref))
    exempt = np.abs(h_re_ref) < thr
    bad = (g != o) & ~exempt
    assert not bad.any(), f"{int(bad.sum())} bit mismatches outside the |Re H| band"
    return int(exempt.sum()), int((g != o).sum())


def check_intensity(I_gpu, I_ref, tol=REL_TOL):
    """P-4: max |dI| / max I and ||dI||_2 / ||I||_2 both <= tol."""
    I_gpu = np.asarray(I_gpu, np.float64)
    d = I_gpu - I_ref
    mx = np.max(np.abs(d)) / np.max(np.abs(I_ref))
    nr = np.linalg.norm(d) / np.linalg.norm(I_ref)
    assert mx <= tol and nr <= tol, f"intensity max-rel {mx:.3e}, norm-rel {nr:.3e}"
    return mx, nr


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def to_np(t):
    return t.detach().cpu().numpy()


def cuda_target(T):
    return torch.from_numpy(np.ascontiguousarray(T, np.float32)).cuda()
