"""Calibration micro-benchmark (test tooling, not product): libholo's unitary fft2
hook vs torch.fft.fft2 (cuFFT) on the same batched complex64 frames."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2004_04049_b200 as hb


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for n, B in [(1024, 8), (1024, 32), (2048, 4), (256, 64)]:
    x = torch.randn(B, n, n, dtype=torch.complex64, device="cuda")
    out = torch.empty_like(x)
    t_cu = timeit(lambda: torch.fft.fft2(x, norm="ortho"))
    t_h = timeit(lambda: hb.fft2(x, out=out))
    hb.profile_enable(True)
    for _ in range(5):
        hb.fft2(x, out=out)
    torch.cuda.synchronize()
    r = {k: hb.profile_read(k) for k in ("fft_rows", "fft_cols")}
    hb.profile_enable(False)
    bytes_ = 4 * B * n * n * 8
    print(f"N={n} B={B}: cuFFT {t_cu:8.1f} us ({bytes_ / t_cu / 1e3:6.0f} GB/s)   holo {t_h:8.1f} us "
          f"({bytes_ / t_h / 1e3:6.0f} GB/s)  rows {r['fft_rows'][1] / r['fft_rows'][0] * 1e3:7.1f} us  "
          f"cols {r['fft_cols'][1] / r['fft_cols'][0] * 1e3:7.1f} us")
