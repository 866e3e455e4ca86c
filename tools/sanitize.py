"""Small calls of every libholo entry point for compute-sanitizer runs (one tool per gpurun
call, as the profiling recipe requires):
    python tools/sanitize.py && compute-sanitizer --tool memcheck python tools/sanitize.py
Sizes N in {64, 256, 1024, 2048}: OSPR with a general (Lemire), power-of-two and wrapping pool,
the on-the-fly source, several chunks, sub-frame shards + row-slice a7 + MSE from sums; GS
continuous and quantised, the one-step hook; fft2 both ways; the randomisation hooks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import Region, blobs_target  # noqa: E402

sizes = [int(x) for x in os.environ.get("SAN_SIZES", "64,256,1024,2048").split(",")]
for n in sizes:
    S = 3 if n >= 1024 else 5
    T = torch.from_numpy(blobs_target(3, n, 6, n / 16, n / 6, Region.upper_half(n))).cuda()
    for L in (1021, 4096, n + 1):
        lut = hb.lut_generate(2004, L)
        r = hb.ospr_generate(T, S, lut, phase_offset=7)
    r2 = hb.ospr_generate(T, S, prng_seed=7, phase_offset=5)
    r3 = hb.ospr_generate(T, S, None)                                   # flat phase (N_LUT = 0)
    os.environ["HOLO_OSPR_CHUNK_BYTES"] = str(n * n * 8)                  # one pair per chunk
    r4 = hb.ospr_generate(T, S, lut)
    del os.environ["HOLO_OSPR_CHUNK_BYTES"]
    # two ranks' shards, emulated C-1 (sum), a7 on the owned rows, C-2, MSE
    p0 = hb.ospr_generate(T, S, lut, sf_range=(0, 2), want_mse=False)
    p1 = hb.ospr_generate(T, S, lut, sf_range=(2, S), want_mse=False)
    tot = (p0.intensity + p1.intensity)[0]
    m0, s0 = hb.ospr_finalize_rows(T, tot[: n // 2].contiguous(), 0, S)
    m1, s1 = hb.ospr_finalize_rows(T, tot[n // 2:].contiguous(), n // 2, S)
    mse = hb.ospr_mse_from_sums(s0 + s1, hb.default_omega(n, "ospr"))
    fm, fmse = hb.ospr_finalize(T, tot[None].contiguous(), S)
    g = hb.gs_generate(T.unsqueeze(0).contiguous(), 2, lut, levels=0)
    g2 = hb.gs_generate(T.unsqueeze(0).contiguous(), 2, lut, levels=16, want_levels=True)
    r0 = hb.debug_randomise(T, lut, 3).unsqueeze(0)
    rk, st = hb.gs_step(r0, T, levels=0)
    z = hb.debug_ospr_pairs(T, S, lut, offset=3)
    x = torch.randn(1, n, n, dtype=torch.complex64, device="cuda")
    y = hb.fft2(x)
    yi = hb.fft2(y, inverse=True)
    torch.cuda.synchronize()
    print(n, float(r.mse[0]), float(r2.mse[0]), float(r3.mse[0]), float(r4.mse[0]), float(mse[0]),
          float(fmse[0]), float(g.mse[0, -1]), float(g2.mse[0, -1]), float(st.mse[0, 0]), flush=True)
