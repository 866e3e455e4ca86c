"""Small OSPR/GS/fft2 calls for compute-sanitizer runs (one tool per run)."""
import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2004_04049_b200 as hb
from holo_synth import blobs_target, Region
for n, S in ((64, 5), (256, 4), (1024, 3)):
    T = torch.from_numpy(blobs_target(3, n, 6, n / 16, n / 6, Region.upper_half(n))).cuda()
    lut = hb.lut_generate(2004, 1021)
    r = hb.ospr_generate(T, S, lut)
    r2 = hb.ospr_generate(T, S, prng_seed=7, phase_offset=5)
    g = hb.gs_generate(T.unsqueeze(0).contiguous(), 2, lut, levels=0)
    g2 = hb.gs_generate(T.unsqueeze(0).contiguous(), 2, lut, levels=16, want_levels=True)
    x = torch.randn(1, n, n, dtype=torch.complex64, device="cuda")
    y = hb.fft2(x)
    torch.cuda.synchronize()
    print(n, float(r.mse[0]), float(r2.mse[0]), float(g.mse[0, -1]), float(g2.mse[0, -1]))
