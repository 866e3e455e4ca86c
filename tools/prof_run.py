"""Small driver for ncu captures: runs the C3 OSPR step and a short C4-shaped GS (gs: 8 frames;
gs64: all 64 frames of C4 in one launch group, its 512 MiB state streaming from HBM)
(profile with -k regex:<kernel> -s <skip> -c <count>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2004_04049_b200 as hb
from holo_synth import LUT_SEED, WORKLOADS, target_for

what = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
if what in ("all", "ospr"):
    w = WORKLOADS["C3"]
    T = torch.from_numpy(target_for(w)).to(dev)
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    for _ in range(reps):
        r = hb.ospr_generate(T, w.n_sub, lut)
    torch.cuda.synchronize()
    print("ospr mse", r.mse.item())
if what == "c5":
    w = WORKLOADS["C5"]
    T = torch.from_numpy(target_for(w)).to(dev)
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    for _ in range(reps):
        r = hb.ospr_generate(T, w.n_sub, lut)
    torch.cuda.synchronize()
    print("c5 mse", r.mse.item())
if what == "n4096":                                   # R-26: one 4096^2 OSPR frame (N_SF = 4) and one GS iteration
    from holo_synth import Region, blobs_target
    n = 4096
    T = torch.from_numpy(blobs_target(3, n, 16, n / 16, n / 6.4, Region.upper_half(n))[None]).to(dev)
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    for _ in range(reps):
        r = hb.ospr_generate(T, 4, lut)
        g = hb.gs_generate(T, 1, lut)
    torch.cuda.synchronize()
    print("n4096 mse", r.mse.item(), g.mse[0, 0].item())
if what in ("all", "gs", "gs64"):
    w = WORKLOADS["C4"]
    nfr = w.frames if what == "gs64" else 8          # gs64: the whole C4 launch group (512 MiB state)
    T = torch.from_numpy(np.stack([target_for(w, b) for b in range(nfr)])).to(dev)
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    for _ in range(reps):
        g = hb.gs_generate(T, 3, lut, levels=0)
    torch.cuda.synchronize()
    print("gs mse", g.mse[:, -1].cpu().numpy())
