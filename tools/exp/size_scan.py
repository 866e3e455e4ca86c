"""OSPR kernel times across N (tooling): one frame set of N_SF sub-frames per N, every kernel
bracketed by libholo's profiling events, reported per pair-pixel so the passes can be compared
across transform sizes (E = 16, 32, 64 values per thread).

    python tools/exp/size_scan.py [n_sub]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import LUT_SEED, Region, blobs_target  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dev = torch.device("cuda", 0)
lut = hb.lut_generate(LUT_SEED, 1 << 16)
for n in (256, 512, 1024, 2048):
    T = torch.from_numpy(blobs_target(3, n, 16, n / 16, n / 6.4, Region.upper_half(n))).to(dev)
    ws = torch.empty(hb.ospr_workspace_bytes(n, 1, S), dtype=torch.uint8, device=dev)
    out = hb.ospr_generate(T, S, lut, workspace=ws)
    reps = 10
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        hb.ospr_generate(T, S, lut, workspace=ws, out=out)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    step_us = a.elapsed_time(b) * 1e3 / reps
    hb.profile_enable(True)
    for _ in range(reps):
        hb.ospr_generate(T, S, lut, workspace=ws, out=out)
    torch.cuda.synchronize()
    times = {}
    for name in hb.kernel_names():
        cnt, ms = hb.profile_read(name)
        if cnt:
            times[name] = 1e3 * ms / reps
    hb.profile_enable(False)
    pp = (S + 1) // 2 * n * n                     # pair-pixels per frame set
    print(f"N={n:5d} step {step_us:8.1f} us  {S / step_us * 1e6:10.0f} sf/s  |  " +
          "  ".join(f"{k} {v:7.1f} us ({1e6 * v / pp:5.2f} ps/pp)" for k, v in times.items()))
