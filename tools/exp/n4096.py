"""Timing of the N = 4096 path (R-26) next to N = 2048, per sub-frame and per GS
frame-iteration, CUDA events around whole calls after warm-up (inputs larger than L2).
python tools/exp/n4096.py [--reps 5]"""
import argparse
import json

import numpy as np
import torch

import paper_2004_04049_b200 as hb
from holo_synth import LUT_SEED, Region, blobs_target


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    out = {}
    for n in (2048, 4096):
        S = 32
        T = torch.from_numpy(blobs_target(3, n, 16, n / 16, n / 6.4, Region.upper_half(n))[None]).cuda()
        ws = torch.empty(hb.ospr_workspace_bytes(n, 1, S), dtype=torch.uint8, device="cuda")
        res = hb.ospr_generate(T, S, lut, workspace=ws)
        ms = timed(lambda: hb.ospr_generate(T, S, lut, workspace=ws, out=res), args.reps)
        B, it = 4, 5
        Tg = torch.from_numpy(np.stack([blobs_target(5 + b, n, 16, n / 16, n / 6.4, Region.full(n))
                                        for b in range(B)])).cuda()
        wsg = torch.empty(hb.gs_workspace_bytes(n, B, it), dtype=torch.uint8, device="cuda")
        g = hb.gs_generate(Tg, it, lut, workspace=wsg)
        gms = timed(lambda: hb.gs_generate(Tg, it, lut, workspace=wsg, out=g), args.reps)
        out[n] = {"ospr_ms_per_frame_S32": ms, "ospr_subframes_per_s": S / ms * 1e3,
                  "gs_ms_4x5": gms, "gs_frame_iters_per_s": B * it / gms * 1e3,
                  "ospr_ns_per_pixel_subframe": ms * 1e6 / (S * n * n)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
