"""the paper's LUT-length experiment (PAPER.md §"Results", P:124-150,
Figs. 5/6) re-run on the GPU hot path.

For every N_LUT in a prime sweep (plus 0, the reference length 1000 of the NMSE, N and
N+1 around the resolution spike, 10007, and the independent-phase "centre image" of
Fig. 6 -- phases drawn on the fly, holo_ospr_generate_prng), and for each of six
synthetic test targets (stand-ins for the USC-SIPI images of Fig. 4, which are not in
the container; image 0 stands in for Mandrill): R independent runs of OSPR with N_SF = 24
binary sub-frames, each run with its own LUT seed ("the average of 100 independent
runs").  Reported per length: mean and standard deviation of the R-12 MSE per image and
the NMSE of P:127,

    NMSE_{image,n} = MSE_{image,n} * MSE_{Mandrill,1000} / MSE_{image,1000},

with its mean over images +- 2 sigma (the red line and grey band of Fig. 5).

Every number comes from the library's C ABI (lut_generate + ospr_generate with the six
targets as six frames of one call).  Writes a CSV and a JSON summary.

    python tools/lut_sweep.py [--n 256] [--runs 100] [--out profiles/r01_f1_lut_sweep_256]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import Region, blobs_target  # noqa: E402

N_SF = 24
REF_LEN = 1000            # the NMSE reference length of P:127 (non-prime, G-4)
N_IMAGES = 6


def primes_upto(m: int):
    sieve = np.ones(m + 1, dtype=bool)
    sieve[:2] = False
    for i in range(2, int(m ** 0.5) + 1):
        if sieve[i]:
            sieve[i * i::i] = False
    return np.nonzero(sieve)[0]


def lengths(n: int, lmax: int):
    """0, every prime <= 100, then primes roughly log-spaced up to lmax, plus the special
    lengths of the paper's discussion (N, N+1, 10007, the reference 1000)."""
    ps = primes_upto(lmax)
    small = [int(p) for p in ps if p <= 100]
    big = [int(p) for p in ps if p > 100]
    picks = set()
    for x in np.geomspace(101, lmax, 60):
        picks.add(min(big, key=lambda p: abs(p - x)))
    special = {0, REF_LEN, n, n + 1, 10007}
    return sorted(set(small) | picks | {s for s in special if s <= lmax})


def targets(n: int):
    """Six seeded synthetic targets over the OSPR region (R-13): image 0 is textured (dense
    small blobs + strong noise) standing in for Mandrill, the others smoother scenes."""
    om = Region.upper_half(n)
    s = n / 64.0
    imgs = [blobs_target(5000, n, 64, 1.0 * s, 3.0 * s, om, noise=0.6)]
    for i in range(1, N_IMAGES):
        imgs.append(blobs_target(5000 + i, n, 4 + 4 * i, 4.0 * s, 10.0 * s, om))
    return np.stack(imgs)


def run(n: int, runs: int, lmax: int, seed0: int = 7000):
    dev = torch.device("cuda", 0)
    T = torch.from_numpy(targets(n)).to(dev)
    F = T.shape[0]
    ws = torch.empty(hb.ospr_workspace_bytes(n, F, N_SF), dtype=torch.uint8, device=dev)
    out = hb.OsprResult(bits=None, intensity=torch.empty((F, n, n), dtype=torch.float32, device=dev),
                        mse=torch.empty(F, dtype=torch.float64, device=dev))
    lens = lengths(n, lmax)
    lut = torch.empty(max(max(lens), 1), dtype=torch.complex64, device=dev)
    keys = [("lut", L) for L in lens] + [("prng", -1)]
    mse = np.zeros((len(keys), runs, F))
    t0 = time.perf_counter()
    for j, (kind, L) in enumerate(keys):
        rows = []
        for r in range(runs):
            seed = seed0 + r
            if kind == "prng":
                hb.ospr_generate(T, N_SF, prng_seed=seed, want_bits=False, workspace=ws, out=out)
            elif L == 0:
                hb.ospr_generate(T, N_SF, None, want_bits=False, workspace=ws, out=out)
            else:
                hb.lut_generate(seed, L, out=lut[:L])
                hb.ospr_generate(T, N_SF, lut[:L], want_bits=False, workspace=ws, out=out)
            rows.append(out.mse.clone())
        mse[j] = torch.stack(rows).cpu().numpy()
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    return keys, mse, secs


def summarise(n, keys, mse, runs, secs, out_prefix):
    ref = [j for j, k in enumerate(keys) if k == ("lut", REF_LEN)][0]
    mref = mse[ref].mean(axis=0)                               # MSE_{image,1000}, per image
    scale = mref[0] / mref                                     # MSE_{Mandrill,1000} / MSE_{image,1000}
    nmse = mse * scale[None, None, :]                          # [len][run][image]
    lines = ["kind,n_lut,mean_nmse,std_nmse_over_images_runs," +
             ",".join(f"mse_img{i}_mean,mse_img{i}_std" for i in range(mse.shape[2]))]
    table = []
    for j, (kind, L) in enumerate(keys):
        v = nmse[j].ravel()
        row = [kind, L if kind == "lut" else "", float(v.mean()), float(v.std())]
        for i in range(mse.shape[2]):
            row += [float(mse[j, :, i].mean()), float(mse[j, :, i].std())]
        table.append(row)
        lines.append(",".join(str(x) for x in row))
    open(out_prefix + ".csv", "w").write("\n".join(lines) + "\n")

    def at(kind, L):
        j = keys.index((kind, L))
        return float(nmse[j].mean())

    indep = at("prng", -1)
    summary = {
        "experiment": "PAPER.md Figs. 5/6 analogue (SURVEY.md §8(f) f1): OSPR, N_SF=24, binary, "
                      f"{n}x{n}, six synthetic targets, {runs} independent runs per length, R-12 MSE over "
                      "Omega normalised as P:127",
        "n": n, "runs": runs, "lengths": len(keys) - 1, "gpu_seconds_wall": secs,
        "ospr_calls": len(keys) * runs, "sub_frames": len(keys) * runs * N_SF * mse.shape[2],
        "nmse_independent": indep,
        "nmse_L0": at("lut", 0),
        "nmse_L=N": at("lut", n) if ("lut", n) in keys else None,
        "nmse_L=N+1": at("lut", n + 1) if ("lut", n + 1) in keys else None,
        "nmse_L=10007": at("lut", 10007) if ("lut", 10007) in keys else None,
        "additional_error_L10007_vs_independent": (at("lut", 10007) / indep - 1.0) if ("lut", 10007) in keys else None,
        "csv": os.path.basename(out_prefix + ".csv"),
    }
    json.dump(summary, open(out_prefix + ".json", "w"), indent=1)
    return summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--runs", type=int, default=100)
    ap.add_argument("--lmax", type=int, default=100003)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    out = a.out or os.path.join(ROOT, "profiles", f"r01_f1_lut_sweep_{a.n}")
    keys, mse, secs = run(a.n, a.runs, a.lmax)
    print(json.dumps(summarise(a.n, keys, mse, a.runs, secs, out), indent=1))


if __name__ == "__main__":
    main()
