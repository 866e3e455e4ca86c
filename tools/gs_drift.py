"""C4 GS trajectory drift: GPU kernel vs the fp64 oracle, next to a numpy complex64
control on the same inputs (SURVEY.md probe A.4c).

For each selected frame b of BASELINE configs[3] (1024^2, 64 frames, 50 iterations,
continuous phase-only, LUT 2^16, cursor b*P):
  * gpu      -- MSE_k of the bench's launch (all 64 frames in one gs_generate call);
  * oracle   -- oracle.gs (fp64, radix-2) from the same inputs;
  * control  -- the same GS loop in numpy complex64 (pocketfft, norm="ortho"), the
                M-1 MSE in fp64 from its fp32 intensity: what a plain fp32 GS does;
  * one-step -- at every iteration, the oracle's step from the GPU's own R_{k-1}
                (gs_step chain, bit-identical to the fused loop).
Writes a JSON summary (per-iteration relative MSE errors) to the path given.

usage: python tools/gs_drift.py OUT.json [--frames 0,31,63] [--lib path/to/libholo.so]
Test/measurement infrastructure: it calls oracle/ (allowed for tools that verify).
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--frames", default="0,31,63")
ap.add_argument("--lib", default=None)
ap.add_argument("--no-onestep", action="store_true")
args = ap.parse_args()

import paper_2004_04049_b200._lib as L  # noqa: E402
if args.lib:
    L.LIB_PATH = os.path.abspath(args.lib)
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import LUT_SEED, WORKLOADS, target_for  # noqa: E402

w = WORKLOADS["C4"]
n, P, iters = w.n, w.n * w.n, w.iters
frames = [int(x) for x in args.frames.split(",")]
region = (0, n, 0, n)
Ts = np.stack([target_for(w, b) for b in range(w.frames)])
lut_o = oracle.lut_build(LUT_SEED, 1 << 16)


def control_c64(T, cursor):
    """Plain complex64 GS (g0-g5 in the oracle's order), numpy pocketfft."""
    idx = (cursor + np.arange(P, dtype=np.int64)) % lut_o.shape[0]
    ph = (lut_o[idx, 0] + 1j * lut_o[idx, 1]).astype(np.complex64).reshape(n, n)
    T32 = T.astype(np.float32)
    R = (T32 * ph).astype(np.complex64)
    mse = []
    t2 = T32.astype(np.float64) ** 2
    for _ in range(iters):
        H = np.fft.ifft2(R, norm="ortho")
        a = np.abs(H)
        h = np.where(a > 0, H / np.where(a > 0, a, 1), np.complex64(1)).astype(np.complex64)
        Rp = np.fft.fft2(h, norm="ortho")
        I = (Rp.real * Rp.real + Rp.imag * Rp.imag).astype(np.float32)
        Id = I.astype(np.float64)
        sc = t2.sum() / Id.sum()
        mse.append(float(np.mean((sc * Id - t2) ** 2)))
        amp = np.abs(Rp)
        R = np.where(amp > 0, T32 * (Rp / np.where(amp > 0, amp, 1)), T32).astype(np.complex64)
    return np.array(mse)


t0 = time.time()
dev = torch.device("cuda", 0)
lg = hb.lut_generate(LUT_SEED, 1 << 16, device=dev)
res = hb.gs_generate(torch.from_numpy(Ts).to(dev), iters, lg, levels=0, want_holo=False)
mse_gpu = res.mse.cpu().numpy()
torch.cuda.synchronize()
print(f"gpu done {time.time() - t0:.1f}s", flush=True)

with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
    fut_or = {b: ex.submit(oracle.gs, Ts[b], iters, lut_o, b * P, 0, region) for b in frames}
    fut_ct = {b: ex.submit(control_c64, Ts[b], b * P) for b in frames}
    onestep = {}
    if not args.no_onestep:
        for b in frames:
            tg = torch.from_numpy(np.ascontiguousarray(Ts[b])).to(dev)
            r = hb.debug_randomise(tg, lg, b * P).unsqueeze(0)
            futs = []
            for k in range(iters):
                r_prev = r[0].cpu().numpy().astype(np.complex128)
                r, st = hb.gs_step(r, tg, levels=0)
                m = float(st.mse.cpu().numpy()[0, 0])
                assert m == mse_gpu[b, k], ("fused != step chain", b, k)
                futs.append((m, ex.submit(oracle.gs_step, r_prev, Ts[b], 0, region)))
            onestep[b] = [abs(m - f.result()["mse"]) / f.result()["mse"] for m, f in futs]
    ref = {b: f.result()["mse"] for b, f in fut_or.items()}
    ctl = {b: f.result() for b, f in fut_ct.items()}
print(f"oracle/control done {time.time() - t0:.1f}s", flush=True)

out = {"what": "C4 GS trajectory MSE, relative error vs the fp64 oracle per iteration",
       "lib": os.path.basename(L.LIB_PATH), "frames": {}}
for b in frames:
    eg = np.abs(mse_gpu[b] - ref[b]) / ref[b]
    ec = np.abs(ctl[b] - ref[b]) / ref[b]
    d = {"gpu_rel": eg.tolist(), "control_c64_rel": ec.tolist(), "oracle_mse": ref[b].tolist(),
         "gpu_max": float(eg.max()), "control_max": float(ec.max()),
         "gpu_argmax": int(eg.argmax()) + 1, "control_argmax": int(ec.argmax()) + 1}
    if b in onestep:
        d["onestep_rel"] = onestep[b]
        d["onestep_max"] = float(max(onestep[b]))
    out["frames"][str(b)] = d
    print(f"frame {b}: gpu max {eg.max():.3e} (it {eg.argmax() + 1}), control max {ec.max():.3e} "
          f"(it {ec.argmax() + 1}), one-step max {d.get('onestep_max', float('nan')):.3e}; "
          f"mse 1 -> 50: {ref[b][0]:.4e} -> {ref[b][-1]:.4e}")
    for k in (1, 10, 20, 30, 40, 50):
        print(f"   it {k:2d}: gpu {eg[k - 1]:.2e}  control {ec[k - 1]:.2e}")
# transform accuracy at 1024^2 on a unit-modulus field (the GS hologram's kind of input)
rng = np.random.default_rng(7)
u = np.exp(2j * np.pi * rng.random((n, n)))
fa = {}
for inv in (False, True):
    ref_f = oracle.fft2(u, inverse=inv)
    g = hb.fft2(torch.from_numpy(u.astype(np.complex64)).to(dev), inverse=inv).cpu().numpy()
    c = (np.fft.ifft2 if inv else np.fft.fft2)(u.astype(np.complex64), norm="ortho")
    nr = lambda x: float(np.linalg.norm(x - ref_f) / np.linalg.norm(ref_f))
    fa["inverse" if inv else "forward"] = {"gpu_norm_rel": nr(g), "numpy_c64_norm_rel": nr(c)}
out["fft2_1024_unit_modulus"] = fa
print("fft2 accuracy", fa)
json.dump(out, open(args.out, "w"), indent=1)
