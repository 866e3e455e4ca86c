import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2004_04049_b200 as hb
from holo_synth import blobs_target, Region
def replay(bits, n):
    b = torch.from_numpy(np.unpackbits(bits.cpu().numpy(), axis=-1)).double().cuda()  # [S][n][n]
    h = 2 * b - 1
    X = torch.fft.fft2(h, norm="ortho")
    return (X.abs() ** 2).mean(0)
for n, S, F in [(2048, 2, 1), (2048, 6, 1), (2048, 8, 1), (1024, 24, 1), (2048, 8, 2)]:
    T = torch.from_numpy(np.stack([blobs_target(9 + f, n, 8, 40.0, 100.0, Region.upper_half(n)) for f in range(F)])).cuda()
    lut = hb.lut_generate(2004, 10007)
    r = hb.ospr_generate(T, S, lut)
    for f in range(F):
        I = replay(r.bits[f], n)
        d = (I - r.intensity[f].double()).abs().max().item() / I.max().item()
        print(n, S, F, f, "rel", d, "chunk", hb.ospr_chunk_pairs(n, S))
from holo_synth import WORKLOADS, target_for, LUT_SEED
w = WORKLOADS["C5"]
Ts = torch.from_numpy(np.stack([target_for(w, f) for f in range(2)])).cuda()
lut = hb.lut_generate(LUT_SEED, 1 << 16)
r = hb.ospr_generate(Ts, w.n_sub, lut)
for f in range(2):
    I = replay(r.bits[f], w.n)
    d = (I - r.intensity[f].double()).abs().max().item() / I.max().item()
    same = [bool(torch.equal(r.bits[f, 0], r.bits[f, s])) for s in range(w.n_sub)]
    print("C5 frame", f, "rel", d, "identical-to-sf0:", "".join("1" if x else "0" for x in same))
