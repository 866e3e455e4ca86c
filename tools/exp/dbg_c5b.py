import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2004_04049_b200 as hb, oracle
from holo_synth import WORKLOADS, target_for, LUT_SEED
w = WORKLOADS["C5"]
Ts = np.stack([target_for(w, f) for f in range(2)])
lg = hb.lut_generate(LUT_SEED, 1 << 16)
res = hb.ospr_generate(torch.from_numpy(Ts).cuda(), w.n_sub, lg)
bits, I = res.bits.cpu().numpy(), res.intensity.cpu().numpy()
for f in range(2):
    Ir = oracle.replay_from_bits(bits[f], w.n)
    d = np.abs(I[f] - Ir); k = np.unravel_index(np.argmax(d), d.shape)
    print("frame", f, "max-rel", d.max() / Ir.max(), "at", k, "I", I[f][k], "ref", Ir[k], "norm-rel", np.linalg.norm(I[f]-Ir)/np.linalg.norm(Ir))
    b = torch.from_numpy(np.unpackbits(bits[f], axis=-1)).double().cuda()
    X = torch.fft.fft2(2 * b - 1, norm="ortho"); It = (X.abs() ** 2).mean(0).cpu().numpy()
    print("   torch replay vs oracle replay max-rel", np.abs(It - Ir).max() / Ir.max())
