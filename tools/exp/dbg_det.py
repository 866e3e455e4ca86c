import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2004_04049_b200 as hb
from holo_synth import WORKLOADS, target_for, LUT_SEED
for name, F in (("C5", 2), ("C3", 1)):
    w = WORKLOADS[name]
    Ts = torch.from_numpy(np.stack([target_for(w, f) for f in range(F)])).cuda()
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    outs = [hb.ospr_generate(Ts, w.n_sub, lut) for _ in range(3)]
    torch.cuda.synchronize()
    for i in (1, 2):
        print(name, "run", i, "bits equal", torch.equal(outs[0].bits, outs[i].bits),
              "I equal", torch.equal(outs[0].intensity, outs[i].intensity),
              "maxdiff I", (outs[0].intensity - outs[i].intensity).abs().max().item(),
              "bits diff bytes", (outs[0].bits != outs[i].bits).sum().item())
