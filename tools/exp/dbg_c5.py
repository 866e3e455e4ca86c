import sys, os, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2004_04049_b200 as hb
from holo_synth import WORKLOADS, target_for, LUT_SEED
w = WORKLOADS["C5"]
lut = hb.lut_generate(LUT_SEED, 1 << 16)
for F in (1, 2):
    Ts = torch.from_numpy(np.stack([target_for(w, f) for f in range(F)])).cuda()
    r = hb.ospr_generate(Ts, w.n_sub, lut)
    torch.cuda.synchronize()
    for f in range(F):
        same = [bool(torch.equal(r.bits[f, 0], r.bits[f, s])) for s in range(w.n_sub)]
        print(os.environ.get("HOLO_PDL", "1"), "F", F, "frame", f, "".join("1" if x else "0" for x in same))
