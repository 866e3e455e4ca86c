"""Pass A split (tooling): the production producer alone (holo_debug_ospr_pairs: conj Z of the
12 C3 pairs written to HBM, no FFT) against the full pass A inside ospr_generate, both
bracketed by libholo's profiling events.   python tools/exp/passa_split.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import LUT_SEED, WORKLOADS, target_for  # noqa: E402

dev = torch.device("cuda", 0)
w = WORKLOADS["C3"]
T = torch.from_numpy(target_for(w)).to(dev)
lut = hb.lut_generate(LUT_SEED, 1 << 16)
for name, fn in (("producer only (Z to HBM)", lambda: hb.debug_ospr_pairs(T, w.n_sub, lut)),
                 ("full step", lambda: hb.ospr_generate(T, w.n_sub, lut))):
    fn()
    torch.cuda.synchronize()
    hb.profile_enable(True)
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    out = {}
    for k in hb.kernel_names():
        c, ms = hb.profile_read(k)
        if c:
            out[k] = round(1e3 * ms / c, 2)
    hb.profile_enable(False)
    print(name, out)
