"""Frame-stream host cost (tooling): wall time of K submit() calls against the device time of
the K frame sets, to tell a host-bound pipeline from a device-bound one."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import LUT_SEED, WORKLOADS, target_for  # noqa: E402

w = WORKLOADS["C3"]
n, S = w.n, w.n_sub
hosts = [torch.from_numpy(target_for(w)).pin_memory() for _ in range(3)]
lut = torch.empty(1 << 16, dtype=torch.complex64, device="cuda")
st = hb.OsprStream(n, S, lut, depth=3, before_each=lambda: hb.lut_generate(LUT_SEED, 1 << 16, out=lut))
for i in range(9):
    st.submit(hosts[i % 3])
st.drain()
K = 50
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(st.h2d)
t0 = time.perf_counter()
for i in range(K):
    st.submit(hosts[i % 3])
t1 = time.perf_counter()
b.record(st.d2h)
torch.cuda.synchronize()
print(f"host {1e6 * (t1 - t0) / K:.1f} us per submit, device {1e3 * a.elapsed_time(b) / K:.1f} us per frame set")
