"""Host cost per OsprStream.submit (the e2e pipeline is host-bound when this exceeds the ~0.11 ms
device time of a C3 frame set): wall time of back-to-back submits, with the bench's a0 hook
through the Python API and through a cached raw ABI call.  python tools/exp/stream_host.py"""
import time

import torch

import paper_2004_04049_b200 as hb
from holo_synth import LUT_SEED, WORKLOADS, target_for
from paper_2004_04049_b200._lib import check, lib

w = WORKLOADS["C3"]
n, S, L = w.n, w.n_sub, 1 << 16
hosts = [torch.from_numpy(target_for(w)).pin_memory() for _ in range(3)]
lut = torch.empty(L, dtype=torch.complex64, device="cuda")
res = {}
for mode in ("none", "raw", "api", "none2", "raw2", "api2"):
    st = hb.OsprStream(n, S, lut, depth=3)
    if mode.startswith("api"):
        st.before_each = lambda: hb.lut_generate(LUT_SEED, L, out=lut)
    elif mode.startswith("raw"):
        fn, ptr, cs = lib().holo_lut_generate, lut.data_ptr(), st.comp.cuda_stream
        st.before_each = lambda: check(fn(LUT_SEED, L, ptr, cs))
    for i in range(10):
        st.submit(hosts[i % 3])
    st.drain()
    torch.cuda.synchronize()
    k = 300
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(st.h2d)
    for i in range(k):
        st.submit(hosts[i % 3])
    t1 = time.perf_counter()
    b.record(st.d2h)
    torch.cuda.synchronize()
    res[mode] = {"host_us_per_submit": (t1 - t0) / k * 1e6, "device_us_per_set": a.elapsed_time(b) / k * 1e3}
print(res)
