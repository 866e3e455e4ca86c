"""Host cost per binding call (argument checks + ctypes), at a size where the GPU work is small:
python tools/exp/api_host.py"""
import time

import torch

import paper_2004_04049_b200 as hb
from holo_synth import LUT_SEED

n, S = 64, 4
T = torch.rand(1, n, n, device="cuda")
lut = hb.lut_generate(LUT_SEED, 256)
ws = torch.empty(hb.ospr_workspace_bytes(n, 1, S), dtype=torch.uint8, device="cuda")
out = hb.OsprResult(bits=torch.empty((1, 2, n, n // 8), dtype=torch.uint8, device="cuda"),
                    intensity=torch.empty((1, n, n), device="cuda"), mse=None)
rows = torch.empty((n // 2, n), device="cuda")
sums = torch.empty(5, dtype=torch.float64, device="cuda")
fws = torch.empty(int(hb.lib().holo_ospr_finalize_workspace_size()), dtype=torch.uint8, device="cuda")
mse = torch.empty(1, dtype=torch.float64, device="cuda")
om = hb.default_omega(n, "ospr")
calls = {
    "lut_generate": lambda: hb.lut_generate(LUT_SEED, 256, out=lut),
    "ospr_generate_shard": lambda: hb.ospr_generate(T, S, lut, sf_range=(0, 2), want_mse=False, workspace=ws, out=out),
    "ospr_finalize_rows": lambda: hb.ospr_finalize_rows(T[0], out.intensity[0, :n // 2], 0, S, out=rows, sums_out=sums,
                                                        workspace=fws),
    "ospr_mse_from_sums": lambda: hb.ospr_mse_from_sums(sums.view(1, 5), om, out=mse),
}
res = {}
for name, fn in calls.items():
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    k = 500
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    res[name] = round((time.perf_counter() - t0) / k * 1e6, 1)
    torch.cuda.synchronize()
print(res)
