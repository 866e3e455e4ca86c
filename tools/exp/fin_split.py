"""Finalize with and without the MSE reduction (tooling), bracketed by libholo's events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2004_04049_b200 as hb  # noqa: E402
from holo_synth import WORKLOADS, target_for  # noqa: E402

w = WORKLOADS["C3"]
T = torch.from_numpy(target_for(w)).cuda()
acc = torch.rand((1, w.n, w.n), device="cuda")
out = torch.empty_like(acc)
mse = torch.empty(1, dtype=torch.float64, device="cuda")
ws = torch.empty(hb.ospr_workspace_bytes(w.n, 1, w.n_sub), dtype=torch.uint8, device="cuda")
for want in (False, True):
    for _ in range(3):
        hb.ospr_finalize(T, acc, w.n_sub, want_mse=want, out=out, mse_out=mse, workspace=ws)
    torch.cuda.synchronize()
    hb.profile_enable(True)
    for _ in range(20):
        hb.ospr_finalize(T, acc, w.n_sub, want_mse=want, out=out, mse_out=mse, workspace=ws)
    torch.cuda.synchronize()
    c, ms = hb.profile_read("ospr_finalize")
    hb.profile_enable(False)
    print("want_mse", want, round(1e3 * ms / c, 2), "us")
