"""The pipelined frame stream (paper_2004_04049_b200.stream): every frame set
it returns must be bit-identical to a direct ospr_generate call at the continuing cursor
off0 + f N_SF N^2 (R-2), whatever the pipeline depth; one frame set is also checked against
the fp64 oracle (P-3 protocol)."""
import numpy as np
import pytest
import torch

import oracle
from holo_synth import LUT_SEED, Region, blobs_target
from parity import check_bits, cuda_target, lut_pair, to_np

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")


def targets(n, k, seed):
    return [blobs_target(seed + i, n, 6, max(1.0, n / 16), max(2.0, n / 6), Region.upper_half(n)) for i in range(k)]


@pytest.mark.parametrize("n,S,L,depth,advance,stride", [
    (256, 6, 1021, 3, True, 1),
    (256, 5, 1021, 2, True, 1),       # odd N_SF: unpaired last sub-frame
    (128, 4, 4096, 1, True, 1),       # depth 1: fully serialised
    (256, 6, 1021, 3, False, 1),      # every frame set at off0
    (256, 6, 1021, 3, True, 4),       # stream 0 of 4 (one per GPU): global frame sets 0, 4, 8, ...
    (1024, 24, 1 << 16, 3, True, 1),  # C3
])
def test_stream_matches_direct_calls(n, S, L, depth, advance, stride):
    off0 = 12345
    lg, _ = lut_pair(LUT_SEED, L)
    Ts = targets(n, 7, 600 + n)
    hosts = [torch.from_numpy(T).pin_memory() for T in Ts]
    st = hb.OsprStream(n, S, lg, depth=depth, phase_offset=off0, advance=advance, frame_stride=stride,
                       want_intensity=True)
    got = []
    for f, h in enumerate(hosts):
        st.submit(h)
        if f >= depth - 1:                       # consume each frame set before its slot is reused
            g = f - depth + 1
            b, m, i = st.result(g)
            got.append((g, b.clone(), m.clone(), i.clone()))
    st.drain()
    for g in range(len(hosts) - depth + 1, len(hosts)):
        b, m, i = st.result(g)
        got.append((g, b.clone(), m.clone(), i.clone()))
    assert [g for g, *_ in got] == list(range(len(hosts)))
    P = n * n
    for g, b, m, i in got:
        ref = hb.ospr_generate(cuda_target(Ts[g]), S, lg, phase_offset=off0 + (g * stride * S * P if advance else 0))
        torch.cuda.synchronize()
        assert torch.equal(b, ref.bits[0].cpu()), g
        assert torch.equal(m, ref.mse.cpu()), g
        assert torch.equal(i, ref.intensity[0].cpu()), g


def test_stream_frame_against_oracle():
    n, S, L, off0 = 64, 4, 257, 99
    lg, lo = lut_pair(LUT_SEED, L)
    Ts = targets(n, 3, 700)
    st = hb.OsprStream(n, S, lg, depth=2, phase_offset=off0)
    for T in Ts:
        st.submit(torch.from_numpy(T).pin_memory())
    bits, _, _ = st.result(2)
    bits = bits.numpy()
    P = n * n
    for s in range(S):
        _, h_re, _ = oracle.ospr_subframe(Ts[2], lo, off0 + (2 * S + s) * P, want_h=True, want_intensity=False)
        check_bits(bits[s], h_re, n)


def test_stream_rejects_stale_frames():
    st = hb.OsprStream(64, 2, None, depth=2)
    h = torch.zeros((64, 64), dtype=torch.float32).pin_memory()
    for _ in range(3):
        st.submit(h)
    with pytest.raises(ValueError):
        st.result(0)                             # slot reused by frame set 2
    st.result(2)
    with pytest.raises(ValueError):
        st.submit(torch.zeros((32, 32), dtype=torch.float32))


def test_native_a0_and_python_sequencer_agree():
    """The native sequencer with a0 per frame set (lut_seed: holo_lut_generate into the pool on the
    compute stream before each frame set) and the Python sequencer with the same a0 as a
    before_each hook give the direct calls' holograms and MSE, bit for bit."""
    n, S, L, off0 = 256, 6, 4099, 777
    Ts = targets(n, 5, 900)
    hosts = [torch.from_numpy(T).pin_memory() for T in Ts]
    lut_a = torch.zeros(L, dtype=torch.complex64, device="cuda")          # garbage-free but not the pool
    lut_b = torch.zeros(L, dtype=torch.complex64, device="cuda")
    nat = hb.OsprStream(n, S, lut_a, depth=2, phase_offset=off0, lut_seed=LUT_SEED)
    py = hb.OsprStream(n, S, lut_b, depth=2, phase_offset=off0,
                       before_each=lambda: hb.lut_generate(LUT_SEED, L, out=lut_b))
    assert nat._native is not None and py._native is None
    ref_lut = hb.lut_generate(LUT_SEED, L)
    for f, h in enumerate(hosts):
        nat.submit(h)
        py.submit(h)
        b1, m1, _ = nat.result(f)
        b2, m2, _ = py.result(f)
        ref = hb.ospr_generate(torch.from_numpy(Ts[f]).cuda(), S, ref_lut, phase_offset=off0 + f * S * n * n)
        assert torch.equal(b1, ref.bits[0].cpu()) and torch.equal(b2, ref.bits[0].cpu()), f
        assert m1.item() == ref.mse.item() and m2.item() == ref.mse.item(), f
    assert nat.done(len(hosts) - 1)
    nat.close()
    with pytest.raises(RuntimeError):
        nat.submit(hosts[0])                     # the native streams are gone
    with pytest.raises(ValueError):
        hb.OsprStream(n, S, lut_a, lut_seed=1, before_each=lambda: None)
