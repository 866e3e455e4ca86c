"""GPU checks of the multi-GPU partition with the real libholo kernels.

* One process, one GPU: every rank's sub-frame shard is computed on the same device, the
  reduce-scatter (C-1) is emulated by summing the shards' partial intensities, a7 runs on
  each owned row slice (holo_ospr_finalize_rows), the five sums are added (C-2) and the MSE
  evaluated (holo_ospr_mse_from_sums): P-8 against the single call.
* The video pipeline (SubframeShardPipeline) on one GPU: world = 1 equals direct calls bit for
  bit; a k-way split with stand-in collectives (each rank's own slice, no exchange) exercises
  the two-stream overlap and the slot reuse against the same arithmetic done synchronously.
* >= 2 GPUs: real NCCL ranks (skipped when fewer GPUs are visible).
"""
import os
import socket

import numpy as np
import pytest
import torch

from holo_synth import LUT_SEED, Region, blobs_target
from parity import REL_TOL, cuda_target, rel, to_np

pytestmark = pytest.mark.gpu

hb = pytest.importorskip("paper_2004_04049_b200")
from paper_2004_04049_b200.parallel import SubframeShardPipeline, subframe_range  # noqa: E402


def _frame(n, seed):
    return blobs_target(seed, n, 8, n / 32, n / 10, Region.upper_half(n))


@pytest.mark.parametrize("n,S,world", [(512, 8, 2), (512, 8, 4), (512, 8, 8), (1024, 12, 4), (1024, 13, 4),
                                       (2048, 32, 8)])
def test_subframe_shards_reduce_scatter_emulated(n, S, world):
    """P-8: shards + C-1 (emulated sum) + a7 on owned rows + C-2 == the single call: bits
    bit-identical, mean intensity within 1e-6 (fp32 reassociation), MSE within 1e-5."""
    T = cuda_target(_frame(n, 40 + n))
    lut = hb.lut_generate(LUT_SEED, 10007)
    om = Region.upper_half(n).as_tuple()
    off = 123457
    ref = hb.ospr_generate(T, S, lut, phase_offset=off)
    total = torch.zeros((1, n, n), dtype=torch.float32, device=T.device)
    for r in range(world):
        b, e = subframe_range(S, world, r)
        if b == e:
            continue                     # more ranks than pairs: this rank adds zeros
        part = hb.ospr_generate(T, S, lut, phase_offset=off, sf_range=(b, e), want_mse=False)
        assert torch.equal(part.bits, ref.bits[:, b:e]), (r, b, e)
        total += part.intensity
    sums = torch.zeros(5, dtype=torch.float64, device=T.device)
    mean = torch.empty_like(total[0])
    for r in range(world):
        r0, r1 = r * n // world, (r + 1) * n // world
        m_r, s_r = hb.ospr_finalize_rows(T, total[0, r0:r1].contiguous(), r0, S, omega=om)
        mean[r0:r1] = m_r
        sums += s_r
    mse = hb.ospr_mse_from_sums(sums, om)
    I_ref = ref.intensity[0].double()
    assert (mean.double() - I_ref).abs().max().item() <= 1e-6 * I_ref.abs().max().item()
    assert rel(mse.item(), ref.mse.item()) <= 1e-5


def test_finalize_rows_whole_frame_equals_finalize():
    """Rows [0, N) reproduce holo_ospr_finalize's mean and MSE (same arithmetic per pixel)."""
    n, S = 256, 6
    T = cuda_target(_frame(n, 7))
    lut = hb.lut_generate(LUT_SEED, 4099)
    part = hb.ospr_generate(T, S, lut, sf_range=(0, S - 1), want_mse=False)   # a partial sum
    om = Region.upper_half(n).as_tuple()
    mean_f, mse_f = hb.ospr_finalize(T, part.intensity, S, omega=om)
    mean_r, sums = hb.ospr_finalize_rows(T, part.intensity[0].clone(), 0, S, omega=om)
    assert torch.equal(mean_r, mean_f[0])
    assert rel(hb.ospr_mse_from_sums(sums, om).item(), mse_f.item()) <= 1e-12


def test_pipeline_world1_equals_direct_calls():
    n, S = 1024, 8
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    Ts = [cuda_target(_frame(n, 60 + f)) for f in range(3)]
    pipe = SubframeShardPipeline(n, S, 1, 0, lut, depth=2, phase_offset=5)
    got = []
    for f in range(5):
        pipe.submit(Ts[f % 3])
        if f >= 1:
            bits, mean, mse = pipe.result(f - 1)
            got.append((bits.clone(), mean.clone(), mse.clone()))
    pipe.drain()
    bits, mean, mse = pipe.result(4)
    got.append((bits.clone(), mean.clone(), mse.clone()))
    for f in range(5):
        ref = hb.ospr_generate(Ts[f % 3], S, lut, phase_offset=5 + f * S * n * n)
        assert torch.equal(got[f][0], ref.bits) and torch.equal(got[f][1], ref.intensity)
        assert torch.equal(got[f][2], ref.mse)


@pytest.mark.parametrize("world", [2, 8])
def test_pipeline_split_streams_match_synchronous(world):
    """Rank 0 of a `world`-way split on one GPU, the collectives replaced by 'keep my own
    slice' (no exchange): every frame's outputs through the two-stream pipeline (depth 2, the
    side stream of frame f overlapping frame f+1's passes) equal the same calls made
    synchronously -- no race between the streams or in the slot reuse."""
    n, S = 2048, 32
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    Ts = [cuda_target(_frame(n, 80 + f)) for f in range(2)]
    nr = n // world

    def own_slice(out, inp):
        out.copy_(inp[:out.numel()])
    pipe = SubframeShardPipeline(n, S, world, 0, lut, depth=2, reduce_scatter=own_slice, all_reduce=lambda t: None)
    outs = []
    for f in range(6):
        pipe.submit(Ts[f % 2])
        if f >= 1:
            b_, m_, s_ = pipe.result(f - 1)
            outs.append((b_.clone(), m_.clone(), s_.clone()))
    pipe.drain()
    b_, m_, s_ = pipe.result(5)
    outs.append((b_.clone(), m_.clone(), s_.clone()))
    om = Region.upper_half(n).as_tuple()
    sb, se = subframe_range(S, world, 0)
    for f in range(6):
        part = hb.ospr_generate(Ts[f % 2][None], S, lut, phase_offset=f * S * n * n, sf_range=(sb, se),
                                want_mse=False)
        mean, sums = hb.ospr_finalize_rows(Ts[f % 2], part.intensity[0, :nr].contiguous(), 0, S, omega=om)
        mean = mean[None]
        mse = hb.ospr_mse_from_sums(sums, om)
        assert torch.equal(outs[f][0], part.bits), f
        assert torch.equal(outs[f][1], mean), f
        assert torch.equal(outs[f][2], mse), f


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _nccl_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        n, S = 2048, 32
        lut = hb.lut_generate(LUT_SEED, 1 << 16)
        Ts = [cuda_target(_frame(n, 80 + f)) for f in range(2)]
        pipe = SubframeShardPipeline(n, S, world, rank, lut, depth=2)
        res = []
        for f in range(3):
            pipe.submit(Ts[f % 2])
        pipe.drain()
        for f in range(1, 3):
            b_, m_, s_ = pipe.result(f)
            res.append((to_np(b_), to_np(m_), float(s_.item())))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), **{f"b{i}": r[0] for i, r in enumerate(res)},
                 **{f"m{i}": r[1] for i, r in enumerate(res)}, mse=np.array([r[2] for r in res]))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_pipeline_nccl_ranks_match_single_gpu(tmp_path):
    """P-8 with real NCCL ranks: bits of every shard identical to the 1-GPU call, the owned
    row slices reassemble its mean intensity (1e-6), and every rank's MSE matches it (1e-5)."""
    import torch.multiprocessing as mp
    world = 1 << (min(torch.cuda.device_count(), 8).bit_length() - 1)   # a power of two: divides N and N_SF
    mp.start_processes(_nccl_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    n, S = 2048, 32
    lut = hb.lut_generate(LUT_SEED, 1 << 16)
    for i, f in enumerate((1, 2)):
        T = cuda_target(_frame(n, 80 + f % 2))
        ref = hb.ospr_generate(T, S, lut, phase_offset=f * S * n * n)
        mean = np.concatenate([o[f"m{i}"][0] for o in outs])
        I_ref = to_np(ref.intensity[0]).astype(np.float64)
        assert np.max(np.abs(mean - I_ref)) <= 1e-6 * np.max(I_ref)
        for r, o in enumerate(outs):
            b, e = subframe_range(S, world, r)
            assert np.array_equal(o[f"b{i}"][0], to_np(ref.bits[0, b:e]))
            assert rel(o["mse"][i], ref.mse.item()) <= 1e-5
