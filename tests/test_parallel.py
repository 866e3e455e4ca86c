"""Multi-rank host logic of paper_2004_04049_b200.parallel on CPU (gloo, world size 2).

The sharding code runs unchanged; its compute callables are replaced by
oracle-backed stand-ins (this is test code: only tests may call the oracle) so
that the partition, the global draw indices, the all-reduce of partial sums
and the finalize-after-reduce order are checked against a single-process
oracle run.
"""
import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from holo_synth import LUT_SEED, Region, blobs_target
from paper_2004_04049_b200.parallel import ShardedGs, ShardedOspr, shard_range

N, NSUB = 32, 7


def test_shard_range_partition():
    for n in (1, 5, 7, 24, 32, 60):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


# ---- oracle-backed stand-ins for the libholo calls (test doubles) -----------------------------

def oracle_ospr_generate(target, n_sub, lut, phase_offset=0, sf_range=None, want_bits=True, want_mse=True,
                         omega=None, workspace=None, out=None):
    T = target.numpy()
    T3 = T if T.ndim == 3 else T[None]
    F, n, _ = T3.shape
    b, e = sf_range
    lo = None if lut is None else lut.numpy()
    inten = np.zeros((F, n, n))
    bits = np.zeros((F, e - b, n, n // 8), np.uint8)
    for f in range(F):
        for s in range(b, e):
            cur = phase_offset + (f * n_sub + s) * n * n
            bi, _, I = oracle.ospr_subframe(T3[f], lo, cur, want_h=False, want_intensity=True)
            bits[f, s - b] = bi
            inten[f] += I
    if out is not None:                  # write into the caller's buffers (graph-style API)
        out.intensity.copy_(torch.from_numpy(inten))
        out.bits.copy_(torch.from_numpy(bits))
        return out
    return SimpleNamespace(intensity=torch.from_numpy(inten), bits=torch.from_numpy(bits), mse=None)


def oracle_ospr_finalize(target, intensity_sum, n_sub, omega=None, want_mse=True, out=None, mse_out=None,
                         workspace=None):
    T = target.numpy()
    T3 = T if T.ndim == 3 else T[None]
    mean = intensity_sum / n_sub
    if out is not None:
        out.copy_(mean)
        mean = out
    region = omega or Region.upper_half(T3.shape[-1]).as_tuple()
    mse = torch.tensor([oracle.mse_m1(mean[f].numpy(), T3[f], region) for f in range(T3.shape[0])],
                       dtype=torch.float64)
    if mse_out is not None:
        mse_out.copy_(mse)
        mse = mse_out
    return mean, mse


def oracle_gs_generate(targets, iters, lut, phase_offset=0, levels=0, **kw):
    T = targets.numpy()
    lo = None if lut is None else lut.numpy()
    n = T.shape[-1]
    mse = np.stack([oracle.gs(T[b], iters, lo, phase_offset + b * n * n, levels, (0, n, 0, n))["mse"]
                    for b in range(T.shape[0])])
    return SimpleNamespace(mse=torch.from_numpy(mse))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ts = np.stack([blobs_target(50 + f, N, 3, 2.0, 5.0, Region.upper_half(N)) for f in range(2)])
        lut = torch.from_numpy(oracle.lut_build(LUT_SEED, 257))
        sh = ShardedOspr(world, rank, generate=oracle_ospr_generate, finalize=oracle_ospr_finalize,
                         all_reduce=lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
        res = sh.run(torch.from_numpy(Ts), NSUB, lut, phase_offset=11)
        # the bench's N > 1 step structure: (shard) -> C-1 -> (finalize) into caller-owned buffers
        b, e = shard_range(NSUB, world, rank)
        buf = SimpleNamespace(bits=torch.zeros((2, e - b, N, N // 8), dtype=torch.uint8),
                              intensity=torch.zeros((2, N, N), dtype=torch.float64), mse=None)
        mse_buf = torch.zeros(2, dtype=torch.float64)
        pre, coll, post = sh.stages(torch.from_numpy(Ts), NSUB, lut, None, buf, mse_buf, phase_offset=11)
        pre()
        coll()
        post()
        gTs = np.stack([blobs_target(70 + b, N, 3, 2.0, 5.0, Region.full(N)) for b in range(5)])
        (fb, fe), gres = ShardedGs(world, rank, generate=oracle_gs_generate).run(
            torch.from_numpy(gTs), 3, lut, phase_offset=5)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), b=res.sf_range[0], e=res.sf_range[1],
                 bits=res.bits.numpy(), inten=res.intensity.numpy(), mse=res.mse.numpy(),
                 fb=fb, fe=fe, gmse=gres.mse.numpy(), st_bits=buf.bits.numpy(), st_inten=buf.intensity.numpy(),
                 st_mse=mse_buf.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_ospr_and_gs_gloo_world2(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    Ts = np.stack([blobs_target(50 + f, N, 3, 2.0, 5.0, Region.upper_half(N)) for f in range(2)])
    lo = oracle.lut_build(LUT_SEED, 257)
    bits_ref, I_ref, mse_ref = oracle.ospr(Ts, NSUB, lo, 11, Region.upper_half(N).as_tuple())
    # shards cover the sub-frames exactly once and reproduce the single-process holograms
    assert [int(o["b"]) for o in outs] == [0, 3] and [int(o["e"]) for o in outs] == [3, NSUB]
    for o in outs:
        assert np.array_equal(o["bits"], bits_ref[:, int(o["b"]):int(o["e"])])
        # every rank holds the all-reduced mean and the MSE computed after the reduction
        assert np.max(np.abs(o["inten"] - I_ref)) <= 1e-12 * I_ref.max()
        assert np.allclose(o["mse"], mse_ref, rtol=1e-12, atol=0)
        # the staged form (pre / collective / post into caller buffers) gives the same result
        assert np.array_equal(o["st_bits"], o["bits"])
        assert np.max(np.abs(o["st_inten"] - I_ref)) <= 1e-12 * I_ref.max()
        assert np.allclose(o["st_mse"], mse_ref, rtol=1e-12, atol=0)
    # GS: frames [0,2) and [2,5), initial phases drawn at the global cursor
    gTs = np.stack([blobs_target(70 + b, N, 3, 2.0, 5.0, Region.full(N)) for b in range(5)])
    full = np.stack([oracle.gs(gTs[b], 3, lo, 5 + b * N * N, 0, (0, N, 0, N))["mse"] for b in range(5)])
    got = np.concatenate([o["gmse"] for o in outs])
    assert [(int(o["fb"]), int(o["fe"])) for o in outs] == [(0, 2), (2, 5)]
    assert np.array_equal(got, full)
