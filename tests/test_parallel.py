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
from paper_2004_04049_b200.parallel import ShardedGs, ShardedOspr, SubframeShardPipeline, shard_range, subframe_range

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


def test_subframe_range_whole_pairs():
    """OSPR shards deal out whole Hermitian pairs (2s, 2s+1): they tile [0, n_sub), never split
    a pair, leave an odd tail on the last rank with pairs, and hold at most one pair more than
    any other rank."""
    for S in (1, 2, 3, 7, 8, 12, 13, 24, 32):
        for world in (1, 2, 3, 4, 8, 16):
            rs = [subframe_range(S, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == S
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert all(b % 2 == 0 for b, e in rs)
            pairs = [(e - b + 1) // 2 for b, e in rs]
            assert max(pairs) - min(pairs) <= 1
            odd = [r for r, (b, e) in enumerate(rs) if (e - b) % 2]
            assert odd == ([] if S % 2 == 0 else [max(r for r, (b, e) in enumerate(rs) if e > b)])


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


def oracle_gs_generate(targets, iters, lut, phase_offset=0, levels=0, **kw):
    T = targets.numpy()
    lo = None if lut is None else lut.numpy()
    n = T.shape[-1]
    mse = np.stack([oracle.gs(T[b], iters, lo, phase_offset + b * n * n, levels, (0, n, 0, n))["mse"]
                    for b in range(T.shape[0])])
    return SimpleNamespace(mse=torch.from_numpy(mse))


def oracle_finalize_rows(target, intensity_sum_rows, row0, n_sub, omega=None, out=None, sums_out=None,
                         workspace=None):
    """Stand-in for holo_ospr_finalize_rows: mean of the owned rows and the five R-12 sums
    over omega restricted to them (fp64)."""
    n = target.shape[-1]
    T = target.numpy().reshape(n, n).astype(np.float64)
    mean = intensity_sum_rows.numpy().astype(np.float64) / n_sub
    rows = mean.shape[0]
    r0, r1, c0, c1 = omega
    y = np.arange(row0, row0 + rows)[:, None]
    x = np.arange(n)[None, :]
    m = (y >= r0) & (y < r1) & (x >= c0) & (x < c1)
    I, t2 = mean[m], T[row0:row0 + rows][m] ** 2
    sums = torch.tensor([I.sum(), (I * I).sum(), (I * t2).sum(), t2.sum(), (t2 * t2).sum()], dtype=torch.float64)
    out.copy_(torch.from_numpy(mean))
    sums_out.copy_(sums)
    return out, sums_out


def oracle_mse_from_sums(sums, omega, out=None):
    """Stand-in for holo_ospr_mse_from_sums on reduced sums [F][5]."""
    cnt = (omega[1] - omega[0]) * (omega[3] - omega[2])
    res = []
    for s in sums.numpy().reshape(-1, 5):
        a = 0.0 if s[0] == 0 else s[3] / s[0]
        res.append(max(a * a * s[1] - 2 * a * s[2] + s[4], 0.0) / cnt)
    out.copy_(torch.tensor(res, dtype=torch.float64))
    return out


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
        sh = ShardedOspr(world, rank, generate=oracle_ospr_generate, finalize_rows=oracle_finalize_rows,
                         mse_from_sums=oracle_mse_from_sums,
                         reduce_scatter=lambda o, i: dist.reduce_scatter_tensor(o, i),
                         all_reduce=lambda t: dist.all_reduce(t, op=dist.ReduceOp.SUM))
        res = sh.run(torch.from_numpy(Ts), NSUB, lut, phase_offset=11)
        gTs = np.stack([blobs_target(70 + b, N, 3, 2.0, 5.0, Region.full(N)) for b in range(5)])
        (fb, fe), gres = ShardedGs(world, rank, generate=oracle_gs_generate).run(
            torch.from_numpy(gTs), 3, lut, phase_offset=5)
        # video frames with sub-frame shards: C-1 reduce-scatter, a7 on the owned rows, C-2 (gloo)
        pipe = SubframeShardPipeline(N, NSUB, world, rank, lut, device="cpu", depth=2, phase_offset=11,
                                     generate=oracle_ospr_generate, finalize_rows=oracle_finalize_rows,
                                     mse_from_sums=oracle_mse_from_sums,
                                     reduce_scatter=lambda o, i: dist.reduce_scatter_tensor(o, i),
                                     all_reduce=lambda t: dist.all_reduce(t))
        vid = []
        for f in range(3):
            pipe.submit(torch.from_numpy(Ts[f % 2].copy()))
            bits_f, mean_f, mse_f = pipe.result(f)
            vid.append((bits_f.numpy().copy(), mean_f.numpy().copy(), float(mse_f[0])))
        np.savez(os.path.join(out_dir, f"vid{rank}.npz"), rows0=pipe.rows[0], rows1=pipe.rows[1],
                 **{f"bits{f}": v[0] for f, v in enumerate(vid)}, **{f"mean{f}": v[1] for f, v in enumerate(vid)},
                 mse=np.array([v[2] for v in vid]))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), b=res.sf_range[0], e=res.sf_range[1],
                 bits=res.bits.numpy(), inten=res.intensity.numpy(), mse=res.mse.numpy(),
                 fb=fb, fe=fe, gmse=gres.mse.numpy(), r0=res.rows[0], r1=res.rows[1])
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
    assert [int(o["b"]) for o in outs] == [0, 4] and [int(o["e"]) for o in outs] == [4, NSUB]
    for o in outs:
        assert np.array_equal(o["bits"], bits_ref[:, int(o["b"]):int(o["e"])])
        # C-1: every rank holds the reduced mean of its owned rows; C-2: the MSE after the reduction
        r0, r1 = int(o["r0"]), int(o["r1"])
        assert np.max(np.abs(o["inten"] - I_ref[:, r0:r1])) <= 1e-6 * I_ref.max()
        assert np.allclose(o["mse"], mse_ref, rtol=1e-6, atol=0)
    assert [(int(o["r0"]), int(o["r1"])) for o in outs] == [(0, N // 2), (N // 2, N)]
    # GS: frames [0,2) and [2,5), initial phases drawn at the global cursor
    gTs = np.stack([blobs_target(70 + b, N, 3, 2.0, 5.0, Region.full(N)) for b in range(5)])
    full = np.stack([oracle.gs(gTs[b], 3, lo, 5 + b * N * N, 0, (0, N, 0, N))["mse"] for b in range(5)])
    got = np.concatenate([o["gmse"] for o in outs])
    assert [(int(o["fb"]), int(o["fe"])) for o in outs] == [(0, 2), (2, 5)]
    assert np.array_equal(got, full)

    # video pipeline (configs[4]'s partition): frame f = target f % 2 at cursor 11 + f N_SF N^2;
    # the owned row slices reassemble the mean, the MSE after C-2 equals the oracle's
    vids = [np.load(tmp_path / f"vid{r}.npz") for r in range(world)]
    for f in range(3):
        bref, Iref, mref = oracle.ospr(Ts[f % 2][None], NSUB, lo, 11 + f * NSUB * N * N,
                                       Region.upper_half(N).as_tuple())
        mean = np.concatenate([v[f"mean{f}"][0] for v in vids])
        assert [(int(v["rows0"]), int(v["rows1"])) for v in vids] == [(0, N // 2), (N // 2, N)]
        assert np.max(np.abs(mean - Iref[0])) <= 1e-6 * Iref.max()     # fp32 buffers
        mean = mean.reshape(N, N)
        for r, v in enumerate(vids):
            b, e = subframe_range(NSUB, world, r)
            assert np.array_equal(v[f"bits{f}"][0], bref[0, b:e])
            assert abs(v["mse"][f] - mref[0]) <= 1e-6 * mref[0]
