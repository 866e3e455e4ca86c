#!/usr/bin/env python3
"""Benchmark of the B200 hot path of arXiv 2004.04049 (OSPR + GS with LUT phase
randomisation), BASELINE.json metric "OSPR 1024^2 binary sub-frames/s & GS
iters/s; achieved HBM GB/s vs peak".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl holo|reference]

One step = one pass of every hot-path row of SURVEY.md §8(a) over one batch:
  OSPR (headline `value`): BASELINE configs[2] (C3) -- a0 LUT build (L = 2^16 by
  default) + a1-a7 for one frame set of N_SF = 24 binary 1024x1024 sub-frames
  (holograms, mean replay intensity, MSE), inputs resident in HBM.
  GS (`gs` block): BASELINE configs[3] (C4) -- 64 frames x 50 iterations at
  1024x1024, continuous phase-only, LUT 2^16.
  C5 video (`c5_video` block): BASELINE configs[4] -- 2048^2 frames, N_SF = 32,
  streamed back to back.
Timing: W untimed warm-up steps, then K steps, each bracketed by a barrier and
torch.cuda.synchronize(); L2 is flushed (256 MiB write) before every timed step;
CUDA events on the launching stream; max over ranks.
Multi-GPU (torchrun, one process per GPU, NCCL):
  * C3 headline (`--ospr-shard frames`, default): rank r runs its own frame set r
    (global cursor, R-2) -- independent problems, no collective, weak scaling;
    `--ospr-shard subframes` splits one frame set's sub-frames over the ranks
    instead (reduce-scatter + a7 on the owned rows + 5-double all-reduce).
  * C5 video: every frame's sub-frames are split over the ranks (configs[4]'s
    partition); C-1 = NCCL reduce-scatter of the partial intensity (each rank owns
    2048/N rows), a7 on the owned rows, C-2 = NCCL all-reduce of five doubles, then
    the MSE, all on a side stream overlapping the next frame's passes.
  * GS: the C4 frames are sharded (no collective).
`--impl reference` times the fp64 CPU oracle (oracle/) on the host cores on the
same workload (the paper has no GPU implementation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "OSPR 1024^2 binary sub-frames/s"
UNIT = "sub-frames/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["holo", "reference"], default="holo")
    ap.add_argument("--lut", type=int, default=1 << 16, help="headline LUT length")
    ap.add_argument("--ospr-shard", choices=["frames", "subframes"], default="frames",
                    help="N > 1: each rank its own C3 frame set (weak, no collective; default) or one frame "
                         "set's sub-frames split across ranks + NCCL reduce-scatter of the partial intensity, "
                         "a7 on the owned rows and an all-reduce of five doubles (strong)")
    ap.add_argument("--no-gs", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gs-steps", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every step eagerly instead of replaying a captured CUDA graph")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        mhz, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                mhz.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(mhz)}


# ---------------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------------
def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_loop(step_fn, k, w, world, flush):
    """W warm-up steps, then K timed steps bracketed as a block by a barrier + device sync on
    both sides.  Inside the block each step is: L2 flush, event, step, event, all enqueued
    on the stream without a host sync, so the host queues step i+1 while the device runs
    step i.  The step time is the sum of the per-step event intervals: device time of the
    steps alone, the flushes between them excluded."""
    import torch
    for _ in range(w):
        step_fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    barrier(world)
    torch.cuda.synchronize()
    evs = []
    for _ in range(k):
        flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        step_fn()
        b.record(s)
        evs.append((a, b))
    torch.cuda.synchronize()
    barrier(world)
    per = [a.elapsed_time(b) for a, b in evs]
    return sum(per), per


HBM_SPEC_GBS = 8000.0   # B200 datasheet HBM3e bandwidth (report both denominators)


def fft_rate(units_per_s, P, paired):
    """FFT GFLOP/s at 5 P log2 P flop per 2D transform of P points (BASELINE north_star's
    count), two transforms (back- and forward-propagation) per unit.  `nominal` counts every
    unit's own transforms; `executed` the transforms actually run (Hermitian pairing packs two
    OSPR sub-frames into one complex transform)."""
    per_unit = 2 * 5 * P * math.log2(P)
    nominal = units_per_s * per_unit / 1e9
    return {"unit": "GFLOP/s", "nominal": nominal, "executed": nominal / 2 if paired else nominal,
            "flop_per_unit_nominal": per_unit, "count": "5 P log2 P per 2D DFT of P points, 2 per unit"}


def graphed(step_fn, enabled):
    """Capture one step (after it has run eagerly once, so every one-off host set-up --
    twiddle tables, shared-memory opt-ins -- is done) into a CUDA graph and return its
    replay; the step's kernels then launch without per-kernel host overhead."""
    if not enabled:
        return step_fn
    import torch
    step_fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step_fn()
    torch.cuda.synchronize()
    return g.replay


def ncu_traffic(kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or (None, None)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = d["kernels"][kernel]
        return e["dram_bytes_per_launch"], d["source"]
    except Exception:
        return None, None


def kernel_times(hb, step_fn, steps, flush, use_graph):
    """{kernel class: launches, total_ms, avg_us} over `steps` steps.  Graph mode captures the
    step once more with libholo's profiling on (event-record nodes around every kernel) and
    reads the events after each replay; eager mode brackets each launch directly."""
    import torch
    acc = {}

    def collect():
        for name in hb.kernel_names():
            cnt, ms = hb.profile_read(name)
            if cnt:
                a = acc.setdefault(name, [0, 0.0])
                a[0] += cnt
                a[1] += ms

    hb.profile_enable(True)
    if use_graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step_fn()
        torch.cuda.synchronize()
        for _ in range(steps):
            flush()
            g.replay()
            torch.cuda.synchronize()
            collect()
    else:
        for _ in range(steps):
            flush()
            step_fn()
        torch.cuda.synchronize()
        collect()
    hb.profile_enable(False)
    if use_graph:
        del g
    return {k: {"launches": v[0], "total_ms": v[1], "avg_us": 1e3 * v[1] / v[0]} for k, v in acc.items()}


def graphed_stages(pre, collective, post, enabled):
    """A step made of local parts around one (eager) collective: pre and post (None: nothing)
    are each captured into a CUDA graph (after one eager run), the collective (NCCL) runs
    eagerly between them; a collective marked `.local` (nothing to exchange) is captured too."""
    post = post or (lambda: None)
    if not enabled:
        def eager():
            pre()
            collective()
            post()
        return eager
    import torch
    pre()
    collective()
    post()
    torch.cuda.synchronize()
    if getattr(collective, "local", False):   # no exchange (one rank): one graph for the whole step
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            pre()
            collective()
            post()
        torch.cuda.synchronize()
        return g.replay
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1):
        pre()
    torch.cuda.synchronize()

    def replay():
        g1.replay()
        collective()
        post()
    return replay


def run_gpu(args):
    import torch
    import paper_2004_04049_b200 as hb
    from holo_synth import LUT_SEED, WORKLOADS, target_for

    world, rank, local = dist_setup(args)
    dev = torch.device("cuda", torch.cuda.current_device())
    props = torch.cuda.get_device_properties(dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        flush_buf.fill_(1)

    # ---------------- OSPR C3 ----------------
    w3 = WORKLOADS["C3"]
    n, S, P = w3.n, w3.n_sub, w3.n * w3.n
    T = torch.from_numpy(target_for(w3)).to(dev)
    from paper_2004_04049_b200.parallel import shard_range, subframe_range  # noqa: F401
    # HOLO_BENCH_FAKE_WORLD=k (testing only, N = 1): run rank 0's shard of a k-way split with a
    # no-op collective, to exercise the N > 1 step structure (graphs around the collective)
    fake = int(os.environ.get("HOLO_BENCH_FAKE_WORLD", "0")) if world == 1 else 0
    mode = "subframes" if fake > 1 else args.ospr_shard
    # frames: rank r runs global frame set r (cursor off0 + r N_SF P, R-2), independent of the
    # others -- no collective; subframes: one frame set's sub-frames split over the ranks, C-1
    frames_mode = (mode == "frames")
    sworld = 1 if frames_mode else (fake if fake > 1 else world)
    srank = 0 if frames_mode else rank
    frame_off = rank * S * P if frames_mode else 0
    sb, se = subframe_range(S, sworld, srank)
    full = (sworld == 1)
    ws = torch.empty(hb.ospr_workspace_bytes(n, 1, S), dtype=torch.uint8, device=dev)
    lut_buf = torch.empty(max(args.lut, 1), dtype=torch.complex64, device=dev)
    out = hb.OsprResult(bits=torch.empty((1, se - sb, n, n // 8), dtype=torch.uint8, device=dev),
                        intensity=torch.empty((1, n, n), dtype=torch.float32, device=dev),
                        mse=torch.empty(1, dtype=torch.float64, device=dev) if full else None)
    mse_buf = torch.empty(1, dtype=torch.float64, device=dev)

    from paper_2004_04049_b200.parallel import ShardedOspr
    stand_in = dict(reduce_scatter=lambda o, i: o.copy_(i[:o.numel()]), all_reduce=lambda t: None)
    sharded = ShardedOspr(sworld, srank, **(stand_in if fake > 1 else {}))
    if not full:
        r0, r1 = sharded.rows(n)
        mean_rows = torch.empty((1, r1 - r0, n), dtype=torch.float32, device=dev)
        sums_buf = torch.zeros((1, 5), dtype=torch.float64, device=dev)
        fin_ws = torch.empty(int(hb.lib().holo_ospr_finalize_workspace_size()), dtype=torch.uint8, device=dev)

    def ospr_stages(L, lut, T_in=None):
        """(pre, exchange) of one OSPR step: a0 + this rank's shard (the whole frame set, a7
        fused, when it is not split); for a split, the exchange C-1 (reduce-scatter of the
        partial intensity) + a7 on the owned rows + C-2 (five doubles) + MSE, eager (NCCL)."""
        Tx = T if T_in is None else T_in

        def pre_a0():
            hb.lut_generate(LUT_SEED, L, out=lut[:L])                               # a0
            if full:
                out.mse = mse_buf
                hb.ospr_generate(Tx, S, lut[:L], phase_offset=frame_off, workspace=ws, out=out)   # a1-a7
            else:
                hb.ospr_generate(Tx, S, lut[:L], phase_offset=frame_off, sf_range=(sb, se), want_mse=False,
                                 workspace=ws, out=out)                             # a1-a6 (shard)

        def exchange():
            if not full:
                sharded.exchange(Tx, out.intensity, S, mean_rows, sums_buf, mse_buf, None, fin_workspace=fin_ws)
        exchange.local = full
        return pre_a0, exchange

    def make_ospr_step(L, lut):
        pre, exch = ospr_stages(L, lut)

        def step():
            pre()
            exch()
        return step

    use_graph = not args.no_graph
    step = make_ospr_step(args.lut, lut_buf)
    l0 = hb.launch_count()
    step()
    launches_per_step = hb.launch_count() - l0                 # libholo kernels in one step
    timed_step = graphed_stages(*ospr_stages(args.lut, lut_buf), None, use_graph)
    with Clocks(local) as clk:
        # the timed block lasts milliseconds; the sampler (100 ms period) sees the clocks of the
        # same step running untimed for 0.6 s right before it (extra warm-up, same load)
        t0 = time.perf_counter()
        for _ in range(5):
            flush()
            timed_step()
        torch.cuda.synchronize()
        n_load = min(20000, int(max_over_ranks(math.ceil(0.6 / max((time.perf_counter() - t0) / 5, 1e-5)), world)))
        for _ in range(n_load):      # the same count on every rank (the step may hold a collective)
            flush()
            timed_step()
        torch.cuda.synchronize()
        total_ms, per = timed_loop(timed_step, args.steps, args.warmup, world, flush)
    launches_timed = launches_per_step * args.steps
    total_ms = max_over_ranks(total_ms, world)
    ms_step = total_ms / args.steps
    sets_per_step = world if frames_mode else 1               # frame sets all ranks finish per step
    value = sets_per_step * S * args.steps / (total_ms / 1e3)

    # per-kernel device time: the same step in the same launch configuration, every kernel
    # bracketed by CUDA events on its launch stream, K more steps after an L2 flush each
    kern = kernel_times(hb, step, args.steps, flush, use_graph and sworld == 1)   # (no NCCL in a graph)
    step_kernel_ms = sum(v["total_ms"] for v in kern.values()) / args.steps

    # roofline of the dominant kernel (algorithmic bytes per launch)
    npairs = (se - sb + 1) // 2
    chunk = hb.ospr_chunk_pairs(n, S)
    nchunks = -(-npairs // chunk)
    np_l = npairs / nchunks                                      # pairs per launch (average)
    nsub_l = (se - sb) / nchunks                                 # sub-frames per launch
    fused_a7 = "ospr_finalize" not in kern                       # N >= 1024: a7 runs inside pass C
    alg_bytes = {                                                # DESIGN.md §7 table
        "ospr_rows_a": 4 * P + 8 * min(args.lut, 2 * np_l * P) + 8 * P * np_l,
        "ospr_cols": 16 * P * np_l + nsub_l * P / 8,
        # pass C: pair rows in; fused a7: T in, intensity out, sign bytes -> packed holograms
        "ospr_rows_c": (8 * P * np_l + 8 * P + 2 * (se - sb) * P / 8) if fused_a7 else
                       (8 * P * np_l + 4 * P + (4 * P if nchunks > 1 else 0) * (nchunks - 1) / nchunks),
        "ospr_finalize": 12 * P + 2 * (se - sb) * P / 8,             # + sign bytes -> packed holograms
    }
    dom = max((k for k in kern if k in alg_bytes), key=lambda k: kern[k]["total_ms"])
    per_launch = alg_bytes[dom]
    achieved = per_launch / (kern[dom]["avg_us"] * 1e-6) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    share = kern[dom]["total_ms"] / args.steps / step_kernel_ms
    traffic, traffic_src = ncu_traffic(dom)

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if frames_mode else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded Gaussian-blob targets, holo_synth; stands in for USC-SIPI images)",
        "config": {"workload": "C3: OSPR 1024x1024 binary, N_SF=24, one frame set per step and GPU (a0 LUT "
                               "build + a1-a7 incl. MSE); BASELINE configs[2]",
                   "n": n, "n_sub": S, "lut_len": args.lut, "lut_seed": LUT_SEED,
                   "l2": "flushed before every timed step (256 MiB write)",
                   "launch": ("CUDA graph replay of the step (captured once)" if sworld == 1 else
                              "CUDA graph replay of the shard, then the eager exchange (NCCL)") if use_graph
                             else "eager launches",
                   "parallelism": (f"frame-set shards x{world}: rank r runs global frame set r (cursor off0 + "
                                   "r*N_SF*N^2), no collective" if frames_mode else
                                   f"sub-frame shards x{sworld} + NCCL reduce-scatter of the partial intensity "
                                   "(C-1), a7 on the owned rows, NCCL all-reduce of 5 doubles (C-2)")},
        "gpu_launches": launches_timed,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "dram_frac": (traffic / (kern[dom]["avg_us"] * 1e-6) / 1e9 / hbm_peak) if traffic else None,
                     "algorithmic_bytes_per_launch": per_launch, "avg_launch_us": kern[dom]["avg_us"],
                     "share_of_step": share, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                     "peak_spec": HBM_SPEC_GBS, "frac_spec": achieved / HBM_SPEC_GBS},
        "fft": fft_rate(value, P, paired=True),
        "kernels": kern,
        "clocks": clk.summary(),
        "device": {"name": props.name, "sms": props.multi_processor_count,
                   "l2_mb": getattr(props, "L2_cache_size", 0) / 2 ** 20},
    }

    # ---------------- LUT sweep of C3 ----------------
    if not args.no_sweep and world == 1:
        sweep = {}
        big = torch.empty(max(w3.lut_lens), dtype=torch.complex64, device=dev)
        # BASELINE's lengths all divide N_SF N^2 (every sub-frame draws the same phases, SURVEY G-8);
        # 65537 (prime) is the non-degenerate control at the same pool size
        for L in tuple(w3.lut_lens) + (65537,):
            st = graphed(make_ospr_step(L, big), use_graph)
            tm, _ = timed_loop(st, max(3, args.steps // 2), 2, world, flush)
            sweep[str(L)] = {"sub_frames_per_s": S * max(3, args.steps // 2) / (tm / 1e3),
                             "ms_per_step": tm / max(3, args.steps // 2), "mse": float(out.mse.item())}
        # no pool at all -- SplitMix64 + R-5 per draw in pass A (bit-identical
        # to the full-length pool above, which it replaces: the paper's memory-vs-compute trade-off)
        def prng_step():
            hb.ospr_generate(T, S, prng_seed=LUT_SEED, workspace=ws, out=out)
        st = graphed(prng_step, use_graph)
        ks = max(3, args.steps // 2)
        tm, _ = timed_loop(st, ks, 2, world, flush)
        sweep["prng"] = {"sub_frames_per_s": S * ks / (tm / 1e3), "ms_per_step": tm / ks,
                         "mse": float(out.mse.item()),
                         "what": "phases drawn on the fly (holo_ospr_generate_prng), no LUT"}
        # P:170's runtime-flexible alternative (R-25): SplitMix64 per draw indexing a 2^q sin/cos table
        for q in (8, 12, 16):
            tbl = torch.empty(1 << q, dtype=torch.complex64, device=dev)

            def table_step(q=q, tbl=tbl):
                hb.phase_table(q, out=tbl)
                hb.ospr_generate(T, S, prng_seed=LUT_SEED, phase_bits=q, table=tbl, workspace=ws, out=out)
            st = graphed(table_step, use_graph)
            tm, _ = timed_loop(st, ks, 2, world, flush)
            sweep[f"prng_table_q{q}"] = {"sub_frames_per_s": S * ks / (tm / 1e3), "ms_per_step": tm / ks,
                                         "mse": float(out.mse.item()),
                                         "what": f"SplitMix64 per draw + a 2^{q}-entry sin/cos table "
                                                 "(holo_ospr_generate_prng_table; phases quantised to "
                                                 f"{1 << q} levels)"}
        result["lut_sweep"] = sweep
        del big

    # ---------------- e2e through the public API with host buffers ----------------
    if not args.no_e2e and frames_mode:
        # the frame stream: pinned host target -> H2D -> a0 + ospr_generate ->
        # D2H of the packed holograms and MSE, per frame set, pipelined over three CUDA streams;
        # rank r streams global frame sets r, r + N, r + 2N, ...
        hosts = [torch.from_numpy(target_for(w3)).pin_memory() for _ in range(3)]
        lut_e2e = torch.empty(max(args.lut, 1), dtype=torch.complex64, device=dev)
        stream = hb.OsprStream(n, S, lut_e2e[:args.lut], depth=3, phase_offset=rank * S * P, frame_stride=world,
                               lut_seed=LUT_SEED)                       # a0 per frame set, native sequencer
        for i in range(args.warmup):
            stream.submit(hosts[i % 3])
        stream.drain()
        torch.cuda.synchronize()
        barrier(world)
        ke = max(args.steps, 60)   # frame sets streamed: amortises the pipeline's fill and drain
        first = stream.f
        reps = []
        for _ in range(3):         # the host is in the loop: the median of three runs
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream.h2d)
            for i in range(ke):
                stream.submit(hosts[i % 3])
            b.record(stream.d2h)
            torch.cuda.synchronize()
            barrier(world)
            reps.append(max_over_ranks(a.elapsed_time(b), world))
        tm = statistics.median(reps)
        mse_e2e = float(stream.result(stream.f - 1)[1][0])
        # the box's own host-link rates for these transfers (copies alone, pinned buffers), so that
        # the e2e number can be read against them: it is bounded by max(kernels, H2D, D2H) per set
        pcie = {}
        dev_t = torch.empty(hosts[0].shape, dtype=torch.float32, device=dev)
        dev_b = torch.empty(stream.bits_host[0].shape, dtype=torch.uint8, device=dev)
        for name, dst, src in (("h2d", dev_t, hosts[0]), ("d2h", stream.bits_host[0], dev_b)):
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                dst.copy_(src, non_blocking=True)
            b.record()
            torch.cuda.synchronize()
            pcie[name + "_gbs"] = 20 * src.numel() * src.element_size() / (a.elapsed_time(b) * 1e-3) / 1e9
        del dev_t, dev_b
        result["e2e"] = {"value": world * S * ke / (tm / 1e3), "unit": UNIT, "frame_sets_timed": ke,
                         "runs_ms": reps, "statistic": "median of 3 runs",
                         "h2d_bytes_per_step": world * hosts[0].numel() * 4,
                         "d2h_bytes_per_step": world * (stream.bits_host[0].numel() + 8),
                         "bytes_per_step": "all ranks (one frame set per rank per step)",
                         "ms_per_step": tm / ke, "frame_sets": [first, stream.f], "mse_last": mse_e2e,
                         "host_link": pcie,
                         "what": "paper_2004_04049_b200.OsprStream (public API): per frame set a pinned host target "
                                 "-> device, a0 LUT build, ospr_generate (a1-a7) with the continuing cursor, packed "
                                 "holograms + MSE -> pinned host; H2D of f+1 and D2H of f-1 overlap the kernels of "
                                 "f (3 CUDA streams, 3 slots, eager launches, one native holo_ospr_stream_submit "
                                 "per frame set); timed by events from the first H2D to the last D2H",
                         "l2": "not flushed between pipelined frame sets; every input of a frame set is produced "
                               "inside it (target by its H2D, LUT by a0)"}
    elif not args.no_e2e:
        T_host = torch.from_numpy(target_for(w3)).pin_memory()
        bits_host = torch.empty(out.bits.shape, dtype=torch.uint8).pin_memory()
        mse_host = torch.empty(1, dtype=torch.float64).pin_memory()
        T_dev = torch.empty_like(T)
        lut_e2e = hb.lut_generate(LUT_SEED, args.lut, device=dev)

        pre, coll = ospr_stages(args.lut, lut_e2e, T_in=T_dev)

        def e2e_pre():
            T_dev.copy_(T_host, non_blocking=True)                              # H2D inputs
            pre()                                                               # a0, a1-a6 (shard)

        def e2e_post():                                                         # (a7 in the exchange)
            mse_host.copy_(mse_buf, non_blocking=True)                          # D2H metric
            bits_host.copy_(out.bits, non_blocking=True)                        # D2H holograms
        tm, _ = timed_loop(graphed_stages(e2e_pre, coll, e2e_post, use_graph), args.steps, args.warmup, world,
                           flush)
        tm = max_over_ranks(tm, world)
        result["e2e"] = {"value": S * args.steps / (tm / 1e3), "unit": UNIT,
                         "h2d_bytes_per_step": T_host.numel() * 4,
                         "d2h_bytes_per_step": bits_host.numel() + 8,
                         "what": "pinned host target -> device, a0 LUT build, ospr_generate (a1-a7), packed "
                                 "holograms + MSE -> host; " + ("CUDA graphs (memcpy + kernel nodes)"
                                                                if use_graph else "eager")}

    # ---------------- OSPR C5 frame sets (2048^2, N_SF = 32) ----------------
    if not args.no_c5 and world == 1:
        w5 = WORKLOADS["C5"]
        n5, S5, P5 = w5.n, w5.n_sub, w5.n * w5.n
        T5 = torch.from_numpy(target_for(w5, rank)).to(dev)     # rank r: frame r of the video
        lut5 = torch.empty(w5.lut_lens[0], dtype=torch.complex64, device=dev)
        ws5 = torch.empty(hb.ospr_workspace_bytes(n5, 1, S5), dtype=torch.uint8, device=dev)
        out5 = hb.OsprResult(bits=torch.empty((1, S5, n5, n5 // 8), dtype=torch.uint8, device=dev),
                             intensity=torch.empty((1, n5, n5), dtype=torch.float32, device=dev),
                             mse=torch.empty(1, dtype=torch.float64, device=dev))

        def c5_step():
            hb.lut_generate(LUT_SEED, w5.lut_lens[0], out=lut5)
            hb.ospr_generate(T5, S5, lut5, phase_offset=rank * S5 * P5, workspace=ws5, out=out5)
        k5 = max(3, args.steps // 4)
        tm5, _ = timed_loop(graphed(c5_step, use_graph), k5, min(args.warmup, 3), world, flush)
        tm5 = max_over_ranks(tm5, world)
        np5 = (S5 + 1) // 2
        bytes5 = 32 * P5 * np5 + 4 * P5 + 12 * P5 + 3 * S5 * P5 / 8   # passes A-C + finalize + sign bytes
        result["c5"] = {
            "metric": "OSPR 2048^2 binary sub-frames/s", "unit": UNIT,
            "value": world * S5 * k5 / (tm5 / 1e3), "ms_per_step": tm5 / k5, "steps": k5,
            "scaling": "weak", "mse": float(out5.mse.item()),
            "step_hbm": {"algorithmic_bytes": bytes5, "achieved_gbs": bytes5 / (tm5 / k5 * 1e-3) / 1e9,
                         "frac": bytes5 / (tm5 / k5 * 1e-3) / 1e9 / hbm_peak},
            "config": {"workload": "C5 frame set: OSPR 2048x2048 binary, N_SF=32, LUT 2^16, one video frame per "
                                   "step and GPU (a0 + a1-a7); BASELINE configs[4] (its 60-frame video is 60 such "
                                   "steps)", "l2": "flushed before every timed step",
                       "launch": "CUDA graph replay" if use_graph else "eager launches"},
        }
        del ws5

    # ---------------- OSPR C5 video: sub-frame shards + C-1/C-2 on a side stream (configs[4]) ----------------
    if not args.no_c5:
        result["c5_video"] = c5_video(args, hb, world, rank, dev, flush)

    # ---------------- GS C4 ----------------
    if not args.no_gs:
        w4 = WORKLOADS["C4"]
        B, iters, n4 = w4.frames, w4.iters, w4.n
        from paper_2004_04049_b200.parallel import shard_range
        fb, fe = shard_range(B, world, rank)
        T4 = torch.from_numpy(np.stack([target_for(w4, b) for b in range(fb, fe)])).to(dev)
        lut4 = torch.empty(1 << 16, dtype=torch.complex64, device=dev)
        ws4 = torch.empty(hb.gs_workspace_bytes(n4, fe - fb, iters), dtype=torch.uint8, device=dev)
        gout = hb.GsResult(holo=torch.empty((fe - fb, n4, n4), dtype=torch.complex64, device=dev), levels=None,
                           intensity=torch.empty((fe - fb, n4, n4), dtype=torch.float32, device=dev),
                           mse=torch.empty((fe - fb, iters), dtype=torch.float64, device=dev),
                           err_e=torch.empty((fe - fb, iters), dtype=torch.float64, device=dev))

        from paper_2004_04049_b200.parallel import ShardedGs
        gsh = ShardedGs(world, rank)

        def gs_step():
            hb.lut_generate(LUT_SEED, 1 << 16, out=lut4)
            hb.gs_generate(T4, iters, lut4, phase_offset=gsh.frame_range(B)[0] * n4 * n4, levels=0,
                           workspace=ws4, out=gout)
        ks = args.gs_steps or max(3, args.steps // 4)
        gs_timed = graphed(gs_step, use_graph)
        gm, _ = timed_loop(gs_timed, ks, min(args.warmup, 3), world, flush)
        gk = kernel_times(hb, gs_step, 1, flush, use_graph)
        gm = max_over_ranks(gm, world)
        P4 = n4 * n4
        g = hb.gs_group_frames(n4, fe - fb)
        gbytes = {"gs_cols": 16 * P4 * g, "gs_rows": 20 * P4 * g}
        gdom = max(gbytes, key=lambda k: gk.get(k, {"total_ms": 0})["total_ms"])
        gach = gbytes[gdom] / (gk[gdom]["avg_us"] * 1e-6) / 1e9
        gtraffic, gtraffic_src = ncu_traffic(gdom)   # DRAM bytes per launch at C4 size (64 frames)
        result["gs"] = {
            "metric": "GS 1024^2 iterations/s", "unit": "frame-iterations/s",
            "value": B * iters * ks / (gm / 1e3), "ms_per_step": gm / ks, "steps": ks,
            "config": {"workload": "C4: GS 1024x1024, 64 frames x 50 iterations, continuous phase-only, "
                                   "LUT 2^16; BASELINE configs[3]", "frames_per_rank": fe - fb,
                       "launch": "CUDA graph replay" if use_graph else "eager launches"},
            "roofline": {"bound": "hbm", "kernel": gdom, "achieved": gach, "peak": hbm_peak, "unit": "GB/s",
                         "frac": gach / hbm_peak, "algorithmic_bytes_per_launch": gbytes[gdom],
                         "avg_launch_us": gk[gdom]["avg_us"], "peak_spec": HBM_SPEC_GBS,
                         "frac_spec": gach / HBM_SPEC_GBS,
                         "traffic": gtraffic, "traffic_source": gtraffic_src,
                         "dram_frac": (gtraffic / (gk[gdom]["avg_us"] * 1e-6) / 1e9 / hbm_peak
                                       if gtraffic else None)},
            "fft": fft_rate(B * iters * ks / (gm / 1e3), P4, paired=False),
            "kernels": gk,
        }

    if rank == 0 and world == 1:
        result["cpu_baseline"] = cpu_baseline(args.lut)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result))


def c5_video(args, hb, world, rank, dev, flush):
    """BASELINE configs[4]: a stream of 2048^2 video frames, N_SF = 32 binary sub-frames each,
    the sub-frames of every frame sharded over the ranks (SubframeShardPipeline): per frame a0 +
    this rank's shard on the compute stream; C-1 reduce-scatter of the partial intensity (each
    rank owns 2048/N rows), a7 on the owned rows, C-2 all-reduce of five doubles and the MSE on
    a side stream, overlapping the next frame's passes.  Timed from the first frame's launch to
    the last frame's MSE (CUDA events, max over ranks).  At N = 1 the same stream runs whole
    frames with the fused a7 and no collective.  HOLO_BENCH_FAKE_SHARDS=k (N = 1, testing only):
    rank 0 of a k-way split with stand-in collectives (own slice, no exchange) -- not a result."""
    import torch
    from holo_synth import LUT_SEED, WORKLOADS, target_for
    from paper_2004_04049_b200.parallel import SubframeShardPipeline
    w5 = WORKLOADS["C5"]
    n5, S5, P5, L5 = w5.n, w5.n_sub, w5.n * w5.n, w5.lut_lens[0]
    fake = int(os.environ.get("HOLO_BENCH_FAKE_SHARDS", "0")) if world == 1 else 0
    sworld = fake if fake > 1 else world
    nt = 4                                                     # distinct seeded targets, cycled
    Ts = [torch.from_numpy(target_for(w5, f)).to(dev) for f in range(nt)]
    lut5 = torch.empty(L5, dtype=torch.complex64, device=dev)
    kw = {}
    if fake > 1:
        kw = dict(reduce_scatter=lambda o, i: o.copy_(i[:o.numel()]), all_reduce=lambda t: None)
    pipe = SubframeShardPipeline(n5, S5, sworld, rank, lut5, depth=2, lut_seed=LUT_SEED, **kw)   # a0 per frame
    kf = max(16, args.steps)                                   # frames streamed per timed run
    for f in range(max(args.warmup, 3)):
        pipe.submit(Ts[f % nt])
    pipe.drain()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    reps = []
    for _ in range(3):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.compute)
        for f in range(kf):
            pipe.submit(Ts[f % nt])
        (pipe.side if sworld > 1 else pipe.compute).wait_stream(pipe.compute)
        b.record(pipe.side if sworld > 1 else pipe.compute)
        torch.cuda.synchronize()
        barrier(world)
        reps.append(max_over_ranks(a.elapsed_time(b), world))
    tm = statistics.median(reps)
    mse_last = float(pipe.result(pipe.f - 1)[2].item())
    # the parts alone: one frame's compute (a0 + shard) and, N > 1, one C-1 reduce-scatter
    sb, se = pipe.sf
    comp = []
    for _ in range(3):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.compute)
        pipe.submit(Ts[0])
        b.record(pipe.compute)
        torch.cuda.synchronize()
        comp.append(a.elapsed_time(b))
    c1 = None
    if world > 1:
        import torch.distributed as dist
        inp = torch.ones(n5 * n5, dtype=torch.float32, device=dev)
        outp = torch.empty(n5 * n5 // world, dtype=torch.float32, device=dev)
        for _ in range(3):
            dist.reduce_scatter_tensor(outp, inp)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            dist.reduce_scatter_tensor(outp, inp)
        b.record()
        torch.cuda.synchronize()
        c1 = max_over_ranks(a.elapsed_time(b) / 10, world)
    return {
        "metric": "OSPR 2048^2 binary sub-frames/s (video stream, sub-frame shards)", "unit": UNIT,
        "value": S5 * kf / (tm / 1e3), "ms_per_frame": tm / kf, "frames_timed": kf, "runs_ms": reps,
        "statistic": "median of 3 runs", "scaling": "strong" if sworld > 1 else "n/a (one GPU)",
        "mse_last_frame": mse_last,
        "shard": {"sub_frames": [sb, se], "owned_rows": list(pipe.rows) if sworld > 1 else [0, n5]},
        "compute_ms_per_frame": statistics.median(comp),
        "c1_reduce_scatter_ms": c1,
        "c1_bytes": 4 * P5 if sworld > 1 else 0,
        "config": {"workload": "C5: OSPR 2048x2048 binary video, N_SF=32, LUT 2^16 (a0 per frame), frames "
                               f"streamed back to back ({nt} seeded targets cycled); BASELINE configs[4]",
                   "partition": (f"sub-frame shards x{sworld} (whole pairs, subframe_range), C-1 NCCL reduce-scatter of the "
                                 "partial intensity (fp32, N^2/world per rank), a7 on the owned rows, C-2 NCCL "
                                 "all-reduce of 5 doubles, MSE -- on a side stream overlapping the next frame"
                                 if sworld > 1 else "whole frames on one GPU, fused a7, no collective") +
                                (" [FAKE: stand-in collectives, not a result]" if fake > 1 else ""),
                   "l2": "flushed once before each timed run of kf frames; each frame's working set (the "
                         "512 MiB pair buffer of 16 pairs) exceeds the 126 MB L2",
                   "launch": "eager launches, two streams"},
    }


# ---------------------------------------------------------------------------------------------
# CPU oracle (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------------------------
def _oracle_frame_set(T, lut, S, region, threads):
    """The oracle as it stands on one C3 frame set: one thread per sub-frame
    (or_ospr_subframe releases the GIL through ctypes), then mean + M-1 MSE."""
    import oracle
    n = T.shape[0]

    def one(s):
        return oracle.ospr_subframe(T, lut, s * n * n, want_h=False, want_intensity=True)[2]

    with ThreadPoolExecutor(max_workers=threads) as ex:
        Is = list(ex.map(one, range(S)))
    I = np.sum(Is, axis=0) / S
    return oracle.mse_m1(I, T, region)


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_one_thread_rate(T, lut, k=2):
    """The oracle's single-thread rate (report 1-thread and all-core rates): k
    sub-frames of the frame set, one after another on one core."""
    import oracle
    n = T.shape[0]
    t0 = time.perf_counter()
    for s in range(k):
        oracle.ospr_subframe(T, lut, s * n * n, want_h=False, want_intensity=True)
    return k / (time.perf_counter() - t0)


def cpu_baseline(L, steps=1):
    import oracle
    from holo_synth import LUT_SEED, WORKLOADS, target_for
    w3 = WORKLOADS["C3"]
    T = target_for(w3)
    lut = oracle.lut_build(LUT_SEED, L)
    threads = min(w3.n_sub, os.cpu_count() or 1)
    t0 = time.perf_counter()
    for _ in range(steps):
        _oracle_frame_set(T, lut, w3.n_sub, w3.omega().as_tuple(), threads)
    dt = time.perf_counter() - t0
    return {"value": w3.n_sub * steps / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{steps} full C3 frame set(s): {w3.n_sub} sub-frames of 1024^2 (apply_phase, radix-2 "
                      f"fp64 IDFT, sign, DFT, |.|^2) + mean + MSE, L={L}, one thread per sub-frame; "
                      f"host nproc={os.cpu_count()}",
            "seconds": dt, "cpu_model": cpu_model(), "value_1_thread": oracle_one_thread_rate(T, lut)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from holo_synth import LUT_SEED, WORKLOADS, target_for
    oracle.build()
    w3 = WORKLOADS["C3"]
    T = target_for(w3)
    lut = oracle.lut_build(LUT_SEED, args.lut)
    threads = min(w3.n_sub, os.cpu_count() or 1)
    steps, warm = max(1, min(args.steps, 3)), min(args.warmup, 1)
    for _ in range(warm):
        _oracle_frame_set(T, lut, w3.n_sub, w3.omega().as_tuple(), threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        _oracle_frame_set(T, lut, w3.n_sub, w3.omega().as_tuple(), threads)
    dt = time.perf_counter() - t0
    v = w3.n_sub * steps / dt
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: OSPR 1024x1024 binary, N_SF=24, one frame set per step; BASELINE configs[2]",
                   "lut_len": args.lut},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{steps} C3 frame set(s) of 24 sub-frames (steps capped at 3 to bound CPU "
                                   f"time), one thread per sub-frame, host nproc={os.cpu_count()}",
                         "cpu_model": cpu_model(), "value_1_thread": oracle_one_thread_rate(T, lut)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
