// passes.cuh -- launch shapes of the two kinds of FFT pass every kernel of libholo
// is built from:
//
//  * row passes: each row transform is owned by the T = R1 threads of one warp
//    (N <= 2048, so T <= 32; N = 4096 has its own two-warp row kernels, rows2w.cuh)
//    and synchronises with __syncwarp() only; warps run
//    independently; rows arrive by 1D TMA (cp.async.bulk) into per-warp slots or are
//    built in place (OSPR pass A), results go straight back (coalesced: lane t holds
//    x = t + R1*m).
//  * column passes: persistent CTAs stream tiles of W (8 or 4) columns x N rows
//    through a three-stage shared-memory ring filled by TMA (cp.async.bulk.tensor.2d,
//    mbarrier completion); the transforms read the tile from shared memory, exchange
//    in place, and the results leave through the stage by one TMA tile store.  At
//    N = 2048 two consumer groups per CTA share the ring (col_pipe_g2_kernel).
#pragma once

#include "fft.cuh"
#include "tma.cuh"

#include <stdlib.h>

#include <type_traits>

// HOLO_L2PF: the fused OSPR pass C at N <= 1024 also prefetches each warp's pair row after the
// next one into L2 (cp.async.bulk.prefetch), so that its TMA load finds it there: 33.7 -> 32.5 us
// at C3 (prefetch distance HOLO_CF_PFD, ospr.cu).  Measured and not kept: the same at N = 2048 (C5 0.617 -> 0.622 ms), in the GS row pass
// (no gain), and for the column pipelines' 2D tiles (cp.async.bulk.prefetch.tensor: OSPR 48.6 ->
// 50.2 us, GS 228 -> 262 us, C5 0.618 -> 0.89 ms).
#ifndef HOLO_L2PF
#define HOLO_L2PF 1
#endif

namespace holo {

// A column-pipeline body may declare `static constexpr bool kPrologue = true` and a
// `prologue(args, ntiles)` that every thread of every CTA runs once, after the CTA's first
// tile loads are issued (so that work overlaps them).  GS reduces the previous row pass's
// metric partials there.
template <class B, class = void>
struct HasPrologue : std::false_type {};
template <class B>
struct HasPrologue<B, std::void_t<decltype(B::kPrologue)>> : std::integral_constant<bool, B::kPrologue> {};

// ---- row pipeline ---------------------------------------------------------------------------
// Warp-persistent, per-warp double-buffered: a work item is GPW = 32/T consecutive rows
// (always 256*E contiguous bytes), fetched by one cp.async.bulk (1D TMA) into the warp's
// next ring slot while the warp transforms the current one.  The slot is then reused in
// place as the exchange buffer (padded layout, GPW * (N + N/R1) elements).
template <int N>
struct RowPipe {
    using P = fft::Plan<N>;
    static constexpr int GPW = 32 / P::T;
    static constexpr int WPC = 4;                               // warps per CTA
    static constexpr uint32_t IN_BYTES = (uint32_t)GPW * N * 8;
    static constexpr uint32_t XCH_BYTES = (uint32_t)GPW * P::SMEM * 8;
    static constexpr uint32_t SLOT_C = ((XCH_BYTES > IN_BYTES ? XCH_BYTES : IN_BYTES) + 127) / 128 * 128;
};

// Per-warp ring of two slots of `slot_bytes` each (+ one mbarrier per slot).
struct WarpRing {
    unsigned char *base;
    uint64_t *bars;
    uint32_t slot_bytes;
    __device__ __forceinline__ unsigned char *slot(int s) const { return base + (size_t)s * slot_bytes; }
};

template <uint32_t SLOT_BYTES, int WPC>
__device__ __forceinline__ WarpRing make_ring(unsigned char *smem_raw)
{
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    WarpRing r;
    r.slot_bytes = SLOT_BYTES;
    r.base = smem_raw + (size_t)warp * 2 * SLOT_BYTES;
    r.bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)WPC * 2 * SLOT_BYTES) + 2 * warp;
    if (lane == 0) {
        tma::mbar_init(&r.bars[0], 1);
        tma::mbar_init(&r.bars[1], 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    return r;
}

template <uint32_t SLOT_BYTES, int WPC>
constexpr size_t ring_smem() { return (size_t)WPC * 2 * SLOT_BYTES + (size_t)WPC * 2 * sizeof(uint64_t); }

// Plain batched row transform, items = GPW-row groups of `in`, results to `out`
// (in place allowed: an item is read completely before it is written).
template <int N, bool INV>
__global__ void __launch_bounds__(RowPipe<N>::WPC * 32)
rows_fft_kernel(const float2 *__restrict__ tw, const float2 *in, float2 *out, int nitems)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    using RP = RowPipe<N>;
    constexpr int R1 = P::R1, E = P::E, GPW = RP::GPW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const WarpRing ring = make_ring<RP::SLOT_C, RP::WPC>(smem_raw);
    const int lane = threadIdx.x & 31, g = lane / R1, t = lane % R1;
    const int stride = gridDim.x * RP::WPC;
    int item = blockIdx.x * RP::WPC + (threadIdx.x >> 5);
    if (lane == 0 && item < nitems) {
        tma::mbar_arrive_expect_tx(&ring.bars[0], RP::IN_BYTES);
        tma::load_1d(ring.slot(0), in + (size_t)item * GPW * N, RP::IN_BYTES, &ring.bars[0]);
    }
    fft::Twiddles<N> twr;
    twr.load(tw, t);
    #pragma unroll 1   // one copy of the transform code (instruction cache)
    for (int k = 0; item < nitems; item += stride, ++k) {
        const int s = k & 1;
        const int nxt = item + stride;
        if (lane == 0 && nxt < nitems) {
            tma::mbar_arrive_expect_tx(&ring.bars[s ^ 1], RP::IN_BYTES);
            tma::load_1d(ring.slot(s ^ 1), in + (size_t)nxt * GPW * N, RP::IN_BYTES, &ring.bars[s ^ 1]);
        }
        tma::mbar_wait(&ring.bars[s], (uint32_t)((k >> 1) & 1));
        float2 *sl = reinterpret_cast<float2 *>(ring.slot(s));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sl[g * N + t + R1 * m];
        // the inverse runs the forward body on conjugates: F^-1{x} = conj(F{conj(x)}) exactly,
        // the same arithmetic as the fused GS row pass (bit-identical gs_step chains)
        if (INV) {
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m].y = -v[m].y;
        }
        fft::fft2pass<N, false, 1, true>(v, sl + g * P::SMEM, t, twr);
        float2 *o = out + ((size_t)item * GPW + g) * N;
#pragma unroll
        for (int r = 0; r < E; ++r)
            o[t + R1 * r] = INV ? make_float2(v[r].x, -v[r].y) : v[r];
        tma::fence_proxy_async_smem();
        __syncwarp();
    }
}

// Host: persistent grid for a row pipeline kernel.
template <typename K>
inline int pipe_grid(K kernel, int threads, size_t smem, int nitems, int wpc)
{
    const int cap = resident_ctas((const void *)kernel, threads, smem);   // SMs x CTAs per SM (cached)
    const int want = (nitems + wpc - 1) / wpc;
    return want < cap ? want : cap;
}

template <int N, bool INV>
holo_status launch_rows_fft(KernelId id, const float2 *tw, const float2 *in, float2 *out, int nrows, cudaStream_t s)
{
    using RP = RowPipe<N>;
    constexpr size_t smem = ring_smem<RP::SLOT_C, RP::WPC>();
    const int nitems = nrows / RP::GPW;
    const int grid = pipe_grid(rows_fft_kernel<N, INV>, RP::WPC * 32, smem, nitems, RP::WPC);
    return launch(id, rows_fft_kernel<N, INV>, dim3(grid), dim3(RP::WPC * 32), smem, s, tw, in, out, nitems);
}

// ---- column pipeline -------------------------------------------------------------------------
// FFT policy per size: the two-pass transform.  (A three-pass E = 16 policy doubles the
// warps per tile but measured 75 vs 52 us for the OSPR column pass at N = 1024: its extra
// shared-memory exchange outweighs the occupancy gain; removed.)
template <int N, bool REG>
struct ColFftFor {
    using type = fft::ColFft2<N, REG>;
};

template <int N, int NSTAGES = 0, int WIDTH = 8>
struct ColPipe {
    static constexpr int W = WIDTH;                        // columns per tile (OSPR: 8 = one packed byte per row)
    // 3 stages: one CTA per SM, tile k+2 loading while tile k computes and tile k-1's store
    // drains; 1 stage: two CTAs per SM overlap each other's loads and stores
    static constexpr int STAGES = NSTAGES > 0 ? NSTAGES : 3;
    static constexpr int PREFETCH = STAGES > 1 ? STAGES - 1 : 1;   // tiles in flight ahead
    using F = typename ColFftFor<N, (STAGES >= 2 && fft::Plan<N>::E <= 32)>::type;
    static constexpr int T = F::T, E = F::E;
    static constexpr int THREADS = W * T;
    static constexpr int BOX_ROWS = N < 256 ? N : 256;    // TMA box limit is 256 per dimension
    static constexpr int NBOX = N / BOX_ROWS;
    static constexpr uint32_t TILE_BYTES = (uint32_t)N * W * 8;
    static constexpr int STAGE_ELEMS = F::SMEM * W;       // padded exchange layout >= dense tile
    static constexpr size_t BAR_OFFSET = (size_t)STAGES * STAGE_ELEMS * sizeof(float2);
    static constexpr size_t SCRATCH_OFFSET = BAR_OFFSET + 64;
    static constexpr size_t SCRATCH_BYTES = (size_t)2 * W * T * (E > 32 ? 8 : 4);   // 2 words per thread
    static constexpr size_t SMEM = SCRATCH_OFFSET + SCRATCH_BYTES;
    static constexpr int TILES_PER_FRAME = N / W;
};

// Persistent TMA-fed column pipeline.  Tile k of this CTA is (frame, ct) =
// (tile / TPF, tile % TPF); its columns [ct*W, ct*W + W) of rows [frame*N, frame*N + N)
// arrive in stage k % STAGES by TMA.  Thread (c, t) = (threadIdx % W, threadIdx / W) gets
// column c at rows t + T*m (the transform's natural map) and hands it to Body::run
// with its slot of the stage buffer for the in-place exchanges, a 2-words-per-thread
// scratch area (ordered by the transform's barriers) and the FFT policy.  The results go
// back through the stage and one TMA tile store (in place); a stage is refilled once
// its store has been read out, PREFETCH tiles ahead.
template <int N, class Body, int NSTAGES>
__global__ void __launch_bounds__(ColPipe<N, NSTAGES, Body::kWidth>::THREADS,
                                  (N <= 2048 && ((ColPipe<N, NSTAGES, Body::kWidth>::STAGES == 1 && N <= 1024) ||
                                                 Body::kWidth < 8)) ? 2 : 1)
col_pipe_kernel(const __grid_constant__ CUtensorMap tmap, int ntiles, const typename Body::Args a, int rev)
{
    HOLO_PDL_ENTRY();
    using CP = ColPipe<N, NSTAGES, Body::kWidth>;
    using F = typename CP::F;
    constexpr int T = CP::T, E = CP::E, W = CP::W, TPF = CP::TILES_PER_FRAME, S = CP::STAGES, PF = CP::PREFETCH;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage0 = reinterpret_cast<float2 *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + CP::BAR_OFFSET);
    uint32_t *scratch = reinterpret_cast<uint32_t *>(smem_raw + CP::SCRATCH_OFFSET);
    const int c = threadIdx.x % W, t = threadIdx.x / W;
    F fft;
    fft.init(a.tw, t);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    // rev: the tiles in reverse order (the last frames / pairs the previous pass wrote, still in
    // L2, come first)
    auto phys = [&](int tile) { return rev ? ntiles - 1 - tile : tile; };
    auto issue = [&](int tile, int s) {
        const int fr = phys(tile) / TPF, ct = phys(tile) % TPF;
        tma::mbar_arrive_expect_tx(&bars[s], CP::TILE_BYTES);
#pragma unroll
        for (int q = 0; q < CP::NBOX; ++q)
            tma::load_2d(stage0 + (size_t)s * CP::STAGE_ELEMS + q * CP::BOX_ROWS * W, &tmap, ct * W,
                         fr * N + q * CP::BOX_ROWS, &bars[s]);
    };
    if (threadIdx.x == 0)
        for (int j = 0; j < PF; ++j) {
            const int tile = blockIdx.x + j * gridDim.x;
            if (tile < ntiles)
                issue(tile, j % S);
        }
    if constexpr (HasPrologue<Body>::value)
        Body::prologue(a, ntiles);
    int k = 0;
    #pragma unroll 1   // one copy of the transform code (instruction cache)
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int s = k % S;
        float2 *st = stage0 + (size_t)s * CP::STAGE_ELEMS;
        tma::mbar_wait(&bars[s], (uint32_t)((k / S) & 1));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = st[(t + T * m) * W + c];
        Body::template run<F, W>(v, st + c, scratch, c, t, phys(tile) / TPF, phys(tile) % TPF, a, fft);
        // results -> the stage in natural [row][col] layout -> one TMA tile store (in place)
        __syncthreads();                   // every thread is done with the exchange data
#pragma unroll
        for (int m = 0; m < E; ++m)
            st[(t + T * m) * W + c] = v[m];
        tma::fence_proxy_async_smem();     // generic writes before the async-proxy store
        __syncthreads();
        if (threadIdx.x == 0) {
            const int fr = phys(tile) / TPF, ct = phys(tile) % TPF;
#pragma unroll
            for (int q = 0; q < CP::NBOX; ++q)
                tma::store_2d(&tmap, ct * W, fr * N + q * CP::BOX_ROWS, st + q * CP::BOX_ROWS * W);
            tma::bulk_commit();
            const int nxt = tile + PF * gridDim.x;   // -> stage (k + PF) % S, last stored by tile k + PF - S
            if (nxt < ntiles) {
                tma::bulk_wait_read<(S > 1 ? 1 : 0)>();
                issue(nxt, (k + PF) % S);
            }
        }
    }
    if (threadIdx.x == 0)
        tma::bulk_wait<0>();               // stores complete before the CTA retires
}

// Grouped variant (N = 2048, where one W-column tile's transform needs E = 64 values per thread
// and a single 4-warp CTA per SM is all the register file and shared memory allow otherwise):
// two consumer groups of W*T threads share one three-buffer ring.  Group g takes the CTA's
// tiles k = g, g + 2, ... (buffer k % 3), syncs on its own named barrier, and its leader stores
// tile k, waits for the store to read out, and refills the same buffer with tile k + 3, which
// the other group transforms next-but-one.  Twice the warps of the plain pipeline per SM.
template <int N, class Body>
struct ColPipeG2 {
    using CP = ColPipe<N, 3, Body::kWidth>;
    using F = fft::ColFft2<N, false>;         // pool twiddles: the register budget of two groups
    static_assert(F::E == CP::E && F::T == CP::T, "same transform shape as the plain pipeline");
    static constexpr int GROUPS = 2, S = 3;
    static constexpr int GT = CP::THREADS, THREADS = GROUPS * GT;
    static constexpr size_t BAR_OFFSET = CP::BAR_OFFSET;
    static constexpr size_t SCRATCH_OFFSET = BAR_OFFSET + 64;
    static constexpr size_t SMEM = SCRATCH_OFFSET + GROUPS * CP::SCRATCH_BYTES;
};

template <int N, class Body>
__global__ void __launch_bounds__(ColPipeG2<N, Body>::THREADS, 1)
col_pipe_g2_kernel(const __grid_constant__ CUtensorMap tmap, int ntiles, const typename Body::Args a, int rev)
{
    HOLO_PDL_ENTRY();
    using G = ColPipeG2<N, Body>;
    using CP = typename G::CP;
    using F = typename G::F;
    constexpr int T = CP::T, E = CP::E, W = CP::W, TPF = CP::TILES_PER_FRAME, S = G::S, GT = G::GT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage0 = reinterpret_cast<float2 *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + G::BAR_OFFSET);
    const int g = threadIdx.x / GT, lt = threadIdx.x % GT;
    uint32_t *scratch = reinterpret_cast<uint32_t *>(smem_raw + G::SCRATCH_OFFSET + (size_t)g * CP::SCRATCH_BYTES);
    const int c = lt % W, t = lt / W;
    F fft;
    fft.init(a.tw, t);
    fft.sync.id = 1 + g;
    fft.sync.n = GT;
    const fft::GroupSync gsync = fft.sync;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    // rev: the tiles in reverse order (the last frames / pairs the previous pass wrote, still in
    // L2, come first)
    auto phys = [&](int tile) { return rev ? ntiles - 1 - tile : tile; };
    auto issue = [&](int tile, int s) {
        const int fr = phys(tile) / TPF, ct = phys(tile) % TPF;
        tma::mbar_arrive_expect_tx(&bars[s], CP::TILE_BYTES);
#pragma unroll
        for (int q = 0; q < CP::NBOX; ++q)
            tma::load_2d(stage0 + (size_t)s * CP::STAGE_ELEMS + q * CP::BOX_ROWS * W, &tmap, ct * W,
                         fr * N + q * CP::BOX_ROWS, &bars[s]);
    };
    if (threadIdx.x == 0)
        for (int j = 0; j < S; ++j) {
            const int tile = blockIdx.x + j * gridDim.x;
            if (tile < ntiles)
                issue(tile, j);
        }
    if constexpr (HasPrologue<Body>::value)
        Body::prologue(a, ntiles);
    #pragma unroll 1   // one copy of the transform code (instruction cache)
    for (int k = g, tile = blockIdx.x + g * gridDim.x; tile < ntiles; k += 2, tile += 2 * gridDim.x) {
        const int s = k % S;
        float2 *st = stage0 + (size_t)s * CP::STAGE_ELEMS;
        tma::mbar_wait(&bars[s], (uint32_t)((k / S) & 1));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = st[(t + T * m) * W + c];
        Body::template run<F, W>(v, st + c, scratch, c, t, phys(tile) / TPF, phys(tile) % TPF, a, fft);
        gsync();                           // every thread of the group is done with the exchange data
#pragma unroll
        for (int m = 0; m < E; ++m)
            st[(t + T * m) * W + c] = v[m];
        tma::fence_proxy_async_smem();     // generic writes before the async-proxy store
        gsync();
        if (lt == 0) {
            const int fr = phys(tile) / TPF, ct = phys(tile) % TPF;
#pragma unroll
            for (int q = 0; q < CP::NBOX; ++q)
                tma::store_2d(&tmap, ct * W, fr * N + q * CP::BOX_ROWS, st + q * CP::BOX_ROWS * W);
            tma::bulk_commit();
            const int nxt = tile + S * gridDim.x;   // tile k + 3: this buffer's next use
            if (nxt < ntiles) {
                tma::bulk_wait_read<0>();           // the store has read the buffer out
                issue(nxt, s);
            }
        }
    }
    if (lt == 0)
        tma::bulk_wait<0>();               // stores complete before the CTA retires
}

// Host: launch the column pipeline over `nframes` frames of `buf` (row-major
// [nframes*N][N] complex64).
template <int N, class Body, int NSTAGES>
holo_status launch_cols_s(KernelId id, const float2 *buf, int nframes, const typename Body::Args &a, cudaStream_t s,
                          int rev)
{
    using CP = ColPipe<N, NSTAGES, Body::kWidth>;
    CUtensorMap map;
    HOLO_TRY(make_tmap_c64(&map, buf, N, (uint64_t)nframes * N, CP::W, CP::BOX_ROWS));
    // persistent grid: SMs x resident CTAs per SM (registers and shared memory both count)
    const int grid = pipe_grid(col_pipe_kernel<N, Body, NSTAGES>, CP::THREADS, CP::SMEM,
                               nframes * CP::TILES_PER_FRAME, 1);
    const int ntiles = nframes * CP::TILES_PER_FRAME;
    return launch(id, col_pipe_kernel<N, Body, NSTAGES>, dim3(grid), dim3(CP::THREADS), CP::SMEM, s, map, ntiles, a,
                  rev);
}

template <int N, class Body>
holo_status launch_cols_g2(KernelId id, const float2 *buf, int nframes, const typename Body::Args &a, cudaStream_t s,
                           int rev)
{
    using G = ColPipeG2<N, Body>;
    using CP = typename G::CP;
    CUtensorMap map;
    HOLO_TRY(make_tmap_c64(&map, buf, N, (uint64_t)nframes * N, CP::W, CP::BOX_ROWS));
    const int ntiles = nframes * CP::TILES_PER_FRAME;
    const int grid = pipe_grid(col_pipe_g2_kernel<N, Body>, G::THREADS, G::SMEM, (ntiles + 1) / 2, 1);
    return launch(id, col_pipe_g2_kernel<N, Body>, dim3(grid), dim3(G::THREADS), G::SMEM, s, map, ntiles, a, rev);
}

// Body::kStages (3 or 1) picks the variant (measured per body); HOLO_COL_STAGES overrides it;
// Body::kGroups = 2 selects the grouped pipeline.
template <int N, class Body>
holo_status launch_cols(KernelId id, const float2 *buf, int nframes, const typename Body::Args &a, cudaStream_t s,
                        bool rev = false)
{
    if constexpr (Body::kGroups == 2) {
        static const bool off = getenv("HOLO_COL_G1") != nullptr;   // experiments: the plain pipeline
        if (!off)
            return launch_cols_g2<N, Body>(id, buf, nframes, a, s, rev);
    }
    static const int env_stages = [] {
        const char *e = getenv("HOLO_COL_STAGES");
        return e ? atoi(e) : 0;
    }();
    const int stages = env_stages ? env_stages : Body::kStages;
    if constexpr (ColPipe<N, 3, Body::kWidth>::SMEM <= 227 * 1024) {   // three stages fit
        if (stages == 3)
            return launch_cols_s<N, Body, 3>(id, buf, nframes, a, s, rev);
    }
    return launch_cols_s<N, Body, 1>(id, buf, nframes, a, s, rev);
}

} // namespace holo
