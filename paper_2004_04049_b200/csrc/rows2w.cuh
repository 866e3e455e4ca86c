// rows2w.cuh -- row passes for N = 4096 (R-26): a 4096-point row transform needs
// R1 = 64 threads (two warps), so the warp-synchronous row pipelines of passes.cuh (one warp per
// row) do not apply.  Here a row is owned by a two-warp group that synchronises on its own named
// barrier; a CTA of 128 threads holds two such groups.  Rows are read and written directly
// (thread t of a group holds x = t + 64 m, a coalesced 512-byte access per warp and m).  These
// kernels favour plainness over speed: N = 4096 is outside every BASELINE configuration.
#pragma once

#include "passes.cuh"

namespace holo {

template <int N>
struct Row2W {
    using P = fft::Plan<N>;
    static_assert(P::T == 64, "two warps per row");
    static constexpr int THREADS = 128, GROUPS = 2;
    static constexpr size_t SMEM = (size_t)GROUPS * P::SMEM * sizeof(float2);   // exchange buffers
};

// The group (0 or 1) of this thread, its index t < 64 within the row, its exchange buffer and
// barrier (named barriers 1 and 2; 0 is __syncthreads).
struct Row2WThread {
    int grp, t;
    fft::GroupSync sync;
};
__device__ __forceinline__ Row2WThread row2w_thread()
{
    Row2WThread r;
    r.grp = threadIdx.x >> 6;
    r.t = threadIdx.x & 63;
    r.sync.id = 1 + r.grp;
    r.sync.n = 64;
    return r;
}

// Forward transform of the row held in v (thread t: elements t + 64 m) in the group's buffer.
template <int N>
__device__ __forceinline__ void row2w_fft(float2 (&v)[fft::Plan<N>::E], float2 *sm, const float2 *__restrict__ tw,
                                          const Row2WThread &rt)
{
    fft::fft2pass_impl<N, false, 1, false>(v, sm, rt.t, fft::TwGlobal<N>{tw + fft::Plan<N>::TW_OFFSET + rt.t},
                                           fft::NoHook(), rt.sync);
}

// Plain batched row transforms (in place allowed): INV runs the forward body on conjugates.
template <int N, bool INV>
__global__ void __launch_bounds__(Row2W<N>::THREADS, 1)
rows2w_fft_kernel(const float2 *__restrict__ tw, const float2 *in, float2 *out, int nrows)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    constexpr int E = P::E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const Row2WThread rt = row2w_thread();
    float2 *sm = reinterpret_cast<float2 *>(smem_raw) + (size_t)rt.grp * P::SMEM;
    #pragma unroll 1
    for (int row = blockIdx.x * 2 + rt.grp; row < nrows; row += gridDim.x * 2) {
        const float2 *src = in + (size_t)row * N + rt.t;
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            v[m] = src[64 * m];
            if (INV)
                v[m].y = -v[m].y;
        }
        row2w_fft<N>(v, sm, tw, rt);
        float2 *dst = out + (size_t)row * N + rt.t;
#pragma unroll
        for (int m = 0; m < E; ++m)
            dst[64 * m] = INV ? make_float2(v[m].x, -v[m].y) : v[m];
    }
}

template <int N, bool INV>
holo_status launch_rows2w_fft(KernelId id, const float2 *tw, const float2 *in, float2 *out, int nrows, cudaStream_t s)
{
    using R = Row2W<N>;
    const int grid = pipe_grid(rows2w_fft_kernel<N, INV>, R::THREADS, R::SMEM, (nrows + 1) / 2, 1);
    return launch(id, rows2w_fft_kernel<N, INV>, dim3(grid), dim3(R::THREADS), R::SMEM, s, tw, in, out, nrows);
}

// Batched row transforms for any supported N: the warp row pipeline (N <= 2048) or two-warp rows.
template <int N, bool INV>
holo_status launch_row_fft(KernelId id, const float2 *tw, const float2 *in, float2 *out, int nrows, cudaStream_t s)
{
    if constexpr (fft::Plan<N>::T > 32)
        return launch_rows2w_fft<N, INV>(id, tw, in, out, nrows, s);
    else
        return launch_rows_fft<N, INV>(id, tw, in, out, nrows, s);
}

} // namespace holo
