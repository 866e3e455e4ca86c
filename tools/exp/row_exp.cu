// Row-pass experiment harness (tooling, not product): variants of the warp-per-row FFT
// pipeline on 12 frames of 1024^2 complex64 (ring slots, twiddle source, warps per CTA,
// transforms per item).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo \
//        tools/exp/row_exp.cu paper_2004_04049_b200/csrc/runtime.cu -lcuda -o tools/exp/row_exp
#include <cstdio>
#include "../../paper_2004_04049_b200/csrc/passes.cuh"

using namespace holo;
constexpr int N = 1024;

// SLOTS ring slots per warp (1: load-wait-compute, 2: double-buffered TMA), REG twiddles in
// registers, WPC warps per CTA, NFFT transforms per row (forward/inverse alternating).
template <int SLOTS, bool REG, int WPC, int NFFT>
__global__ void __launch_bounds__(WPC * 32)
row_kernel(const float2 *__restrict__ tw, const float2 *in, float2 *out, int nitems)
{
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E;
    constexpr uint32_t IN_BYTES = N * 8, SLOT = ((P::SMEM * 8) + 127) / 128 * 128;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = lane;
    unsigned char *base = smem_raw + (size_t)warp * SLOTS * SLOT;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)WPC * SLOTS * SLOT) + SLOTS * warp;
    if (lane == 0) {
        for (int s = 0; s < SLOTS; ++s)
            tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    const int stride = gridDim.x * WPC;
    int item = blockIdx.x * WPC + warp;
    if (lane == 0 && item < nitems) {
        tma::mbar_arrive_expect_tx(&bars[0], IN_BYTES);
        tma::load_1d(base, in + (size_t)item * N, IN_BYTES, &bars[0]);
    }
    fft::Twiddles<N, REG> twr;
    twr.load(tw, t);
#pragma unroll 1
    for (int k = 0; item < nitems; item += stride, ++k) {
        const int s = SLOTS == 2 ? (k & 1) : 0;
        const int nxt = item + stride;
        if (SLOTS == 2 && lane == 0 && nxt < nitems) {
            tma::mbar_arrive_expect_tx(&bars[s ^ 1], IN_BYTES);
            tma::load_1d(base + (s ^ 1) * SLOT, in + (size_t)nxt * N, IN_BYTES, &bars[s ^ 1]);
        }
        tma::mbar_wait(&bars[s], (uint32_t)((SLOTS == 2 ? (k >> 1) : k) & 1));
        float2 *sl = reinterpret_cast<float2 *>(base + s * SLOT);
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sl[t + R1 * m];
#pragma unroll 1
        for (int h = 0; h < NFFT; ++h) {
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m].y = -v[m].y;
            fft::fft2pass<N, false, 1, true>(v, sl, t, twr);
        }
        __syncwarp();
        if (SLOTS == 1 && lane == 0 && nxt < nitems) {   // refill as soon as the exchange is read
            tma::mbar_arrive_expect_tx(&bars[0], IN_BYTES);
            tma::load_1d(base, in + (size_t)nxt * N, IN_BYTES, &bars[0]);
        }
        float2 *o = out + (size_t)item * N;
#pragma unroll
        for (int m = 0; m < E; ++m)
            o[t + R1 * m] = v[m];
    }
}

template <int SLOTS, bool REG, int WPC, int NFFT>
void run(const float2 *tw, const float2 *in, float2 *out, int nframes, int reps)
{
    using P = fft::Plan<N>;
    constexpr uint32_t SLOT = ((P::SMEM * 8) + 127) / 128 * 128;
    const size_t smem = (size_t)WPC * SLOTS * SLOT + (size_t)WPC * SLOTS * 8;
    auto kern = row_kernel<SLOTS, REG, WPC, NFFT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPC * 32, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    const int nitems = nframes * N;
    const int grid = 148 * per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i)
        kern<<<grid, WPC * 32, smem>>>(tw, in, out, nitems);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i)
        kern<<<grid, WPC * 32, smem>>>(tw, in, out, nitems);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("SLOTS=%d REG=%d WPC=%d NFFT=%d regs=%d per_sm=%d (warps/SM %d): %8.2f us  %s\n", SLOTS, (int)REG, WPC,
           NFFT, fa.numRegs, per_sm, per_sm * WPC, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    const int nframes = 12;
    float2 *in, *out;
    cudaMalloc(&in, (size_t)nframes * N * N * 8);
    cudaMalloc(&out, (size_t)nframes * N * N * 8);
    cudaMemset(in, 0, (size_t)nframes * N * N * 8);
    const float2 *tw;
    fft::twiddles(&tw);
    for (int rep = 0; rep < 2; ++rep) {
        run<2, true, 4, 1>(tw, in, out, nframes, 20);
        run<2, false, 4, 1>(tw, in, out, nframes, 20);
        run<1, true, 4, 1>(tw, in, out, nframes, 20);
        run<1, false, 4, 1>(tw, in, out, nframes, 20);
        run<1, false, 8, 1>(tw, in, out, nframes, 20);
        run<2, false, 8, 1>(tw, in, out, nframes, 20);
        run<2, true, 4, 2>(tw, in, out, nframes, 20);
        run<2, false, 4, 2>(tw, in, out, nframes, 20);
        run<1, false, 4, 2>(tw, in, out, nframes, 20);
        run<1, false, 8, 2>(tw, in, out, nframes, 20);
        run<1, true, 4, 0>(tw, in, out, nframes, 20);
        run<2, true, 4, 0>(tw, in, out, nframes, 20);
    }
    return 0;
}
