// Column-pass experiment (tooling): tile width W (columns per tile) x stages x CTAs per SM,
// 2 FFTs per column (IFFT -> FFT, conj trick), TMA load + TMA store, 12 frames of 1024^2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -lineinfo \
//        tools/exp/colw_exp.cu paper_2004_04049_b200/csrc/runtime.cu -o tools/exp/colw_exp
#include <cstdio>
#include "../../paper_2004_04049_b200/csrc/passes.cuh"

using namespace holo;
constexpr int N = 1024;

template <int W, int S, bool REG>
__global__ void __launch_bounds__(W * 32)
colw_kernel(const __grid_constant__ CUtensorMap tmap, int ntiles, const float2 *tw)
{
    using F = fft::ColFft2<N, REG>;
    constexpr int T = F::T, E = F::E, TPF = N / W, BOX = 256, NBOX = N / BOX;
    constexpr int STAGE = F::SMEM * W;
    constexpr uint32_t TILE_BYTES = (uint32_t)N * W * 8;
    constexpr int PF = S > 1 ? S - 1 : 1;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage0 = reinterpret_cast<float2 *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)S * STAGE * 8);
    const int c = threadIdx.x % W, t = threadIdx.x / W;
    F fft;
    fft.init(tw, t);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int tile, int s) {
        const int fr = tile / TPF, ct = tile % TPF;
        tma::mbar_arrive_expect_tx(&bars[s], TILE_BYTES);
        for (int q = 0; q < NBOX; ++q)
            tma::load_2d(stage0 + (size_t)s * STAGE + q * BOX * W, &tmap, ct * W, fr * N + q * BOX, &bars[s]);
    };
    if (threadIdx.x == 0)
        for (int j = 0; j < PF; ++j)
            if (blockIdx.x + j * gridDim.x < ntiles)
                issue(blockIdx.x + j * gridDim.x, j % S);
    int k = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int s = k % S;
        float2 *st = stage0 + (size_t)s * STAGE;
        tma::mbar_wait(&bars[s], (uint32_t)((k / S) & 1));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = st[(t + T * m) * W + c];
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            fft.template run<false, W>(v, st + c, t);
            if (h == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    v[r] = make_float2(v[r].x >= 0.f ? 1.f : -1.f, v[r].y <= 0.f ? 1.f : -1.f);
            }
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < E; ++m)
            st[(t + T * m) * W + c] = v[m];
        tma::fence_proxy_async_smem();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int fr = tile / TPF, ct = tile % TPF;
            for (int q = 0; q < NBOX; ++q)
                tma::store_2d(&tmap, ct * W, fr * N + q * BOX, st + q * BOX * W);
            tma::bulk_commit();
            const int nxt = tile + PF * gridDim.x;
            if (nxt < ntiles) {
                tma::bulk_wait_read<(S > 1 ? 1 : 0)>();
                issue(nxt, (k + PF) % S);
            }
        }
    }
    if (threadIdx.x == 0)
        tma::bulk_wait<0>();
}

template <int W, int S, bool REG>
void run(const float2 *tw, float2 *buf, int nframes, int reps)
{
    CUtensorMap map;
    make_tmap_c64(&map, buf, N, (uint64_t)nframes * N, W, 256);
    const size_t smem = (size_t)S * fft::ColFft2<N, REG>::SMEM * W * 8 + 64;
    auto kern = colw_kernel<W, S, REG>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W * 32, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    const int ntiles = nframes * (N / W), grid = 148 * per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i)
        kern<<<grid, W * 32, smem>>>(map, ntiles, tw);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i)
        kern<<<grid, W * 32, smem>>>(map, ntiles, tw);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("W=%d S=%d REG=%d regs=%d per_sm=%d warps/SM=%d: %8.2f us  %s\n", W, S, (int)REG, fa.numRegs, per_sm,
           per_sm * W, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    const int nframes = 12;
    float2 *buf;
    cudaMalloc(&buf, (size_t)nframes * N * N * 8);
    cudaMemset(buf, 0, (size_t)nframes * N * N * 8);
    const float2 *tw;
    fft::twiddles(&tw);
    for (int rep = 0; rep < 2; ++rep) {
        run<8, 3, true>(tw, buf, nframes, 20);
        run<4, 3, true>(tw, buf, nframes, 20);
        run<4, 2, true>(tw, buf, nframes, 20);
        run<4, 3, false>(tw, buf, nframes, 20);
        run<2, 3, true>(tw, buf, nframes, 20);
        run<2, 4, true>(tw, buf, nframes, 20);
        run<16, 1, true>(tw, buf, nframes, 20);
    }
    return 0;
}
