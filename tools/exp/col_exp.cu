// Column-pass experiment harness (tooling, not product): times variants of the TMA-fed
// column pipeline on 12 frames of 1024^2 complex64 to locate the bottleneck.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -lineinfo tools/exp/col_exp.cu paper_2004_04049_b200/csrc/runtime.cu (includes ospr.cu) -lcuda -o /tmp/col_exp
#include <cstdio>
#include <vector>
#include "../../paper_2004_04049_b200/csrc/ospr.cu"

using namespace holo;

constexpr int N = 1024;

// NFFT transforms (IFFT/FFT alternating through one body), STORE: 0 direct STG, 1 STS + TMA store
template <int NFFT, int STORE, int STAGES>
__global__ void __launch_bounds__(256, 1)
exp_kernel(const __grid_constant__ CUtensorMap tmap, int ntiles, const float2 *tw, float2 *buf)
{
    using CP = ColPipe<N, 2>;
    using F = fft::ColFft2<N, true>;
    constexpr int T = CP::T, E = CP::E, W = CP::W, TPF = CP::TILES_PER_FRAME;
    constexpr int STAGE_ELEMS = CP::STAGE_ELEMS;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage0 = reinterpret_cast<float2 *>(smem_raw);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw + (size_t)STAGES * STAGE_ELEMS * 8);
    const int c = threadIdx.x % W, t = threadIdx.x / W;
    F fft;
    fft.init(tw, t);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            tma::mbar_init(&bars[s], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int tile, int s) {
        const int fr = tile / TPF, ct = tile % TPF;
        tma::mbar_arrive_expect_tx(&bars[s], CP::TILE_BYTES);
#pragma unroll
        for (int q = 0; q < CP::NBOX; ++q)
            tma::load_2d(stage0 + (size_t)s * STAGE_ELEMS + q * CP::BOX_ROWS * W, &tmap, ct * W,
                         fr * N + q * CP::BOX_ROWS, &bars[s]);
    };
    const int PRE = STORE == 1 ? STAGES - 1 : STAGES;   // prefetch distance
    if (threadIdx.x == 0)
        for (int s = 0; s < PRE; ++s) {
            const int tile = blockIdx.x + s * gridDim.x;
            if (tile < ntiles)
                issue(tile, s);
        }
    int k = 0;
#pragma unroll 1
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int s = k % STAGES;
        float2 *st = stage0 + (size_t)s * STAGE_ELEMS;
        tma::mbar_wait(&bars[s], (uint32_t)((k / STAGES) & 1));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = st[(t + T * m) * W + c];
#pragma unroll 1
        for (int h = 0; h < NFFT; ++h) {
#pragma unroll
            for (int r = 0; r < E; ++r)
                v[r].y = -v[r].y;
            fft.template run<false, W>(v, st + c, t);
        }
        if (STORE == 0) {
            __syncthreads();
            const int nxt = tile + STAGES * gridDim.x;
            if (threadIdx.x == 0 && nxt < ntiles)
                issue(nxt, s);
            float2 *o = buf + ((size_t)(tile / TPF) * N + t) * N + (tile % TPF) * W + c;
#pragma unroll
            for (int m = 0; m < E; ++m)
                o[(size_t)T * m * N] = v[m];
        } else {
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m)
                st[(t + T * m) * W + c] = v[m];
            tma::fence_proxy_async_smem();
            __syncthreads();
            if (threadIdx.x == 0) {
                const int fr = tile / TPF, ct = tile % TPF;
#pragma unroll
                for (int q = 0; q < CP::NBOX; ++q)
                    tma::store_2d(&tmap, ct * W, fr * N + q * CP::BOX_ROWS, st + q * CP::BOX_ROWS * W);
                tma::bulk_commit();
                // refill the stage freed longest ago: tile + (STAGES-1) goes to stage (k-1) % STAGES
                const int nxt = tile + (STAGES - 1) * gridDim.x;
                if (nxt < ntiles) {
                    tma::bulk_wait_read<1>();
                    issue(nxt, (k + STAGES - 1) % STAGES);
                }
            }
        }
    }
    if (STORE == 1 && threadIdx.x == 0)
        tma::bulk_wait<0>();
}

template <int NFFT, int STORE, int STAGES>
float run(const float2 *tw, float2 *buf, int nframes, int reps)
{
    CUtensorMap map;
    make_tmap_c64(&map, buf, N, (uint64_t)nframes * N, 8, 256);
    const size_t smem = (size_t)STAGES * ColPipe<N, 2>::STAGE_ELEMS * 8 + 64;
    auto kern = exp_kernel<NFFT, STORE, STAGES>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    const int ntiles = nframes * (N / 8);
    const int grid = 148 * per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i)
        kern<<<grid, 256, smem>>>(map, ntiles, tw, buf);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i)
        kern<<<grid, 256, smem>>>(map, ntiles, tw, buf);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("NFFT=%d STORE=%s STAGES=%d per_sm=%d: %8.2f us/launch (%d frames)  %s\n", NFFT,
           STORE ? "tma" : "stg", STAGES, per_sm, 1e3 * ms / reps, nframes, cudaGetErrorString(e));
    return ms;
}

void run_ospr(const float2 *tw, float2 *buf, uint8_t *bits, int npairs, int reps)
{
    typename OsprColBody<N>::Args ca{tw, buf, bits, npairs, 1};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i)
        launch_cols<N, OsprColBody<N>>(K_OSPR_COLS, buf, npairs, ca, 0);
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i)
        launch_cols<N, OsprColBody<N>>(K_OSPR_COLS, buf, npairs, ca, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("OSPR body bits=%s: %8.2f us/launch  %s\n", bits ? "yes" : "no", 1e3 * ms / reps,
           cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    const int nframes = 12;
    float2 *buf;
    cudaMalloc(&buf, (size_t)nframes * N * N * 8);
    cudaMemset(buf, 0, (size_t)nframes * N * N * 8);
    const float2 *tw;
    fft::twiddles(&tw);
    uint8_t *bits;
    cudaMalloc(&bits, (size_t)2 * nframes * N * N / 8);
    for (int rep = 0; rep < 2; ++rep) {
        run<0, 0, 2>(tw, buf, nframes, 20);
        run<0, 1, 3>(tw, buf, nframes, 20);
        run<1, 0, 2>(tw, buf, nframes, 20);
        run<1, 1, 3>(tw, buf, nframes, 20);
        run<2, 0, 2>(tw, buf, nframes, 20);
        run<2, 1, 3>(tw, buf, nframes, 20);
        run<2, 1, 2>(tw, buf, nframes, 20);
        run_ospr(tw, buf, nullptr, nframes, 20);
        run_ospr(tw, buf, bits, nframes, 20);
    }
    return 0;
}
