// ospr.cu -- One-Step Phase-Retrieval (Fig. 2 right, P:47, P:53;
// steps a1-a7 of DESIGN.md §1) as three fused FFT passes per chunk of
// sub-frame pairs plus a finalize pass per frame.
//
//   pass A  ospr_rows_a  prologue: R_s = T * lut[(base_s + p) mod L] for the two
//                        sub-frames a, b of a pair at pixels (y, x) and (-y, -x),
//                        Hermitian parts packed as Z = Herm(R_a) + i Herm(R_b)
//                        (so F^-1{Z} = Re H_a + i Re H_b);
//                        row IFFT; write Z (complex64).
//   pass B  ospr_cols    column IFFT -> H; a4: bit_a = Re H >= 0, bit_b = Im H >= 0,
//                        packed MSB-first via warp ballots; h' = (+-1) + i(+-1);
//                        column FFT of h'; write back in place.
//   pass C  ospr_rows_c  row FFT -> X = F{h'_a} + i F{h'_b}; accumulate |X|^2/N^2
//                        over the chunk's pairs in registers; one RMW of the
//                        frame accumulator A per chunk.
//   finalize             I[k] = (A[k] + A[-k]) / 2 / N_SF  (= sum_s |F{h'_s}|^2 / N_SF,
//                        DESIGN.md §5) and the fp64 MSE partial sums over Omega.
//
// All 1/sqrt(N) factors of Eqs. (1)-(2) are dropped inside the passes: a positive
// scale does not change sign(Re H), and the forward scale 1/N^2 on |X|^2 is an
// exact power of two applied in pass C.
#include "fft.cuh"

namespace holo {

constexpr int kMaxChunk = 16;
constexpr int kFinBlocks = 592;   // finalize CTAs per frame (fixed => deterministic sums)
constexpr int kFinThreads = 256;

template <int N>
struct RowCfg {
    using P = fft::Plan<N>;
    static constexpr int RPC = (N >= 2048) ? 4 : ((256 / P::T) < N ? (256 / P::T) : N);
    static constexpr int THREADS = RPC * P::T;
    static constexpr size_t SMEM = (size_t)RPC * P::SMEM * sizeof(float2);
};

template <int N>
struct ColCfg {
    using P = fft::Plan<N>;
    static constexpr int W = 8;    // columns per CTA = one packed byte per row
    static constexpr int THREADS = W * P::T;
    static constexpr size_t SMEM = (size_t)W * P::SMEM * sizeof(float2);
};

struct PairBases {
    uint32_t a[kMaxChunk];
    uint32_t b[kMaxChunk];
};

// ---- pass A ------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(RowCfg<N>::THREADS)
ospr_rows_a_kernel(const float2 *__restrict__ tw, const float *__restrict__ T, const float2 *__restrict__ lut, LutIndexer ix,
                   PairBases bases, int npairs, int last_has_b, float2 *__restrict__ buf)
{
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E, RPC = RowCfg<N>::RPC;
    extern __shared__ float2 smem[];
    const int lr = threadIdx.x / R1, t = threadIdx.x % R1;
    const int g = blockIdx.x * RPC + lr;
    const bool active = g < npairs * N;
    const int pair = active ? g / N : 0;
    const int y = g % N, ym = (N - y) & (N - 1);
    const bool has_b = (pair < npairs - 1) || last_has_b;
    float2 v[E];
    if (active) {
        const float *Ty = T + (size_t)y * N;
        const float *Tm = T + (size_t)ym * N;
        if (lut != nullptr) {
            const uint32_t rya = ix.mod_any((uint64_t)bases.a[pair] + (uint64_t)y * N);
            const uint32_t rma = ix.mod_any((uint64_t)bases.a[pair] + (uint64_t)ym * N);
            const uint32_t ryb = ix.mod_any((uint64_t)bases.b[pair] + (uint64_t)y * N);
            const uint32_t rmb = ix.mod_any((uint64_t)bases.b[pair] + (uint64_t)ym * N);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int x = t + R1 * m, xm = (N - x) & (N - 1);
                const float t1 = __ldg(Ty + x), t2 = __ldg(Tm + xm);
                const float2 ca1 = lut_at(lut, ix.mod(rya + x));
                const float2 ca2 = lut_at(lut, ix.mod(rma + xm));
                // 2 Herm(R_a)[y][x] = R_a[y][x] + conj(R_a[-y][-x])
                float2 za = make_float2(t1 * ca1.x + t2 * ca2.x, t1 * ca1.y - t2 * ca2.y);
                float2 zb = make_float2(0.f, 0.f);
                if (has_b) {
                    const float2 cb1 = lut_at(lut, ix.mod(ryb + x));
                    const float2 cb2 = lut_at(lut, ix.mod(rmb + xm));
                    zb = make_float2(t1 * cb1.x + t2 * cb2.x, t1 * cb1.y - t2 * cb2.y);
                }
                v[m] = make_float2(za.x - zb.y, za.y + zb.x);
            }
        } else {   // flat phase (N_LUT = 0): R = T, Herm(R) = (T + T(-p)) / 2
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int x = t + R1 * m, xm = (N - x) & (N - 1);
                const float h = __ldg(Ty + x) + __ldg(Tm + xm);
                v[m] = make_float2(h, has_b ? h : 0.f);
            }
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = make_float2(0.f, 0.f);
    }
    fft::fft2pass<N, true, 1>(v, smem + lr * P::SMEM, t, tw);
    if (active) {
        float2 *out = buf + ((size_t)pair * N + y) * N;
#pragma unroll
        for (int r = 0; r < E; ++r)
            out[t + R1 * r] = v[r];
    }
}

// ---- pass B ------------------------------------------------------------------------------
__device__ __forceinline__ uint8_t msb_first8(unsigned bits8) { return (uint8_t)(__brev(bits8) >> 24); }

template <int N>
__global__ void __launch_bounds__(ColCfg<N>::THREADS)
ospr_cols_kernel(const float2 *__restrict__ tw, float2 *__restrict__ buf, int npairs, int last_has_b, uint8_t *__restrict__ bits)
{
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E, W = ColCfg<N>::W;
    constexpr size_t FRAME_BYTES = (size_t)N * N / 8;
    extern __shared__ float2 smem[];
    const int c = threadIdx.x % W, t = threadIdx.x / W;
    const int tile = blockIdx.x, pair = blockIdx.y;
    const bool has_b = (pair < npairs - 1) || last_has_b;
    float2 *col = buf + (size_t)pair * N * N + tile * W + c;
    float2 v[E];
#pragma unroll
    for (int m = 0; m < E; ++m)
        v[m] = col[(size_t)(t + R1 * m) * N];
    fft::fft2pass<N, true, W>(v, smem + c, t, tw);           // v[r] = H at row t + R1*r
    const int grp = (threadIdx.x & 31) / W;
    uint8_t *ba = bits ? bits + (size_t)(2 * pair) * FRAME_BYTES + tile : nullptr;
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const bool pa = v[r].x >= 0.0f;                  // a4; -0.0 -> +1 (R-7)
        const bool pb = v[r].y >= 0.0f;
        const unsigned ma = __ballot_sync(0xffffffffu, pa);
        const unsigned mb = __ballot_sync(0xffffffffu, pb);
        if (ba != nullptr && c == 0) {
            const size_t off = (size_t)(t + R1 * r) * (N / 8);
            ba[off] = msb_first8((ma >> (W * grp)) & 0xFFu);
            if (has_b)
                ba[FRAME_BYTES + off] = msb_first8((mb >> (W * grp)) & 0xFFu);
        }
        v[r] = make_float2(pa ? 1.0f : -1.0f, has_b ? (pb ? 1.0f : -1.0f) : 0.0f);
    }
    fft::fft2pass<N, false, W>(v, smem + c, t, tw);
#pragma unroll
    for (int r = 0; r < E; ++r)
        col[(size_t)(t + R1 * r) * N] = v[r];
}

// ---- pass C ------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(RowCfg<N>::THREADS)
ospr_rows_c_kernel(const float2 *__restrict__ tw, const float2 *__restrict__ buf, int npairs, float *__restrict__ acc, int accumulate)
{
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E, RPC = RowCfg<N>::RPC;
    extern __shared__ float2 smem[];
    const int lr = threadIdx.x / R1, t = threadIdx.x % R1;
    const int y = blockIdx.x * RPC + lr;
    float a[E];
#pragma unroll
    for (int r = 0; r < E; ++r)
        a[r] = 0.0f;
    for (int p = 0; p < npairs; ++p) {
        const float2 *row = buf + ((size_t)p * N + y) * N;
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = row[t + R1 * m];
        fft::fft2pass<N, false, 1>(v, smem + lr * P::SMEM, t, tw);
#pragma unroll
        for (int r = 0; r < E; ++r)
            a[r] += v[r].x * v[r].x + v[r].y * v[r].y;
    }
    constexpr float inv_p = 1.0f / ((float)N * (float)N);   // exact power of two
    float *out = acc + (size_t)y * N;
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const float val = a[r] * inv_p;
        out[t + R1 * r] = accumulate ? out[t + R1 * r] + val : val;
    }
}

// ---- finalize + MSE -----------------------------------------------------------------------
__device__ __forceinline__ void block_reduce_store(double (&s)[5], int nvals, double *dst)
{
    __shared__ double red[32][5];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = 0; i < nvals; ++i) {
        double x = s[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0)
            red[w][i] = x;
    }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        for (int i = 0; i < nvals; ++i) {
            double x = lane < nw ? red[lane][i] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                x += __shfl_down_sync(0xffffffffu, x, o);
            if (lane == 0)
                dst[i] = x;
        }
    }
}

// intensity[k] = (A[k] + A[-k]) * scale (symmetrise = 1) or A[k] * scale; optional
// fp64 partial sums (sum I, sum I^2, sum I T^2, sum T^2, sum T^4) over Omega.
__global__ void __launch_bounds__(kFinThreads)
ospr_finalize_kernel(const float *__restrict__ acc, const float *__restrict__ T, int n, int symmetrise,
                     float scale, float *out, holo_region om, double *__restrict__ parts)
{
    const int P = n * n;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < P; k += gridDim.x * blockDim.x) {
        const int y = k / n, x = k - y * n;
        float I;
        if (symmetrise) {
            const int km = ((n - y) & (n - 1)) * n + ((n - x) & (n - 1));
            I = (acc[k] + acc[km]) * scale;
        } else {
            I = acc[k] * scale;
        }
        out[k] = I;
        if (parts != nullptr && y >= om.row0 && y < om.row1 && x >= om.col0 && x < om.col1) {
            const double Id = I, tt = T[k], t2 = tt * tt;
            s[0] += Id;
            s[1] += Id * Id;
            s[2] += Id * t2;
            s[3] += t2;
            s[4] += t2 * t2;
        }
    }
    if (parts != nullptr)
        block_reduce_store(s, 5, parts + (size_t)blockIdx.x * 5);
}

// One CTA per frame: fixed-order reduction of nblk x 5 partial sums, then R-12:
// a = S_T2 / S_I (0 if S_I = 0); mse = (a^2 S_II - 2 a S_IT2 + S_T4) / |Omega|.
__global__ void __launch_bounds__(256)
mse_reduce_kernel(const double *__restrict__ parts, int nblk, size_t frame_stride, double inv_count,
                  double *__restrict__ mse)
{
    const double *p = parts + (size_t)blockIdx.x * frame_stride;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nblk; b += blockDim.x)
        for (int i = 0; i < 5; ++i)
            s[i] += p[(size_t)b * 5 + i];
    __shared__ double out[5];
    block_reduce_store(s, 5, out);
    __syncthreads();
    if (threadIdx.x == 0) {
        const double a = out[0] == 0.0 ? 0.0 : out[3] / out[0];
        const double sum = a * a * out[1] - 2.0 * a * out[2] + out[4];
        mse[blockIdx.x] = (sum > 0.0 ? sum : 0.0) * inv_count;
    }
}

// ---- host orchestration -------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int ospr_chunk_pairs(int n, int n_sub)
{
    const size_t frame = (size_t)n * n * sizeof(float2);
    size_t budget = 64ull << 20;   // pair buffers kept L2-resident between passes
    if (const char *e = getenv("HOLO_OSPR_CHUNK_BYTES"))
        budget = strtoull(e, nullptr, 10);
    long c = (long)(budget / frame);
    const int npairs = (n_sub + 1) / 2;
    if (c < 1)
        c = 1;
    if (c > kMaxChunk)
        c = kMaxChunk;
    if (c > npairs)
        c = npairs;
    return (int)c;
}

struct OsprWs {
    float2 *buf;
    float *acc;
    double *parts;
};

static size_t ospr_ws_layout(int n, int n_sub, char *base, OsprWs *w)
{
    const size_t P = (size_t)n * n;
    const int chunk = ospr_chunk_pairs(n, n_sub);
    size_t off = 0;
    const size_t o_buf = off;
    off = align256(off + (size_t)chunk * P * sizeof(float2));
    const size_t o_acc = off;
    off = align256(off + P * sizeof(float));
    const size_t o_parts = off;
    off = align256(off + (size_t)kFinBlocks * 5 * sizeof(double));
    if (w) {
        w->buf = (float2 *)(base + o_buf);
        w->acc = (float *)(base + o_acc);
        w->parts = (double *)(base + o_parts);
    }
    return off;
}

static uint32_t draw_base(uint64_t phase_offset, uint64_t sf_global, uint64_t P, uint64_t L)
{
    if (L == 0)
        return 0;
    unsigned __int128 g = (unsigned __int128)phase_offset + (unsigned __int128)sf_global * P;
    return (uint32_t)(g % L);
}

static int fin_grid(int n)
{
    const int want = (n * n + kFinThreads - 1) / kFinThreads;
    return want < kFinBlocks ? want : kFinBlocks;
}

holo_status finalize_frame(const float *acc, const float *T, int n, int symmetrise, float scale,
                           float *out, holo_region om, double *parts, double *mse, cudaStream_t s)
{
    const int grid = fin_grid(n);
    HOLO_TRY(launch(K_OSPR_FINALIZE, ospr_finalize_kernel, dim3(grid), dim3(kFinThreads), 0, s, acc, T,
                    n, symmetrise, scale, out, om, mse ? parts : (double *)nullptr));
    if (mse) {
        const double cnt = (double)(om.row1 - om.row0) * (double)(om.col1 - om.col0);
        HOLO_TRY(launch(K_MSE_REDUCE, mse_reduce_kernel, dim3(1), dim3(256), 0, s, (const double *)parts,
                        grid, (size_t)0, 1.0 / cnt, mse));
    }
    return HOLO_OK;
}

template <int N>
static holo_status ospr_run(const float2 *tw, const float *target, int n_frames, int n_sub, const float2 *lut, uint64_t n_lut,
                            uint64_t phase_offset, int sf_begin, int sf_end, uint8_t *holo_bits,
                            float *intensity, double *mse, holo_region om, void *ws, cudaStream_t s)
{
    using RC = RowCfg<N>;
    using CC = ColCfg<N>;
    constexpr size_t P = (size_t)N * N;
    OsprWs w;
    ospr_ws_layout(N, n_sub, (char *)ws, &w);
    const int chunk = ospr_chunk_pairs(N, n_sub);
    const int nsh = sf_end - sf_begin;
    const int npairs_total = (nsh + 1) / 2;
    const bool full = (sf_begin == 0 && sf_end == n_sub);
    const LutIndexer ix = LutIndexer::make(n_lut ? (uint32_t)n_lut : 1u, N);
    for (int f = 0; f < n_frames; ++f) {
        const float *Tf = target + (size_t)f * P;
        for (int c0 = 0; c0 < npairs_total; c0 += chunk) {
            const int np = (npairs_total - c0) < chunk ? (npairs_total - c0) : chunk;
            PairBases pb;
            for (int p = 0; p < np; ++p) {
                const int sa = sf_begin + 2 * (c0 + p), sb = sa + 1;
                pb.a[p] = draw_base(phase_offset, (uint64_t)f * n_sub + sa, P, n_lut);
                pb.b[p] = sb < sf_end ? draw_base(phase_offset, (uint64_t)f * n_sub + sb, P, n_lut) : 0u;
            }
            const int last_sa = sf_begin + 2 * (c0 + np - 1);
            const int last_has_b = (last_sa + 1) < sf_end;
            uint8_t *bits = holo_bits ? holo_bits + ((size_t)f * nsh + 2 * (size_t)c0) * (P / 8) : nullptr;
            const int rows = np * N;
            HOLO_TRY(launch(K_OSPR_ROWS_A, ospr_rows_a_kernel<N>, dim3((rows + RC::RPC - 1) / RC::RPC),
                            dim3(RC::THREADS), RC::SMEM, s, tw, Tf, lut, ix, pb, np, last_has_b, w.buf));
            HOLO_TRY(launch(K_OSPR_COLS, ospr_cols_kernel<N>, dim3(N / CC::W, np), dim3(CC::THREADS),
                            CC::SMEM, s, tw, w.buf, np, last_has_b, bits));
            HOLO_TRY(launch(K_OSPR_ROWS_C, ospr_rows_c_kernel<N>, dim3(N / RC::RPC), dim3(RC::THREADS),
                            RC::SMEM, s, tw, (const float2 *)w.buf, np, w.acc, c0 > 0 ? 1 : 0));
        }
        const float scale = full ? 0.5f / (float)n_sub : 0.5f;
        HOLO_TRY(finalize_frame(w.acc, Tf, N, 1, scale, intensity + (size_t)f * P, om, w.parts,
                                (full && mse) ? mse + f : nullptr, s));
    }
    return HOLO_OK;
}

holo_status check_n(int n)
{
    if (n < 16 || n > 2048 || (n & (n - 1)) != 0)
        return set_error(HOLO_ERR_INVALID_ARG, "n must be a power of two in [16, 2048], got %d", n);
    return HOLO_OK;
}

holo_status check_region(holo_region om, int n)
{
    if (om.row0 < 0 || om.col0 < 0 || om.row1 > n || om.col1 > n || om.row0 >= om.row1 || om.col0 >= om.col1)
        return set_error(HOLO_ERR_INVALID_ARG, "region [%d,%d)x[%d,%d) empty or outside [0,%d)^2", om.row0,
                         om.row1, om.col0, om.col1, n);
    return HOLO_OK;
}

} // namespace holo

using namespace holo;

extern "C" size_t holo_ospr_workspace_size(int32_t n, int32_t n_frames, int32_t n_sub)
{
    (void)n_frames;
    if (check_n(n) != HOLO_OK || n_sub < 1)
        return 0;
    return ospr_ws_layout(n, n_sub, nullptr, nullptr);
}

extern "C" holo_status holo_ospr_generate(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                          const holo_c64 *lut, uint64_t n_lut, uint64_t phase_offset,
                                          int32_t sf_begin, int32_t sf_end, uint8_t *holo_bits,
                                          float *intensity, double *mse, holo_region omega, void *ws,
                                          size_t ws_bytes, holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(n_frames >= 1 && n_sub >= 1, "n_frames and n_sub must be >= 1 (got %d, %d)", n_frames, n_sub);
    HOLO_CHECK_ARG(0 <= sf_begin && sf_begin < sf_end && sf_end <= n_sub,
                   "sub-frame range [%d,%d) must be a non-empty part of [0,%d)", sf_begin, sf_end, n_sub);
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    HOLO_CHECK_ARG((lut == nullptr) == (n_lut == 0), "lut must be NULL iff n_lut == 0");
    HOLO_CHECK_ARG(target != nullptr && intensity != nullptr, "target and intensity are required");
    const bool full = (sf_begin == 0 && sf_end == n_sub);
    HOLO_CHECK_ARG(full || mse == nullptr, "mse must be NULL for a partial sub-frame range");
    HOLO_TRY(check_region(omega, n));
    HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
    const size_t need = holo_ospr_workspace_size(n, n_frames, n_sub);
    if (ws_bytes < need)
        return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    const float2 *tw = nullptr;
    HOLO_TRY(fft::twiddles(&tw));
    cudaStream_t s = (cudaStream_t)stream;
    const float2 *l = (const float2 *)lut;
#define HOLO_OSPR_CASE(NN)                                                                         \
    case NN:                                                                                       \
        return ospr_run<NN>(tw, target, n_frames, n_sub, l, n_lut, phase_offset, sf_begin, sf_end,     \
                            holo_bits, intensity, mse, omega, ws, s);
    switch (n) {
        HOLO_OSPR_CASE(16)
        HOLO_OSPR_CASE(32)
        HOLO_OSPR_CASE(64)
        HOLO_OSPR_CASE(128)
        HOLO_OSPR_CASE(256)
        HOLO_OSPR_CASE(512)
        HOLO_OSPR_CASE(1024)
        HOLO_OSPR_CASE(2048)
    default:
        return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
    }
#undef HOLO_OSPR_CASE
}

extern "C" holo_status holo_ospr_finalize(const float *target, const float *intensity_sum, int32_t n,
                                          int32_t n_frames, int32_t n_sub, holo_region omega,
                                          float *intensity_mean, double *mse, void *ws, size_t ws_bytes,
                                          holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(n_frames >= 1 && n_sub >= 1, "n_frames and n_sub must be >= 1");
    HOLO_CHECK_ARG(target && intensity_sum && intensity_mean, "target, intensity_sum, intensity_mean required");
    HOLO_TRY(check_region(omega, n));
    const size_t need = (size_t)kFinBlocks * 5 * sizeof(double);
    if (mse) {
        HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
        if (ws_bytes < need)
            return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    }
    const size_t P = (size_t)n * n;
    for (int f = 0; f < n_frames; ++f)
        HOLO_TRY(finalize_frame(intensity_sum + f * P, target + f * P, n, 0, 1.0f / (float)n_sub,
                                intensity_mean + f * P, omega, (double *)ws, mse ? mse + f : nullptr,
                                (cudaStream_t)stream));
    return HOLO_OK;
}
