// hooks.cu -- test hooks of the C ABI (not on the hot path): a plain unitary 2D
// DFT/IDFT (Eqs. (1)-(2)) built from the same FFT device code as the
// fused passes, and step a2 (randomisation) alone for bit-exact probing.
#include "rows2w.cuh"

namespace holo {

template <int N, bool INV>
struct HookColBody {
    static constexpr int kStages = 3;   // measured best column-pipeline variant for this body
    static constexpr int kWidth = N >= 4096 ? 4 : 8;   // columns per tile (4096: one 133 KB stage)
    static constexpr int kGroups = 1;
    struct Args {
        const float2 *tw;
        float2 *buf;
        float scale;
    };
    template <class F, int W>
    static __device__ __forceinline__ void run(float2 (&v)[F::E], float2 *sm, uint32_t *, int c, int t, int fr,
                                               int tile,
                                               const Args &a, const F &fft)
    {
        constexpr int R1 = F::T, E = F::E;   // element m of thread t = row t + R1*m; W columns per tile
        fft.template run<INV, W>(v, sm, t);
#pragma unroll
        for (int r = 0; r < E; ++r)
            v[r] = make_float2(v[r].x * a.scale, v[r].y * a.scale);   // stored by the pipeline (TMA)
    }
};

template <int N>
static holo_status fft2_run(const float2 *tw, const float2 *in, float2 *out, int batch, int inverse, cudaStream_t s)
{
    const int nrows = batch * N;
    const float scale = 1.0f / (float)N;   // unitary: 1/sqrt(N*N), an exact power of two
    if (inverse) {
        HOLO_TRY((launch_row_fft<N, true>(K_FFT_ROWS, tw, in, out, nrows, s)));
        typename HookColBody<N, true>::Args a{tw, out, scale};
        HOLO_TRY((launch_cols<N, HookColBody<N, true>>(K_FFT_COLS, out, batch, a, s)));
    } else {
        HOLO_TRY((launch_row_fft<N, false>(K_FFT_ROWS, tw, in, out, nrows, s)));
        typename HookColBody<N, false>::Args a{tw, out, scale};
        HOLO_TRY((launch_cols<N, HookColBody<N, false>>(K_FFT_COLS, out, batch, a, s)));
    }
    return HOLO_OK;
}

__global__ void __launch_bounds__(256)
randomise_kernel(const float *__restrict__ T, int P, const float2 *__restrict__ lut, LutIndexer ix, uint32_t base,
                 float2 *__restrict__ r_out)
{
    HOLO_PDL_ENTRY();
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
        const float t = T[p];
        if (lut == nullptr) {
            r_out[p] = make_float2(t, 0.0f);
        } else {
            const float2 c = lut_at(lut, ix.mod_any((uint64_t)base + (uint64_t)p));
            r_out[p] = make_float2(t * c.x, t * c.y);   // a2, fp32 products
        }
    }
}

holo_status check_n(int n);

} // namespace holo

using namespace holo;

extern "C" holo_status holo_fft2(const holo_c64 *in, holo_c64 *out, int32_t n, int32_t batch, int32_t inverse,
                                 holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(in != nullptr && out != nullptr, "in/out is NULL");
    HOLO_CHECK_ARG(batch >= 1, "batch must be >= 1");
    const float2 *tw = nullptr;
    HOLO_TRY(fft::twiddles(&tw));
    const float2 *i = (const float2 *)in;
    float2 *o = (float2 *)out;
    cudaStream_t s = (cudaStream_t)stream;
    switch (n) {
    case 16: return fft2_run<16>(tw, i, o, batch, inverse, s);
    case 32: return fft2_run<32>(tw, i, o, batch, inverse, s);
    case 64: return fft2_run<64>(tw, i, o, batch, inverse, s);
    case 128: return fft2_run<128>(tw, i, o, batch, inverse, s);
    case 256: return fft2_run<256>(tw, i, o, batch, inverse, s);
    case 512: return fft2_run<512>(tw, i, o, batch, inverse, s);
    case 1024: return fft2_run<1024>(tw, i, o, batch, inverse, s);
    case 2048: return fft2_run<2048>(tw, i, o, batch, inverse, s);
    case 4096: return fft2_run<4096>(tw, i, o, batch, inverse, s);
    default: return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
    }
}

extern "C" holo_status holo_debug_randomise(const float *target, int32_t n, const holo_c64 *lut, uint64_t n_lut,
                                            uint64_t offset, holo_c64 *r_out, holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(target != nullptr && r_out != nullptr, "target/r_out is NULL");
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    HOLO_CHECK_ARG((lut == nullptr) == (n_lut == 0), "lut must be NULL iff n_lut == 0");
    const LutIndexer ix = LutIndexer::make(n_lut ? (uint32_t)n_lut : 1u, n);
    const uint32_t base = n_lut ? (uint32_t)(offset % n_lut) : 0u;
    const int P = n * n;
    const int grid = (P + 255) / 256 < 1184 ? (P + 255) / 256 : 1184;
    return launch(K_RANDOMISE, randomise_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, target, P,
                  (const float2 *)lut, ix, base, (float2 *)r_out);
}
