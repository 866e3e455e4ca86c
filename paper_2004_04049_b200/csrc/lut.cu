// lut.cu -- step a0: generation of the phase pool ("Random numbers can be
// generated at compile time to fill the LUT").
//
// Entry k = recipe R-5 applied to u_k = high word of SplitMix64 output k (R-3,
// R-4).  The recipe is fixed to the operation (every product and sum is an
// explicit round-to-nearest double intrinsic, so nvcc cannot contract it into
// FMAs) so that the pool is bit-identical to any other implementation of R-5,
// in particular the fp64 CPU oracle (R-5; parity P-1).
#include "common.cuh"

namespace holo {

__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t k)
{
    uint64_t z = seed + (k + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Taylor polynomials on [0, pi/4] in Horner form: sin to x^17, cos to x^16.
__device__ __forceinline__ double r5_sin(double x, double s)
{
    double p = 1.0 / 355687428096000.0;
    p = __dadd_rn(-1.0 / 1307674368000.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 6227020800.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 39916800.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 362880.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 5040.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 120.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 6.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0, __dmul_rn(s, p));
    return __dmul_rn(x, p);
}

__device__ __forceinline__ double r5_cos(double s)
{
    double p = 1.0 / 20922789888000.0;
    p = __dadd_rn(-1.0 / 87178291200.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 479001600.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 3628800.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 40320.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 720.0, __dmul_rn(s, p));
    p = __dadd_rn(1.0 / 24.0, __dmul_rn(s, p));
    p = __dadd_rn(-1.0 / 2.0, __dmul_rn(s, p));
    return __dadd_rn(1.0, __dmul_rn(s, p));
}

// (cos, sin) of 2 pi u / 2^32 by R-5: octant reduction with reflection of odd
// octants, one multiply by fl(pi/2^31), polynomials, exact quadrant fix-up,
// RN-even rounding to fp32 and -0 -> +0.
__device__ __forceinline__ float2 r5_phase(uint32_t u)
{
    const uint32_t o = u >> 29;
    uint32_t f = u & 0x1FFFFFFFu;
    if (o & 1u)
        f = 0x20000000u - f;
    const double x = __dmul_rn((double)f, 3.14159265358979323846264338327950288 / 2147483648.0);
    const double s = __dmul_rn(x, x);
    const double S = r5_sin(x, s), Cc = r5_cos(s);
    double c, sn;
    switch (o) {
    case 0: c = Cc;  sn = S;   break;
    case 1: c = S;   sn = Cc;  break;
    case 2: c = -S;  sn = Cc;  break;
    case 3: c = -Cc; sn = S;   break;
    case 4: c = -Cc; sn = -S;  break;
    case 5: c = -S;  sn = -Cc; break;
    case 6: c = S;   sn = -Cc; break;
    default: c = Cc; sn = -S;  break;
    }
    float cf = __double2float_rn(c), sf = __double2float_rn(sn);
    if (cf == 0.0f)
        cf = 0.0f;
    if (sf == 0.0f)
        sf = 0.0f;
    return make_float2(cf, sf);
}

// Grid-stride over entries; 64-bit counter (full-length pools exceed 2^24).
__global__ void __launch_bounds__(256) lut_generate_kernel(uint64_t seed, uint64_t n_lut, float2 *lut)
{
    HOLO_PDL_ENTRY();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_lut; k += stride)
        lut[k] = r5_phase((uint32_t)(splitmix64_at(seed, k) >> 32));
}

} // namespace holo

using namespace holo;

extern "C" holo_status holo_lut_generate(uint64_t seed, uint64_t n_lut, holo_c64 *lut, holo_stream stream)
{
    HOLO_CHECK_ARG(n_lut >= 1 && n_lut < (1ull << 31), "n_lut must be in [1, 2^31), got %llu",
                   (unsigned long long)n_lut);
    HOLO_CHECK_ARG(lut != nullptr, "lut is NULL");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // 8 resident 256-thread CTAs per SM, grid-stride beyond that.
    uint64_t want = (n_lut + 255) / 256;
    uint64_t cap = (uint64_t)sms * 8;
    unsigned grid = (unsigned)(want < cap ? want : cap);
    return launch(K_LUT_GENERATE, lut_generate_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream,
                  seed, n_lut, (float2 *)lut);
}
