// phase.cuh -- the phase source of step a0 in device code: SplitMix64 in counter
// form (R-4) and recipe R-5 for (cos, sin) of 2 pi u / 2^32 (R-3), every product and
// sum an explicit round-to-nearest double intrinsic so that nvcc cannot contract it
// into FMAs.  Used by lut_generate (the pool, "generated at compile time") and by
// the on-the-fly PRNG source of pass A (holo_ospr_generate_prng),
// which therefore reproduce each other bit for bit (R-4 prefix property, c3 #15).
#pragma once

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


// Phase of global draw index k of the stream `seed`: lut_generate(seed, L)[k] for any L > k.
__device__ __forceinline__ float2 prng_phase(uint64_t seed, uint64_t k)
{
    return r5_phase((uint32_t)(splitmix64_at(seed, k) >> 32));
}

} // namespace holo
