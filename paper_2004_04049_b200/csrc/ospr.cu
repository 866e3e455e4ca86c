// ospr.cu -- One-Step Phase-Retrieval (Fig. 2 right, P:47, P:53;
// steps a1-a7 of DESIGN.md §1) as three fused FFT passes per chunk of
// sub-frame pairs plus a finalize pass per frame.
//
//   pass A  ospr_rows_a(2)  R_s = T * lut[(base_s + p) mod L] (or the on-the-fly
//                        source, LUT_PRNG) for the two sub-frames a, b of a pair at
//                        pixels p and -p, Hermitian parts packed as Z = 2 Herm(R_a)
//                        + 2i Herm(R_b) (so F^-1{Z} = 2 (Re H_a + i Re H_b),
//                        DESIGN.md §5), built (conjugated) in shared memory and
//                        row-IFFTed in the same kernel; N >= 1024: a warp pair per
//                        mirrored row pair (ospr_rows_a2_kernel).
//   pass B  ospr_cols    column IFFT -> H; a4: bit_a = Re H >= 0, bit_b = Im H >= 0,
//                        8x8 bit transposes into tile-major sign bytes;
//                        h' = (+-1) + i(+-1); column FFT of h'; TMA store in place.
//   pass C  ospr_rows_c  row FFT -> X = F{h'_a} + i F{h'_b}; accumulate |X|^2/N^2
//                        over the chunk's pairs in registers; one RMW of the
//                        frame accumulator A per chunk; on the frame's last chunk
//                        extra CTAs turn the sign bytes into packed holograms (R-8).
//   finalize             I[k] = (A[k] + A[-k]) / 2 / N_SF  (= sum_s |F{h'_s}|^2 / N_SF,
//                        DESIGN.md §5) and the fp64 MSE over Omega (last-CTA
//                        fixed-order reduction).
//
// All 1/sqrt(N) factors of Eqs. (1)-(2) are dropped inside the passes: a positive
// scale does not change sign(Re H), and the forward scale 1/N^2 on |X|^2 is an
// exact power of two applied in pass C.
#include <type_traits>

#include "passes.cuh"
#include "phase.cuh"
#include "rows2w.cuh"

namespace holo {

constexpr int kMaxChunk = 64;

// Device address of this translation unit's one-entry pool {1 + 0i} (common.cuh).
static holo_status flat_lut(const float2 **p)
{
    void *a = nullptr;
    cudaError_t e = cudaGetSymbolAddress(&a, k_flat_lut);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaGetSymbolAddress(k_flat_lut)");
    *p = (const float2 *)a;
    return HOLO_OK;
}

constexpr int kFinBlocks = 592;   // finalize CTAs per frame (fixed => deterministic sums; 4 per SM)
constexpr int kFinThreads = 256;
constexpr size_t kFinWsBytes = (size_t)kFinBlocks * 5 * sizeof(double) + 256;   // partial sums + ticket


// ---- randomisation (a1, a2) with Hermitian pairing ---------------------------------------------
// For an unordered pixel pair {p, -p} of one sub-frame pair (a, b), T and the LUT are read once:
//   Ha = R_a(p) + conj(R_a(-p)) = 2 Herm(R_a)(p),   Hb likewise,   R_s = T * lut[(base_s + p) mod L]
//   Z(p) = Ha + i Hb,   Z(-p) = conj(Ha) + i conj(Hb)   (the Hermitian parts are conjugate-symmetric)
// so that F^-1{Z} = 2 (Re H_a + i Re H_b) after pass A.
// Draw base of global sub-frame s: (off + s * N^2) mod L with off, N^2 reduced mod L on the
// host (all operands < 2^31, so the 64-bit product cannot overflow).
__device__ __forceinline__ uint32_t subframe_base(uint32_t off_mod, uint64_t s, uint32_t p_mod, const LutIndexer &ix)
{
    return ix.mod64((uint64_t)off_mod + (uint64_t)ix.mod64(s) * (uint64_t)p_mod);
}

// conj(Z) at the pixel pair {p1, p2 = -p1} of one sub-frame pair (a, b) from T (t1, t2) and the
// phase factors a1, a2 (sub-frame a) and b1, b2 (sub-frame b) at p1, p2.
struct ZPair {
    float2 z1, z2;
};
__device__ __forceinline__ ZPair z_pair(float t1, float t2, float tb1, float tb2, float2 a1, float2 a2, float2 b1,
                                        float2 b2)
{
    // Ha = t1 a1 + t2 conj(a2),  Hb = tb1 b1 + tb2 conj(b2)  (tb = t, or 0 for an absent b)
    const float2 ha = f2::fma(conjf2(a2), f2::bc(t2), f2::mul(a1, f2::bc(t1)));
    const float2 hb = f2::fma(conjf2(b2), f2::bc(tb2), f2::mul(b1, f2::bc(tb1)));
    // Z(p) = Ha + i Hb,  Z(-p) = conj(Ha) + i conj(Hb) = (Ha.x + Hb.y, Hb.x - Ha.y); returned
    // CONJUGATED (sign flips folded into the adds' operand modifiers): pass A transforms
    // conj(Z) with the forward body, F^-1{Z} = conj(F{conj(Z)}).
    return ZPair{cadd(conjf2(ha), make_float2(-hb.y, -hb.x)), cadd(ha, make_float2(hb.y, -hb.x))};
}

// LUT index base of row y of a sub-frame whose draws start at base: (base + y N) mod L.
__device__ __forceinline__ uint32_t row_base(uint32_t base, int y, int n, const LutIndexer &ix)
{
    return ix.mod32(base + (uint32_t)y * (uint32_t)n);   // base < L < 2^31, y n < 2^22: no overflow
}

// ---- pass A: randomisation (a1, a2) with Hermitian pairing, fused into the row IFFT --------------
// A warp unit is ROWS rows of one sub-frame pair made of ROWS/2 mirrored row pairs
// {y, -y mod N}: item 0 = rows {0, N/2} (each its own mirror), item k > 0 = rows {k, N-k}.
// The warp first builds Z for all the unit's rows in its shared-memory slot, reading T
// and the LUT once per pixel pair {p, -p} (coalesced rows, L1/L2-resident), then
// row-IFFTs them GPW rows per round and writes the result (no Z round trip through HBM).
template <int N>
struct RowA {
    using P = fft::Plan<N>;
    static constexpr int GPW = 32 / P::T;                        // rows per FFT round
    static constexpr int ROWS = GPW < 2 ? 2 : GPW;               // rows per unit
    static constexpr int ROUNDS = ROWS / GPW;
    static constexpr int IPU = ROWS / 2;                         // mirrored row pairs per unit
    static constexpr int UNITS_PER_PAIR = (N / 2) / IPU;
    static constexpr int WPC = 4;
    static constexpr uint32_t SLOT = ((uint32_t)ROWS * P::SMEM * 8 + 127) / 128 * 128;
    static constexpr size_t SMEM = (size_t)WPC * SLOT;
};

// The phase source of pass A: the LUT (modes LUT_WRAP / LUT_POW2 / LUT_GENERAL, index
// (off + s N^2 + p) mod L) or, in mode LUT_PRNG, SplitMix64 + recipe R-5 evaluated per
// draw (index off + s N^2 + p, no wrap): bit-identical to a LUT longer than every index.
struct PhaseSrc {
    const float2 *lut;         // the pool, or (LUT_PRNG_TABLE) the 2^q sin/cos table
    LutIndexer ix;
    uint32_t off_mod, p_mod;   // phase_offset mod L, N^2 mod L
    uint64_t seed, off;        // LUT_PRNG(_TABLE): stream seed, phase_offset
    uint32_t shift;            // LUT_PRNG_TABLE: 32 - q (the table index is the code's top q bits)
};

template <int N, int LMODE>
struct PhaseRows {
    static constexpr bool kStream = LMODE == LUT_PRNG || LMODE == LUT_PRNG_TABLE;   // no pool, no wrap
    using Base = typename std::conditional<kStream, uint64_t, uint32_t>::type;
    // draw index of pixel 0 of global sub-frame s (mod L for the LUT)
    static __device__ __forceinline__ Base subframe(const PhaseSrc &ps, uint64_t s)
    {
        if constexpr (kStream)
            return ps.off + s * (uint64_t)N * N;
        else
            return subframe_base(ps.off_mod, s, ps.p_mod, ps.ix);
    }
    static __device__ __forceinline__ Base row(const PhaseSrc &ps, Base sb, int y)
    {
        if constexpr (kStream)
            return sb + (uint64_t)y * N;
        else
            return row_base(sb, y, N, ps.ix);
    }
    static __device__ __forceinline__ float2 at(const PhaseSrc &ps, Base rb, int x)
    {
        if constexpr (LMODE == LUT_PRNG)
            return prng_phase(ps.seed, rb + (uint64_t)x);
        else if constexpr (LMODE == LUT_PRNG_TABLE)   // PRNG + a small sin/cos table (R-25)
            return __ldg(ps.lut + ((uint32_t)(splitmix64_at(ps.seed, rb + (uint64_t)x) >> 32) >> ps.shift));
        else
            return __ldg(ps.lut + ps.ix.template mod_t<LMODE>(rb + (uint32_t)x));
    }
};

template <int N, int LMODE, bool ZOUT = false>
__global__ void __launch_bounds__(RowA<N>::WPC * 32)
ospr_rows_a_kernel(const float2 *__restrict__ tw, const float *__restrict__ T, const PhaseSrc ps, uint64_t sf_first,
                   int npairs, int last_pair_has_b, float2 *__restrict__ buf, unsigned *zc)
{
    HOLO_PDL_ENTRY();
    if (zc != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
        *zc = 0u;                        // the frame's fused-finalize ticket (pass C, last chunk)
    using P = fft::Plan<N>;
    using RA = RowA<N>;
    using PR = PhaseRows<N, LMODE>;
    using Base = typename PR::Base;
    constexpr int R1 = P::R1, E = P::E, GPW = RA::GPW, IPU = RA::IPU;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane / R1, t = lane % R1;
    float2 *sl = reinterpret_cast<float2 *>(smem_raw + (size_t)warp * RA::SLOT);
    fft::Twiddles<N> twr;
    twr.load(tw, t);
    const int nunits = npairs * RA::UNITS_PER_PAIR;
    #pragma unroll 1
    for (int u = blockIdx.x * RA::WPC + warp; u < nunits; u += gridDim.x * RA::WPC) {
        const int pair = u / RA::UNITS_PER_PAIR, k0 = (u % RA::UNITS_PER_PAIR) * IPU;
        const bool has_b = (pair < npairs - 1) || last_pair_has_b;
        const Base ba = PR::subframe(ps, sf_first + 2 * (uint64_t)pair);
        const Base bb = PR::subframe(ps, sf_first + 2 * (uint64_t)pair + 1);
        const float bsc = has_b ? 1.0f : 0.0f;   // an absent sub-frame b contributes R_b = 0
        // build Z: row slot 2i holds row y, slot 2i+1 its mirror row ym (padded stride P::SMEM).
        // Rows 0 and N/2 are their own mirrors: their pairs are x <-> N - x, x in [0, N/2].
#pragma unroll 1
        for (int j = 0; j < 2 * IPU; j += 2) {
            const int k = k0 + j / 2;
            float2 *s0 = sl + (size_t)j * P::SMEM, *s1 = s0 + P::SMEM;
            if (k > 0) {   // pixel pairs (k, x) <-> (N - k, N - x), x < N: N/32 per lane
                const int y = k, ym = N - k;
                const Base a1 = PR::row(ps, ba, y), a2 = PR::row(ps, ba, ym);
                const Base b1 = PR::row(ps, bb, y), b2 = PR::row(ps, bb, ym);
                const float *T1 = T + (size_t)y * N, *T2 = T + (size_t)ym * N;
                constexpr int M = N < 32 ? 1 : N / 32;
                if constexpr (LMODE == LUT_WRAP && N >= 64) {
                    // No index of the four LUT rows wraps (the usual case; always for L a
                    // multiple of N with an aligned offset): every load of the row pair is a
                    // fixed offset from a per-lane base pointer, no per-pixel index arithmetic.
                    const uint32_t lim = ps.ix.L - (uint32_t)N;
                    if (a1 <= lim && a2 <= lim && b1 <= lim && b2 <= lim) {
                        const float2 *LA1 = ps.lut + a1 + lane, *LB1 = ps.lut + b1 + lane;
                        const float2 *LA2 = ps.lut + a2 + (N - lane), *LB2 = ps.lut + b2 + (N - lane);
                        const float *T1l = T1 + lane, *T2l = T2 + (N - lane);
                        float2 *S0 = s0 + lane, *S1 = s1 + (N - lane);
                        {   // m = 0: the mirror of x = 0 is 0, not N
                            const int xm = (N - lane) & (N - 1);
                            const float t1 = T1l[0], t2 = T2[xm];
                            const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, LA1[0], ps.lut[a2 + xm], LB1[0],
                                                   ps.lut[b2 + xm]);
                            S0[0] = z.z1;
                            s1[xm] = z.z2;
                        }
#pragma unroll 16
                        for (int m = 1; m < M; ++m) {
                            const float t1 = T1l[32 * m], t2 = T2l[-32 * m];
                            const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, LA1[32 * m], LA2[-32 * m], LB1[32 * m],
                                                   LB2[-32 * m]);
                            S0[32 * m] = z.z1;
                            S1[-32 * m] = z.z2;
                        }
                        continue;
                    }
                }
#pragma unroll (LMODE == LUT_PRNG ? 2 : 16)
                for (int m = 0; m < M; ++m) {
                    const int x = lane + 32 * m;
                    if (N < 32 && x >= N)
                        break;
                    const int xm = (N - x) & (N - 1);
                    const float t1 = T1[x], t2 = T2[xm];
                    const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a2, xm),
                                           PR::at(ps, b1, x), PR::at(ps, b2, xm));
                    s0[x] = z.z1;
                    s1[xm] = z.z2;
                }
            } else {       // rows 0 and N/2: pairs (yy, x) <-> (yy, N - x), x <= N/2
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const int yy = h ? N / 2 : 0;
                    float2 *d = h ? s1 : s0;
                    const Base a1 = PR::row(ps, ba, yy), b1 = PR::row(ps, bb, yy);
                    const float *T1 = T + (size_t)yy * N;
                    for (int x = lane; x <= N / 2; x += 32) {
                        const int xm = (N - x) & (N - 1);
                        const float t1 = T1[x], t2 = T1[xm];
                        const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a1, xm),
                                               PR::at(ps, b1, x), PR::at(ps, b1, xm));
                        d[x] = z.z1;
                        d[xm] = z.z2;
                    }
                }
            }
        }
        __syncwarp();
        // row IFFT, GPW rows per round: F^-1{x} = conj(F{conj(x)}) (one transform body)
#pragma unroll 1
        for (int r = 0; r < RA::ROUNDS; ++r) {
            const int slot = r * GPW + g;
            float2 *sg = sl + (size_t)slot * P::SMEM;
            float2 v[E];
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = sg[t + R1 * m];                       // conj(Z), built so by the producer
            if constexpr (!ZOUT)                             // ZOUT: the test hook writes conj(Z) itself
                fft::fft2pass<N, false, 1, true>(v, sg, t, twr);
            const int k = k0 + slot / 2;
            const int y = (slot & 1) ? (k > 0 ? N - k : N / 2) : k;
            float2 *o = buf + ((size_t)pair * N + y) * N;
#pragma unroll
            for (int m = 0; m < E; ++m)
                o[t + R1 * m] = v[m];   // conj of the row IFFT (the pair buffer is kept conjugated)
        }
        __syncwarp();
    }
}

// Pass A for N >= 1024 (one row per warp item): a unit {y, N - y} is shared by a PAIR of warps.
// Each warp builds the Z pixel pairs of one half of the columns (both rows), the pair meets at
// a named barrier, then each warp row-IFFTs one of the two rows in place.  One row slot per warp
// (instead of two) and pool twiddles (instead of registers) let half again as many warps reside
// per SM, to hide the producer's L2 latency.
template <int N>
struct RowA2 {
    using P = fft::Plan<N>;
    static_assert(32 / P::T == 1, "one row per warp item");
    static constexpr int WPC = 4, UPC = WPC / 2;                 // warps, units per CTA
    static constexpr uint32_t SLOT = ((uint32_t)P::SMEM * 8 + 127) / 128 * 128;   // one row
    static constexpr size_t SMEM = (size_t)WPC * SLOT;
    static constexpr int UNITS_PER_PAIR = N / 2;
};

#ifndef HOLO_A2_MINB2048
#define HOLO_A2_MINB2048 3
#endif
template <int N, int LMODE, bool ZOUT = false>
__global__ void __launch_bounds__(RowA2<N>::WPC * 32, (N == 2048 && HOLO_A2_MINB2048) ? HOLO_A2_MINB2048 : 0)
ospr_rows_a2_kernel(const float2 *__restrict__ tw, const float *__restrict__ T, const PhaseSrc ps, uint64_t sf_first,
                    int npairs, int last_pair_has_b, float2 *__restrict__ buf, unsigned *zc)
{
    HOLO_PDL_ENTRY();
    if (zc != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
        *zc = 0u;                        // the frame's fused-finalize ticket (pass C, last chunk)
    using P = fft::Plan<N>;
    using RA = RowA2<N>;
    using PR = PhaseRows<N, LMODE>;
    using Base = typename PR::Base;
    constexpr int R1 = P::R1, E = P::E, M = N / 32, MH = M / 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = lane;
    const int up = warp >> 1, h = warp & 1;                      // unit slot in the CTA, half
    float2 *s0 = reinterpret_cast<float2 *>(smem_raw + (size_t)(2 * up) * RA::SLOT);
    float2 *s1 = reinterpret_cast<float2 *>(smem_raw + (size_t)(2 * up + 1) * RA::SLOT);
    // pass-2 twiddles factorised into registers (no loads per transform; 20 registers instead of 62
    // at N = 1024: 42.4 -> 39.9 us at C3; at N = 2048 capped at 168 registers for three CTAs per SM:
    // C5 0.634 -> 0.620 ms)
#ifndef HOLO_A2_TWF_MAXN
#define HOLO_A2_TWF_MAXN 2048
#endif
    using TwSrc = typename std::conditional<(N <= HOLO_A2_TWF_MAXN), fft::TwFact<N>, fft::TwGlobal<N>>::type;
    TwSrc twp;
    if constexpr (N <= HOLO_A2_TWF_MAXN)
        twp.load(tw, t);
    else
        twp.p = tw + P::TW_OFFSET + t;
    const int nunits = npairs * RA::UNITS_PER_PAIR;
    #pragma unroll 1
    for (int u = blockIdx.x * RA::UPC + up; u < nunits; u += gridDim.x * RA::UPC) {
        const int pair = u / RA::UNITS_PER_PAIR, k = u % RA::UNITS_PER_PAIR;
        const bool has_b = (pair < npairs - 1) || last_pair_has_b;
        const Base ba = PR::subframe(ps, sf_first + 2 * (uint64_t)pair);
        const Base bb = PR::subframe(ps, sf_first + 2 * (uint64_t)pair + 1);
        const float bsc = has_b ? 1.0f : 0.0f;   // an absent sub-frame b contributes R_b = 0
        const int y = k, ym = k > 0 ? N - k : N / 2;
        if (k > 0) {   // pixel pairs (y, x) <-> (ym, N - x), this warp: x in [h N/2, (h+1) N/2)
            const int x0 = h * (N / 2);
            const Base a1 = PR::row(ps, ba, y), a2 = PR::row(ps, ba, ym);
            const Base b1 = PR::row(ps, bb, y), b2 = PR::row(ps, bb, ym);
            const float *T1 = T + (size_t)y * N, *T2 = T + (size_t)ym * N;
            bool fast = false;
            if constexpr (LMODE == LUT_WRAP) {
                const uint32_t lim = ps.ix.L - (uint32_t)N;
                fast = a1 <= lim && a2 <= lim && b1 <= lim && b2 <= lim;
            }
            if (fast) {   // no LUT row wraps: fixed offsets from per-lane base pointers
                const int xl = x0 + lane;
                const float2 *LA1 = ps.lut + (uint32_t)a1 + xl, *LB1 = ps.lut + (uint32_t)b1 + xl;
                const float2 *LA2 = ps.lut + (uint32_t)a2 + (N - xl), *LB2 = ps.lut + (uint32_t)b2 + (N - xl);
                const float *T1l = T1 + xl, *T2l = T2 + (N - xl);
                float2 *S0 = s0 + xl, *S1 = s1 + (N - xl);
                {   // m = 0: the mirror of x = 0 is 0, not N
                    const int xm = (N - xl) & (N - 1);
                    const float t1 = T1l[0], t2 = T2[xm];
                    const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, LA1[0], ps.lut[(uint32_t)a2 + xm], LB1[0],
                                           ps.lut[(uint32_t)b2 + xm]);
                    S0[0] = z.z1;
                    s1[xm] = z.z2;
                }
                if (has_b) {   // (every pair but an unpaired tail: no R_b scaling in the loop)
#pragma unroll
                    for (int m = 1; m < MH; ++m) {
                        const float t1 = T1l[32 * m], t2 = T2l[-32 * m];
                        const ZPair z = z_pair(t1, t2, t1, t2, LA1[32 * m], LA2[-32 * m], LB1[32 * m], LB2[-32 * m]);
                        S0[32 * m] = z.z1;
                        S1[-32 * m] = z.z2;
                    }
                } else {
#pragma unroll 4
                    for (int m = 1; m < MH; ++m) {
                        const float t1 = T1l[32 * m], t2 = T2l[-32 * m];
                        const ZPair z = z_pair(t1, t2, 0.0f, 0.0f, LA1[32 * m], LA2[-32 * m], LB1[32 * m],
                                               LB2[-32 * m]);
                        S0[32 * m] = z.z1;
                        S1[-32 * m] = z.z2;
                    }
                }
            } else {
#pragma unroll (LMODE == LUT_PRNG ? 2 : 8)
                for (int m = 0; m < MH; ++m) {
                    const int x = x0 + lane + 32 * m, xm = (N - x) & (N - 1);
                    const float t1 = T1[x], t2 = T2[xm];
                    const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a2, xm),
                                           PR::at(ps, b1, x), PR::at(ps, b2, xm));
                    s0[x] = z.z1;
                    s1[xm] = z.z2;
                }
            }
        } else {       // unit 0: rows 0 and N/2, each its own mirror; this warp builds row h
            const int yy = h ? N / 2 : 0;
            float2 *d = h ? s1 : s0;
            const Base a1 = PR::row(ps, ba, yy), b1 = PR::row(ps, bb, yy);
            const float *T1 = T + (size_t)yy * N;
            for (int x = lane; x <= N / 2; x += 32) {
                const int xm = (N - x) & (N - 1);
                const float t1 = T1[x], t2 = T1[xm];
                const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a1, xm),
                                       PR::at(ps, b1, x), PR::at(ps, b1, xm));
                d[x] = z.z1;
                d[xm] = z.z2;
            }
        }
        asm volatile("bar.sync %0, 64;" ::"r"(1 + up) : "memory");   // both halves of Z are built
        // row IFFT of row (h ? ym : y) in place: F^-1{x} = conj(F{conj(x)})
        float2 *sg = h ? s1 : s0;
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sg[t + R1 * m];                           // conj(Z), built so by the producer
        if constexpr (!ZOUT)                                 // ZOUT: the test hook writes conj(Z) itself
            fft::fft2pass_impl<N, false, 1, true>(v, sg, t, twp);
        float2 *o = buf + ((size_t)pair * N + (h ? ym : y)) * N;
#pragma unroll
        for (int m = 0; m < E; ++m)
            o[t + R1 * m] = v[m];       // conj of the row IFFT (the pair buffer is kept conjugated)
        asm volatile("bar.sync %0, 64;" ::"r"(1 + up) : "memory");   // both rows read before reuse
    }
}

// Pass A for N = 4096 (a row transform spans two warps, R-26): one CTA of four warps per unit
// {y, N - y}.  All four warps build Z for the unit's pixel pairs (a quarter of the columns
// each) into two row slots, then warps 0-1 row-IFFT row y and warps 2-3 row N - y, each pair
// on its own named barrier.  Same phase indexing and Z arithmetic as ospr_rows_a2_kernel.
template <int N>
struct RowA4 {
    using P = fft::Plan<N>;
    static_assert(P::T == 64, "two warps per row");
    static constexpr int THREADS = 128;
    static constexpr uint32_t SLOT = ((uint32_t)P::SMEM * 8 + 127) / 128 * 128;   // one row
    static constexpr size_t SMEM = 2 * (size_t)SLOT;
    static constexpr int UNITS_PER_PAIR = N / 2;
};

template <int N, int LMODE, bool ZOUT = false>
__global__ void __launch_bounds__(RowA4<N>::THREADS, 3)
ospr_rows_a4_kernel(const float2 *__restrict__ tw, const float *__restrict__ T, const PhaseSrc ps, uint64_t sf_first,
                    int npairs, int last_pair_has_b, float2 *__restrict__ buf)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    using RA = RowA4<N>;
    using PR = PhaseRows<N, LMODE>;
    using Base = typename PR::Base;
    constexpr int R1 = P::R1, E = P::E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *s0 = reinterpret_cast<float2 *>(smem_raw);
    float2 *s1 = reinterpret_cast<float2 *>(smem_raw + RA::SLOT);
    const int tid = threadIdx.x, grp = tid >> 6, t = tid & 63;
    const fft::GroupSync gsync{1 + grp, 64};
    const int nunits = npairs * RA::UNITS_PER_PAIR;
    #pragma unroll 1
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int pair = u / RA::UNITS_PER_PAIR, k = u % RA::UNITS_PER_PAIR;
        const bool has_b = (pair < npairs - 1) || last_pair_has_b;
        const Base ba = PR::subframe(ps, sf_first + 2 * (uint64_t)pair);
        const Base bb = PR::subframe(ps, sf_first + 2 * (uint64_t)pair + 1);
        const float bsc = has_b ? 1.0f : 0.0f;   // an absent sub-frame b contributes R_b = 0
        const int y = k, ym = k > 0 ? N - k : N / 2;
        if (k > 0) {   // pixel pairs (y, x) <-> (ym, N - x) for every x
            const Base a1 = PR::row(ps, ba, y), a2 = PR::row(ps, ba, ym);
            const Base b1 = PR::row(ps, bb, y), b2 = PR::row(ps, bb, ym);
            const float *T1 = T + (size_t)y * N, *T2 = T + (size_t)ym * N;
            bool fast = false;
            if constexpr (LMODE == LUT_WRAP) {
                const uint32_t lim = ps.ix.L - (uint32_t)N;
                fast = a1 <= lim && a2 <= lim && b1 <= lim && b2 <= lim;
            }
            if (fast) {   // no LUT row wraps: plain offsets from the row bases
                const float2 *LA1 = ps.lut + (uint32_t)a1, *LA2 = ps.lut + (uint32_t)a2;
                const float2 *LB1 = ps.lut + (uint32_t)b1, *LB2 = ps.lut + (uint32_t)b2;
#pragma unroll 8
                for (int x = tid; x < N; x += RA::THREADS) {
                    const int xm = (N - x) & (N - 1);
                    const float t1 = T1[x], t2 = T2[xm];
                    const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, LA1[x], LA2[xm], LB1[x], LB2[xm]);
                    s0[x] = z.z1;
                    s1[xm] = z.z2;
                }
            } else {
#pragma unroll 4
                for (int x = tid; x < N; x += RA::THREADS) {
                    const int xm = (N - x) & (N - 1);
                    const float t1 = T1[x], t2 = T2[xm];
                    const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a2, xm),
                                           PR::at(ps, b1, x), PR::at(ps, b2, xm));
                    s0[x] = z.z1;
                    s1[xm] = z.z2;
                }
            }
        } else {       // unit 0: rows 0 and N/2, each its own mirror; group grp builds row grp
            const int yy = grp ? N / 2 : 0;
            float2 *d = grp ? s1 : s0;
            const Base a1 = PR::row(ps, ba, yy), b1 = PR::row(ps, bb, yy);
            const float *T1 = T + (size_t)yy * N;
            for (int x = t; x <= N / 2; x += 64) {
                const int xm = (N - x) & (N - 1);
                const float t1 = T1[x], t2 = T1[xm];
                const ZPair z = z_pair(t1, t2, t1 * bsc, t2 * bsc, PR::at(ps, a1, x), PR::at(ps, a1, xm),
                                       PR::at(ps, b1, x), PR::at(ps, b1, xm));
                d[x] = z.z1;
                d[xm] = z.z2;
            }
        }
        __syncthreads();                                     // Z of both rows is built
        float2 *sg = grp ? s1 : s0;
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sg[t + R1 * m];                           // conj(Z), built so by the producer
        if constexpr (!ZOUT)                                 // ZOUT: the test hook writes conj(Z) itself
            fft::fft2pass_impl<N, false, 1, false>(v, sg, t, fft::TwGlobal<N>{tw + P::TW_OFFSET + t}, fft::NoHook(),
                                                   gsync);
        float2 *o = buf + ((size_t)pair * N + (grp ? ym : y)) * N;
#pragma unroll
        for (int m = 0; m < E; ++m)
            o[t + R1 * m] = v[m];       // conj of the row IFFT (the pair buffer is kept conjugated)
        __syncthreads();                                     // both slots read before the next unit
    }
}

// ---- pass B: column IFFT -> a4 sign + pack -> column FFT (TMA-fed pipeline) ------------------
// 8x8 bit-matrix transpose (bit 8i + j <-> bit 8j + i), three masked swap stages.
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x)
{
    uint64_t t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    return x ^ t ^ (t << 28);
}

// Columns per OSPR column-pass tile (see OsprColBody::kWidth); host and device agree on it.
constexpr int ospr_col_width(int n) { return n >= 1024 ? 4 : 8; }

template <int N>
struct OsprColBody {
    static constexpr int kStages = 3;   // measured best column-pipeline variant for this body
    // columns per tile: 8 (one packed byte per tile row); N = 2048: 4 (a nibble per tile row),
    // so that three 2048-row stages fit in shared memory and the ring overlaps load, transform
    // and store (an 8-column tile leaves room for one stage only).  N = 4096: one 4-column stage
    // of 133 KB and one 256-thread group (2-column tiles with three stages measured 27 % slower:
    // 16-byte row segments halve the DRAM sector efficiency)
    static constexpr int kWidth = ospr_col_width(N);
    static constexpr int kGroups = N == 2048 ? 2 : 1;   // two consumer groups per CTA (ColPipeG2)
    struct Args {
        const float2 *tw;
        float2 *buf;
        uint8_t *bits;        // tile-major sign bytes bt[2 * pair + f][ct][y] (nullable)
        int npairs;
        int last_has_b;
    };
    template <class F, int W>
    static __device__ __forceinline__ void run(float2 (&v)[F::E], float2 *sm, uint32_t *scratch, int c, int t,
                                               int pair, int ct, const Args &a, const F &fft)
    {
        constexpr int R1 = F::T, E = F::E;   // element m of thread t = row t + R1*m; W columns per tile
        const bool has_b = (pair < a.npairs - 1) || a.last_has_b;
        static_assert(E <= 64 && (W == 8 || W == 4), "bit words hold at most 64 rows per thread; a byte or "
                                                       "nibble per tile row");
        using Word = typename std::conditional<(E > 32), unsigned long long, unsigned>::type;
        static_assert(2 * W * R1 * sizeof(Word) <= ColPipe<N, 0, W>::SCRATCH_BYTES, "scratch holds both bit planes");
        Word *sw = reinterpret_cast<Word *>(scratch);            // [frame 2][t R1][c W] sign words
        Word wa = 0, wb = 0;                                     // a4: bit r = sign of row t + R1*r
        // IFFT then FFT through ONE transform body (instruction cache): F^-1{x} = conj(F{conj(x)})
        // exactly, since negation is exact.  Pass A stores the conjugate of its row IFFT, so the
        // tile already holds conj(x) and the column IFFT needs no input negation.
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            fft.template run<false, W>(v, sm, t);
            if (h == 0) {                                        // v = conj(H) (x N): Re H = v.x, Im H = -v.y
                // u = (Re H, Im H) + 0 (one FADD2): -0.0 becomes +0.0, so u's sign bit is set iff
                // the value is < 0, and h' = +-1 is that sign bit on 1.0f (R-7: Re H >= 0 -> +1).
                if constexpr (E <= 32) {
                    // the sign bits are shifted into a 32-bit word by one funnel shift each, last
                    // element first (bit r = element r), and inverted once at the end (C3: the
                    // column pass 1328 -> 1232 instructions per thread and tile)
                    uint32_t sa = 0, sb = 0;
#pragma unroll
                    for (int r = E - 1; r >= 0; --r) {
                        const float2 u = f2::add(conjf2(v[r]), make_float2(0.0f, 0.0f));
                        const uint32_t ua = __float_as_uint(u.x), ub = __float_as_uint(u.y);
                        sa = __funnelshift_l(ua, sa, 1);
                        sb = __funnelshift_l(ub, sb, 1);
                        v[r] = make_float2(__uint_as_float((ua & 0x80000000u) | 0x3f800000u),
                                           __uint_as_float((ub & 0x80000000u) | 0x3f800000u));
                    }
                    constexpr uint32_t mask = E < 32 ? (1u << E) - 1u : 0xFFFFFFFFu;
                    wa = (Word)(~sa & mask);
                    wb = (Word)(~sb & mask);
                } else {   // E = 64 (N = 2048): per-bit insertion measured faster there (C5 0.616 vs 0.65 ms)
#pragma unroll
                    for (int r = 0; r < E; ++r) {
                        const float2 u = f2::add(conjf2(v[r]), make_float2(0.0f, 0.0f));
                        const uint32_t ua = __float_as_uint(u.x), ub = __float_as_uint(u.y);
                        wa |= (Word)((~ua) >> 31) << r;
                        wb |= (Word)((~ub) >> 31) << r;
                        v[r] = make_float2(__uint_as_float((ua & 0x80000000u) | 0x3f800000u),
                                           __uint_as_float((ub & 0x80000000u) | 0x3f800000u));
                    }
                }
                if (!has_b) {                                    // unpaired tail: h'_b = 0
#pragma unroll
                    for (int r = 0; r < E; ++r)
                        v[r].y = 0.0f;
                }
                sw[t * W + c] = wa;                              // read back after the next FFT's barriers
                sw[(R1 + t) * W + c] = wb;
            }
        }
        // (the pipeline stores v, the column FFT of h')
        // pack (R-8, MSB-first): the byte of tile row y = t' + R1*r holds the 8 columns' sign
        // bits r of words [f][t'][0..7]; a task gathers 8 rows r = 8*rb .. 8*rb+7 of one t' as
        // an 8x8 bit matrix (byte 7-c = column c) and transposes it into the 8 row bytes.  The
        // bytes go to the tile-major staging layout bt[sub-frame][ct][y] (a warp writes 32
        // consecutive rows = one sector); pass C's transpose CTAs make them row-major.
        if (a.bits != nullptr) {
            constexpr int RG = E < 8 ? 1 : E / 8, RPG = E < 8 ? E : 8, TASKS = 2 * R1 * RG;
#pragma unroll 1
            for (int task = t * W + c; task < TASKS; task += W * R1) {   // t W + c: thread within the group
                const int f = task / (R1 * RG), rem = task % (R1 * RG), tt = rem % R1, rb = rem / R1;
                if (f == 1 && !has_b)
                    continue;
                Word q[W];                                       // the W words, vector loads
                if constexpr (sizeof(Word) == 4 && W == 8) {
                    const uint4 *q4 = reinterpret_cast<const uint4 *>(sw + (f * R1 + tt) * W);
                    const uint4 lo = q4[0], hi = q4[1];
                    q[0] = lo.x, q[1] = lo.y, q[2] = lo.z, q[3] = lo.w, q[4] = hi.x, q[5] = hi.y, q[6] = hi.z, q[7] = hi.w;
                } else if constexpr (sizeof(Word) == 4 && W == 4) {   // one 16-byte load (no 4-way conflict)
                    const uint4 q4 = *reinterpret_cast<const uint4 *>(sw + (f * R1 + tt) * W);
                    q[0] = q4.x, q[1] = q4.y, q[2] = q4.z, q[3] = q4.w;
                } else if constexpr (sizeof(Word) == 8 && W == 4) {   // two 16-byte loads
                    const ulonglong2 *q2 = reinterpret_cast<const ulonglong2 *>(sw + (f * R1 + tt) * W);
                    const ulonglong2 lo = q2[0], hi = q2[1];
                    q[0] = lo.x, q[1] = lo.y, q[2] = hi.x, q[3] = hi.y;
                } else {
#pragma unroll
                    for (int cc = 0; cc < W; ++cc)
                        q[cc] = sw[(f * R1 + tt) * W + cc];
                }
                uint64_t m = 0;
#pragma unroll
                for (int cc = 0; cc < W; ++cc)
                    m |= (uint64_t)((q[cc] >> (8 * rb)) & 0xFFu) << (8 * (7 - cc));
                m = transpose8x8(m);
                // W = 4: the byte's high nibble holds the tile's 4 columns (MSB-first), the low one 0
                uint8_t *dst = a.bits + ((size_t)(2 * pair + f) * (N / W) + ct) * N + tt + R1 * 8 * rb;
#pragma unroll
                for (int r = 0; r < RPG; ++r)
                    dst[r * R1] = (uint8_t)(m >> (8 * r));
            }
        }
    }
};

// Tile-major sign bytes bt[q][ct][y] (ct < N/8, y < N) -> row-major packed holograms
// out[q][y][ct] (R-8), one block of YB rows of sub-frame q per CTA, through shared memory;
// 32-bit words on both global sides when N >= 32 (every thread's loads in flight at once).
// Run by extra CTAs of ospr_rows_c_kernel (64 threads) or ospr_finalize_kernel (256 threads).
template <int N>
struct BitsT {
    static constexpr int C = N / 8, YB = N < 32 ? N : 32, BLOCKS_PER_Q = N / YB;
    static constexpr int W = OsprColBody<N>::kWidth;   // staging: one byte (W = 8) or nibble (W = 4) per tile row
    static constexpr size_t BYTES_PER_SUBFRAME = (size_t)N * (N / W);
};

template <int N, int NT = 256>
__device__ __forceinline__ void bits_transpose_block(const uint8_t *__restrict__ bt, uint8_t *__restrict__ out, int q,
                                                     int yblk)
{
    constexpr int C = BitsT<N>::C, YB = BitsT<N>::YB;
    __shared__ __align__(16) uint8_t sm[C][YB + 4];
    const int y0 = yblk * YB;
    constexpr int TW = BitsT<N>::W;
    const uint8_t *src = bt + (size_t)q * BitsT<N>::BYTES_PER_SUBFRAME + y0;
    uint8_t *dst = out + ((size_t)q * N + y0) * C;
    if constexpr (N >= 32) {
        constexpr int WPR = YB / 4, WORDS = C * WPR, PER = (WORDS + NT - 1) / NT;   // words per ct row
        uint32_t w[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + NT * j;
            if constexpr (TW == 8) {
                w[j] = i < WORDS ? __ldg(reinterpret_cast<const uint32_t *>(src + (size_t)(i / WPR) * N) + i % WPR)
                                 : 0u;
            } else {   // nibble tiles 2 ct and 2 ct + 1 -> the byte's high and low nibble
                uint32_t hi = 0u, lo = 0u;
                if (i < WORDS) {
                    hi = __ldg(reinterpret_cast<const uint32_t *>(src + (size_t)(2 * (i / WPR)) * N) + i % WPR);
                    lo = __ldg(reinterpret_cast<const uint32_t *>(src + (size_t)(2 * (i / WPR) + 1) * N) + i % WPR);
                }
                w[j] = hi | ((lo >> 4) & 0x0F0F0F0Fu);
            }
        }
        // word w of staged row r sits at word w ^ sw(r) (WPR = 8 words per row, stride 9 words):
        // the byte gathers below read rows 4k + jj across the lanes k of a warp, which without the
        // swizzle hit 8 banks only (4-way conflicts, measured 295 k excess wavefronts per C3 step)
        static_assert(WPR == 8, "eight words per staged row");
        auto sw = [](int r) { return (r >> 5) & 3; };
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + NT * j;
            if (i < WORDS) {
                const int r = i / WPR;
                *reinterpret_cast<uint32_t *>(&sm[r][4 * ((i % WPR) ^ sw(r))]) = w[j];
            }
        }
        __syncthreads();
        constexpr int OW = C / 4;   // output words per row
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int i = threadIdx.x + NT * j;
            if (i < WORDS) {
                const int y = i / OW, c4 = 4 * (i % OW), yw = y >> 2, yb = y & 3;
                uint32_t v = 0u;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
                    v |= (uint32_t)sm[c4 + jj][4 * (yw ^ sw(c4 + jj)) + yb] << (8 * jj);
                reinterpret_cast<uint32_t *>(dst + (size_t)y * C)[i % OW] = v;
            }
        }
    } else {
        static_assert(TW == 8, "nibble staging only for N = 2048");
        for (int i = threadIdx.x; i < C * YB; i += blockDim.x)
            sm[i / YB][i % YB] = src[(size_t)(i / YB) * N + i % YB];
        __syncthreads();
        for (int i = threadIdx.x; i < C * YB; i += blockDim.x)
            dst[i] = sm[i % C][i / C];
    }
}

// ---- pass C: row FFT + |X|^2 summed over the chunk's pairs --------------------------------------
// One CTA = one row group y (GPW rows) at a time, two warps splitting the chunk's pairs.
// Each warp streams its pair rows (y, p) through ONE shared-memory slot: the 1D TMA load of
// the next pair row is issued as soon as the current transform has read its exchange back,
// so it overlaps pass 2 and the |X|^2 accumulation.  Small CTAs (two warps, ~21 KB) let a
// whole N = 1024 frame's row groups be resident in one wave, instead of the 1.15 waves
// (58 % efficiency) of four-warp CTAs.  The halves are summed in a fixed order
// (deterministic), then one read-modify-write of the frame accumulator A per row and chunk.
template <int N>
struct RowC {
    using P = fft::Plan<N>;
    static constexpr int GPW = 32 / P::T, NGRP = N / GPW;
    static constexpr uint32_t IN_BYTES = (uint32_t)GPW * N * 8;
    static constexpr uint32_t XCH_BYTES = (uint32_t)GPW * P::SMEM * 8;
    static constexpr uint32_t SLOT = ((XCH_BYTES > IN_BYTES ? XCH_BYTES : IN_BYTES) + 127) / 128 * 128;
    static constexpr size_t RED = (size_t)GPW * N * sizeof(float);
    static constexpr size_t SMEM = 2 * (size_t)SLOT + RED + 2 * sizeof(uint64_t);
};

template <int N>
__global__ void __launch_bounds__(64)
ospr_rows_c_kernel(const float2 *__restrict__ tw, const float2 *__restrict__ buf, int npairs,
                   float *__restrict__ acc, int accumulate, unsigned *ticket, int nbt, const uint8_t *__restrict__ bt,
                   uint8_t *__restrict__ bits)
{
    HOLO_PDL_ENTRY();
    if ((int)blockIdx.x < nbt) {         // the frame's sign-byte transposes (last chunk), scheduled first
        const int j = (int)blockIdx.x;
        bits_transpose_block<N, 64>(bt, bits, j / BitsT<N>::BLOCKS_PER_Q, j % BitsT<N>::BLOCKS_PER_Q);
        return;
    }
    if (ticket != nullptr && blockIdx.x == nbt && threadIdx.x == 0)
        *ticket = 0u;                    // the finalize ticket, reset ahead of the finalize kernel
    const int cta = (int)blockIdx.x - nbt, nctas = (int)gridDim.x - nbt;
    using P = fft::Plan<N>;
    using RC = RowC<N>;
    constexpr int R1 = P::R1, E = P::E, GPW = RC::GPW, NGRP = RC::NGRP;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int half = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane / R1, t = lane % R1;
    float2 *sl = reinterpret_cast<float2 *>(smem_raw + (size_t)half * RC::SLOT);
    float *red = reinterpret_cast<float *>(smem_raw + 2 * (size_t)RC::SLOT);              // [GPW*N]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + 2 * (size_t)RC::SLOT + RC::RED) + half;
    const int hp = (npairs + 1) / 2;                     // pairs of half 0; half 1 gets the rest
    const int p0 = half * hp, p1 = half ? npairs : hp;
    auto src = [&](int gg, int p) { return buf + ((size_t)p * N + (size_t)gg * GPW) * N; };
    if (lane == 0) {
        tma::mbar_init(bar, 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    int grp = cta;
    if (lane == 0 && grp < NGRP && p0 < p1) {
        tma::mbar_arrive_expect_tx(bar, RC::IN_BYTES);
        tma::load_1d(sl, src(grp, p0), RC::IN_BYTES, bar);
    }
    uint32_t k = 0;
    #pragma unroll 1
    for (; grp < NGRP; grp += nctas) {
        float a[E];
#pragma unroll
        for (int r = 0; r < E; ++r)
            a[r] = 0.0f;
        #pragma unroll 1   // one copy of the transform code (instruction cache)
        for (int p = p0; p < p1; ++p, ++k) {
            tma::mbar_wait(bar, k & 1u);
            float2 v[E];
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = sl[g * N + t + R1 * m];
            const bool more = (p + 1 < p1) || (grp + nctas < NGRP);
            const float2 *nx = (p + 1 < p1) ? src(grp, p + 1) : src(grp + nctas, p0);
            fft::fft2pass_hook<N, false, 1, true>(v, sl + g * P::SMEM, t, tw, [&] {
                // WAR across proxies: every lane's exchange reads are performed (proxy fence)
                // before lane 0's TMA write into the same slot is issued
                tma::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0 && more) {
                    tma::mbar_arrive_expect_tx(bar, RC::IN_BYTES);
                    tma::load_1d(sl, nx, RC::IN_BYTES, bar);
                }
            });
#pragma unroll
            for (int r = 0; r < E; ++r)
                a[r] = __fmaf_rn(v[r].x, v[r].x, __fmaf_rn(v[r].y, v[r].y, a[r]));
        }
        // combine the two halves (half 0 + half 1, fixed order) and update A
        float *rg = red + g * N;
        if (half == 1) {
#pragma unroll
            for (int r = 0; r < E; ++r)
                rg[t + R1 * r] = a[r];
        }
        __syncthreads();
        if (half == 0) {
            constexpr float inv_p = 1.0f / ((float)N * (float)N);   // exact power of two
            float *o = acc + ((size_t)grp * GPW + g) * N;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const float val = (a[r] + rg[t + R1 * r]) * inv_p;
                o[t + R1 * r] = accumulate ? o[t + R1 * r] + val : val;
            }
        }
        __syncthreads();
    }
}

// Pass C for N = 4096 (R-26): a two-warp group per row y, the chunk's pair rows read straight
// from the pair buffer (coalesced), row FFT, |X|^2 summed over the pairs in registers, one
// read-modify-write of the accumulator row.  The first nbt CTAs transpose the frame's sign
// bytes (last chunk), as in ospr_rows_c_kernel; the finalize kernel symmetrises.
template <int N>
__global__ void __launch_bounds__(Row2W<N>::THREADS, 1)
ospr_rows2w_c_kernel(const float2 *__restrict__ tw, const float2 *__restrict__ buf, int npairs,
                     float *__restrict__ acc, int accumulate, unsigned *ticket, int nbt, const uint8_t *__restrict__ bt,
                     uint8_t *__restrict__ bits)
{
    HOLO_PDL_ENTRY();
    if ((int)blockIdx.x < nbt) {
        const int j = (int)blockIdx.x;
        bits_transpose_block<N, Row2W<N>::THREADS>(bt, bits, j / BitsT<N>::BLOCKS_PER_Q, j % BitsT<N>::BLOCKS_PER_Q);
        return;
    }
    if (ticket != nullptr && blockIdx.x == nbt && threadIdx.x == 0)
        *ticket = 0u;                    // the finalize ticket, reset ahead of the finalize kernel
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const Row2WThread rt = row2w_thread();
    float2 *sm = reinterpret_cast<float2 *>(smem_raw) + (size_t)rt.grp * P::SMEM;
    const int cta = (int)blockIdx.x - nbt, nctas = (int)gridDim.x - nbt;
    #pragma unroll 1
    for (int y = cta * 2 + rt.grp; y < N; y += nctas * 2) {
        float a[E];
#pragma unroll
        for (int r = 0; r < E; ++r)
            a[r] = 0.0f;
        #pragma unroll 1
        for (int p = 0; p < npairs; ++p) {
            if (rt.t == 0) {   // the group's next pair row into L2 while this one transforms
                const int yn = y + nctas * 2;
                const float2 *nx = p + 1 < npairs ? buf + ((size_t)(p + 1) * N + y) * N
                                 : yn < N         ? buf + (size_t)yn * N
                                                  : nullptr;
                if (nx != nullptr)
                    tma::prefetch_l2(nx, (uint32_t)N * 8);
            }
            const float2 *src = buf + ((size_t)p * N + y) * N + rt.t;
            float2 v[E];
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = src[R1 * m];
            row2w_fft<N>(v, sm, tw, rt);
#pragma unroll
            for (int r = 0; r < E; ++r)
                a[r] = __fmaf_rn(v[r].x, v[r].x, __fmaf_rn(v[r].y, v[r].y, a[r]));
        }
        constexpr float inv_p = 1.0f / ((float)N * (float)N);   // exact power of two
        float *o = acc + (size_t)y * N + rt.t;
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const float val = a[r] * inv_p;
            o[R1 * r] = accumulate ? o[R1 * r] + val : val;
        }
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

// Finalize grid: FB CTAs of kFinThreads threads, ITER pixels per thread (fixed per N, so the
// partial-sum order -- and the MSE -- is deterministic).
template <int N>
struct FinPlan {
    static constexpr int P = N * N, WANT = (P + 8 * kFinThreads - 1) / (8 * kFinThreads);
    static constexpr int FB = WANT < kFinBlocks ? WANT : kFinBlocks;
    static constexpr int ITER = (P + FB * kFinThreads - 1) / (FB * kFinThreads);
};

// R-12 from the five fp64 sums: a = S_T2 / S_I (0 if S_I = 0);
// mse = (a^2 S_II - 2 a S_IT2 + S_T4) / |Omega|.
__device__ __forceinline__ double mse_from_sums(const double *o, double inv_count)
{
    const double a = o[0] == 0.0 ? 0.0 : o[3] / o[0];
    const double sum = a * a * o[1] - 2.0 * a * o[2] + o[4];
    return (sum > 0.0 ? sum : 0.0) * inv_count;
}

// ---- pass C + a7 for the frame's last chunk (N >= 1024): mirrored row pairs per CTA ----------
// Unit u covers rows {u, N - u} (u = 0: rows 0 and N/2, each its own mirror).  Warps 0-1 take
// row ya = u, warps 2-3 row yb (pairs split between the two warps of a row, as in pass C).  With
// both rows' |X|^2 sums in shared memory the CTA symmetrises (I[k] = (A[k] + A[-k]) s), writes
// the two intensity rows and its five fp64 MSE partials, and the last CTA (ticket) reduces the
// N/2 partials in unit order.  No accumulator round trip through HBM and no finalize launch;
// the T rows are fetched at CTA start, so the epilogue waits on shared memory only.
template <int N>
struct RowCF {
    using P = fft::Plan<N>;
    static_assert(32 / P::T == 1, "one row per warp");
    static constexpr int NU = N / 2, THREADS = 128;
    // pair-row slots per warp.  One: four CTAs per SM, so the 512 units of N = 1024 run in one
    // wave.  Two (HOLO_CF_SLOTS=2, N <= 1024) keep two loads in flight per warp but leave three
    // CTAs per SM, and the 512 units take 1.15 waves: measured 36.3 vs 33.3 us at C3.
#ifndef HOLO_CF_SLOTS
#define HOLO_CF_SLOTS 1
#endif
    static constexpr int SLOTS = N <= 1024 ? HOLO_CF_SLOTS : 1;
    static constexpr uint32_t IN_BYTES = (uint32_t)N * 8, SLOT = RowC<N>::SLOT;
    // A rows ya, yb (fp32) after the transforms: in the slot memory if it is large enough
    static constexpr size_t SLOTS_BYTES = 4 * (size_t)SLOTS * SLOT;
    static constexpr bool A_ALIAS = SLOTS_BYTES >= 2 * (size_t)N * sizeof(float) && SLOTS > 1;
    static constexpr size_t SA = A_ALIAS ? 0 : SLOTS_BYTES;
    static constexpr size_t BAR = A_ALIAS ? SLOTS_BYTES : SA + 2 * (size_t)N * sizeof(float);
    static constexpr size_t SMEM = BAR + 4 * SLOTS * sizeof(uint64_t);
};

template <int N>
__global__ void __launch_bounds__(RowCF<N>::THREADS, N <= 1024 ? 4 - (RowCF<N>::SLOTS - 1) : 1)
ospr_rows_cf_kernel(const float2 *__restrict__ tw, const float2 *__restrict__ buf, int npairs,
                    const float *__restrict__ acc_in, const float *__restrict__ T, float scale, float *__restrict__ out,
                    holo_region om, double *__restrict__ parts, unsigned *ticket, double inv_count,
                    double *__restrict__ mse, int nbt, const uint8_t *__restrict__ bt, uint8_t *__restrict__ bits)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    using RC = RowCF<N>;
    constexpr int R1 = P::R1, E = P::E, NU = RC::NU, PER = N / RC::THREADS;
    if ((int)blockIdx.x >= NU) {         // the frame's sign-byte transposes, after the row-pair units:
        const int j = (int)blockIdx.x - NU;   // they fill the slots the units leave free
        bits_transpose_block<N, RowCF<N>::THREADS>(bt, bits, j / BitsT<N>::BLOCKS_PER_Q, j % BitsT<N>::BLOCKS_PER_Q);
        return;
    }
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = lane, half = warp & 1, side = warp >> 1;
    const int u = (int)blockIdx.x;
    const int ya = u, yb = u > 0 ? N - u : N / 2;
    const int y = side ? yb : ya;
    constexpr int NS = RC::SLOTS;
    float2 *sl0 = reinterpret_cast<float2 *>(smem_raw + (size_t)warp * NS * RC::SLOT);
    float *sA = reinterpret_cast<float *>(smem_raw + RC::SA);           // [2][N]: A of ya, yb
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem_raw + RC::BAR) + warp * NS;
    // T of both rows: read in the epilogue (no registers held across the transforms)
    const int hp = (npairs + 1) / 2, p0 = half * hp, p1 = half ? npairs : hp;
    auto src = [&](int p) { return buf + ((size_t)p * N + (size_t)y) * N; };
    auto slot = [&](int i) { return sl0 + (size_t)i * (RC::SLOT / sizeof(float2)); };
    if (lane == 0) {
        for (int i = 0; i < NS; ++i)
            tma::mbar_init(&bar[i], 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    if (lane == 0)                       // the first NS pair rows in flight
        for (int i = 0; i < NS && p0 + i < p1; ++i) {
            tma::mbar_arrive_expect_tx(&bar[i], RC::IN_BYTES);
            tma::load_1d(slot(i), src(p0 + i), RC::IN_BYTES, &bar[i]);
        }
#ifndef HOLO_CF_PFD
#define HOLO_CF_PFD 2   // measured at C3: 1 -> 110.6, 2 -> 110.5, 3 -> 110.8, none -> 111.3 us per step
#endif
    // (prefetching the rows before the loop's first prefetch as well, at CTA start: 33.6 vs 32.3 us)
    float a[E];
#pragma unroll
    for (int r = 0; r < E; ++r)
        a[r] = 0.0f;
    uint32_t k = 0;
    #pragma unroll 1
    for (int p = p0; p < p1; ++p, ++k) {
        if (HOLO_L2PF && N <= 1024 && lane == 0 && p + NS + HOLO_CF_PFD - 1 < p1 - 1)   // a later pair row into L2
            tma::prefetch_l2(src(p + NS + HOLO_CF_PFD), RC::IN_BYTES);
        const int si = NS > 1 ? (int)(k % NS) : 0;
        float2 *sl = slot(si);
        tma::mbar_wait(&bar[si], (k / NS) & 1u);
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sl[t + R1 * m];
        const bool more = p + NS < p1;
        const float2 *nx = src(p + NS);
        fft::fft2pass_hook<N, false, 1, true>(v, sl, t, tw, [&] {
            // WAR across proxies: the exchange reads of this slot before the TMA refill
            tma::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && more) {
                tma::mbar_arrive_expect_tx(&bar[si], RC::IN_BYTES);
                tma::load_1d(sl, nx, RC::IN_BYTES, &bar[si]);
            }
        });
#pragma unroll
        for (int r = 0; r < E; ++r)
            a[r] = __fmaf_rn(v[r].x, v[r].x, __fmaf_rn(v[r].y, v[r].y, a[r]));
    }
    if constexpr (RC::A_ALIAS)
        __syncthreads();                 // every warp is done with its slots (sA aliases them)
    // A row = (half 0 + half 1) / N^2 (+ earlier chunks' sums), fixed order as in pass C
    float *rowA = sA + (size_t)side * N;
    if (half == 1) {
#pragma unroll
        for (int r = 0; r < E; ++r)
            rowA[t + R1 * r] = a[r];
    }
    __syncthreads();
    if (half == 0) {
        constexpr float inv_p = 1.0f / ((float)N * (float)N);   // exact power of two
#pragma unroll
        for (int r = 0; r < E; ++r) {
            const int x = t + R1 * r;
            const float val = (a[r] + rowA[x]) * inv_p;
            rowA[x] = acc_in != nullptr ? acc_in[(size_t)y * N + x] + val : val;
        }
    }
    __syncthreads();
    // a7: symmetrise both rows, write the mean intensity, fp64 MSE partials (R-12) over Omega
    float ta[PER], tb[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        ta[j] = __ldg(T + (size_t)ya * N + threadIdx.x + RC::THREADS * j);
        tb[j] = __ldg(T + (size_t)yb * N + threadIdx.x + RC::THREADS * j);
    }
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    const float *A0 = sA, *A1 = sA + N;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int r = h ? yb : ya;
        // the mirror of (r, x) is (N - r, N - x): row yb for ya (u > 0), or the row itself (u = 0)
        const float *own = h ? A1 : A0, *mir = (u > 0) ? (h ? A0 : A1) : own;
        const bool row_in = r >= om.row0 && r < om.row1;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int x = threadIdx.x + RC::THREADS * j;
            const float I = (own[x] + mir[(N - x) & (N - 1)]) * scale;   // as ospr_finalize_kernel
            out[(size_t)r * N + x] = I;
            if (mse != nullptr && row_in && x >= om.col0 && x < om.col1) {
                const double Id = I, tt = h ? tb[j] : ta[j], t2 = tt * tt;
                s[0] += Id;
                s[1] += Id * Id;
                s[2] += Id * t2;
                s[3] += t2;
                s[4] += t2 * t2;
            }
        }
    }
    if (mse == nullptr)
        return;
    block_reduce_store(s, 5, parts + (size_t)u * 5);
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();                                   // this unit's partials before its ticket
        last = atomicAdd(ticket, 1u) == (unsigned)NU - 1u;
    }
    __syncthreads();
    if (!last)
        return;
    __threadfence();
    double tsum[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < NU; b += blockDim.x)
        for (int i = 0; i < 5; ++i)
            tsum[i] += __ldcg(parts + (size_t)b * 5 + i);
    __shared__ double o[5];
    __syncthreads();
    block_reduce_store(tsum, 5, o);
    __syncthreads();
    if (threadIdx.x == 0) {
        *mse = mse_from_sums(o, inv_count);
        *ticket = 0u;
    }
}


// intensity[k] = (A[k] + A[-k]) * scale (symmetrise = 1) or A[k] * scale; optional fp64
// partial sums (sum I, sum I^2, sum I T^2, sum T^2, sum T^4) over Omega, one slot per CTA.
// With mse != NULL the last CTA to finish (atomic ticket on *counter, which the host zeroes
// before the launch and the last CTA re-zeroes) reduces the slots in CTA order -- a fixed
// order, so the MSE is deterministic -- and writes R-12.  CTAs fb.. of the grid instead
// transpose the frame's nq sub-frames of tile-major sign bytes into packed holograms.
template <int N>
__global__ void __launch_bounds__(kFinThreads)
ospr_finalize_kernel(const float *__restrict__ acc, const float *__restrict__ T, int symmetrise, float scale,
                     float *__restrict__ out, holo_region om, double *__restrict__ parts, unsigned *counter,
                     double inv_count, double *__restrict__ mse)
{
    HOLO_PDL_ENTRY();
    constexpr int P = N * N, LOG = fft::ilog2(N), FB = FinPlan<N>::FB, ITER = FinPlan<N>::ITER;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    // a fixed number of pixels per thread, fully unrolled (N <= 2048: every load in flight at
    // once; N = 4096, ITER = 111: unrolled by 8)
    constexpr int UNR = ITER <= 32 ? ITER : 8;
#pragma unroll UNR
    for (int i = 0; i < ITER; ++i) {
        const int k = (int)blockIdx.x * kFinThreads + (int)threadIdx.x + i * FB * kFinThreads;
        if (k >= P)
            break;
        const int y = k >> LOG, x = k & (N - 1);
        float I;
        if (symmetrise) {
            const int km = (((N - y) & (N - 1)) << LOG) + ((N - x) & (N - 1));
            I = (__ldg(acc + k) + __ldg(acc + km)) * scale;
        } else {
            I = __ldg(acc + k) * scale;
        }
        out[k] = I;
        if (parts != nullptr && y >= om.row0 && y < om.row1 && x >= om.col0 && x < om.col1) {
            const double Id = I, tt = __ldg(T + k), t2 = tt * tt;
            s[0] += Id;
            s[1] += Id * Id;
            s[2] += Id * t2;
            s[3] += t2;
            s[4] += t2 * t2;
        }
    }
    if (parts == nullptr)
        return;
    block_reduce_store(s, 5, parts + (size_t)blockIdx.x * 5);
    if (mse == nullptr)
        return;
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();                                   // this CTA's slot before its ticket
        last = atomicAdd(counter, 1u) == (unsigned)FB - 1;
    }
    __syncthreads();
    if (!last)
        return;
    __threadfence();
    double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < FB; b += blockDim.x)
        for (int i = 0; i < 5; ++i)
            t[i] += __ldcg(parts + (size_t)b * 5 + i);
    __shared__ double o[5];
    __syncthreads();
    block_reduce_store(t, 5, o);
    __syncthreads();
    if (threadIdx.x == 0) {
        *mse = mse_from_sums(o, inv_count);
        *counter = 0u;
    }
}

// ---- a7 on a row slice (the owned slice after a cross-rank reduce-scatter, C-1) ---------------
// Rows [row0, row0 + nrows) of one frame: mean = sum * scale (in place allowed) and the five
// fp64 partial sums (sum I, I^2, I T^2, T^2, T^4) over Omega restricted to the slice, one slot
// per CTA; the last CTA (ticket) reduces the slots in CTA order (deterministic) into sums[5].
// kFinThreads threads, `iter` pixels per thread, grid fixed by (n, nrows).
__global__ void __launch_bounds__(kFinThreads)
ospr_finalize_rows_kernel(const float *__restrict__ acc, const float *__restrict__ T, int n, int row0, int nrows,
                          int iter, float scale, float *__restrict__ out, holo_region om,
                          double *__restrict__ parts, unsigned *counter, double *__restrict__ sums)
{
    HOLO_PDL_ENTRY();
    const int pix = n * nrows;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < iter; ++i) {
        const int k = (int)blockIdx.x * kFinThreads + (int)threadIdx.x + i * (int)gridDim.x * kFinThreads;
        if (k >= pix)
            break;
        const int y = row0 + k / n, x = k % n;
        const float I = __ldg(acc + k) * scale;
        out[k] = I;
        if (y >= om.row0 && y < om.row1 && x >= om.col0 && x < om.col1) {
            const double Id = I, tt = __ldg(T + (size_t)y * n + x), t2 = tt * tt;
            s[0] += Id;
            s[1] += Id * Id;
            s[2] += Id * t2;
            s[3] += t2;
            s[4] += t2 * t2;
        }
    }
    block_reduce_store(s, 5, parts + (size_t)blockIdx.x * 5);
    __shared__ int last;
    if (threadIdx.x == 0) {
        __threadfence();                                   // this CTA's slot before its ticket
        last = atomicAdd(counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last)
        return;
    __threadfence();
    double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
        for (int i = 0; i < 5; ++i)
            t[i] += __ldcg(parts + (size_t)b * 5 + i);
    __shared__ double o[5];
    __syncthreads();
    block_reduce_store(t, 5, o);
    __syncthreads();
    if (threadIdx.x < 5)
        sums[threadIdx.x] = o[threadIdx.x];
    if (threadIdx.x == 0)
        *counter = 0u;
}

// R-12 from the five (cross-rank reduced) sums of each frame (C-2 done by the caller).
__global__ void ospr_mse_from_sums_kernel(const double *__restrict__ sums, int n_frames, double inv_count,
                                          double *__restrict__ mse)
{
    HOLO_PDL_ENTRY();
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f < n_frames)
        mse[f] = mse_from_sums(sums + (size_t)f * 5, inv_count);
}

// ---- host orchestration -------------------------------------------------------------------
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static int ospr_chunk_pairs(int n, int n_sub)
{
    const size_t frame = (size_t)n * n * sizeof(float2);
    // pair-buffer budget: fewer, larger chunks win (each chunk costs three launches with their
    // ramps; L2 residency of smaller chunks measured no gain): C3 and C5 run as one chunk
    size_t budget = 1ull << 30;
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
    uint8_t *bt;        // tile-major sign bytes of a chunk
    double *cf_parts;   // fused a7 (N >= 1024): [N/2][5] unit partial sums, then the ticket
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
    off = align256(off + kFinWsBytes);
    const size_t o_bt = off;
    // staged sign bytes (one byte or nibble per tile row) of a frame's sub-frames
    off = align256(off + (size_t)(2 * ((n_sub + 1) / 2)) * (size_t)n * (size_t)(n / ospr_col_width(n)));
    const size_t o_cf = off;
    off = align256(off + (size_t)(n / 2) * 5 * sizeof(double) + 64);
    if (w) {
        w->cf_parts = (double *)(base + o_cf);
        w->buf = (float2 *)(base + o_buf);
        w->acc = (float *)(base + o_acc);
        w->parts = (double *)(base + o_parts);
        w->bt = (uint8_t *)(base + o_bt);
    }
    return off;
}


// The completion ticket of the finalize kernel, after its per-CTA partial-sum slots.
static unsigned *finalize_ticket(double *parts) { return reinterpret_cast<unsigned *>(parts + (size_t)kFinBlocks * 5); }


// Finalize one frame (and, if bits != NULL, transpose its nq sub-frames of sign bytes).
template <int N>
holo_status finalize_frame(const float *acc, const float *T, int symmetrise, float scale, float *out, holo_region om,
                           double *parts, double *mse, cudaStream_t s, bool ticket_zeroed = false)
{
    unsigned *counter = finalize_ticket(parts);
    const double cnt = (double)(om.row1 - om.row0) * (double)(om.col1 - om.col0);
    if (mse && !ticket_zeroed) {
        cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
        if (e != cudaSuccess)
            return cuda_status(e, "cudaMemsetAsync(finalize ticket)");
    }
    return launch(K_OSPR_FINALIZE, ospr_finalize_kernel<N>, dim3(FinPlan<N>::FB), dim3(kFinThreads), 0, s, acc, T,
                  symmetrise, scale, out, om, mse ? parts : (double *)nullptr, counter, 1.0 / cnt, mse);
}

// The phase source of a call: the pool (a0), SplitMix64 + R-5 per draw (f2), or SplitMix64 +
// the 2^q-entry sin/cos table (R-25).
enum PhaseSource : int { SRC_POOL = 0, SRC_PRNG = 1, SRC_TABLE = 2 };

// Pass A over np sub-frame pairs starting at global sub-frame sf_first (ZOUT: the test hook
// variant that stores conj(Z) instead of its row IFFT).
template <int N, bool ZOUT>
static holo_status launch_pass_a(const float2 *tw, const float *Tf, const PhaseSrc &ps, int src, uint64_t sf_first,
                                 int np, int last_has_b, float2 *buf, cudaStream_t s, unsigned *zc = nullptr)
{
    if constexpr (fft::Plan<N>::T > 32) {   // N = 4096: two warps per row
        using RA = RowA4<N>;
        auto kern = src == SRC_PRNG          ? ospr_rows_a4_kernel<N, LUT_PRNG, ZOUT>
                  : src == SRC_TABLE         ? ospr_rows_a4_kernel<N, LUT_PRNG_TABLE, ZOUT>
                  : ps.ix.mode == LUT_WRAP ? ospr_rows_a4_kernel<N, LUT_WRAP, ZOUT>
                  : ps.ix.mode == LUT_POW2 ? ospr_rows_a4_kernel<N, LUT_POW2, ZOUT>
                                           : ospr_rows_a4_kernel<N, LUT_GENERAL, ZOUT>;
        (void)zc;
        const int grid = pipe_grid(kern, RA::THREADS, RA::SMEM, np * RA::UNITS_PER_PAIR, 1);
        return launch(ZOUT ? K_RANDOMISE : K_OSPR_ROWS_A, kern, dim3(grid), dim3(RA::THREADS), RA::SMEM, s, tw, Tf, ps,
                      sf_first, np, last_has_b, buf);
    } else if constexpr (N >= 1024) {
        using RA2 = RowA2<N>;
        auto kern = src == SRC_PRNG          ? ospr_rows_a2_kernel<N, LUT_PRNG, ZOUT>
                  : src == SRC_TABLE         ? ospr_rows_a2_kernel<N, LUT_PRNG_TABLE, ZOUT>
                  : ps.ix.mode == LUT_WRAP ? ospr_rows_a2_kernel<N, LUT_WRAP, ZOUT>
                  : ps.ix.mode == LUT_POW2 ? ospr_rows_a2_kernel<N, LUT_POW2, ZOUT>
                                           : ospr_rows_a2_kernel<N, LUT_GENERAL, ZOUT>;
        const int grid = pipe_grid(kern, RA2::WPC * 32, RA2::SMEM, np * RA2::UNITS_PER_PAIR, RA2::UPC);
        return launch(ZOUT ? K_RANDOMISE : K_OSPR_ROWS_A, kern, dim3(grid), dim3(RA2::WPC * 32), RA2::SMEM, s, tw,
                      Tf, ps, sf_first, np, last_has_b, buf, zc);
    } else {
        using RA = RowA<N>;
        auto kern = src == SRC_PRNG          ? ospr_rows_a_kernel<N, LUT_PRNG, ZOUT>
                  : src == SRC_TABLE         ? ospr_rows_a_kernel<N, LUT_PRNG_TABLE, ZOUT>
                  : ps.ix.mode == LUT_WRAP ? ospr_rows_a_kernel<N, LUT_WRAP, ZOUT>
                  : ps.ix.mode == LUT_POW2 ? ospr_rows_a_kernel<N, LUT_POW2, ZOUT>
                                           : ospr_rows_a_kernel<N, LUT_GENERAL, ZOUT>;
        const int grid = pipe_grid(kern, RA::WPC * 32, RA::SMEM, np * RA::UNITS_PER_PAIR, RA::WPC);
        return launch(ZOUT ? K_RANDOMISE : K_OSPR_ROWS_A, kern, dim3(grid), dim3(RA::WPC * 32), RA::SMEM, s, tw, Tf,
                      ps, sf_first, np, last_has_b, buf, zc);
    }
}

// The phase source of a call (host side).
// src = SRC_TABLE: lut is the 2^q sin/cos table and n_lut = q (the phase bits).
static holo_status make_phase_src(int n, const float2 *lut, uint64_t n_lut, int src, uint64_t seed,
                                  uint64_t phase_offset, PhaseSrc *ps)
{
    const uint64_t P = (uint64_t)n * n;
    ps->shift = src == SRC_TABLE ? 32u - (uint32_t)n_lut : 0u;
    if (src != SRC_POOL)
        n_lut = 0;
    ps->ix = LutIndexer::make(n_lut ? (uint32_t)n_lut : 1u, n);
    ps->lut = lut;                      // N_LUT = 0: the one-entry pool {1 + 0i} (L = 1, R-6)
    if (lut == nullptr && src == SRC_POOL)
        HOLO_TRY(flat_lut(&ps->lut));
    ps->off_mod = n_lut ? (uint32_t)(phase_offset % n_lut) : 0u;
    ps->p_mod = n_lut ? (uint32_t)(P % n_lut) : 0u;
    ps->seed = seed;
    ps->off = phase_offset;
    return HOLO_OK;
}

template <int N>
static holo_status ospr_run(const float2 *tw, const float *target, int n_frames, int n_sub, const float2 *lut, uint64_t n_lut,
                            int src, uint64_t seed, uint64_t phase_offset, int sf_begin, int sf_end,
                            uint8_t *holo_bits, float *intensity, double *mse, holo_region om, void *ws, cudaStream_t s)
{
    constexpr size_t P = (size_t)N * N;
    OsprWs w;
    ospr_ws_layout(N, n_sub, (char *)ws, &w);
    const int chunk = ospr_chunk_pairs(N, n_sub);
    const int nsh = sf_end - sf_begin;
    const int npairs_total = (nsh + 1) / 2;
    const bool full = (sf_begin == 0 && sf_end == n_sub);
    PhaseSrc ps;
    HOLO_TRY(make_phase_src(N, lut, n_lut, src, seed, phase_offset, &ps));
    // a7 fused into the last chunk's pass C when one warp owns a row (N >= 1024); else its own kernel
    constexpr bool kWide = fft::Plan<N>::T > 32;   // N = 4096: two-warp rows (R-26)
    constexpr bool kFuse = !kWide && RowC<N>::GPW == 1;
    const float scale = full ? 0.5f / (float)n_sub : 0.5f;
    for (int f = 0; f < n_frames; ++f) {
        const float *Tf = target + (size_t)f * P;
        for (int c0 = 0; c0 < npairs_total; c0 += chunk) {
            const int np = (npairs_total - c0) < chunk ? (npairs_total - c0) : chunk;
            const int last_sa = sf_begin + 2 * (c0 + np - 1);
            const int last_has_b = (last_sa + 1) < sf_end;
            uint8_t *bt = holo_bits ? w.bt + 2 * (size_t)c0 * BitsT<N>::BYTES_PER_SUBFRAME : nullptr;
            unsigned *cf_ticket = reinterpret_cast<unsigned *>(w.cf_parts + (size_t)(N / 2) * 5);
            const bool last = c0 + np >= npairs_total;
            {
                const uint64_t sf_first = (uint64_t)f * n_sub + (uint64_t)sf_begin + 2 * (uint64_t)c0;
                HOLO_TRY((launch_pass_a<N, false>(tw, Tf, ps, src, sf_first, np, last_has_b, w.buf, s,
                                                  (kFuse && last) ? cf_ticket : nullptr)));
            }
            typename OsprColBody<N>::Args ca{tw, w.buf, bt, np, last_has_b};
            // tiles in reverse order: pass A wrote the last pairs last, so they are still in L2 (measured
            // C3: column pass 51.4 -> 49.0 us)
            HOLO_TRY((launch_cols<N, OsprColBody<N>>(K_OSPR_COLS, w.buf, np, ca, s, true)));
            bool fused = false;
            if constexpr (kFuse) {
                if (last) {   // pass C + a7 fused: mirrored row pairs per CTA
                fused = true;
                using RC = RowCF<N>;
                const int nbt = holo_bits ? nsh * BitsT<N>::BLOCKS_PER_Q : 0;
                const double cnt = (double)(om.row1 - om.row0) * (double)(om.col1 - om.col0);
                HOLO_TRY(launch(K_OSPR_ROWS_C, ospr_rows_cf_kernel<N>, dim3(nbt + RC::NU), dim3(RC::THREADS), RC::SMEM,
                                s, tw, (const float2 *)w.buf, np, c0 > 0 ? (const float *)w.acc : (const float *)nullptr,
                                Tf, scale, intensity + (size_t)f * P, om, w.cf_parts, cf_ticket, 1.0 / cnt,
                                (full && mse) ? mse + f : (double *)nullptr, nbt, (const uint8_t *)w.bt,
                                holo_bits ? holo_bits + (size_t)f * nsh * (P / 8) : nullptr));
                }
            }
            if constexpr (kWide) {
                using R = Row2W<N>;
                const int nbt = (last && holo_bits) ? nsh * BitsT<N>::BLOCKS_PER_Q : 0;
                const int grid = pipe_grid(ospr_rows2w_c_kernel<N>, R::THREADS, R::SMEM, N / 2, 1);
                HOLO_TRY(launch(K_OSPR_ROWS_C, ospr_rows2w_c_kernel<N>, dim3(nbt + grid), dim3(R::THREADS), R::SMEM, s,
                                tw, (const float2 *)w.buf, np, w.acc, c0 > 0 ? 1 : 0, finalize_ticket(w.parts), nbt,
                                (const uint8_t *)w.bt, holo_bits ? holo_bits + (size_t)f * nsh * (P / 8) : nullptr));
            } else if (!fused) {
                using RC = RowC<N>;
                const int nbt = (last && holo_bits) ? nsh * BitsT<N>::BLOCKS_PER_Q : 0;
                const int grid = pipe_grid(ospr_rows_c_kernel<N>, 64, RC::SMEM, RC::NGRP, 1);
                HOLO_TRY(launch(K_OSPR_ROWS_C, ospr_rows_c_kernel<N>, dim3(nbt + grid), dim3(64), RC::SMEM, s, tw,
                                (const float2 *)w.buf, np, w.acc, c0 > 0 ? 1 : 0, finalize_ticket(w.parts), nbt,
                                (const uint8_t *)w.bt, holo_bits ? holo_bits + (size_t)f * nsh * (P / 8) : nullptr));
            }
        }
        if (!kFuse)
            HOLO_TRY(finalize_frame<N>(w.acc, Tf, 1, scale, intensity + (size_t)f * P, om, w.parts,
                                       (full && mse) ? mse + f : nullptr, s, true));
    }
    return HOLO_OK;
}

holo_status check_n(int n)
{
    if (n < 16 || n > 4096 || (n & (n - 1)) != 0)
        return set_error(HOLO_ERR_INVALID_ARG, "n must be a power of two in [16, 4096], got %d", n);
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

extern "C" size_t holo_ospr_finalize_workspace_size(void) { return kFinWsBytes; }

extern "C" int32_t holo_ospr_chunk_pairs(int32_t n, int32_t n_sub)
{
    if (check_n(n) != HOLO_OK || n_sub < 1)
        return 0;
    return ospr_chunk_pairs(n, n_sub);
}

static holo_status ospr_entry(const float *target, int32_t n, int32_t n_frames, int32_t n_sub, const holo_c64 *lut,
                              uint64_t n_lut, int src, uint64_t seed, uint64_t phase_offset, int32_t sf_begin,
                              int32_t sf_end, uint8_t *holo_bits, float *intensity, double *mse, holo_region omega,
                              void *ws, size_t ws_bytes, holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(n_frames >= 1 && n_sub >= 1, "n_frames and n_sub must be >= 1 (got %d, %d)", n_frames, n_sub);
    HOLO_CHECK_ARG(0 <= sf_begin && sf_begin < sf_end && sf_end <= n_sub,
                   "sub-frame range [%d,%d) must be a non-empty part of [0,%d)", sf_begin, sf_end, n_sub);
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    if (src == SRC_TABLE)
        HOLO_CHECK_ARG(lut != nullptr && n_lut >= 1 && n_lut <= 16, "the sin/cos table is required, phase_bits in [1, 16]");
    else
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
#define HOLO_OSPR_CASE(NN)                                                                                 \
    case NN:                                                                                               \
        return ospr_run<NN>(tw, target, n_frames, n_sub, l, n_lut, src, seed, phase_offset, sf_begin, sf_end, \
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
        HOLO_OSPR_CASE(4096)
    default:
        return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
    }
#undef HOLO_OSPR_CASE
}

extern "C" holo_status holo_ospr_generate(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                          const holo_c64 *lut, uint64_t n_lut, uint64_t phase_offset,
                                          int32_t sf_begin, int32_t sf_end, uint8_t *holo_bits,
                                          float *intensity, double *mse, holo_region omega, void *ws,
                                          size_t ws_bytes, holo_stream stream)
{
    return ospr_entry(target, n, n_frames, n_sub, lut, n_lut, SRC_POOL, 0, phase_offset, sf_begin, sf_end, holo_bits,
                      intensity, mse, omega, ws, ws_bytes, stream);
}

extern "C" holo_status holo_ospr_generate_prng(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                               uint64_t seed, uint64_t phase_offset, int32_t sf_begin,
                                               int32_t sf_end, uint8_t *holo_bits, float *intensity, double *mse,
                                               holo_region omega, void *ws, size_t ws_bytes, holo_stream stream)
{
    return ospr_entry(target, n, n_frames, n_sub, nullptr, 0, SRC_PRNG, seed, phase_offset, sf_begin, sf_end, holo_bits,
                      intensity, mse, omega, ws, ws_bytes, stream);
}

extern "C" holo_status holo_ospr_generate_prng_table(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                                     uint64_t seed, const holo_c64 *table, int32_t phase_bits,
                                                     uint64_t phase_offset, int32_t sf_begin, int32_t sf_end,
                                                     uint8_t *holo_bits, float *intensity, double *mse,
                                                     holo_region omega, void *ws, size_t ws_bytes, holo_stream stream)
{
    HOLO_CHECK_ARG(phase_bits >= 1 && phase_bits <= 16, "phase_bits must be in [1, 16], got %d", phase_bits);
    return ospr_entry(target, n, n_frames, n_sub, table, (uint64_t)phase_bits, SRC_TABLE, seed, phase_offset,
                      sf_begin, sf_end, holo_bits, intensity, mse, omega, ws, ws_bytes, stream);
}

extern "C" holo_status holo_debug_ospr_pairs(const float *target, int32_t n, int32_t n_sub, const holo_c64 *lut,
                                             uint64_t n_lut, int32_t use_prng, uint64_t prng_seed,
                                             uint64_t phase_offset, int32_t sf_begin, int32_t sf_end,
                                             holo_c64 *z_out, holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(target != nullptr && z_out != nullptr, "target/z_out is NULL");
    HOLO_CHECK_ARG(n_sub >= 1 && 0 <= sf_begin && sf_begin < sf_end && sf_end <= n_sub,
                   "sub-frame range [%d,%d) must be a non-empty part of [0,%d)", sf_begin, sf_end, n_sub);
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    HOLO_CHECK_ARG(use_prng >= 0 && use_prng <= 2, "use_prng must be 0 (pool), 1 (on the fly) or 2 (table)");
    if (use_prng == SRC_TABLE)
        HOLO_CHECK_ARG(lut != nullptr && n_lut >= 1 && n_lut <= 16, "table mode: lut = the table, n_lut = phase_bits");
    else
        HOLO_CHECK_ARG((lut == nullptr) == (n_lut == 0), "lut must be NULL iff n_lut == 0");
    HOLO_CHECK_ARG(use_prng != SRC_PRNG || lut == nullptr, "use_prng excludes a LUT");
    const float2 *tw = nullptr;
    HOLO_TRY(fft::twiddles(&tw));
    const int src = use_prng;
    PhaseSrc ps;
    HOLO_TRY(make_phase_src(n, (const float2 *)lut, n_lut, src, prng_seed, phase_offset, &ps));
    const int npairs = (sf_end - sf_begin + 1) / 2;
    const int last_has_b = (sf_begin + 2 * (npairs - 1) + 1) < sf_end;
    cudaStream_t s = (cudaStream_t)stream;
    float2 *z = (float2 *)z_out;
#define HOLO_PAIRS_CASE(NN)                                                                                  \
    case NN:                                                                                                 \
        return launch_pass_a<NN, true>(tw, target, ps, src, (uint64_t)sf_begin, npairs, last_has_b, z, s);
    switch (n) {
        HOLO_PAIRS_CASE(16)
        HOLO_PAIRS_CASE(32)
        HOLO_PAIRS_CASE(64)
        HOLO_PAIRS_CASE(128)
        HOLO_PAIRS_CASE(256)
        HOLO_PAIRS_CASE(512)
        HOLO_PAIRS_CASE(1024)
        HOLO_PAIRS_CASE(2048)
        HOLO_PAIRS_CASE(4096)
    default:
        return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
    }
#undef HOLO_PAIRS_CASE
}

extern "C" holo_status holo_ospr_finalize_rows(const float *target, const float *intensity_sum_rows, int32_t n,
                                               int32_t row0, int32_t row1, int32_t n_sub, holo_region omega,
                                               float *intensity_mean_rows, double *sums, void *ws, size_t ws_bytes,
                                               holo_stream stream)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(0 <= row0 && row0 < row1 && row1 <= n, "row slice [%d,%d) must be a non-empty part of [0,%d)",
                   row0, row1, n);
    HOLO_CHECK_ARG(n_sub >= 1, "n_sub must be >= 1");
    HOLO_CHECK_ARG(target && intensity_sum_rows && intensity_mean_rows && sums,
                   "target, intensity_sum_rows, intensity_mean_rows and sums are required");
    HOLO_TRY(check_region(omega, n));
    HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
    if (ws_bytes < kFinWsBytes)
        return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, kFinWsBytes);
    const int nrows = row1 - row0, pix = n * nrows;
    int fb = (pix + 8 * kFinThreads - 1) / (8 * kFinThreads);
    if (fb > kFinBlocks)
        fb = kFinBlocks;
    const int iter = (pix + fb * kFinThreads - 1) / (fb * kFinThreads);
    double *parts = (double *)ws;
    unsigned *counter = finalize_ticket(parts);
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaMemsetAsync(finalize ticket)");
    return launch(K_OSPR_FINALIZE, ospr_finalize_rows_kernel, dim3(fb), dim3(kFinThreads), 0, s,
                  intensity_sum_rows, target, n, row0, nrows, iter, 1.0f / (float)n_sub, intensity_mean_rows, omega, parts,
                  counter, sums);
}

extern "C" holo_status holo_ospr_mse_from_sums(const double *sums, int32_t n_frames, holo_region omega, double *mse,
                                               holo_stream stream)
{
    HOLO_CHECK_ARG(sums != nullptr && mse != nullptr, "sums and mse are required");
    HOLO_CHECK_ARG(n_frames >= 1, "n_frames must be >= 1");
    HOLO_CHECK_ARG(omega.row0 < omega.row1 && omega.col0 < omega.col1, "omega is empty");
    const double cnt = (double)(omega.row1 - omega.row0) * (double)(omega.col1 - omega.col0);
    return launch(K_MSE_REDUCE, ospr_mse_from_sums_kernel, dim3((n_frames + 127) / 128), dim3(128), 0,
                  (cudaStream_t)stream, sums, n_frames, 1.0 / cnt, mse);
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
    const size_t need = kFinWsBytes;
    if (mse) {
        HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
        if (ws_bytes < need)
            return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    }
    const size_t P = (size_t)n * n;
    cudaStream_t s = (cudaStream_t)stream;
    for (int f = 0; f < n_frames; ++f) {
        const float *a = intensity_sum + f * P, *t = target + f * P;
        float *o = intensity_mean + f * P;
        double *m = mse ? mse + f : nullptr, *parts = (double *)ws;
#define HOLO_FIN_CASE(NN)                                                                                  \
    case NN:                                                                                               \
        HOLO_TRY(finalize_frame<NN>(a, t, 0, 1.0f / (float)n_sub, o, omega, parts, m, s)); \
        break;
        switch (n) {
            HOLO_FIN_CASE(16)
            HOLO_FIN_CASE(32)
            HOLO_FIN_CASE(64)
            HOLO_FIN_CASE(128)
            HOLO_FIN_CASE(256)
            HOLO_FIN_CASE(512)
            HOLO_FIN_CASE(1024)
            HOLO_FIN_CASE(2048)
            HOLO_FIN_CASE(4096)
        default:
            return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
        }
#undef HOLO_FIN_CASE
    }
    return HOLO_OK;
}
