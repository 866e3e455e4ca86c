// fft.cuh -- the register/shared-memory FFT machinery of libholo (sm_100a).
//
// Evaluates the unitary DFT pair of PAPER.md Eqs. (1)-(2) up to the
// 1/sqrt(N) scale, which the callers fold into their epilogues.
//
// A length-N transform (N = R1*R2, R1 <= R2, both powers of two) is done by
// T = R1 cooperating threads, each holding E = R2 complex values in registers,
// in two Stockham passes with one exchange through shared memory:
//   pass 1: thread t holds x[t + R1*m], m < R2, and runs Q = R2/R1 radix-R1
//           DFTs over the slots {b + Q*r}, writing y[(t + R1*b)*R1 + r];
//   pass 2: thread t reads y[t + R1*r], r < R2, multiplies by W_N^{r*t} and runs
//           one radix-R2 DFT; output element t + R1*r lands in slot r.
// Input and output use the same thread<->element map, so a transform can be
// followed by another one in registers (OSPR column pass: IFFT -> sign -> FFT).
// The exchange index i is stored at (i + i/R1)*IL: the +i/R1 pad makes both the
// strided pass-1 stores and the contiguous pass-2 loads bank-conflict free, and
// IL interleaves the buffers of IL independent columns (column kernels).
//
// The radix-R DFTs are compile-time codelets (recursive radix-4/radix-2 DIT)
// whose twiddles W_R^k are constexpr; the trivial ones (1, -1, +-i, (+-1+-i)/sqrt2)
// cost no multiplies.
#pragma once

#include "common.cuh"

namespace holo {
namespace fft {

// ---- compile-time trigonometry (for codelet twiddles only) --------------------------------
constexpr double kPi = 3.141592653589793238462643383279502884;

constexpr double sin_red(double x)
{
    double s = x * x, t = x, r = x;
    for (int i = 1; i <= 12; ++i) {
        t *= -s / ((2.0 * i) * (2.0 * i + 1.0));
        r += t;
    }
    return r;
}
constexpr double cos_red(double x)
{
    double s = x * x, t = 1.0, r = 1.0;
    for (int i = 1; i <= 12; ++i) {
        t *= -s / ((2.0 * i - 1.0) * (2.0 * i));
        r += t;
    }
    return r;
}

struct CS {
    double c, s;
};

// cos, sin of 2*pi*k/n by exact octant reduction of the rational k/n.
constexpr CS cs2pi(long long k, long long n)
{
    k %= n;
    if (k < 0)
        k += n;
    long long e = 8 * k;
    long long o = e / n;
    long long rem = e - o * n;
    double f = (o & 1) ? (double)(n - rem) / (double)n : (double)rem / (double)n;
    double x = f * (kPi / 4.0);
    double S = sin_red(x), C = cos_red(x);
    switch (o) {
    case 0: return CS{C, S};
    case 1: return CS{S, C};
    case 2: return CS{-S, C};
    case 3: return CS{-C, S};
    case 4: return CS{-C, -S};
    case 5: return CS{-S, -C};
    case 6: return CS{S, -C};
    default: return CS{C, -S};
    }
}

// x * W_R^K with W_R = exp(-2 pi i / R) (forward) or exp(+2 pi i / R) (inverse).
template <int R, int K, bool INV>
__device__ __forceinline__ float2 tw_mul(float2 x)
{
    constexpr int k = ((K % R) + R) % R;
    if constexpr (k == 0) {
        return x;
    } else if constexpr (2 * k == R) {
        return make_float2(-x.x, -x.y);
    } else if constexpr (4 * k == R) {          // fwd -i, inv +i
        return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
    } else if constexpr (4 * k == 3 * R) {      // fwd +i, inv -i
        return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
    } else if constexpr ((8 * k) % R == 0) {    // odd multiples of pi/4: (+-1 +-i)/sqrt2
        constexpr CS w = cs2pi(INV ? k : -k, R);
        constexpr float h = 0.70710678118654752440f;
        // x + i x = (x.x - x.y, x.y + x.x), x - i x = (x.x + x.y, x.y - x.x): one FADD2 + one FMUL2
        if constexpr (w.c > 0 && w.s > 0)
            return f2::mul(cadd(x, cmul_i(x)), f2::bc(h));
        else if constexpr (w.c > 0)
            return f2::mul(csub(x, cmul_i(x)), f2::bc(h));
        else if constexpr (w.s > 0)
            return f2::mul(csub(x, cmul_i(x)), f2::bc(-h));
        else
            return f2::mul(cadd(x, cmul_i(x)), f2::bc(-h));
    } else {
        constexpr CS w = cs2pi(INV ? k : -k, R);
        return cmul_cs(x, (float)w.c, (float)w.s);
    }
}

// In-place DFT of the R values v[0], v[S], ..., v[(R-1)S] (natural order in and out).
template <int R, int S, bool INV>
struct Dft {
    template <int K>
    static __device__ __forceinline__ void comb4(float2 *v, float2 *t)
    {
        if constexpr (K < R / 4) {
            float2 a = v[4 * S * K];
            float2 b = tw_mul<R, K, INV>(v[S + 4 * S * K]);
            float2 c = tw_mul<R, 2 * K, INV>(v[2 * S + 4 * S * K]);
            float2 d = tw_mul<R, 3 * K, INV>(v[3 * S + 4 * S * K]);
            float2 apc = cadd(a, c), amc = csub(a, c), bpd = cadd(b, d), bmd = csub(b, d);
            // W_4 * (b - d): forward W_4 = -i, inverse +i
            float2 wbmd = INV ? make_float2(-bmd.y, bmd.x) : make_float2(bmd.y, -bmd.x);
            t[K] = cadd(apc, bpd);
            t[K + R / 4] = cadd(amc, wbmd);
            t[K + R / 2] = csub(apc, bpd);
            t[K + 3 * R / 4] = csub(amc, wbmd);
            comb4<K + 1>(v, t);
        }
    }
    template <int K>
    static __device__ __forceinline__ void comb2(float2 *v, float2 *t)
    {
        if constexpr (K < R / 2) {
            float2 a = v[2 * S * K];
            float2 b = tw_mul<R, K, INV>(v[S + 2 * S * K]);
            t[K] = cadd(a, b);
            t[K + R / 2] = csub(a, b);
            comb2<K + 1>(v, t);
        }
    }
    static __device__ __forceinline__ void run(float2 *v)
    {
        if constexpr (R == 1) {
        } else if constexpr (R == 2) {
            float2 a = v[0], b = v[S];
            v[0] = cadd(a, b);
            v[S] = csub(a, b);
        } else if constexpr (R % 4 == 0) {
            Dft<R / 4, 4 * S, INV>::run(v);
            Dft<R / 4, 4 * S, INV>::run(v + S);
            Dft<R / 4, 4 * S, INV>::run(v + 2 * S);
            Dft<R / 4, 4 * S, INV>::run(v + 3 * S);
            float2 t[R];
            comb4<0>(v, t);
#pragma unroll
            for (int i = 0; i < R; ++i)
                v[S * i] = t[i];
        } else {
            Dft<R / 2, 2 * S, INV>::run(v);
            Dft<R / 2, 2 * S, INV>::run(v + S);
            float2 t[R];
            comb2<0>(v, t);
#pragma unroll
            for (int i = 0; i < R; ++i)
                v[S * i] = t[i];
        }
    }
};

// ---- plan ---------------------------------------------------------------------------------
constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n / 2); }

template <int N>
struct Plan {
    static_assert(N >= 16 && N <= 4096 && (N & (N - 1)) == 0, "N must be a power of two in [16, 4096]");
    static constexpr int LOG = ilog2(N);
    static constexpr int R1 = 1 << (LOG / 2);       // threads per transform
    static constexpr int R2 = N / R1;               // values per thread (E)
    static constexpr int E = R2;
    static constexpr int T = R1;
    static constexpr int Q = R2 / R1;               // pass-1 DFTs per thread (1 or 2)
    static constexpr int SMEM = N + N / R1;         // padded exchange buffer, complex elements
    static constexpr int TW_OFFSET = N - 16;        // offset of this N in the twiddle pool
};

// Pass-2 twiddles: g_tw[TW_OFFSET(N) + r*R1 + t] = W_N^{r*t} (forward sign), r < R2, t < R1.
// Laid out r-major so that the R1 threads of a transform read consecutive entries.
// Pool size: sum over N = 16..4096 of N = 8176 entries.  Built once per device by
// holo::fft::twiddles() (host libm in double, rounded to fp32) in library-owned
// device memory; kernels receive the pool pointer as an argument.
constexpr int kTwPool = 8192;   // 8176 two-pass entries (N = 16 .. 4096)
holo_status twiddles(const float2 **pool);

__device__ __forceinline__ int pad_index(int i, int r1) { return i + i / r1; }

// Read-only load the compiler may neither hoist nor merge with an earlier load of the same
// address: keeps two transforms in one kernel from pinning the 2*(R2-1) twiddle registers
// of the first across the work in between (register pressure -> occupancy).
__device__ __forceinline__ float2 ldg_nocse(const float2 *p)
{
    float2 v;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// The R2 pass-2 twiddles W_N^{r*t} (forward sign) of transform role t.  REG = true keeps
// them in registers across every transform a thread performs with that role (2*(R2-1)
// registers); REG = false re-reads them from the L1-resident pool per transform.
template <int N, bool REG = (Plan<N>::E <= 32)>
struct Twiddles {
    float2 w[REG ? Plan<N>::R2 : 1];
    const float2 *p;
    __device__ __forceinline__ void load(const float2 *__restrict__ twp, int t)
    {
        using P = Plan<N>;
        p = twp + P::TW_OFFSET + t;
        if constexpr (REG) {
#pragma unroll
            for (int r = 0; r < P::R2; ++r)
                w[r] = __ldg(p + r * P::R1);
        }
    }
    __device__ __forceinline__ float2 get(int r) const
    {
        if constexpr (REG)
            return w[r];
        else
            return ldg_nocse(p + r * Plan<N>::R1);
    }
};

// Two-pass FFT of one length-N transform held by T = R1 threads (see header).
// `sm` points at this transform's exchange buffer (element i at sm[(i + i/R1)*IL]).
// WS = true: the T threads of the transform live in one warp (T <= 32, row kernels)
// and synchronise with __syncwarp(), so warps run independently; WS = false: the
// threads span warps (column tiles) and every thread of the CTA must call this
// together (__syncthreads()).
struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};

// Barrier of a transform whose threads span warps (WS = false): the whole CTA (id = 0) or a
// named barrier over the n threads of one consumer group (id > 0; grouped column pipeline).
struct GroupSync {
    int id = 0, n = 0;
    __device__ __forceinline__ void operator()() const
    {
        if (id == 0)
            __syncthreads();
        else
            asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    }
};

// `after_exchange` runs once every value has been read back from the exchange buffer, before
// the pass-2 DFT: a caller refilling the buffer by TMA from there on must first order those
// reads before the async-proxy write (fence.proxy.async + __syncwarp; WS = true only).
template <int N, bool INV, int IL, bool WS, class TwSrc, class Hook = NoHook>
__device__ __forceinline__ void fft2pass_impl(float2 (&v)[Plan<N>::E], float2 *sm, int t, const TwSrc &tws,
                                              const Hook &after_exchange = Hook(), const GroupSync &gs = GroupSync())
{
    using P = Plan<N>;
    constexpr int R1 = P::R1, R2 = P::R2, Q = P::Q;
#pragma unroll
    for (int b = 0; b < Q; ++b)
        Dft<R1, Q, INV>::run(v + b);
    if (WS)
        __syncwarp();
    else
        gs();                               // previous readers of sm are done
#pragma unroll
    for (int b = 0; b < Q; ++b)
#pragma unroll
        for (int r = 0; r < R1; ++r) {
            const int i = (t + R1 * b) * R1 + r;
            sm[(i + t + R1 * b) * IL] = v[b + Q * r];   // i/R1 == t + R1*b
        }
    if (WS)
        __syncwarp();
    else
        gs();
#pragma unroll
    for (int r = 0; r < R2; ++r) {
        const int i = t + R1 * r;
        float2 x = sm[(i + r) * IL];                       // i/R1 == r
        if (r > 0) {
            float2 w = tws(r);
            if (INV)
                w.y = -w.y;
            x = cmul(x, w);
        }
        v[r] = x;
    }
    after_exchange();
    Dft<R2, 1, INV>::run(v);
}

template <int N>
struct TwGlobal {
    const float2 *p;
    __device__ __forceinline__ float2 operator()(int r) const { return ldg_nocse(p + r * Plan<N>::R1); }
};

template <int N, bool REG>
struct TwRegs {
    const Twiddles<N, REG> &tw;
    __device__ __forceinline__ float2 operator()(int r) const { return tw.get(r); }
};

// Twiddles read from the global pool (L1-resident) per transform.
template <int N, bool INV, int IL, bool WS = false>
__device__ __forceinline__ void fft2pass(float2 (&v)[Plan<N>::E], float2 *sm, int t,
                                         const float2 *__restrict__ twp)
{
    fft2pass_impl<N, INV, IL, WS>(v, sm, t, TwGlobal<N>{twp + Plan<N>::TW_OFFSET + t});
}

// Pass-2 twiddles W_N^{r t} factorised as W_N^{8a t} * W_N^{b t} (r = 8a + b, b < 8): the
// (R2/8 - 1) + 7 factors of role t are loaded from the pool once and kept in registers
// (20 registers at N = 1024 instead of 62 for the full set); each twiddle with a, b > 0 costs
// one complex multiply (one extra rounding, ~1 ulp) instead of a load per transform.
template <int N>
struct TwFact {
    static constexpr int R1 = Plan<N>::R1, R2 = Plan<N>::R2, NA = (R2 + 7) / 8;
    float2 lo[8], hi[NA];
    __device__ __forceinline__ void load(const float2 *__restrict__ twp, int t)
    {
        const float2 *p = twp + Plan<N>::TW_OFFSET + t;
#pragma unroll
        for (int b = 1; b < 8 && b < R2; ++b)
            lo[b] = __ldg(p + b * R1);
#pragma unroll
        for (int a = 1; a < NA; ++a)
            hi[a] = __ldg(p + 8 * a * R1);
    }
    __device__ __forceinline__ float2 operator()(int r) const
    {
        const int a = r / 8, b = r % 8;
        if (a == 0)
            return lo[b];
        if (b == 0)
            return hi[a];
        return cmul(hi[a], lo[b]);
    }
};

// Twiddles from the pool, with a hook after the exchange (see fft2pass_impl).
template <int N, bool INV, int IL, bool WS, class Hook>
__device__ __forceinline__ void fft2pass_hook(float2 (&v)[Plan<N>::E], float2 *sm, int t, const float2 *__restrict__ twp,
                                              const Hook &after_exchange)
{
    fft2pass_impl<N, INV, IL, WS>(v, sm, t, TwGlobal<N>{twp + Plan<N>::TW_OFFSET + t}, after_exchange);
}

// Twiddles prepared by the caller (Twiddles<N>::load once per role).
template <int N, bool INV, int IL, bool WS = false, bool REG = true>
__device__ __forceinline__ void fft2pass(float2 (&v)[Plan<N>::E], float2 *sm, int t, const Twiddles<N, REG> &tw)
{
    fft2pass_impl<N, INV, IL, WS>(v, sm, t, TwRegs<N, REG>{tw});
}

// FFT policies for the column pipeline: element m of thread t is row t + T*m.
template <int N, bool REG>
struct ColFft2 {
    using P = Plan<N>;
    static constexpr int E = P::E, T = P::T, SMEM = P::SMEM;
    Twiddles<N, REG> tw;
    GroupSync sync;                          // CTA-wide unless the pipeline runs consumer groups
    __device__ __forceinline__ void init(const float2 *twp, int t) { tw.load(twp, t); }
    template <bool INV, int IL>
    __device__ __forceinline__ void run(float2 (&v)[E], float2 *sm, int t) const
    {
        fft2pass_impl<N, INV, IL, false>(v, sm, t, TwRegs<N, REG>{tw}, NoHook(), sync);
    }
};


} // namespace fft
} // namespace holo
