// common.cuh -- shared plumbing of libholo: status reporting, kernel launch
// accounting / profiling, complex helpers, fast modulo.  Product code; it shares
// nothing with oracle/ (DESIGN.md §2).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/holo.h"

namespace holo {

// ---- status ------------------------------------------------------------------------
holo_status set_error(holo_status st, const char *fmt, ...);
holo_status cuda_status(cudaError_t e, const char *where);

#define HOLO_CHECK_ARG(cond, ...)                                                          \
    do {                                                                                   \
        if (!(cond))                                                                       \
            return ::holo::set_error(HOLO_ERR_INVALID_ARG, __VA_ARGS__);                   \
    } while (0)

#define HOLO_TRY(expr)                                                                     \
    do {                                                                                   \
        holo_status _st = (expr);                                                          \
        if (_st != HOLO_OK)                                                                \
            return _st;                                                                    \
    } while (0)

// ---- kernel classes (profiling names) ----------------------------------------------------
enum KernelId : int {
    K_LUT_GENERATE = 0,
    K_OSPR_ROWS_A,      // T x LUT for a sub-frame pair (Hermitian pairing) + row IFFT
    K_OSPR_COLS,        // column IFFT + sign quantise + bit pack + column FFT
    K_OSPR_ROWS_C,      // row FFT + |.|^2 accumulate over the chunk's pairs
    K_OSPR_FINALIZE,    // symmetrise/scale + MSE + sign bytes -> packed holograms
    K_MSE_REDUCE,       // fixed-order reduction of partial sums -> MSE
    K_GS_ROWS_INIT,     // T x LUT (or R_in) + row IFFT
    K_GS_COLS,          // column IFFT + phase constraint + column FFT
    K_GS_ROWS,          // row FFT + metrics + amplitude replacement + row IFFT
    K_FFT_ROWS,         // test hook
    K_FFT_COLS,         // test hook
    K_RANDOMISE,        // test hook
    K_NUM_KERNELS
};
extern const char *const kKernelNames[K_NUM_KERNELS];

// Records profiling events (if enabled) around a launch and counts it.
void prof_before(KernelId id, cudaStream_t s);
void prof_after(KernelId id, cudaStream_t s);
void count_launch();
holo_status ensure_smem(const void *fn, size_t smem);
// SMs x resident CTAs per SM of `fn` at (threads, smem) on the current device; cached, and
// opts the kernel in to `smem` bytes of dynamic shared memory first.
int resident_ctas(const void *fn, int threads, size_t smem);

// Programmatic dependent launch (PDL): every library kernel is launched with programmatic
// stream serialisation and begins with HOLO_PDL_ENTRY: it waits for the previous kernel in
// the stream to complete and flush (griddepcontrol.wait) before touching memory, and each
// CTA signals on its way out (any return path) that the next kernel may be scheduled
// (griddepcontrol.launch_dependents).  The next pass's launch and prologue thus overlap
// this pass's tail instead of following a full drain; ordering is unchanged.  (Signalling
// at entry instead measured slower: early dependents' waiting CTAs share the SMs with the
// running pass.)
struct PdlExitTrigger {
    __device__ __forceinline__ ~PdlExitTrigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
};
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define HOLO_PDL_ENTRY()                        \
    ::holo::PdlExitTrigger holo_pdl_exit_trigger_; \
    ::holo::pdl_wait()
bool pdl_enabled();   // HOLO_PDL=0 launches without the attribute (griddepcontrol then no-ops)

template <typename... KArgs, typename... Args>
holo_status launch(KernelId id, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t s, Args... args)
{
    if (grid.x == 0 || grid.y == 0 || grid.z == 0)
        return HOLO_OK;
    if (smem > 0)
        HOLO_TRY(ensure_smem((const void *)kernel, smem));   // cached per kernel and device
    prof_before(id, s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    if (e == cudaSuccess)
        e = cudaGetLastError();
    prof_after(id, s);
    count_launch();
    if (e != cudaSuccess)
        return cuda_status(e, kKernelNames[id]);
    return HOLO_OK;
}

// ---- complex helpers ---------------------------------------------------------------
// Complex arithmetic on sm_100's packed fp32 pipe: one complex add is one
// add.rn.f32x2 (SASS FADD2), one complex multiply one mul.rn.f32x2 + one
// fma.rn.f32x2 (FMUL2 + FFMA2), the swaps, broadcasts and sign flips folding into
// operand modifiers.  Each lane is an IEEE round-to-nearest fp32 operation, and the
// explicit PTX leaves the compiler nothing to contract, so every instantiation of a
// transform performs bit-identical arithmetic (the fused GS loop equals chained
// gs_step calls, tests/test_gpu_gs.py).
namespace f2 {
__device__ __forceinline__ unsigned long long pk(float2 a)
{
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 up(unsigned long long r)
{
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
__device__ __forceinline__ float2 add(float2 a, float2 b)
{
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return up(r);
}
__device__ __forceinline__ float2 sub(float2 a, float2 b)
{
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return up(r);
}
__device__ __forceinline__ float2 mul(float2 a, float2 b)
{
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return up(r);
}
__device__ __forceinline__ float2 fma(float2 a, float2 b, float2 c)
{
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return up(r);
}
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
} // namespace f2

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2::add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return f2::sub(a, b); }
// i*a = (-a.y, a.x)
__device__ __forceinline__ float2 cmul_i(float2 a) { return make_float2(-a.y, a.x); }
// a*b = (a.x b.x - a.y b.y, a.x b.y + a.y b.x): t = a*b.x (rounded), then fma(i*a, b.y, t)
__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return f2::fma(cmul_i(a), f2::bc(b.y), f2::mul(a, f2::bc(b.x)));
}
// a * (c + i s) for compile-time c, s (immediate operands)
__device__ __forceinline__ float2 cmul_cs(float2 a, float c, float s)
{
    return f2::fma(cmul_i(a), f2::bc(s), f2::mul(a, f2::bc(c)));
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// 1/sqrt(x) for normal x > 0: one SFU instruction (rsqrt.approx.ftz, relative error
// below 2^-22).  Callers treat x < kFltMin (zero, or a denormal the SFU flushes) as zero.
__device__ __forceinline__ float rsqrt_sfu(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
constexpr float kFltMin = 1.17549435082228750797e-38f;   // smallest normal fp32

// 1/sqrt(x), IEEE round-to-nearest (correctly rounded; the SFU estimate plus a Newton fix-up).
__device__ __forceinline__ float rsqrt_rn(float x) { return __frsqrt_rn(x); }

// ---- cyclic LUT index (step a1) ----------------------------------------------------------
// idx = (rowbase + x) mod L for rowbase < L, x < N, evaluated per pixel without a
// hardware divide: L >= N needs at most one subtraction; a power-of-two L is a mask;
// otherwise Lemire's fastmod (exact for 32-bit operands).  An empty pool (N_LUT = 0,
// R-6) is indexed as the one-entry pool {1 + 0i} (L = 1, mask 0).
// LUT_PRNG: no pool, R-5 per draw; LUT_PRNG_TABLE: a draw's top q code bits index a 2^q table (ospr.cu)
enum LutMode : int { LUT_WRAP = 0, LUT_POW2 = 1, LUT_GENERAL = 2, LUT_PRNG = 3, LUT_PRNG_TABLE = 4 };
struct LutIndexer {
    uint32_t L;       // N_LUT (> 0)
    uint32_t mode;    // LutMode
    uint64_t M;       // ceil(2^64 / L) for LUT_GENERAL
    __host__ static LutIndexer make(uint32_t L, uint32_t n)
    {
        LutIndexer r;
        r.L = L;
        r.M = (L & (L - 1)) ? UINT64_MAX / L + 1 : 0;   // Lemire constant (non-powers of two)
        if (L >= n)
            r.mode = LUT_WRAP;
        else if ((L & (L - 1)) == 0)
            r.mode = LUT_POW2;
        else
            r.mode = LUT_GENERAL;
        return r;
    }
    // compile-time mode: branch-free per-pixel index
    template <int MODE>
    __device__ __forceinline__ uint32_t mod_t(uint32_t a) const
    {
        if constexpr (MODE == LUT_WRAP)
            return a >= L ? a - L : a;
        else if constexpr (MODE == LUT_POW2)
            return a & (L - 1);
        else
            return (uint32_t)__umul64hi(M * (uint64_t)a, (uint64_t)L);
    }
    __device__ __forceinline__ uint32_t mod(uint32_t a) const
    {
        if (mode == LUT_WRAP)
            return mod_t<LUT_WRAP>(a);
        if (mode == LUT_POW2)
            return mod_t<LUT_POW2>(a);
        return mod_t<LUT_GENERAL>(a);
    }
    // a mod L for any 32-bit a (per-row bases): mask, or Lemire's fastmod with M = ceil(2^64 / L)
    __device__ __forceinline__ uint32_t mod32(uint32_t a) const
    {
        if ((L & (L - 1)) == 0)
            return a & (L - 1);
        return (uint32_t)__umul64hi(M * (uint64_t)a, (uint64_t)L);
    }
    // a mod L for any 64-bit a (per-sub-frame bases): Barrett with B = floor(2^64 / L) = M - 1
    // (L not a power of two); q = floor(a B / 2^64) is floor(a / L) or one less, so a single
    // conditional subtract finishes.  A hardware-free replacement of the 64-bit '%' subroutine,
    // whose dependent chain cost thousands of cycles per warp unit in pass A.
    __device__ __forceinline__ uint32_t mod64(uint64_t a) const
    {
        if ((L & (L - 1)) == 0)
            return (uint32_t)(a & (uint64_t)(L - 1));
        const uint64_t q = __umul64hi(a, M - 1);
        uint64_t r = a - q * (uint64_t)L;
        if (r >= L)
            r -= L;
        return (uint32_t)r;
    }
    // general a (may exceed 2L)
    __device__ __forceinline__ uint32_t mod_any(uint64_t a) const { return mod64(a); }
};

// Phase factor for pool entry idx.
__device__ __forceinline__ float2 lut_at(const float2 *__restrict__ lut, uint32_t idx)
{
    return __ldg(lut + idx);
}

// The one-entry pool {1 + 0i} standing for N_LUT = 0 (flat phase, R-6).
// (16-byte aligned, two copies: pass A may stage it by a 16-byte bulk copy)
static __device__ __align__(16) const float2 k_flat_lut[2] = {{1.0f, 0.0f}, {1.0f, 0.0f}};

} // namespace holo
