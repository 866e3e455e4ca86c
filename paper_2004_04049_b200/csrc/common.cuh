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
    K_OSPR_RANDOMISE,   // T x LUT for a sub-frame pair, Hermitian pairing (streaming)
    K_OSPR_ROWS_A,      // row IFFT
    K_OSPR_COLS,        // column IFFT + sign quantise + bit pack + column FFT
    K_OSPR_ROWS_C,      // row FFT + |.|^2 accumulate over the chunk's pairs
    K_OSPR_FINALIZE,    // symmetrise/scale + MSE partial sums
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

template <typename... KArgs, typename... Args>
holo_status launch(KernelId id, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t s, Args... args)
{
    if (grid.x == 0 || grid.y == 0 || grid.z == 0)
        return HOLO_OK;
    if (smem > 48 * 1024)
        HOLO_TRY(ensure_smem((const void *)kernel, smem));
    prof_before(id, s);
    kernel<<<grid, block, smem, s>>>(args...);
    cudaError_t e = cudaGetLastError();
    prof_after(id, s);
    count_launch();
    if (e != cudaSuccess)
        return cuda_status(e, kKernelNames[id]);
    return HOLO_OK;
}

// ---- complex helpers ---------------------------------------------------------------
// The FFT arithmetic is written with explicit round-to-nearest intrinsics so that the
// compiler cannot contract it differently in different kernels: every instantiation of a
// transform performs bit-identical arithmetic (the fused GS loop equals chained gs_step
// calls, tests/test_gpu_gs.py).
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y)); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return make_float2(__fmaf_rn(a.x, b.x, -__fmul_rn(a.y, b.y)), __fmaf_rn(a.x, b.y, __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// 1/sqrt(x) for x > 0: hardware estimate + one Newton step (about 1 ulp; a few
// branch-free instructions instead of the IEEE sqrt + divide sequences, whose code
// size per unrolled element overflows the instruction cache).
__device__ __forceinline__ float rsqrt_nr(float x)
{
    const float r = rsqrtf(x);
    return __fmul_rn(r, __fmaf_rn(__fmul_rn(-0.5f, x), __fmul_rn(r, r), 1.5f));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

// ---- cyclic LUT index (step a1) ----------------------------------------------------------
// idx = (rowbase + x) mod L for rowbase < L, x < N, evaluated per pixel without a
// hardware divide: L >= N needs at most one subtraction; a power-of-two L is a mask;
// otherwise Lemire's fastmod (exact for 32-bit operands).
struct LutIndexer {
    uint32_t L;       // N_LUT (> 0)
    uint32_t mode;    // 0: L >= N (single wrap); 1: power of two; 2: general
    uint64_t M;       // ceil(2^64 / L) for mode 2
    __host__ static LutIndexer make(uint32_t L, uint32_t n)
    {
        LutIndexer r;
        r.L = L;
        r.M = (L & (L - 1)) ? UINT64_MAX / L + 1 : 0;   // Lemire constant (non-powers of two)
        if (L >= n)
            r.mode = 0;
        else if ((L & (L - 1)) == 0)
            r.mode = 1;
        else
            r.mode = 2;
        return r;
    }
    __device__ __forceinline__ uint32_t mod(uint32_t a) const
    {
        if (mode == 0)
            return a >= L ? a - L : a;
        if (mode == 1)
            return a & (L - 1);
        return (uint32_t)__umul64hi(M * (uint64_t)a, (uint64_t)L);
    }
    // general a (may exceed 2L): used once per row
    __device__ __forceinline__ uint32_t mod_any(uint64_t a) const { return (uint32_t)(a % L); }
};

// Phase factor for pool entry idx (flat 1+0i when the pool is empty, R-6).
__device__ __forceinline__ float2 lut_at(const float2 *__restrict__ lut, uint32_t idx)
{
    return __ldg(lut + idx);
}

} // namespace holo
