// lut.cu -- step a0: generation of the phase pool ("Random numbers can be
// generated at compile time to fill the LUT").
//
// Entry k = recipe R-5 applied to u_k = high word of SplitMix64 output k (R-3,
// R-4).  The recipe is fixed to the operation (every product and sum is an
// explicit round-to-nearest double intrinsic, so nvcc cannot contract it into
// FMAs) so that the pool is bit-identical to any other implementation of R-5,
// in particular the fp64 CPU oracle (R-5; parity P-1).
#include "phase.cuh"

namespace holo {

// Grid-stride over entries; 64-bit counter (full-length pools exceed 2^24).
__global__ void __launch_bounds__(256) lut_generate_kernel(uint64_t seed, uint64_t n_lut, float2 *lut)
{
    HOLO_PDL_ENTRY();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_lut; k += stride)
        lut[k] = prng_phase(seed, k);
}

// The sin/cos table of the quantised PRNG source (R-25): entry k = R-5 at the angle code
// k << (32 - q), i.e. (cos, sin) of 2 pi k / 2^q, for k < 2^q.
__global__ void __launch_bounds__(256) phase_table_kernel(int q, float2 *tbl)
{
    HOLO_PDL_ENTRY();
    const uint32_t m = 1u << q;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < m; k += gridDim.x * blockDim.x)
        tbl[k] = r5_phase(k << (32 - q));
}

} // namespace holo

using namespace holo;

extern "C" holo_status holo_phase_table(int32_t phase_bits, holo_c64 *table, holo_stream stream)
{
    HOLO_CHECK_ARG(phase_bits >= 1 && phase_bits <= 16, "phase_bits must be in [1, 16], got %d", phase_bits);
    HOLO_CHECK_ARG(table != nullptr, "table is NULL");
    const unsigned m = 1u << phase_bits, grid = (m + 255) / 256;
    return launch(K_LUT_GENERATE, phase_table_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, phase_bits,
                  (float2 *)table);
}

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
