// gs.cu -- Gerchberg-Saxton (Fig. 2 left; steps g0-g6 of
// DESIGN.md §1) as two fused FFT passes per iteration over groups of frames
// (C4: one group of 64 frames, a 512 MiB state streamed from HBM).
//
//   gs_rows_init  g0: R_0 = T * lut[(base_b + p) mod L] (or a given R_{k-1} for the
//                 one-step hook); row IFFT -> state; fp64 sums of T^2, T^4 over Omega.
//   gs_cols       column IFFT -> H_k; g2 constraint (H/|H| or nearest of Q levels);
//                 last iteration writes h / level outputs; column FFT -> state.
//   gs_rows       row FFT -> R'_k (x 1/N); g4: I_k = |R'_k|^2, fp64 partial sums of
//                 I, I^2, d^2, d I (d = a0 I - T^2) over Omega and (|R'_k| - T)^2 over
//                 the plane; g5: R_k = T R'_k/|R'_k|; row IFFT -> state (or R_k / I_k).
//                 The warp finishing a frame's last row item reduces the frame's item
//                 partials in a fixed order -> MSE_k (R-12), E_k (ticket per frame).
//
// The 1/sqrt(N) factors of the inverse transforms are dropped: the constraint
// and the amplitude replacement are invariant to a positive scale.
#include "rows2w.cuh"

namespace holo {

constexpr int kMaxGroup = 64;
constexpr int kGsParts = 5;   // per-item metric partial sums (gs_rows_kernel)

template <int N>
struct GsRowCfg {
    static constexpr bool kWide = fft::Plan<N>::T > 32;   // N = 4096: two warps per row (gs_rows2w_kernel)
    // partial-sum slots per frame and iteration: one per row item, or (4096) one per warp
    static constexpr int NBLK = kWide ? 2 * N : N / RowPipe<N>::GPW;
};


__device__ __forceinline__ void block_reduce_n(double *s, int nvals, double *dst)
{
    __shared__ double red[32][kGsParts];
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

__device__ __forceinline__ bool in_region(int y, int x, const holo_region &om)
{
    return y >= om.row0 && y < om.row1 && x >= om.col0 && x < om.col1;
}

// The normalisations of g2 (H / |H|) and g5 (T R' / |R'|, |R'|).  HOLO_GS_NORM selects the
// reciprocal square root: 0 = the SFU estimate (rel. error < 2^-22; default), 1 = correctly
// rounded (__frsqrt_rn) then RN products, 2 = RN sqrt then RN divisions.  Measured at C4
// (tools/gs_drift.py, profiles/r02_gs_drift.json): the 50-iteration MSE trajectory and the
// one-step error are the same for all three (the fp32 transforms' rounding dominates), while
// 1 and 2 slow the GS passes by 40-50 %, so the default is 0 (R-22).
#ifndef HOLO_GS_NORM
#define HOLO_GS_NORM 0
#endif
__device__ __forceinline__ float2 gs_unit(float2 h, float m2)
{
#if HOLO_GS_NORM == 2
    const float s = __fsqrt_rn(m2);
    return make_float2(__fdiv_rn(h.x, s), __fdiv_rn(h.y, s));
#else
    return f2::mul(h, f2::bc(HOLO_GS_NORM == 0 ? rsqrt_sfu(m2) : rsqrt_rn(m2)));
#endif
}
// |X| and T / |X| for m2 = |X|^2 (both 0 when m2 is below the smallest normal: R-16's zero case).
struct GsAmp {
    float mag, g;
};
__device__ __forceinline__ GsAmp gs_amp(float m2, float tt, bool nz)
{
#if HOLO_GS_NORM == 2
    const float s = nz ? __fsqrt_rn(m2) : 0.0f;
    return GsAmp{s, nz ? __fdiv_rn(tt, s) : 0.0f};
#else
    const float rr = nz ? (HOLO_GS_NORM == 0 ? rsqrt_sfu(m2) : rsqrt_rn(m2)) : 0.0f;
    return GsAmp{__fmul_rn(m2, rr), __fmul_rn(tt, rr)};
#endif
}

// ---- g0: R_0 = T * lut[(base_b + p) mod L] (or a given R_in) -> state; T sums over Omega -----------
// CTAs per frame of the prepare kernel (fixed => deterministic sums; 256 keep small batches at
// HBM speed: 4 frames of 4096^2 took 600 us with 64)
constexpr int kGsTBlocks = 256;

__device__ __forceinline__ uint32_t gs_lut_mod(uint32_t a, const LutIndexer &ix)
{
    return (ix.L & (ix.L - 1)) == 0 ? (a & (ix.L - 1)) : (uint32_t)__umul64hi(ix.M * (uint64_t)a, (uint64_t)ix.L);
}

template <int N>
__global__ void __launch_bounds__(256)
gs_prepare_kernel(const float *__restrict__ T, const float2 *__restrict__ lut, LutIndexer ix, uint32_t off_mod,
                  uint32_t p_mod, uint64_t frame0, const float2 *__restrict__ r_in, holo_region om,
                  float2 *__restrict__ state, double *__restrict__ tparts)
{
    HOLO_PDL_ENTRY();
    constexpr int P = N * N;
    const int fr = blockIdx.y;
    const float *Tf = T + (size_t)fr * P;
    float2 *S = state + (size_t)fr * P;
    uint32_t base = 0;
    if (lut != nullptr)
        base = ix.mod64((uint64_t)off_mod + (uint64_t)ix.mod64(frame0 + fr) * (uint64_t)p_mod);
    double s[2] = {0.0, 0.0};
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
        const float t = __ldg(Tf + p);
        float2 R;
        if (r_in != nullptr) {
            R = r_in[(size_t)fr * P + p];
        } else if (lut != nullptr) {
            const float2 c = __ldg(lut + gs_lut_mod(base + (uint32_t)p, ix));
            R = make_float2(__fmul_rn(t, c.x), __fmul_rn(t, c.y));   // a2, exact fp32 products
        } else {
            R = make_float2(t, 0.0f);
        }
        S[p] = conjf2(R);   // the state is kept conjugated (row passes transform conj(R) forward)
        const int y = p / N, x = p % N;
        if (in_region(y, x, om)) {
            const double td = t, t2 = td * td;
            s[0] += t2;
            s[1] += t2 * t2;
        }
    }
    block_reduce_n(s, 2, tparts + ((size_t)fr * kGsTBlocks + blockIdx.x) * 2);
}

// g0 fused with the first row transform (N <= 2048): items are GPW-row groups, as in the row
// pipeline; each warp builds conj(R_0) of its rows straight into registers (the same products
// as gs_prepare_kernel), row-FFTs them (F{conj(R_0)}, as rows_fft_kernel) and writes the state
// once, and stores its fp64 partial sums of T^2, T^4 over Omega per item (reduced per frame in a
// fixed order by gs_tsum_kernel).  Saves the prepare kernel's state write and the row FFT's read.
template <int N>
__global__ void __launch_bounds__(RowPipe<N>::WPC * 32, N <= 1024 ? 4 : 1)
gs_init_rows_kernel(const float2 *__restrict__ tw, const float *__restrict__ T, const float2 *__restrict__ lut,
                    LutIndexer ix, uint32_t off_mod, uint32_t p_mod, uint64_t frame0,
                    const float2 *__restrict__ r_in, holo_region om, float2 *__restrict__ state,
                    double *__restrict__ tparts, int nitems)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    using RP = RowPipe<N>;
    constexpr int R1 = P::R1, E = P::E, GPW = RP::GPW, NGRP = N / GPW;
    constexpr uint32_t XB = (RP::XCH_BYTES + 127) / 128 * 128;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane / R1, t = lane % R1;
    float2 *sl = reinterpret_cast<float2 *>(smem_raw + (size_t)warp * XB);
    fft::Twiddles<N, false> twr;                         // pool twiddles: four CTAs per SM at N = 1024
    twr.load(tw, t);
    #pragma unroll 1
    for (int item = blockIdx.x * RP::WPC + warp; item < nitems; item += gridDim.x * RP::WPC) {
        const int fr = item / NGRP, grp = item % NGRP, y = grp * GPW + g;
        const size_t rofs = ((size_t)fr * N + y) * N;
        uint32_t base = 0;
        if (lut != nullptr)
            base = ix.mod64((uint64_t)off_mod + (uint64_t)ix.mod64(frame0 + fr) * (uint64_t)p_mod);
        const bool row_in = y >= om.row0 && y < om.row1;
        double s2 = 0.0, s4 = 0.0;
        float2 v[E];
        float tv[E];
        // one branch per source around whole unrolled loops, so that every load of the row is in
        // flight at once (per-element branches serialised the loads: 0.95 ms vs 0.19 ms at C4)
#pragma unroll
        for (int m = 0; m < E; ++m)
            tv[m] = __ldg(T + rofs + t + R1 * m);
        if (r_in != nullptr) {
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = conjf2(r_in[rofs + t + R1 * m]);
        } else if (lut != nullptr) {
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = __ldg(lut + gs_lut_mod(base + (uint32_t)(y * N + t + R1 * m), ix));
#pragma unroll
            for (int m = 0; m < E; ++m)   // a2, exact fp32 products; the state is kept conjugated
                v[m] = make_float2(__fmul_rn(tv[m], v[m].x), -__fmul_rn(tv[m], v[m].y));
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m)
                v[m] = make_float2(tv[m], -0.0f);
        }
        if (row_in) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int x = t + R1 * m;
                if (x >= om.col0 && x < om.col1) {
                    const double td = tv[m], t2 = td * td;
                    s2 += t2;
                    s4 += t2 * t2;
                }
            }
        }
        fft::fft2pass<N, false, 1, true>(v, sl + g * P::SMEM, t, twr);   // F{conj(R_0)}
#pragma unroll
        for (int m = 0; m < E; ++m)
            state[rofs + t + R1 * m] = v[m];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s2 += __shfl_down_sync(0xffffffffu, s2, o);
            s4 += __shfl_down_sync(0xffffffffu, s4, o);
        }
        if (lane == 0) {
            tparts[((size_t)fr * NGRP + grp) * 2] = s2;
            tparts[((size_t)fr * NGRP + grp) * 2 + 1] = s4;
        }
    }
}

// g4 of iteration k for the frames of a launch group (pointers offset to the group).
struct GsMetrics {
    const float *a0;      // [G] prior a0 = sum_Omega T^2 / |Omega| (gs_tsum_kernel)
    const double *tsum;   // [G][2] sum_Omega T^2, T^4
    const double *parts;  // [G][nblk][kGsParts] the row pass's item partial sums
    double *mse, *err_e;  // [G][iters] outputs (nullable)
    int nframes, nblk, iters, k;
    double inv_count;     // 1 / |Omega|
};

// R-12 for frame fr from its item partials, reduced in a fixed order by the whole CTA: a =
// S_T2 / S_I and, about the prior a0 the partials were taken at (d = a0 I - T^2),
//   sum (a I - T^2)^2 = S_dd + 2 (a - a0) S_dI + (a - a0)^2 S_II;   S_I = 0: a = 0, sum = S_T4.
__device__ __forceinline__ void gs_frame_metrics(const GsMetrics &gm, int fr)
{
    const double *pp = gm.parts + (size_t)fr * gm.nblk * kGsParts;
    double s[kGsParts] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < gm.nblk; i += blockDim.x)
#pragma unroll
        for (int j = 0; j < kGsParts; ++j)
            s[j] += pp[(size_t)i * kGsParts + j];
    __shared__ double o[kGsParts];
    block_reduce_n(s, kGsParts, o);
    __syncthreads();
    if (threadIdx.x == 0) {
        const double sT2 = gm.tsum[2 * fr], sT4 = gm.tsum[2 * fr + 1];
        double sum = sT4;
        if (o[0] != 0.0) {
            const double da = sT2 / o[0] - (double)gm.a0[fr];
            sum = o[2] + 2.0 * da * o[3] + da * da * o[1];
        }
        if (gm.mse)
            gm.mse[(size_t)fr * gm.iters + gm.k] = (sum > 0.0 ? sum : 0.0) * gm.inv_count;
        if (gm.err_e)
            gm.err_e[(size_t)fr * gm.iters + gm.k] = o[4];
    }
}

// The last iteration's metrics (earlier ones are reduced in the next column pass's prologue).
__global__ void __launch_bounds__(256)
gs_mse_kernel(const GsMetrics gm)
{
    HOLO_PDL_ENTRY();
    gs_frame_metrics(gm, blockIdx.x);
}

// ---- column pass: IFFT -> constraint -> FFT (TMA-fed pipeline) ----------------------------------
template <int N, bool QUANT>
struct GsColBody {
    static constexpr int kStages = 3;   // measured best column-pipeline variant for this body
    // columns per tile (4 measured 6 % slower for this body); N = 4096: 4, one 133 KB stage
    // (2-column tiles on three stages, two groups: 26 % slower, half-sector row segments)
    static constexpr int kWidth = N >= 4096 ? 4 : 8;
    static constexpr int kGroups = 1;
    static constexpr bool kPrologue = true;
    struct Args {
        const float2 *tw;
        float2 *buf;          // the group's state (updated in place)
        int levels;
        const float2 *qtab;   // Q-entry level table (QUANT only)
        float2 *holo;
        uint8_t *lev;
        GsMetrics pend;       // metrics of the previous row pass to reduce (pend.parts NULL: none)
    };
    // The previous iteration's per-frame metric reductions go to the CTAs that own one tile
    // fewer than the others (ntiles mod grid of them own one more), so they add nothing to the
    // pass's critical path; the reductions overlap the CTAs' first TMA tile loads.
    static __device__ __forceinline__ void prologue(const Args &a, int ntiles)
    {
        if (a.pend.parts == nullptr)
            return;
        const int rem = ntiles % (int)gridDim.x;
        for (int fr = ((int)blockIdx.x + (int)gridDim.x - rem) % (int)gridDim.x; fr < a.pend.nframes;
             fr += (int)gridDim.x)
            gs_frame_metrics(a.pend, fr);
    }
    template <class F, int W>
    static __device__ __forceinline__ void run(float2 (&v)[F::E], float2 *sm, uint32_t *, int c, int t, int fr,
                                               int tile,
                                               const Args &a, const F &fft)
    {
        constexpr int R1 = F::T, E = F::E;   // element m of thread t = row t + R1*m; W columns per tile
        const size_t fofs = (size_t)fr * N * N;
        const int levels = a.levels;
        const float q_over_2pi = (float)levels * 0.15915494309189533577f;
        // IFFT then FFT through ONE transform body (instruction cache): F^-1{x} = conj(F{conj(x)});
        // the state is kept conjugated by the row passes, so the tile already holds conj(x)
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            fft.template run<false, W>(v, sm, t);
            if (h == 1)
                break;
            int jl[QUANT ? E : 1];                             // level indices (QUANT)
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const float2 hk = make_float2(v[r].x, -v[r].y);  // H_k (x N)
                float2 o;
                if constexpr (!QUANT) {
                    const float m2 = __fmaf_rn(hk.x, hk.x, __fmul_rn(hk.y, hk.y));
                    o = m2 < kFltMin ? make_float2(1.0f, 0.0f)               // R-16: H = 0 -> +1
                                     : gs_unit(hk, m2);                      // H / |H|
                } else {
                    float th = atan2f(hk.y, hk.x);
                    if (th < 0.0f)
                        th += 6.28318530717958647692f;
                    int j = (int)floorf(th * q_over_2pi + 0.5f);
                    if (j >= levels)
                        j -= levels;
                    jl[r] = j;
                    o = a.qtab[j];                             // (cos, sin)(2 pi j / Q), built by gs_qtab
                }
                v[r] = o;
            }
            if (a.holo != nullptr || a.lev != nullptr) {       // last iteration only: g6 outputs
                const size_t base = fofs + (size_t)t * N + tile * W + c;
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const size_t idx = base + (size_t)R1 * r * N;
                    if (a.holo != nullptr)
                        a.holo[idx] = v[r];
                    if constexpr (QUANT) {
                        if (a.lev != nullptr)
                            a.lev[idx] = (uint8_t)jl[r];
                    }
                }
            }
        }
        // (the pipeline stores v, the column FFT of h_k, with a TMA tile store)
    }
};

// Level table exp(2 pi i j / Q), j < Q, in double then rounded (R-15).
__global__ void gs_qtab_kernel(int levels, float2 *__restrict__ qtab)
{
    HOLO_PDL_ENTRY();
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < levels; j += gridDim.x * blockDim.x) {
        double sn, cs;
        sincospi(2.0 * (double)j / (double)levels, &sn, &cs);
        qtab[j] = make_float2((float)cs, (float)sn);
    }
}

// ---- row pass: FFT -> metrics -> amplitude replacement -> IFFT (row pipeline) ---------------------
enum GsRowMode : int { GS_FUSED = 0, GS_LAST = 1, GS_STEP = 2 };

// Items are GPW-row groups of the group's frames (NGRP = N / GPW per frame); each item's
// fp64 partial sums (I, I^2, d^2, d I over Omega with d = a0 I - T^2; (|R'| - T)^2 over the
// plane) go to parts[frame][grp] for a fixed-order reduction in the next column pass's
// prologue (GsColBody::prologue), or by gs_mse_kernel after the last iteration.
template <int N, int MODE>
__global__ void __launch_bounds__(RowPipe<N>::WPC * 32)
gs_rows_kernel(const float2 *__restrict__ tw, float2 *state, const float *__restrict__ T, int nitems, holo_region om,
               float *__restrict__ inten, float2 *__restrict__ r_out, const float *__restrict__ a0,
               double *__restrict__ parts, int rev)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    using RP = RowPipe<N>;
    constexpr int R1 = P::R1, E = P::E, GPW = RP::GPW, NGRP = N / GPW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const WarpRing ring = make_ring<RP::SLOT_C, RP::WPC>(smem_raw);
    const int lane = threadIdx.x & 31, g = lane / R1, t = lane % R1;
    const int stride = gridDim.x * RP::WPC;
    int item = blockIdx.x * RP::WPC + (threadIdx.x >> 5);
    if (lane == 0 && item < nitems) {
        tma::mbar_arrive_expect_tx(&ring.bars[0], RP::IN_BYTES);
        tma::load_1d(ring.slot(0), state + (size_t)(rev ? nitems - 1 - item : item) * GPW * N, RP::IN_BYTES,
                     &ring.bars[0]);
    }
    fft::Twiddles<N, false> twr;                          // pool twiddles (register budget)
    twr.load(tw, t);
    constexpr float inv_n = 1.0f / (float)N;                 // exact power of two
    static_assert(E <= 64, "one column-mask bit per element");
    uint64_t colmask = 0;                                     // bit r: column t + R1 r lies in Omega
#pragma unroll
    for (int r = 0; r < E; ++r)
        colmask |= (uint64_t)(t + R1 * r >= om.col0 && t + R1 * r < om.col1) << r;
    #pragma unroll 1   // one copy of the transform code (instruction cache)
    for (int k = 0; item < nitems; item += stride, ++k) {
        const int s = k & 1;
        const int nxt = item + stride;
        if (lane == 0 && nxt < nitems) {
            tma::mbar_arrive_expect_tx(&ring.bars[s ^ 1], RP::IN_BYTES);
            tma::load_1d(ring.slot(s ^ 1), state + (size_t)(rev ? nitems - 1 - nxt : nxt) * GPW * N, RP::IN_BYTES,
                         &ring.bars[s ^ 1]);
        }
        // rev: items in reverse order (the frames the column pass wrote last, still in L2, first)
        const int pit = rev ? nitems - 1 - item : item;
        const int fr = pit / NGRP, grp = pit % NGRP;
        const int y = grp * GPW + g;
        const size_t rofs = ((size_t)fr * N + y) * N;
        tma::mbar_wait(&ring.bars[s], (uint32_t)((k >> 1) & 1));
        float2 *sl = reinterpret_cast<float2 *>(ring.slot(s));
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = sl[g * N + t + R1 * m];
        // forward FFT, then (FUSED) the inverse through the same transform body:
        // F^-1{x} = conj(F{conj(x)}) exactly (instruction cache: one copy of the FFT code)
#pragma unroll 1
        for (int h = 0; h < (MODE == GS_FUSED ? 2 : 1); ++h) {
            float tv[E];
            if (h == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    tv[r] = __ldg(T + rofs + t + R1 * r);       // in flight during the FFT
            }
            // h = 0: X = N R'_k;  h = 1: F{conj(R_k)} = N conj(F^-1{R_k}), stored as is (the state
            // is kept conjugated; the column pass then needs no input negation)
            fft::fft2pass<N, false, 1, true>(v, sl + g * P::SMEM, t, twr);
            if (h == 1) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    state[rofs + t + R1 * r] = v[r];
                break;
            }
            // g4 metrics.  R-12 needs sum (a I - T^2)^2 with a = sum T^2 / sum I, known only after
            // the pass; it is accumulated about the frame's prior a0 = sum_Omega T^2 / |Omega| (for
            // the full plane this IS a, by Parseval: sum I = sum |h|^2 = N^2) as
            //   sum (a I - T^2)^2 = S_dd + 2 (a - a0) S_dI + (a - a0)^2 S_II,  d = a0 I - T^2,
            // so no large terms cancel (gs_frame_metrics).  fp32 partial sums over this thread's E
            // elements (all terms of S_dd, S_II positive), then fp64 across lanes, rows, frames.
            // The sums run on m2 = |X|^2 = N^2 I (I = m2 / N^2 is an exact power-of-two scaling, so
            // sum m2 / N^2 is bit-identical to sum I); the scales are applied in fp64 afterwards.
            float fe = 0.0f, sI = 0.0f, sII = 0.0f, sDD = 0.0f, sDI = 0.0f;
            const float a0n = __fmul_rn(a0[fr], inv_n * inv_n);       // a0 / N^2 (exact)
            const uint64_t in_om = (y >= om.row0 && y < om.row1) ? colmask : 0u;   // bit r: x in Omega
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int x = t + R1 * r;
                const float2 X = v[r];
                // explicit rounding: identical arithmetic in every instantiation (fused == step)
                const float m2 = __fmaf_rn(X.x, X.x, __fmul_rn(X.y, X.y));
                const bool nz = m2 >= kFltMin;
                const float tt = tv[r];
                const GsAmp ga = gs_amp(m2, tt, nz);
                const float d = __fmaf_rn(ga.mag, inv_n, -tt);              // |R'_k| - T
                fe = __fmaf_rn(d, d, fe);
                if ((in_om >> r) & 1u) {
                    const float dd = __fmaf_rn(a0n, m2, -__fmul_rn(tt, tt));   // a0 I - T^2
                    sI = __fadd_rn(sI, m2);
                    sII = __fmaf_rn(m2, m2, sII);
                    sDD = __fmaf_rn(dd, dd, sDD);
                    sDI = __fmaf_rn(dd, m2, sDI);
                }
                if (MODE == GS_LAST || MODE == GS_STEP) {
                    if (inten != nullptr)
                        inten[rofs + x] = __fmul_rn(m2, inv_n * inv_n);
                }
                if (MODE != GS_LAST)   // conj(R_k), R_k = T X / |X| (R-16: |R'| = 0 -> T)
                    v[r] = nz ? f2::mul(conjf2(X), f2::bc(ga.g)) : make_float2(tt, -0.0f);
            }
            constexpr double i2 = 1.0 / ((double)N * N), i4 = i2 * i2;   // exact
            double sums[kGsParts] = {(double)sI * i2, (double)sII * i4, (double)sDD, (double)sDI * i2, (double)fe};
            // warp reduction of the item's sums (lanes of all GPW rows of the item)
#pragma unroll
            for (int i = 0; i < kGsParts; ++i) {
                double x = sums[i];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    x += __shfl_down_sync(0xffffffffu, x, o);
                sums[i] = x;
            }
            if (lane == 0) {
                double *dst = parts + ((size_t)fr * NGRP + grp) * kGsParts;
#pragma unroll
                for (int i = 0; i < kGsParts; ++i)
                    dst[i] = sums[i];
            }
            if (MODE == GS_STEP) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    r_out[rofs + t + R1 * r] = conjf2(v[r]);   // R_k itself
            }
        }
        tma::fence_proxy_async_smem();
        __syncwarp();
    }
}

// Row pass for N = 4096 (R-26): a two-warp group per row (item = row, frame-major), rows read and
// written straight from the state (coalesced).  Same arithmetic per element as gs_rows_kernel;
// each warp's fp64 partial sums go to its own slot parts[frame][2 y + warp] (NBLK = 2 N).
template <int N, int MODE>
__global__ void __launch_bounds__(Row2W<N>::THREADS, 1)
gs_rows2w_kernel(const float2 *__restrict__ tw, float2 *state, const float *__restrict__ T, int nrows, holo_region om,
                 float *__restrict__ inten, float2 *__restrict__ r_out, const float *__restrict__ a0,
                 double *__restrict__ parts, int rev)
{
    HOLO_PDL_ENTRY();
    using P = fft::Plan<N>;
    constexpr int R1 = P::R1, E = P::E, NBLK = GsRowCfg<N>::NBLK;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const Row2WThread rt = row2w_thread();
    float2 *sm = reinterpret_cast<float2 *>(smem_raw) + (size_t)rt.grp * P::SMEM;
    const int t = rt.t, lane = threadIdx.x & 31, wig = t >> 5;   // warp within the row group
    constexpr float inv_n = 1.0f / (float)N;
    static_assert(E <= 64, "one column-mask bit per element");
    uint64_t colmask = 0;
#pragma unroll
    for (int r = 0; r < E; ++r)
        colmask |= (uint64_t)(t + R1 * r >= om.col0 && t + R1 * r < om.col1) << r;
    #pragma unroll 1
    for (int item = blockIdx.x * 2 + rt.grp; item < nrows; item += gridDim.x * 2) {
        const int pit = rev ? nrows - 1 - item : item;
        const int fr = pit / N, y = pit % N;
        const size_t rofs = ((size_t)fr * N + y) * N;
        float2 v[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            v[m] = state[rofs + t + R1 * m];
        #pragma unroll 1
        for (int h = 0; h < (MODE == GS_FUSED ? 2 : 1); ++h) {
            float tv[E];
            if (h == 0) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    tv[r] = __ldg(T + rofs + t + R1 * r);
            }
            row2w_fft<N>(v, sm, tw, rt);
            if (h == 1) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    state[rofs + t + R1 * r] = v[r];
                break;
            }
            float fe = 0.0f, sI = 0.0f, sII = 0.0f, sDD = 0.0f, sDI = 0.0f;
            const float a0n = __fmul_rn(a0[fr], inv_n * inv_n);
            const uint64_t in_om = (y >= om.row0 && y < om.row1) ? colmask : 0u;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const int x = t + R1 * r;
                const float2 X = v[r];
                const float m2 = __fmaf_rn(X.x, X.x, __fmul_rn(X.y, X.y));
                const bool nz = m2 >= kFltMin;
                const float tt = tv[r];
                const GsAmp ga = gs_amp(m2, tt, nz);
                const float d = __fmaf_rn(ga.mag, inv_n, -tt);
                fe = __fmaf_rn(d, d, fe);
                if ((in_om >> r) & 1u) {
                    const float dd = __fmaf_rn(a0n, m2, -__fmul_rn(tt, tt));
                    sI = __fadd_rn(sI, m2);
                    sII = __fmaf_rn(m2, m2, sII);
                    sDD = __fmaf_rn(dd, dd, sDD);
                    sDI = __fmaf_rn(dd, m2, sDI);
                }
                if (MODE == GS_LAST || MODE == GS_STEP) {
                    if (inten != nullptr)
                        inten[rofs + x] = __fmul_rn(m2, inv_n * inv_n);
                }
                if (MODE != GS_LAST)
                    v[r] = nz ? f2::mul(conjf2(X), f2::bc(ga.g)) : make_float2(tt, -0.0f);
            }
            constexpr double i2 = 1.0 / ((double)N * N), i4 = i2 * i2;
            double sums[kGsParts] = {(double)sI * i2, (double)sII * i4, (double)sDD, (double)sDI * i2, (double)fe};
#pragma unroll
            for (int i = 0; i < kGsParts; ++i) {
                double x = sums[i];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    x += __shfl_down_sync(0xffffffffu, x, o);
                sums[i] = x;
            }
            if (lane == 0) {
                double *dst = parts + ((size_t)fr * NBLK + 2 * y + wig) * kGsParts;
#pragma unroll
                for (int i = 0; i < kGsParts; ++i)
                    dst[i] = sums[i];
            }
            if (MODE == GS_STEP) {
#pragma unroll
                for (int r = 0; r < E; ++r)
                    r_out[rofs + t + R1 * r] = conjf2(v[r]);
            }
        }
    }
}

// One CTA per frame of a launch group: fixed-order sum of the prepare kernel's T partials ->
// tsum[frame] = (sum T^2, sum T^4) over Omega and the prior a0 = sum T^2 / |Omega| that the
// row pass takes its metric partials about (exactly R-12's a for the full plane, by Parseval).
__global__ void __launch_bounds__(256)
gs_tsum_kernel(const double *__restrict__ tparts, int nparts, double inv_count, double *__restrict__ tsum,
               float *__restrict__ a0)
{
    HOLO_PDL_ENTRY();
    const int fr = blockIdx.x;
    double u[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {   // fixed order
        const double *q = tparts + ((size_t)fr * nparts + i) * 2;
        u[0] += q[0];
        u[1] += q[1];
    }
    __shared__ double o[2];
    block_reduce_n(u, 2, o);
    __syncthreads();
    if (threadIdx.x == 0) {
        tsum[2 * fr] = o[0];
        tsum[2 * fr + 1] = o[1];
        a0[fr] = (float)(o[0] * inv_count);
    }
}

// ---- host orchestration --------------------------------------------------------------------------
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

static int gs_group(int n, int batch)
{
    const size_t frame = (size_t)n * n * sizeof(float2);
    size_t budget = 512ull << 20;  // frames per launch group (measured: larger groups amortise pass tails)
    if (const char *e = getenv("HOLO_GS_GROUP_BYTES"))
        budget = strtoull(e, nullptr, 10);
    long g = (long)(budget / frame);
    if (g < 1)
        g = 1;
    if (g > kMaxGroup)
        g = kMaxGroup;
    if (g > batch)
        g = batch;
    return (int)g;
}

static int gs_nblk(int n)
{
    switch (n) {
    case 16: return GsRowCfg<16>::NBLK;
    case 32: return GsRowCfg<32>::NBLK;
    case 64: return GsRowCfg<64>::NBLK;
    case 128: return GsRowCfg<128>::NBLK;
    case 256: return GsRowCfg<256>::NBLK;
    case 512: return GsRowCfg<512>::NBLK;
    case 1024: return GsRowCfg<1024>::NBLK;
    case 2048: return GsRowCfg<2048>::NBLK;
    default: return GsRowCfg<4096>::NBLK;
    }
}

struct GsWs {
    float2 *qtab;
    float2 *state;
    double *parts;    // [G][NBLK][kGsParts] row-pass item partials of the current iteration
    double *tparts;   // [G][max(kGsTBlocks, N)][2] init partials of sum T^2, T^4 (per CTA or per row item)
    double *tsum;     // [G][2]
    float *a0;        // [G]
};

static size_t gs_ws_layout(int n, int batch, char *base, GsWs *w)
{
    const size_t P = (size_t)n * n;
    const int G = gs_group(n, batch), nblk = gs_nblk(n);
    size_t off = 0;
    const size_t o_qtab = off;
    off = al256(off + 65536 * sizeof(float2));
    const size_t o_state = off;
    off = al256(off + (size_t)G * P * sizeof(float2));
    const size_t o_parts = off;
    off = al256(off + (size_t)G * nblk * kGsParts * sizeof(double));
    const size_t o_tparts = off;
    off = al256(off + (size_t)G * (n > kGsTBlocks ? n : kGsTBlocks) * 2 * sizeof(double));
    const size_t o_tsum = off;
    off = al256(off + (size_t)G * 2 * sizeof(double));
    const size_t o_a0 = off;
    off = al256(off + (size_t)G * sizeof(float));

    if (w) {
        w->qtab = (float2 *)(base + o_qtab);
        w->state = (float2 *)(base + o_state);
        w->parts = (double *)(base + o_parts);
        w->tparts = (double *)(base + o_tparts);
        w->tsum = (double *)(base + o_tsum);
        w->a0 = (float *)(base + o_a0);
    }
    return off;
}

holo_status check_n(int n);
holo_status check_region(holo_region om, int n);


// Runs `iters` iterations for all frames (gs_generate, r_in == NULL) or one step
// from r_in (gs_step, iters == 1, r_out != NULL).
template <int N>
static holo_status gs_run(const float2 *tw, const float *target, int batch, int iters, const float2 *lut, uint64_t n_lut,
                          uint64_t phase_offset, int levels, const float2 *r_in, float2 *r_out, float2 *holo,
                          uint8_t *holo_levels, float *intensity, double *mse, double *err_e, holo_region om,
                          void *ws, cudaStream_t s)
{
    constexpr size_t P = (size_t)N * N;
    GsWs w;
    gs_ws_layout(N, batch, (char *)ws, &w);
    const int G = gs_group(N, batch);
    const LutIndexer ix = LutIndexer::make(n_lut ? (uint32_t)n_lut : 1u, N);
    const uint32_t off_mod = n_lut ? (uint32_t)(phase_offset % n_lut) : 0u;
    const uint32_t p_mod = n_lut ? (uint32_t)(P % n_lut) : 0u;
    const double inv_cnt = 1.0 / ((double)(om.row1 - om.row0) * (double)(om.col1 - om.col0));
    if (levels > 0)
        HOLO_TRY(launch(K_GS_COLS, gs_qtab_kernel, dim3((levels + 255) / 256), dim3(256), 0, s, levels, w.qtab));
    for (int g0 = 0; g0 < batch; g0 += G) {
        const int ng = (batch - g0) < G ? (batch - g0) : G;
        if constexpr (!GsRowCfg<N>::kWide) {   // g0 fused with the first row FFT
            using RP = RowPipe<N>;
            constexpr size_t smem = (size_t)RP::WPC * ((RP::XCH_BYTES + 127) / 128 * 128);
            const int nitems = ng * (N / RP::GPW);
            const int grid = pipe_grid(gs_init_rows_kernel<N>, RP::WPC * 32, smem, nitems, RP::WPC);
            HOLO_TRY(launch(K_GS_ROWS_INIT, gs_init_rows_kernel<N>, dim3(grid), dim3(RP::WPC * 32), smem, s, tw,
                            target + g0 * P, lut, ix, off_mod, p_mod, (uint64_t)g0,
                            r_in ? r_in + g0 * P : (const float2 *)nullptr, om, w.state, w.tparts, nitems));
            HOLO_TRY(launch(K_MSE_REDUCE, gs_tsum_kernel, dim3(ng), dim3(256), 0, s, (const double *)w.tparts,
                            N / RP::GPW, inv_cnt, w.tsum, w.a0));
        } else {
            HOLO_TRY(launch(K_GS_ROWS_INIT, gs_prepare_kernel<N>, dim3(kGsTBlocks, ng), dim3(256), 0, s,
                            target + g0 * P, lut, ix, off_mod, p_mod, (uint64_t)g0,
                            r_in ? r_in + g0 * P : (const float2 *)nullptr, om, w.state,
                            w.tparts));
            HOLO_TRY(launch(K_MSE_REDUCE, gs_tsum_kernel, dim3(ng), dim3(256), 0, s, (const double *)w.tparts,
                            kGsTBlocks, inv_cnt, w.tsum, w.a0));
            HOLO_TRY((launch_row_fft<N, false>(K_GS_ROWS_INIT, tw, w.state, w.state, ng * N, s)));   // F{conj(R_0)}
        }
        using RP = RowPipe<N>;
        const float *Tg = target + g0 * P;
        GsMetrics gm{w.a0, w.tsum, w.parts, mse ? mse + (size_t)g0 * iters : (double *)nullptr,
                     err_e ? err_e + (size_t)g0 * iters : (double *)nullptr, ng, GsRowCfg<N>::NBLK, iters, 0, inv_cnt};
        const bool metrics = mse != nullptr || err_e != nullptr;
        // the row pass takes its items in reverse order and the column pass in forward order, so
        // each pass starts on the frames the previous one wrote last, still in L2 (measured at C4:
        // 127.5 k -> 130 k frame-iterations/s)
        constexpr int rev_rows = 1;
        for (int k = 0; k < iters; ++k) {
            const bool last = (k == iters - 1);
            GsMetrics pend = gm;              // iteration k-1's partials, reduced in this pass's prologue
            pend.k = k - 1;
            if (k == 0 || !metrics)
                pend.parts = nullptr;
            if (levels == 0) {
                typename GsColBody<N, false>::Args ca{tw, w.state, 0, nullptr,
                                                      (last && holo) ? holo + g0 * P : (float2 *)nullptr, nullptr, pend};
                HOLO_TRY((launch_cols<N, GsColBody<N, false>>(K_GS_COLS, w.state, ng, ca, s)));
            } else {
                typename GsColBody<N, true>::Args ca{tw, w.state, levels, w.qtab,
                                                     (last && holo) ? holo + g0 * P : (float2 *)nullptr,
                                                     (last && holo_levels) ? holo_levels + g0 * P : (uint8_t *)nullptr,
                                                     pend};
                HOLO_TRY((launch_cols<N, GsColBody<N, true>>(K_GS_COLS, w.state, ng, ca, s)));
            }
            float *ig = intensity ? intensity + g0 * P : (float *)nullptr;
            const float *a0 = w.a0;
            if constexpr (GsRowCfg<N>::kWide) {
                using R = Row2W<N>;
                const int nrows = ng * N;
                auto kern = r_out != nullptr ? gs_rows2w_kernel<N, GS_STEP>
                          : last             ? gs_rows2w_kernel<N, GS_LAST>
                                             : gs_rows2w_kernel<N, GS_FUSED>;
                const int grid = pipe_grid(kern, R::THREADS, R::SMEM, (nrows + 1) / 2, 1);
                HOLO_TRY(launch(K_GS_ROWS, kern, dim3(grid), dim3(R::THREADS), R::SMEM, s, tw, w.state, Tg, nrows, om,
                                (r_out != nullptr || last) ? ig : (float *)nullptr,
                                r_out ? r_out + g0 * P : (float2 *)nullptr, a0, w.parts, rev_rows));
                continue;
            } else {
            constexpr size_t smem = ring_smem<RP::SLOT_C, RP::WPC>();
            const int nitems = ng * GsRowCfg<N>::NBLK;
            if (r_out != nullptr) {
                const int grid = pipe_grid(gs_rows_kernel<N, GS_STEP>, RP::WPC * 32, smem, nitems, RP::WPC);
                HOLO_TRY(launch(K_GS_ROWS, gs_rows_kernel<N, GS_STEP>, dim3(grid), dim3(RP::WPC * 32), smem, s, tw,
                                w.state, Tg, nitems, om, ig, r_out + g0 * P, a0, w.parts, rev_rows));
            } else if (last) {
                const int grid = pipe_grid(gs_rows_kernel<N, GS_LAST>, RP::WPC * 32, smem, nitems, RP::WPC);
                HOLO_TRY(launch(K_GS_ROWS, gs_rows_kernel<N, GS_LAST>, dim3(grid), dim3(RP::WPC * 32), smem, s, tw,
                                w.state, Tg, nitems, om, ig, (float2 *)nullptr, a0, w.parts, rev_rows));
            } else {
                const int grid = pipe_grid(gs_rows_kernel<N, GS_FUSED>, RP::WPC * 32, smem, nitems, RP::WPC);
                HOLO_TRY(launch(K_GS_ROWS, gs_rows_kernel<N, GS_FUSED>, dim3(grid), dim3(RP::WPC * 32), smem, s, tw,
                                w.state, Tg, nitems, om, (float *)nullptr, (float2 *)nullptr, a0, w.parts,
                                rev_rows));
            }
            }
        }
        if (metrics) {
            gm.k = iters - 1;
            HOLO_TRY(launch(K_MSE_REDUCE, gs_mse_kernel, dim3(ng), dim3(256), 0, s, (const GsMetrics)gm));
        }
    }
    return HOLO_OK;
}

static holo_status gs_dispatch(const float2 *tw, int n, const float *target, int batch, int iters, const float2 *lut, uint64_t n_lut,
                               uint64_t off, int levels, const float2 *r_in, float2 *r_out, float2 *holo,
                               uint8_t *lev, float *inten, double *mse, double *err_e, holo_region om, void *ws,
                               cudaStream_t s)
{
#define HOLO_GS_CASE(NN)                                                                                  \
    case NN:                                                                                              \
        return gs_run<NN>(tw, target, batch, iters, lut, n_lut, off, levels, r_in, r_out, holo, lev, inten,   \
                          mse, err_e, om, ws, s);
    switch (n) {
        HOLO_GS_CASE(16)
        HOLO_GS_CASE(32)
        HOLO_GS_CASE(64)
        HOLO_GS_CASE(128)
        HOLO_GS_CASE(256)
        HOLO_GS_CASE(512)
        HOLO_GS_CASE(1024)
        HOLO_GS_CASE(2048)
        HOLO_GS_CASE(4096)
    default:
        return set_error(HOLO_ERR_UNSUPPORTED, "n = %d", n);
    }
#undef HOLO_GS_CASE
}

} // namespace holo

using namespace holo;

extern "C" size_t holo_gs_workspace_size(int32_t n, int32_t batch, int32_t iters)
{
    if (check_n(n) != HOLO_OK || batch < 1 || iters < 1)
        return 0;
    (void)iters;
    return gs_ws_layout(n, batch, nullptr, nullptr);
}

static holo_status gs_check_common(const float *target, int32_t n, int32_t batch, int32_t levels, holo_region om,
                                   uint8_t *holo_levels)
{
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(target != nullptr, "target is NULL");
    HOLO_CHECK_ARG(batch >= 1, "batch must be >= 1");
    if (levels < 0 || levels == 1 || levels > 65535)
        return set_error(HOLO_ERR_UNSUPPORTED, "levels must be 0 or in [2, 65535], got %d", levels);
    HOLO_CHECK_ARG(holo_levels == nullptr || (levels >= 2 && levels <= 256),
                   "holo_levels needs 2 <= levels <= 256");
    HOLO_TRY(check_region(om, n));
    return HOLO_OK;
}

extern "C" int32_t holo_gs_group_frames(int32_t n, int32_t batch)
{
    if (check_n(n) != HOLO_OK || batch < 1)
        return 0;
    return gs_group(n, batch);
}

extern "C" holo_status holo_gs_generate(const float *target, int32_t n, int32_t batch, int32_t iters,
                                        const holo_c64 *lut, uint64_t n_lut, uint64_t phase_offset, int32_t levels,
                                        holo_c64 *holo, uint8_t *holo_levels, float *intensity, double *mse,
                                        double *err_e, holo_region omega, void *ws, size_t ws_bytes,
                                        holo_stream stream)
{
    HOLO_TRY(gs_check_common(target, n, batch, levels, omega, holo_levels));
    HOLO_CHECK_ARG(iters >= 1, "iters must be >= 1");
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    HOLO_CHECK_ARG((lut == nullptr) == (n_lut == 0), "lut must be NULL iff n_lut == 0");
    HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
    const size_t need = holo_gs_workspace_size(n, batch, iters);
    if (ws_bytes < need)
        return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    const float2 *tw = nullptr;
    HOLO_TRY(fft::twiddles(&tw));
    return gs_dispatch(tw, n, target, batch, iters, (const float2 *)lut, n_lut, phase_offset, levels, nullptr, nullptr,
                       (float2 *)holo, holo_levels, intensity, mse, err_e, omega, ws, (cudaStream_t)stream);
}

extern "C" holo_status holo_gs_step(const holo_c64 *r_in, const float *target, int32_t n, int32_t batch,
                                    int32_t levels, holo_c64 *r_out, holo_c64 *holo, uint8_t *holo_levels,
                                    float *intensity, double *mse, double *err_e, holo_region omega, void *ws,
                                    size_t ws_bytes, holo_stream stream)
{
    HOLO_TRY(gs_check_common(target, n, batch, levels, omega, holo_levels));
    HOLO_CHECK_ARG(r_in != nullptr && r_out != nullptr, "r_in and r_out are required");
    HOLO_CHECK_ARG((const void *)r_in != (const void *)r_out, "r_in and r_out must not alias");
    HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
    const size_t need = holo_gs_workspace_size(n, batch, 1);
    if (ws_bytes < need)
        return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    const float2 *tw = nullptr;
    HOLO_TRY(fft::twiddles(&tw));
    return gs_dispatch(tw, n, target, batch, 1, nullptr, 0, 0, levels, (const float2 *)r_in, (float2 *)r_out,
                       (float2 *)holo, holo_levels, intensity, mse, err_e, omega, ws, (cudaStream_t)stream);
}
