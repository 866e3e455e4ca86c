/*
 * holo.h -- C ABI of libholo, the B200 (sm_100a) hot path of arXiv 2004.04049,
 * "Lookup tables for phase randomisation in Gerchberg-Saxton and One-Step
 * Phase-Retrieval holography".
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * the CPU-program spec written from it; "R-k" = reading k in
 * DESIGN.md §3, which fixes what the paper leaves open.
 *
 * Conventions for every call
 *  - All array arguments are DEVICE pointers into memory the caller
 *    allocated and owns (in practice torch tensors).  The library never
 *    allocates, frees or retains caller memory.  Its only own state is a
 *    32 KB FFT twiddle table per device (allocated on the first call on that
 *    device, which therefore must not run under CUDA-graph stream capture),
 *    launch counters and optional profiling events.
 *  - Every call is asynchronous on `stream` (NULL = the legacy default
 *    stream): argument checks happen on the host before anything is
 *    enqueued; results are valid once the stream has completed.
 *  - Calls are thread-safe across distinct workspaces and streams.  Two
 *    calls sharing a workspace must be ordered by the caller.
 *  - Kernels are launched with programmatic stream serialisation (PDL): a
 *    kernel may be scheduled while its predecessor in the stream drains, but
 *    waits for it to complete before touching memory, so stream order is
 *    kept exactly (HOLO_PDL=0 in the environment launches them plainly).
 *    Every call may be captured into a CUDA graph after a first eager call
 *    on the device.
 *  - Images are row-major data[y][x], x fastest (R-10); complex values are
 *    interleaved (re, im) fp32 pairs (`holo_c64`); DC is at [0][0] with no
 *    shift (R-10); the DFT pair is unitary, 1/sqrt(Nx*Ny) in both
 *    directions (Eqs. (1)-(2); R-9).
 *  - N (`n`) must be a power of two in [16, 4096] (square frames); other
 *    sizes return HOLO_ERR_INVALID_ARG.
 *  - On any status other than HOLO_OK nothing has been enqueued except for
 *    HOLO_ERR_CUDA, which reports a launch failure (some work may have been
 *    enqueued before it); holo_last_error() then returns a message for
 *    the calling thread.  No C++ exception crosses this boundary.
 */
#ifndef HOLO_H
#define HOLO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HOLO_OK = 0,
    HOLO_ERR_INVALID_ARG = 1, /* size, pointer or range argument out of contract   */
    HOLO_ERR_UNSUPPORTED = 2, /* valid request this build does not implement        */
    HOLO_ERR_WORKSPACE = 3,   /* ws_bytes smaller than the matching *_workspace_size */
    HOLO_ERR_CUDA = 4         /* CUDA runtime error (message from cudaGetErrorString) */
} holo_status;

/* complex64: one pixel of a complex field (H, R, R' of P:45) or one LUT entry. */
typedef struct {
    float re, im;
} holo_c64;

/* The CUDA stream type (identical to cudaStream_t); NULL = legacy default stream. */
typedef struct CUstream_st *holo_stream;

/* Half-open region [row0,row1) x [col0,col1) of the replay plane over which
 * the error is measured (R-13: OSPR uses rows [1, N/2) x all columns, the
 * "top portion of the replay field" of P:158 without the self-conjugate rows;
 * GS uses the full plane).  Must be non-empty and inside [0,N)^2. */
typedef struct {
    int32_t row0, row1, col0, col1;
} holo_region;

/* Message for the calling thread's last non-OK status ("" if none). */
const char *holo_last_error(void);

/* Library version string, e.g. "holo 0.1.0 sm_100a". */
const char *holo_version(void);

/* ------------------------------------------------------------------------
 * a0 -- the phase pool.  P:68: "Random numbers can be generated at compile
 * time to fill the LUT which then acts as a pool of random numbers for
 * algorithms to sequentially draw from."
 *
 * lut[k] = (cos phi_k, sin phi_k), phi_k = 2*pi*u_k/2^32, u_k = the high 32
 * bits of output k of SplitMix64 seeded with `seed` (R-3, R-4), evaluated by
 * the fixed fp64 recipe R-5 and rounded to fp32 (-0 stored as +0).  Entry k
 * depends only on (seed, k), so LUT(seed, L1) is a prefix of LUT(seed, L2).
 *   seed    generator seed
 *   n_lut   number of entries, 1 <= n_lut < 2^31 (0 is INVALID_ARG: the
 *           N_LUT = 0 "flat" case of P:139 needs no table, see n_lut below)
 *   lut     [n_lut] holo_c64, device, written
 * ------------------------------------------------------------------------ */
holo_status holo_lut_generate(uint64_t seed, uint64_t n_lut, holo_c64 *lut, holo_stream stream);

/* ------------------------------------------------------------------------
 * OSPR -- One-Step Phase-Retrieval (Fig. 2 right).
 * For frame f in [0, n_frames) and sub-frame s in [sf_begin, sf_end):
 *   a1  draw index of pixel p = y*N + x:
 *         g = phase_offset + (f*n_sub + s)*N^2 + p,   phase = lut[g mod n_lut]
 *       ("cycled through sequentially with successive frames and
 *       sub-frames continuing from where the previous left off"; R-1, R-2);
 *       n_lut = 0 means the flat phase 1+0i (R-6, "N_LUT is 0");
 *   a2  R_s = T_f * phase                      ("adding random phase")
 *   a3  H_s = F^-1{R_s}                        (Eq. (2))
 *   a4  H'_s = +1 if Re H_s >= 0 else -1       ("nearest acceptable
 *       value" on a binary {0, pi} SLM; tie and -0.0 -> +1, R-7)
 *   a5  R'_s = F{H'_s}                         (Eq. (1))
 *   a6  sum over s of |R'_s|^2                 ("time averaging")
 *   a7  MSE (R-12): a = sum_Omega T^2 / sum_Omega I;
 *       mse = mean_Omega (a I - T^2)^2  (sum_Omega I = 0 -> a = 0).
 * Sub-frames are processed two at a time through one complex FFT
 * ("Hermitian pairing"); an odd count leaves one unpaired.
 *
 *   target      [n_frames][n][n] fp32 amplitude T, values in [0, 1] (R-11)
 *   n           N, power of two in [16, 4096]
 *   n_frames    >= 1
 *   n_sub       N_SF, sub-frames per frame, >= 1
 *   lut         [n_lut] holo_c64 (NULL iff n_lut == 0)
 *   n_lut       N_LUT, 0 <= n_lut < 2^31
 *   phase_offset  global draw index of pixel 0 of frame 0 sub-frame 0
 *   sf_begin, sf_end  this call's shard of the sub-frames,
 *               0 <= sf_begin < sf_end <= n_sub (multi-GPU: each rank passes
 *               its own range; draw indices stay global)
 *   holo_bits   [n_frames][sf_end-sf_begin][n][n/8] packed H', row-major,
 *               MSB-first, +1 -> 1 (R-8); NULL = not written
 *   intensity   [n_frames][n][n] fp32: the mean replay intensity
 *               (1/n_sub) sum_s |R'_s|^2 if the range is all of [0, n_sub),
 *               otherwise the partial SUM over the shard (finish with
 *               holo_ospr_finalize after the cross-rank reduction)
 *   mse         [n_frames] fp64, NULL = not computed; must be NULL for a
 *               partial range (MSE is nonlinear in I)
 *   omega       error region
 *   ws, ws_bytes  device workspace of at least holo_ospr_workspace_size(...)
 * ------------------------------------------------------------------------ */
size_t holo_ospr_workspace_size(int32_t n, int32_t n_frames, int32_t n_sub);

/* Plan query (instrumentation): the number of sub-frame pairs each chunk of
 * holo_ospr_generate(n, ..., n_sub, ...) transforms per pass (DESIGN.md §5:
 * at most 64 pairs within a 1 GiB pair-buffer budget, which
 * HOLO_OSPR_CHUNK_BYTES overrides); 0 for invalid n or n_sub. */
int32_t holo_ospr_chunk_pairs(int32_t n, int32_t n_sub);

holo_status holo_ospr_generate(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                               const holo_c64 *lut, uint64_t n_lut, uint64_t phase_offset,
                               int32_t sf_begin, int32_t sf_end, uint8_t *holo_bits,
                               float *intensity, double *mse, holo_region omega, void *ws,
                               size_t ws_bytes, holo_stream stream);

/* OSPR with the phases drawn on the fly instead of read from a pool (SURVEY.md
 * §8(f) f2; the paper's memory-vs-compute trade-off):
 * the phase of global draw index g = phase_offset + (f*n_sub + s)*n^2 + p is
 * recipe R-5 of the high word of SplitMix64(seed, g) -- entry g of
 * holo_lut_generate(seed, L) for every L > g -- evaluated in pass A for every
 * pixel, with no wrap.  Results are therefore bit-identical to
 * holo_ospr_generate with a pool generated from the same seed and longer than
 * every draw index ("a LUT the same length as the number of random
 * numbers").  Every other argument, output and error as
 * holo_ospr_generate. */
holo_status holo_ospr_generate_prng(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                    uint64_t seed, uint64_t phase_offset, int32_t sf_begin,
                                    int32_t sf_end, uint8_t *holo_bits, float *intensity, double *mse,
                                    holo_region omega, void *ws, size_t ws_bytes, holo_stream stream);

/* The paper's runtime-flexible alternative ("PRNGs with LUTs for sin
 * and cosine functions are expected to remain the dominant technique";
 * reading R-25): the draws of holo_ospr_generate_prng, their phases quantised
 * to 2^phase_bits levels so that (cos, sin) comes from a small table instead
 * of the recipe: draw g uses table[u_g >> (32 - phase_bits)], u_g the high
 * word of SplitMix64(seed, g).
 *   holo_phase_table   table[k] = R-5 at the angle code k << (32 - phase_bits),
 *                      i.e. (cos, sin)(2 pi k / 2^phase_bits), k < 2^phase_bits;
 *                      table: device, 2^phase_bits holo_c64, 16-byte aligned
 *   holo_ospr_generate_prng_table  as holo_ospr_generate_prng, with `table`
 *                      (from holo_phase_table with the same phase_bits; read
 *                      only) replacing the per-draw recipe
 * phase_bits in [1, 16], else INVALID_ARG. */
holo_status holo_phase_table(int32_t phase_bits, holo_c64 *table, holo_stream stream);
holo_status holo_ospr_generate_prng_table(const float *target, int32_t n, int32_t n_frames, int32_t n_sub,
                                          uint64_t seed, const holo_c64 *table, int32_t phase_bits,
                                          uint64_t phase_offset, int32_t sf_begin, int32_t sf_end,
                                          uint8_t *holo_bits, float *intensity, double *mse,
                                          holo_region omega, void *ws, size_t ws_bytes, holo_stream stream);

/* Mean intensity and MSE from a summed intensity (after the caller's
 * cross-rank sum of holo_ospr_generate partial sums): intensity_mean =
 * intensity_sum / n_sub (in place allowed), mse as step a7.
 * intensity_sum, intensity_mean: [n_frames][n][n]; mse: [n_frames] or NULL;
 * ws: only needed if mse != NULL, at least holo_ospr_finalize_workspace_size()
 * bytes (per-CTA fp64 partial sums and a completion ticket; any
 * holo_ospr_workspace_size buffer is large enough).  Reductions run in a fixed
 * order: the result is deterministic. */
size_t holo_ospr_finalize_workspace_size(void);
holo_status holo_ospr_finalize(const float *target, const float *intensity_sum, int32_t n,
                               int32_t n_frames, int32_t n_sub, holo_region omega,
                               float *intensity_mean, double *mse, void *ws, size_t ws_bytes,
                               holo_stream stream);

/* Step a7 on one frame's row slice, for sub-frame shards finished by a
 * reduce-scatter (each rank owns rows [row0, row1) of the
 * summed intensity) and a 5-double all-reduce (C-2):
 *   intensity_mean_rows = intensity_sum_rows / n_sub   (in place allowed)
 *   sums[5] = (sum I, sum I^2, sum I T^2, sum T^2, sum T^4) over omega
 *             restricted to the slice, fp64, fixed reduction order
 * The MSE is nonlinear in I (P:64 averages intensities, R-12 normalises the
 * average), so ranks add their `sums` (C-2) and only then evaluate
 * holo_ospr_mse_from_sums.  target [n][n] (the whole frame);
 * intensity_sum_rows, intensity_mean_rows [row1-row0][n]; sums: 5 doubles of
 * device memory; ws: holo_ospr_finalize_workspace_size() bytes.
 * INVALID_ARG for an empty or out-of-range slice; WORKSPACE if ws is short. */
holo_status holo_ospr_finalize_rows(const float *target, const float *intensity_sum_rows, int32_t n,
                                    int32_t row0, int32_t row1, int32_t n_sub, holo_region omega,
                                    float *intensity_mean_rows, double *sums, void *ws, size_t ws_bytes,
                                    holo_stream stream);

/* R-12 from reduced sums: mse[f] = (a^2 S_II - 2 a S_IT2 + S_T4) / |omega| with
 * a = S_T2 / S_I (0 if S_I = 0), for sums [n_frames][5] as written by
 * holo_ospr_finalize_rows and summed over the ranks (device pointers). */
holo_status holo_ospr_mse_from_sums(const double *sums, int32_t n_frames, holo_region omega, double *mse,
                                    holo_stream stream);

/* ------------------------------------------------------------------------
 * GS -- Gerchberg-Saxton (Fig. 2 left), frames independent.
 * For frame b in [0, batch):
 *   g0  R_0 = T_b * lut[(phase_offset + b*N^2 + p) mod n_lut]  (the LUT is
 *       used for the initial random phase only; n_lut = 0 -> flat)
 *   for k = 1..iters:
 *   g1    H_k  = F^-1{R_{k-1}}
 *   g2    h_k  = constraint(H_k): levels = 0 -> H/|H| (H = 0 -> +1, R-16);
 *                levels = Q > 0 -> exp(2 pi i j/Q),
 *                j = floor(wrap(arg H) Q/2pi + 1/2) mod Q  (R-14, R-15)
 *   g3    R'_k = F{h_k}
 *   g4    I_k = |R'_k|^2; mse[b][k-1] (R-12 over omega);
 *         err_e[b][k-1] = sum_all (|R'_k| - T)^2  (the GS error that the
 *         error-reduction property makes non-increasing)
 *   g5    R_k = T R'_k / |R'_k|  (|R'_k| = 0 -> T, R-16)
 *   g6  outputs after iteration `iters`.
 *
 *   target       [batch][n][n] fp32
 *   levels       0 (continuous phase-only) or Q in [2, 65535]
 *   holo         [batch][n][n] holo_c64, final h (unit modulus); NULL = skip
 *   holo_levels  [batch][n][n] uint8 level index j, only if 2 <= Q <= 256;
 *                NULL = skip
 *   intensity    [batch][n][n] fp32 final I; NULL = skip
 *   mse, err_e   [batch][iters] fp64; NULL = skip
 * ------------------------------------------------------------------------ */
size_t holo_gs_workspace_size(int32_t n, int32_t batch, int32_t iters);

/* Plan query (instrumentation): frames per launch group of holo_gs_generate(n,
 * batch, ...) (HOLO_GS_GROUP_BYTES overrides the 512 MiB budget);
 * 0 for invalid n or batch. */
int32_t holo_gs_group_frames(int32_t n, int32_t batch);

holo_status holo_gs_generate(const float *target, int32_t n, int32_t batch, int32_t iters,
                             const holo_c64 *lut, uint64_t n_lut, uint64_t phase_offset,
                             int32_t levels, holo_c64 *holo, uint8_t *holo_levels, float *intensity,
                             double *mse, double *err_e, holo_region omega, void *ws,
                             size_t ws_bytes, holo_stream stream);

/* ------------------------------------------------------------------------
 * Test hooks (not on the hot path; same kernels / device functions).
 * ------------------------------------------------------------------------ */

/* Unitary 2D DFT (inverse = 0, Eq. (1)) or IDFT (inverse = 1, Eq. (2)) of
 * `batch` n x n fields.  in and out may alias. */
holo_status holo_fft2(const holo_c64 *in, holo_c64 *out, int32_t n, int32_t batch,
                      int32_t inverse, holo_stream stream);

/* Step a2 alone: r_out[p] = target[p] * lut[(offset + p) mod n_lut] (flat if
 * n_lut == 0), one n x n frame, fp32 products (P-2 bit-exactness probe). */
holo_status holo_debug_randomise(const float *target, int32_t n, const holo_c64 *lut,
                                 uint64_t n_lut, uint64_t offset, holo_c64 *r_out,
                                 holo_stream stream);

/* Test hook: pass A's randomisation stage alone (steps a1, a2 exactly as
 * holo_ospr_generate runs them, same kernels with the FFT skipped).  For the
 * sub-frames [sf_begin, sf_end) of frame 0, taken two at a time (a, b), writes
 * z_out[pair][n][n] = conj(Z) with Z(p) = (R_a(p) + conj(R_a(-p))) +
 * i (R_b(p) + conj(R_b(-p))), R_s = T * lut[(phase_offset + s n^2 + p) mod n_lut]
 * (R_b = 0 for an unpaired last sub-frame): the Hermitian pairing of
 * DESIGN.md §5.  use_prng != 0 (lut NULL): the phases of holo_ospr_generate_prng
 * with stream prng_seed instead.  Errors as holo_ospr_generate. */
holo_status holo_debug_ospr_pairs(const float *target, int32_t n, int32_t n_sub, const holo_c64 *lut,
                                  uint64_t n_lut, int32_t use_prng, uint64_t prng_seed,
                                  uint64_t phase_offset, int32_t sf_begin, int32_t sf_end,
                                  holo_c64 *z_out, holo_stream stream);

/* One GS iteration (g1-g5) from r_in = R_{k-1} for `batch` frames: writes
 * r_out = R_k and, if non-NULL, holo = h_k, holo_levels, intensity = I_k,
 * mse[b], err_e[b].  Bit-identical to iteration k of holo_gs_generate when
 * r_in is that call's R_{k-1}.  ws: holo_gs_workspace_size(n, batch, 1). */
holo_status holo_gs_step(const holo_c64 *r_in, const float *target, int32_t n, int32_t batch,
                         int32_t levels, holo_c64 *r_out, holo_c64 *holo, uint8_t *holo_levels,
                         float *intensity, double *mse, double *err_e, holo_region omega,
                         void *ws, size_t ws_bytes, holo_stream stream);

/* ------------------------------------------------------------------------
 * OSPR frame stream for a binary SLM (PAPER.md P:162:
 * a 1024x1024 ferroelectric display shows the N_SF binary sub-frames of each
 * video frame; P:72 / R-2: frame set f continues the phase cursor).
 *
 * A stream owns three non-blocking CUDA streams (h2d, comp, d2h) and per-slot
 * events; everything else is the caller's.  holo_ospr_stream_submit enqueues
 * frame set f in slot f mod depth: H2D of the target, [a0] +
 * holo_ospr_generate (a1-a7) at cursor phase_offset + f * frame_stride *
 * n_sub * n^2 (advance = 0: phase_offset for every f), D2H of the packed
 * holograms, the MSE and optionally the intensity.  Consecutive frame sets'
 * copies overlap each other's kernels; the host never blocks in submit.
 * ------------------------------------------------------------------------ */

typedef struct holo_ospr_stream holo_ospr_stream;   /* opaque */

/* slots: depth * 7 pointers, per slot in this order:
 *   t_dev      device float [n][n]            target of the slot's frame set
 *   bits_dev   device uint8 [n_sub][n][n/8]    packed holograms (R-8)
 *   inten_dev  device float [n][n]            mean replay intensity
 *   mse_dev    device double [1]
 *   bits_host  host (pinned) uint8 [n_sub][n][n/8]
 *   mse_host   host (pinned) double [1]
 *   inten_host host (pinned) float [n][n], or NULL (intensity not shipped)
 * lut: device pool of n_lut entries (NULL iff n_lut == 0); regen_lut != 0
 *   regenerates it (holo_lut_generate(lut_seed, n_lut), step a0) on the
 *   compute stream before each frame set.  ws: holo_ospr_workspace_size(n, 1,
 *   n_sub) bytes, used by one frame set at a time.  depth in [1, 16].
 * All buffers must stay valid until holo_ospr_stream_destroy.  Errors:
 *   INVALID_ARG (sizes, NULL buffers, region), WORKSPACE, CUDA. */
holo_status holo_ospr_stream_create(int32_t n, int32_t n_sub, int32_t depth, const holo_c64 *lut,
                                    uint64_t n_lut, int32_t regen_lut, uint64_t lut_seed,
                                    uint64_t phase_offset, uint64_t frame_stride, int32_t advance,
                                    holo_region omega, void *const *slots, void *ws, size_t ws_bytes,
                                    holo_ospr_stream **out);

/* Enqueue the next frame set from target_host (float [n][n]; pinned for an
 * asynchronous copy; the caller keeps it unchanged until the frame set is
 * done).  *frame (nullable) receives its index f.  Slot reuse waits on the
 * device for the slot's previous frame set, never on the host. */
holo_status holo_ospr_stream_submit(holo_ospr_stream *st, const float *target_host, int64_t *frame);

/* Block until frame set `frame` (one of the last `depth` submitted) has its
 * outputs in the slot's host buffers, valid until frame + depth is submitted. */
holo_status holo_ospr_stream_wait(holo_ospr_stream *st, int64_t frame);

/* 1 if frame set `frame`'s outputs are in host memory, 0 if pending, -1 if
 * it is not among the last `depth` submitted (or on a CUDA error). */
int32_t holo_ospr_stream_done(holo_ospr_stream *st, int64_t frame);

/* Block until every submitted frame set is complete. */
holo_status holo_ospr_stream_drain(holo_ospr_stream *st);

/* The stream's three CUDA streams (h2d, comp, d2h), e.g. to record timing
 * events or to order other work after a frame set; owned by the stream. */
holo_status holo_ospr_stream_handles(holo_ospr_stream *st, holo_stream *h2d, holo_stream *comp, holo_stream *d2h);

/* Drain and release the stream's CUDA streams and events (NULL: no-op). */
void holo_ospr_stream_destroy(holo_ospr_stream *st);

/* ------------------------------------------------------------------------
 * Instrumentation.
 * ------------------------------------------------------------------------ */

/* Number of kernels this library has launched in this process. */
uint64_t holo_launch_count(void);

/* Kernel timing: while enabled, every kernel launch of the library is
 * bracketed by CUDA events recorded on its launch stream.  holo_profile_read
 * synchronises those events and returns, for the kernel class `name` (e.g.
 * "ospr_cols"), the number of launches and their summed device time in ms
 * since the last enable; returns HOLO_ERR_INVALID_ARG for an unknown name.
 * Launches made while the stream is being captured into a CUDA graph are
 * bracketed by event-record nodes (cudaEventRecordExternal) instead, so after
 * each replay of that graph holo_profile_read returns the replay's times; the
 * graph must not outlive the next holo_profile_enable(1), which recycles the
 * events. */
holo_status holo_profile_enable(int32_t on);
holo_status holo_profile_read(const char *name, uint64_t *launches, double *total_ms);

/* Comma-separated list of the kernel class names holo_profile_read knows. */
const char *holo_kernel_names(void);

#ifdef __cplusplus
}
#endif

#endif /* HOLO_H */
