// stream.cu -- the OSPR frame stream for a binary SLM (the
// 1024x1024 ferroelectric display showing N_SF binary sub-frames per video frame), as native
// host code behind the C ABI: one holo_ospr_stream_submit per frame set enqueues
//
//   h2d  : target f (pinned host) -> slot f mod depth               (copy engine)
//   comp : [a0: lut <- holo_lut_generate(seed, L)] + ospr_generate   (libholo kernels)
//   d2h  : packed holograms + MSE [+ intensity] of f -> pinned host   (copy engine)
//
// on three library-owned non-blocking streams ordered by events only, so frame set f's copies
// overlap the kernels of f - 1 and f + 1 and the host never blocks in submit.  Frame set f uses
// the continuing cursor phase_offset + f * frame_stride * N_SF * N^2 (R-2).  Buffers are
// the caller's (device slots, pinned host slots, workspace); the stream only sequences them.
#include <cuda_runtime.h>

#include <new>

#include "common.cuh"

namespace holo {
holo_status check_n(int n);
holo_status check_region(holo_region om, int n);
}

constexpr int kMaxStreamDepth = 16;
constexpr int kSlotPtrs = 7;   // t_dev, bits_dev, inten_dev, mse_dev, bits_host, mse_host, inten_host

struct holo_ospr_stream {
    int n = 0, n_sub = 0, depth = 0;
    const holo_c64 *lut = nullptr;
    uint64_t n_lut = 0, lut_seed = 0, off0 = 0, stride = 1;
    int regen = 0, advance = 1;
    holo_region omega{};
    void *slot[kMaxStreamDepth][kSlotPtrs] = {};
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t h2d_done[kMaxStreamDepth] = {}, comp_done[kMaxStreamDepth] = {}, d2h_done[kMaxStreamDepth] = {};
    bool used[kMaxStreamDepth] = {};
    int64_t f = 0;
    int device = 0;
};

using namespace holo;

static void stream_release(holo_ospr_stream *st)
{
    if (st->h2d)
        cudaStreamSynchronize(st->h2d);
    if (st->comp)
        cudaStreamSynchronize(st->comp);
    if (st->d2h)
        cudaStreamSynchronize(st->d2h);
    for (int s = 0; s < kMaxStreamDepth; ++s) {
        if (st->h2d_done[s])
            cudaEventDestroy(st->h2d_done[s]);
        if (st->comp_done[s])
            cudaEventDestroy(st->comp_done[s]);
        if (st->d2h_done[s])
            cudaEventDestroy(st->d2h_done[s]);
    }
    if (st->h2d)
        cudaStreamDestroy(st->h2d);
    if (st->comp)
        cudaStreamDestroy(st->comp);
    if (st->d2h)
        cudaStreamDestroy(st->d2h);
    delete st;
}

extern "C" holo_status holo_ospr_stream_create(int32_t n, int32_t n_sub, int32_t depth, const holo_c64 *lut,
                                               uint64_t n_lut, int32_t regen_lut, uint64_t lut_seed,
                                               uint64_t phase_offset, uint64_t frame_stride, int32_t advance,
                                               holo_region omega, void *const *slots, void *ws, size_t ws_bytes,
                                               holo_ospr_stream **out)
{
    HOLO_CHECK_ARG(out != nullptr, "out is NULL");
    *out = nullptr;
    HOLO_TRY(check_n(n));
    HOLO_CHECK_ARG(n_sub >= 1, "n_sub must be >= 1");
    HOLO_CHECK_ARG(depth >= 1 && depth <= kMaxStreamDepth, "depth must be in [1, %d], got %d", kMaxStreamDepth, depth);
    HOLO_CHECK_ARG(n_lut < (1ull << 31), "n_lut must be < 2^31");
    HOLO_CHECK_ARG((lut == nullptr) == (n_lut == 0), "lut must be NULL iff n_lut == 0");
    HOLO_CHECK_ARG(!regen_lut || n_lut >= 1, "regen_lut needs a pool (n_lut >= 1)");
    HOLO_TRY(check_region(omega, n));
    HOLO_CHECK_ARG(slots != nullptr, "slots is NULL");
    for (int s = 0; s < depth; ++s)
        for (int k = 0; k < kSlotPtrs - 1; ++k)   // inten_host (k = 6) is optional
            HOLO_CHECK_ARG(slots[s * kSlotPtrs + k] != nullptr, "slot %d buffer %d is NULL", s, k);
    HOLO_CHECK_ARG(ws != nullptr, "workspace is NULL");
    const size_t need = holo_ospr_workspace_size(n, 1, n_sub);
    if (ws_bytes < need)
        return set_error(HOLO_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, need);
    holo_ospr_stream *st = new (std::nothrow) holo_ospr_stream();
    if (st == nullptr)
        return set_error(HOLO_ERR_INVALID_ARG, "out of host memory");
    st->n = n, st->n_sub = n_sub, st->depth = depth, st->lut = lut, st->n_lut = n_lut;
    st->regen = regen_lut != 0, st->lut_seed = lut_seed, st->off0 = phase_offset, st->stride = frame_stride;
    st->advance = advance != 0, st->omega = omega, st->ws = ws, st->ws_bytes = ws_bytes;
    for (int s = 0; s < depth; ++s)
        for (int k = 0; k < kSlotPtrs; ++k)
            st->slot[s][k] = slots[s * kSlotPtrs + k];
    cudaError_t e = cudaGetDevice(&st->device);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&st->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&st->comp, cudaStreamNonBlocking);
    if (e == cudaSuccess)
        e = cudaStreamCreateWithFlags(&st->d2h, cudaStreamNonBlocking);
    for (int s = 0; s < depth && e == cudaSuccess; ++s) {
        e = cudaEventCreateWithFlags(&st->h2d_done[s], cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&st->comp_done[s], cudaEventDisableTiming);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&st->d2h_done[s], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        stream_release(st);
        return cuda_status(e, "holo_ospr_stream_create");
    }
    *out = st;
    return HOLO_OK;
}

#define HOLO_CUDA(call)                                    \
    do {                                                   \
        const cudaError_t e_ = (call);                     \
        if (e_ != cudaSuccess)                             \
            return cuda_status(e_, #call);                 \
    } while (0)

static holo_status stream_submit(holo_ospr_stream *st, const float *target_host, int64_t *frame);

extern "C" holo_status holo_ospr_stream_submit(holo_ospr_stream *st, const float *target_host, int64_t *frame)
{
    HOLO_CHECK_ARG(st != nullptr && target_host != nullptr, "stream/target_host is NULL");
    int cur = -1;   // the library's kernels launch on the current device: the stream's, for this call
    HOLO_CUDA(cudaGetDevice(&cur));
    if (cur != st->device)
        HOLO_CUDA(cudaSetDevice(st->device));
    const holo_status r = stream_submit(st, target_host, frame);
    if (cur != st->device)
        cudaSetDevice(cur);
    return r;
}

static holo_status stream_submit(holo_ospr_stream *st, const float *target_host, int64_t *frame)
{
    const int64_t f = st->f;
    const int s = (int)(f % st->depth);
    const size_t P = (size_t)st->n * st->n;
    float *t_dev = (float *)st->slot[s][0];
    uint8_t *bits_dev = (uint8_t *)st->slot[s][1];
    float *inten_dev = (float *)st->slot[s][2];
    double *mse_dev = (double *)st->slot[s][3];
    if (st->used[s]) {
        // slot reuse: its previous frame set must have read its target (comp) and shipped its
        // outputs (d2h) before they are overwritten
        HOLO_CUDA(cudaStreamWaitEvent(st->h2d, st->comp_done[s], 0));
        HOLO_CUDA(cudaStreamWaitEvent(st->comp, st->d2h_done[s], 0));
    }
    HOLO_CUDA(cudaMemcpyAsync(t_dev, target_host, P * sizeof(float), cudaMemcpyHostToDevice, st->h2d));
    HOLO_CUDA(cudaEventRecord(st->h2d_done[s], st->h2d));
    HOLO_CUDA(cudaStreamWaitEvent(st->comp, st->h2d_done[s], 0));
    if (st->regen)   // a0: the pool of this frame set
        HOLO_TRY(holo_lut_generate(st->lut_seed, st->n_lut, (holo_c64 *)st->lut, (holo_stream)st->comp));
    const uint64_t off = st->off0 + (st->advance ? (uint64_t)f * st->stride * (uint64_t)st->n_sub * P : 0ull);
    HOLO_TRY(holo_ospr_generate(t_dev, st->n, 1, st->n_sub, st->lut, st->n_lut, off, 0, st->n_sub, bits_dev, inten_dev,
                                mse_dev, st->omega, st->ws, st->ws_bytes, (holo_stream)st->comp));
    HOLO_CUDA(cudaEventRecord(st->comp_done[s], st->comp));
    HOLO_CUDA(cudaStreamWaitEvent(st->d2h, st->comp_done[s], 0));
    HOLO_CUDA(cudaMemcpyAsync(st->slot[s][4], bits_dev, (size_t)st->n_sub * P / 8, cudaMemcpyDeviceToHost, st->d2h));
    HOLO_CUDA(cudaMemcpyAsync(st->slot[s][5], mse_dev, sizeof(double), cudaMemcpyDeviceToHost, st->d2h));
    if (st->slot[s][6] != nullptr)
        HOLO_CUDA(cudaMemcpyAsync(st->slot[s][6], inten_dev, P * sizeof(float), cudaMemcpyDeviceToHost, st->d2h));
    HOLO_CUDA(cudaEventRecord(st->d2h_done[s], st->d2h));
    st->used[s] = true;
    st->f = f + 1;
    if (frame != nullptr)
        *frame = f;
    return HOLO_OK;
}

static holo_status window_slot(const holo_ospr_stream *st, int64_t f, int *s)
{
    HOLO_CHECK_ARG(st != nullptr, "stream is NULL");
    HOLO_CHECK_ARG(f >= st->f - st->depth && f < st->f && f >= 0,
                   "frame set %lld is not among the last %d submitted", (long long)f, st->depth);
    *s = (int)(f % st->depth);
    return HOLO_OK;
}

extern "C" holo_status holo_ospr_stream_wait(holo_ospr_stream *st, int64_t frame)
{
    int s = 0;
    HOLO_TRY(window_slot(st, frame, &s));
    HOLO_CUDA(cudaEventSynchronize(st->d2h_done[s]));
    return HOLO_OK;
}

extern "C" int32_t holo_ospr_stream_done(holo_ospr_stream *st, int64_t frame)
{
    int s = 0;
    if (window_slot(st, frame, &s) != HOLO_OK)
        return -1;
    const cudaError_t e = cudaEventQuery(st->d2h_done[s]);
    if (e == cudaSuccess)
        return 1;
    if (e == cudaErrorNotReady)
        return 0;
    cuda_status(e, "holo_ospr_stream_done");
    return -1;
}

extern "C" holo_status holo_ospr_stream_drain(holo_ospr_stream *st)
{
    HOLO_CHECK_ARG(st != nullptr, "stream is NULL");
    HOLO_CUDA(cudaStreamSynchronize(st->h2d));
    HOLO_CUDA(cudaStreamSynchronize(st->comp));
    HOLO_CUDA(cudaStreamSynchronize(st->d2h));
    return HOLO_OK;
}

extern "C" holo_status holo_ospr_stream_handles(holo_ospr_stream *st, holo_stream *h2d, holo_stream *comp,
                                                holo_stream *d2h)
{
    HOLO_CHECK_ARG(st != nullptr && h2d != nullptr && comp != nullptr && d2h != nullptr, "NULL argument");
    *h2d = (holo_stream)st->h2d;
    *comp = (holo_stream)st->comp;
    *d2h = (holo_stream)st->d2h;
    return HOLO_OK;
}

extern "C" void holo_ospr_stream_destroy(holo_ospr_stream *st)
{
    if (st != nullptr)
        stream_release(st);
}
