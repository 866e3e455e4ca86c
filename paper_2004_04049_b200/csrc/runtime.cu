// runtime.cu -- libholo host runtime: status strings, launch accounting,
// event-based kernel profiling, per-device twiddle tables, version.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "fft.cuh"
#include "tma.cuh"

namespace holo {

const char *const kKernelNames[K_NUM_KERNELS] = {
    "lut_generate", "ospr_rows_a", "ospr_cols", "ospr_rows_c", "ospr_finalize", "mse_reduce",
    "gs_rows_init", "gs_cols",     "gs_rows",   "fft_rows",    "fft_cols",      "randomise",
};

static thread_local std::string t_error;

holo_status set_error(holo_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_error = buf;
    return st;
}

holo_status cuda_status(cudaError_t e, const char *where)
{
    return set_error(HOLO_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ---- launch accounting and profiling -------------------------------------------------------
static std::atomic<uint64_t> g_launches{0};
static std::mutex g_prof_mu;
static std::atomic<bool> g_prof_on{false};
struct ProfRec {
    int id;
    cudaEvent_t a, b;
};
static std::vector<ProfRec> g_recs;
static std::vector<cudaEvent_t> g_event_pool;
static thread_local cudaEvent_t t_pending = nullptr;

static cudaEvent_t take_event()
{
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

bool pdl_enabled()
{
    static const bool on = [] {
        const char *e = getenv("HOLO_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// Inside a stream capture the events become event-record nodes of the graph
// (cudaEventRecordExternal), so every replay re-times the captured kernels.
static void record(cudaEvent_t e, cudaStream_t s)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
        cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else
        cudaEventRecord(e, s);
}

void prof_before(KernelId id, cudaStream_t s)
{
    (void)id;
    if (!g_prof_on.load(std::memory_order_relaxed))
        return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    t_pending = take_event();
    record(t_pending, s);
}

void prof_after(KernelId id, cudaStream_t s)
{
    if (!g_prof_on.load(std::memory_order_relaxed) || t_pending == nullptr)
        return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = take_event();
    record(b, s);
    g_recs.push_back(ProfRec{(int)id, t_pending, b});
    t_pending = nullptr;
}

static std::mutex g_smem_mu;
static std::set<std::pair<int, const void *>> g_smem_done;

holo_status ensure_smem(const void *fn, size_t smem)
{
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_smem_mu);
    auto key = std::make_pair(dev, fn);
    if (g_smem_done.count(key))
        return HOLO_OK;
    // opt in to the largest dynamic size this kernel can have next to its static shared memory
    // (static + dynamic above 48 KB needs the opt-in even when the dynamic part alone is below)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fn);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaFuncGetAttributes");
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int dyn = optin - (int)fa.sharedSizeBytes;
    if ((size_t)dyn < smem)
        return set_error(HOLO_ERR_CUDA, "kernel needs %zu + %zu bytes of shared memory > %d", smem, fa.sharedSizeBytes,
                         optin);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    static const int carveout = [] {   // HOLO_CARVEOUT=percent: shared-memory share of L1 (experiments)
        const char *c = getenv("HOLO_CARVEOUT");
        return c ? atoi(c) : -1;
    }();
    if (carveout >= 0) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        if (e != cudaSuccess)
            return cuda_status(e, "cudaFuncSetAttribute(PreferredSharedMemoryCarveout)");
    }
    g_smem_done.insert(key);
    return HOLO_OK;
}

static std::mutex g_occ_mu;
static std::map<std::tuple<int, const void *, int, size_t>, int> g_occ;

int resident_ctas(const void *fn, int threads, size_t smem)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(dev, fn, threads, smem);
    {
        std::lock_guard<std::mutex> lk(g_occ_mu);
        auto it = g_occ.find(key);
        if (it != g_occ.end())
            return it->second;
    }
    if (smem > 0)
        ensure_smem(fn, smem);
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    const int cap = sms * (per_sm < 1 ? 1 : per_sm);
    std::lock_guard<std::mutex> lk(g_occ_mu);
    g_occ[key] = cap;
    return cap;
}

namespace fft {

static std::mutex g_tw_mu;
static std::map<int, float2 *> g_tw_dev;

holo_status twiddles(const float2 **pool)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_tw_mu);
    auto it = g_tw_dev.find(dev);
    if (it != g_tw_dev.end()) {
        *pool = it->second;
        return HOLO_OK;
    }
    std::vector<float2> host(kTwPool, make_float2(0.f, 0.f));
    for (int lg = 4; lg <= 12; ++lg) {
        int n = 1 << lg, r1 = 1 << (lg / 2), r2 = n / r1, off = n - 16;
        for (int r = 0; r < r2; ++r)
            for (int t = 0; t < r1; ++t) {
                long long m = ((long long)r * t) % n;
                double a = -2.0 * 3.14159265358979323846 * (double)m / (double)n;
                host[off + r * r1 + t] = make_float2((float)std::cos(a), (float)std::sin(a));
            }
    }
    float2 *d = nullptr;
    e = cudaMalloc(&d, sizeof(float2) * kTwPool);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaMalloc(twiddles)");
    e = cudaMemcpy(d, host.data(), sizeof(float2) * kTwPool, cudaMemcpyHostToDevice);
    if (e != cudaSuccess)
        return cuda_status(e, "cudaMemcpy(twiddles)");
    g_tw_dev[dev] = d;
    *pool = d;
    return HOLO_OK;
}

} // namespace fft

// ---- TMA tensor maps (driver entry point fetched through the runtime; no -lcuda) -------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

holo_status make_tmap_c64(CUtensorMap *map, const void *base, uint64_t cols, uint64_t rows, uint32_t box_cols,
                          uint32_t box_rows)
{
    auto fn = encode_fn();
    if (!fn)
        return set_error(HOLO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 8};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return set_error(HOLO_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return HOLO_OK;
}

} // namespace holo

using namespace holo;

extern "C" const char *holo_last_error(void) { return t_error.c_str(); }

extern "C" const char *holo_version(void) { return "holo 0.1.0 sm_100a"; }

extern "C" uint64_t holo_launch_count(void) { return g_launches.load(); }

extern "C" holo_status holo_profile_enable(int32_t on)
{
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (on) {
        for (auto &r : g_recs) {
            cudaEventSynchronize(r.b);
            g_event_pool.push_back(r.a);
            g_event_pool.push_back(r.b);
        }
        g_recs.clear();
    }
    g_prof_on.store(on != 0);
    return HOLO_OK;
}

extern "C" holo_status holo_profile_read(const char *name, uint64_t *launches, double *total_ms)
{
    int id = -1;
    for (int k = 0; k < K_NUM_KERNELS; ++k)
        if (name && std::string(name) == kKernelNames[k])
            id = k;
    if (id < 0)
        return set_error(HOLO_ERR_INVALID_ARG, "unknown kernel name '%s'", name ? name : "(null)");
    std::lock_guard<std::mutex> lk(g_prof_mu);
    uint64_t n = 0;
    double ms = 0.0;
    for (auto &r : g_recs) {
        if (r.id != id)
            continue;
        cudaError_t e = cudaEventSynchronize(r.b);
        if (e != cudaSuccess)
            return cuda_status(e, "cudaEventSynchronize");
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        ms += t;
        ++n;
    }
    if (launches)
        *launches = n;
    if (total_ms)
        *total_ms = ms;
    return HOLO_OK;
}

extern "C" const char *holo_kernel_names(void)
{
    static std::string s;
    static std::once_flag f;
    std::call_once(f, [] {
        for (int k = 0; k < K_NUM_KERNELS; ++k) {
            if (k)
                s += ",";
            s += kKernelNames[k];
        }
    });
    return s.c_str();
}
