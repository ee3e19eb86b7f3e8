// Context lifetime, host<->device transfers (AoS <-> SoA) and the C-ABI
// entry points of libmm_admm (declared in include/mm_admm.h).
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <stdarg.h>

#include <atomic>
#include <condition_variable>
#include <mutex>
#include <sched.h>
#include <string.h>
#include <thread>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges per pipeline stage
#include <vector>

#include "mm_internal.cuh"

int mm_fail(mm_ctx *ctx, int code, const char *fmt, ...) {
    if (ctx) {
        char buf[1024];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        ctx->err = buf;
    }
    return code;
}

// Device memory comes from the device's stream-ordered pool, which keeps up
// to kPoolKeepBytes of freed memory reserved for the process (like a caching
// allocator): a context created after another was destroyed -- a solve on
// host buffers after another -- reuses mapped memory instead of paying
// cudaMalloc's page mapping again.
static const uint64_t kPoolKeepBytes = (uint64_t)48 << 30;
static bool g_pool_ready[64];
static int g_use_pool = -1;

int mm_alloc(mm_ctx *ctx, void **ptr, size_t bytes) {
    if (bytes == 0) bytes = 8;
    if (g_use_pool < 0) {
        const char *e = getenv("MM_DEVICE_POOL");
        g_use_pool = (e && e[0] == '0') ? 0 : 1;
    }
    if (!g_use_pool) {
        cudaError_t e = cudaMalloc(ptr, bytes);
        if (e != cudaSuccess)
            return mm_fail(ctx, MM_ERR_CUDA, "cudaMalloc(%zu) failed: %s", bytes,
                           cudaGetErrorString(e));
        ctx->bytes += (int64_t)bytes;
        return MM_OK;
    }
    const int dev = ctx->device;
    if (dev >= 0 && dev < 64 && !g_pool_ready[dev]) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = kPoolKeepBytes;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
        g_pool_ready[dev] = true;
    }
    cudaError_t e = cudaMallocAsync(ptr, bytes, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);  // usable from any stream
    if (e != cudaSuccess)
        return mm_fail(ctx, MM_ERR_CUDA, "device allocation of %zu B failed: %s", bytes,
                       cudaGetErrorString(e));
    ctx->bytes += (int64_t)bytes;
    return MM_OK;
}

void mm_free(mm_ctx *ctx, void *p) {
    if (!p) return;
    if (g_use_pool) cudaFreeAsync(p, ctx->stream);
    else cudaFree(p);
}

int mm_ensure_partials(mm_ctx *ctx, int64_t nblocks) {
    if (nblocks <= ctx->partials_cap) return MM_OK;
    if (ctx->partials) {
        mm_free(ctx, ctx->partials);
        ctx->bytes -= ctx->partials_cap * MM_MAX_PARTIALS * (int64_t)sizeof(double);
    }
    ctx->partials = nullptr;
    int rc = mm_alloc(ctx, (void **)&ctx->partials, sizeof(double) * MM_MAX_PARTIALS * nblocks);
    if (rc) return rc;
    ctx->partials_cap = nblocks;
    return MM_OK;
}

// The reduction result slot: single-grid and point-set contexts map it from
// pinned host memory, so the last block of a reducing kernel writes the sums
// straight to the host (no copy launch, no copy on the GPU timeline); slab
// contexts keep it in device memory.
//
// Destroyed single-grid / point-set contexts park their stream and mapped
// result slot here for the next context on the same device: pinned
// allocation (~1.3 ms) and stream creation (~0.3 ms) dominate creating a
// small context (config 1 creates one per study).
struct Recycled {
    int device;
    cudaStream_t stream;
    double *host_out;
};
static std::mutex g_recycle_mu;
static std::vector<Recycled> g_recycle;

static bool take_recycled(mm_ctx *ctx) {
    std::lock_guard<std::mutex> lk(g_recycle_mu);
    for (size_t i = 0; i < g_recycle.size(); ++i) {
        if (g_recycle[i].device != ctx->device) continue;
        ctx->stream = g_recycle[i].stream;
        ctx->host_out = g_recycle[i].host_out;
        g_recycle.erase(g_recycle.begin() + (long)i);
        return true;
    }
    return false;
}

// true: the stream and the slot are parked (the caller must not free them)
static bool park_recycled(mm_ctx *ctx) {
    if (!ctx->red_mapped || ctx->slab_mode || !ctx->stream || !ctx->host_out) return false;
    if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    std::lock_guard<std::mutex> lk(g_recycle_mu);
    if (g_recycle.size() >= 8) return false;
    g_recycle.push_back({ctx->device, ctx->stream, ctx->host_out});
    return true;
}

static int alloc_red_out(mm_ctx *ctx) {
    // three slots: reductions, K1's sums of a pipelined step, k_decide's copy
    if (!ctx->host_out)
        MM_CUDA(ctx, cudaHostAlloc((void **)&ctx->host_out, sizeof(double) * 3 * MM_MAX_PARTIALS,
                                   cudaHostAllocMapped));
    MM_CUDA(ctx, cudaHostGetDevicePointer((void **)&ctx->red_out, ctx->host_out, 0));
    ctx->red_mapped = true;
    return MM_OK;
}

int mm_fetch_reduction(mm_ctx *ctx, int K, double *out) {
    if (!ctx->red_mapped)
        MM_CUDA(ctx, cudaMemcpyAsync(ctx->host_out, ctx->red_out, sizeof(double) * K,
                                     cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    memcpy(out, ctx->host_out, sizeof(double) * K);
    mm_drain_timings(ctx);
    return MM_OK;
}

static cudaEvent_t pool_get(mm_ctx *ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// NVTX ranges around every pipeline stage (host-side launch windows, for
// nsys / ncu --nvtx), on when MM_NVTX=1 in the environment at context creation
static const char *const kStageName[MM_NSTAGE] = {
    "mm:local", "mm:row_fwd", "mm:col_fwd", "mm:col_solve", "mm:col_inv", "mm:row_inv",
    "mm:grad", "mm:frozen", "mm:other", "mm:fused", "mm:plane"};

static bool nvtx_on() {
    static const bool on = [] {
        const char *e = getenv("MM_NVTX");
        return e && atoi(e) != 0;
    }();
    return on;
}

void mm_stage_begin(mm_ctx *ctx, int stage, cudaEvent_t *ev) {
    *ev = nullptr;
    if (nvtx_on()) nvtxRangePushA(kStageName[stage]);
    if (!ctx->prof_on) return;
    *ev = pool_get(ctx);
    cudaEventRecord(*ev, ctx->stream);
}

void mm_stage_end(mm_ctx *ctx, int stage, cudaEvent_t ev, int nlaunch) {
    if (nvtx_on()) nvtxRangePop();
    ctx->launches[stage] += nlaunch;
    if (!ctx->prof_on || !ev) return;
    cudaEvent_t b = pool_get(ctx);
    cudaEventRecord(b, ctx->stream);
    ctx->pending.push_back({stage, ev, b});
    ctx->prof_launches[stage] += nlaunch;
}

void mm_drain_timings(mm_ctx *ctx) {
    for (auto &p : ctx->pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess)
            ctx->prof_ms[p.stage] += ms;
        ctx->event_pool.push_back(p.a);
        ctx->event_pool.push_back(p.b);
    }
    ctx->pending.clear();
}

// ---------------------------------------------------------------------------
// AoS <-> SoA
// ---------------------------------------------------------------------------
__global__ void k_aos_to_soa(const double *__restrict__ src, double *__restrict__ dst,
                             int64_t p0, int64_t np, int ncomp, int64_t M) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t tot = np * ncomp;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = i / ncomp;
        int c = (int)(i - p * ncomp);
        dst[(int64_t)c * M + p0 + p] = src[i];
    }
}

__global__ void k_aos_add_soa(const double *__restrict__ src, double *__restrict__ dst,
                              int64_t p0, int64_t np, int ncomp, int64_t M) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t tot = np * ncomp;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = i / ncomp;
        int c = (int)(i - p * ncomp);
        const int64_t o = (int64_t)c * M + p0 + p;
        dst[o] = __dadd_rn(dst[o], src[i]);  // numpy's F + dF, one rounding
    }
}

__global__ void k_soa_to_aos(const double *__restrict__ src, double *__restrict__ dst,
                             int64_t p0, int64_t np, int ncomp, int64_t M) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t tot = np * ncomp;
    for (; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = i / ncomp;
        int c = (int)(i - p * ncomp);
        dst[i] = src[(int64_t)c * M + p0 + p];
    }
}

static int field_info(mm_ctx *ctx, int field, double ***slot, int *ncomp) {
    const int d = ctx->dim, D = ctx->D;
    switch (field) {
        case MM_FIELD_F: *slot = &ctx->F; *ncomp = D; break;
        case MM_FIELD_G: *slot = &ctx->G; *ncomp = D; break;
        case MM_FIELD_LAM: *slot = &ctx->Lam; *ncomp = D; break;
        case MM_FIELD_UT: *slot = &ctx->Ut; *ncomp = d; break;
        case MM_FIELD_PREV_F: *slot = &ctx->prevF; *ncomp = D; break;
        case MM_FIELD_MOD_A: *slot = &ctx->modA; *ncomp = 1; break;
        case MM_FIELD_MOD_B: *slot = &ctx->modB; *ncomp = 1; break;
        case MM_FIELD_ANG: *slot = &ctx->ang; *ncomp = d == 2 ? 1 : 2; break;
        case MM_FIELD_CHART:
            if (d != 3) return mm_fail(ctx, MM_ERR_CONFIG, "chart exists only in 3D");
            *slot = &ctx->chart; *ncomp = 9; break;
        case MM_FIELD_PINC: *slot = &ctx->pinc; *ncomp = 1; break;
        case MM_FIELD_N0: *slot = &ctx->n0; *ncomp = d; break;
        case MM_FIELD_FF: *slot = &ctx->ff; *ncomp = d; break;
        case MM_FIELD_PREV_ANG: *slot = &ctx->prevAng; *ncomp = d == 2 ? 1 : 2; break;
        case MM_FIELD_PREV_CHART:
            if (d != 3) return mm_fail(ctx, MM_ERR_CONFIG, "chart exists only in 3D");
            *slot = &ctx->prevChart; *ncomp = 9; break;
        case MM_FIELD_PREV_PINC: *slot = &ctx->prevPinc; *ncomp = 1; break;
        default: return mm_fail(ctx, MM_ERR_CONFIG, "unknown field id %d", field);
    }
    return MM_OK;
}

static int ensure_field(mm_ctx *ctx, double **slot, int ncomp) {
    if (*slot) return MM_OK;
    int rc = mm_alloc(ctx, (void **)slot, sizeof(double) * ncomp * ctx->M);
    if (rc) return rc;
    MM_CUDA(ctx, cudaMemsetAsync(*slot, 0, sizeof(double) * ncomp * ctx->M, ctx->stream));
    return MM_OK;
}

// Host staging.  Transfers move CHUNK-byte pieces through a device stage
// (AoS <-> SoA transpose on the GPU) and, for pageable host memory, through
// two pinned halves shared by every context of the process: while the DMA of
// chunk i runs, host threads copy chunk i +- 1 between the caller's array and
// the other half (multi-threaded: both the memcpy bandwidth and the page
// faults of freshly allocated destinations scale with threads).  Pinned
// caller memory is DMA'd directly.
static const size_t kChunkBytes = (size_t)128 << 20;

struct PinnedPool {
    std::mutex mu;
    char *half[2] = {nullptr, nullptr};
    size_t cap = 0;
};
static PinnedPool g_pinned;

static int host_threads() {
    static int nt = 0;
    if (!nt) {
        cpu_set_t set;
        int c = 0;
        if (sched_getaffinity(0, sizeof set, &set) == 0) c = CPU_COUNT(&set);
        nt = std::max(1, std::min(c, 16));
    }
    return nt;
}

// Persistent host copy pool (created on first use, never torn down): a copy
// is cut into one contiguous part per thread, taken from an atomic counter by
// the workers and the calling thread, so per-chunk thread start-up does not
// eat into the overlap with the DMA of the next chunk.
class CopyPool {
  public:
    explicit CopyPool(int nworkers) {
        for (int i = 0; i < nworkers; ++i) std::thread([this] { worker(); }).detach();
    }
    void copy(void *dst, const void *src, size_t bytes, int nparts) {
        // one contiguous part per thread: each thread faults in its own range
        const size_t part = (((bytes + nparts - 1) / nparts) + 4095) & ~(size_t)4095;
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = (char *)dst;
            src_ = (const char *)src;
            bytes_ = bytes;
            part_ = part;
            njobs_ = (int)((bytes + part - 1) / part);
            next_.store(0);
            remaining_.store(njobs_);
            ++gen_;
        }
        cv_.notify_all();
        run();
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return remaining_.load() == 0; });
    }

  private:
    void run() {
        int j;
        while ((j = next_.fetch_add(1)) < njobs_) {
            const size_t off = (size_t)j * part_;
            memcpy(dst_ + off, src_ + off, std::min(part_, bytes_ - off));
            if (remaining_.fetch_sub(1) == 1) {
                std::lock_guard<std::mutex> lk(mu_);
                done_.notify_all();
            }
        }
    }
    void worker() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            run();
        }
    }
    std::mutex mu_;
    std::condition_variable cv_, done_;
    char *dst_ = nullptr;
    const char *src_ = nullptr;
    size_t bytes_ = 0, part_ = 1;
    int njobs_ = 0;
    std::atomic<int> next_{0}, remaining_{0};
    uint64_t gen_ = 0;
};

static void par_memcpy(void *dst, const void *src, size_t bytes) {
    const int nt = host_threads();
    if (nt <= 1 || bytes < ((size_t)4 << 20)) {
        memcpy(dst, src, bytes);
        return;
    }
    static CopyPool *pool = new CopyPool(nt - 1);  // intentionally never destroyed
    pool->copy(dst, src, bytes, nt);
}

static int ensure_stage(mm_ctx *ctx, int64_t ndoubles) {
    if (ndoubles <= ctx->stage_cap) return MM_OK;
    if (ctx->stage) {
        mm_free(ctx, ctx->stage);
        ctx->bytes -= ctx->stage_cap * 8;
    }
    ctx->stage = nullptr;
    int rc = mm_alloc(ctx, (void **)&ctx->stage, sizeof(double) * ndoubles);
    if (rc) return rc;
    ctx->stage_cap = ndoubles;
    if (!ctx->xfer_ev[0]) {
        MM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->xfer_ev[0], cudaEventDisableTiming));
        MM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->xfer_ev[1], cudaEventDisableTiming));
    }
    return MM_OK;
}

static int ensure_pinned(mm_ctx *ctx, size_t bytes) {  // caller holds g_pinned.mu
    if (bytes <= g_pinned.cap) return MM_OK;
    for (int h = 0; h < 2; ++h) {
        if (g_pinned.half[h]) cudaFreeHost(g_pinned.half[h]);
        g_pinned.half[h] = nullptr;
    }
    g_pinned.cap = 0;
    for (int h = 0; h < 2; ++h)
        MM_CUDA(ctx, cudaMallocHost((void **)&g_pinned.half[h], bytes));
    g_pinned.cap = bytes;
    return MM_OK;
}

static bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

static void launch_xpose(mm_ctx *ctx, bool to_soa, bool add, double *dev, int64_t p0, int64_t np,
                         int ncomp, int64_t cs) {
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((np * ncomp + threads - 1) / threads, 148 * 32);
    if (!to_soa)
        k_soa_to_aos<<<blocks, threads, 0, ctx->stream>>>(dev, ctx->stage, p0, np, ncomp, cs);
    else if (add)
        k_aos_add_soa<<<blocks, threads, 0, ctx->stream>>>(ctx->stage, dev, p0, np, ncomp, cs);
    else
        k_aos_to_soa<<<blocks, threads, 0, ctx->stream>>>(ctx->stage, dev, p0, np, ncomp, cs);
}

// component stride of a field's device storage (u_tilde keeps ghost planes
// on a slab)
static int64_t field_cs(const mm_ctx *ctx, int field) {
    return field == MM_FIELD_UT ? ctx->uM : ctx->M;
}

static int transfer(mm_ctx *ctx, double *dev, int ncomp, const double *hsrc, double *hdst,
                    bool add = false, int64_t cs = -1) {
    const int64_t M = ctx->M;
    if (cs < 0) cs = M;
    const int64_t chunk_pts =
        std::max<int64_t>(1, std::min<int64_t>(M, (int64_t)(kChunkBytes / (8 * ncomp))));
    int rc = ensure_stage(ctx, chunk_pts * ncomp);
    if (rc) return rc;
    const bool up = hsrc != nullptr;
    const bool pinned = is_pinned(up ? (const void *)hsrc : (const void *)hdst);
    const int64_t nchunk = (M + chunk_pts - 1) / chunk_pts;
    auto span = [&](int64_t i, int64_t &p0, int64_t &np) {
        p0 = i * chunk_pts;
        np = std::min(chunk_pts, M - p0);
    };
    if (pinned) {
        for (int64_t i = 0; i < nchunk; ++i) {
            int64_t p0, np;
            span(i, p0, np);
            const size_t bytes = sizeof(double) * np * ncomp;
            if (up) {
                MM_CUDA(ctx, cudaMemcpyAsync(ctx->stage, hsrc + p0 * ncomp, bytes,
                                             cudaMemcpyHostToDevice, ctx->stream));
                launch_xpose(ctx, true, add, dev, p0, np, ncomp, cs);
            } else {
                launch_xpose(ctx, false, false, dev, p0, np, ncomp, cs);
                MM_CUDA(ctx, cudaMemcpyAsync(hdst + p0 * ncomp, ctx->stage, bytes,
                                             cudaMemcpyDeviceToHost, ctx->stream));
            }
            MM_LAUNCH_CHECK(ctx);
        }
        MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        return MM_OK;
    }
    std::lock_guard<std::mutex> lock(g_pinned.mu);
    if ((rc = ensure_pinned(ctx, kChunkBytes))) return rc;
    if (up) {
        for (int64_t i = 0; i < nchunk; ++i) {
            int64_t p0, np;
            span(i, p0, np);
            const size_t bytes = sizeof(double) * np * ncomp;
            const int h = (int)(i & 1);
            // the DMA that last read this half (chunk i - 2) must be done
            if (i >= 2) MM_CUDA(ctx, cudaEventSynchronize(ctx->xfer_ev[h]));
            par_memcpy(g_pinned.half[h], hsrc + p0 * ncomp, bytes);
            MM_CUDA(ctx, cudaMemcpyAsync(ctx->stage, g_pinned.half[h], bytes,
                                         cudaMemcpyHostToDevice, ctx->stream));
            MM_CUDA(ctx, cudaEventRecord(ctx->xfer_ev[h], ctx->stream));
            launch_xpose(ctx, true, add, dev, p0, np, ncomp, cs);
            MM_LAUNCH_CHECK(ctx);
        }
    } else {
        for (int64_t i = 0; i <= nchunk; ++i) {
            if (i < nchunk) {
                int64_t p0, np;
                span(i, p0, np);
                const int h = (int)(i & 1);
                launch_xpose(ctx, false, false, dev, p0, np, ncomp, cs);
                MM_LAUNCH_CHECK(ctx);
                MM_CUDA(ctx, cudaMemcpyAsync(g_pinned.half[h], ctx->stage,
                                             sizeof(double) * np * ncomp,
                                             cudaMemcpyDeviceToHost, ctx->stream));
                MM_CUDA(ctx, cudaEventRecord(ctx->xfer_ev[h], ctx->stream));
            }
            if (i >= 1) {  // copy out chunk i - 1 while chunk i is in flight
                int64_t p0, np;
                span(i - 1, p0, np);
                const int h = (int)((i - 1) & 1);
                MM_CUDA(ctx, cudaEventSynchronize(ctx->xfer_ev[h]));
                par_memcpy(hdst + p0 * ncomp, g_pinned.half[h], sizeof(double) * np * ncomp);
            }
        }
    }
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return MM_OK;
}

// ---------------------------------------------------------------------------
// twiddles (long double on the host, rounded once)
// ---------------------------------------------------------------------------
static std::vector<double2> twiddle_table(int N) {
    std::vector<double2> t(N > 0 ? N : 1);
    for (int k = 0; k < N; ++k) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * (long double)k / N;
        t[k].x = (double)cosl(a);
        t[k].y = (double)sinl(a);
    }
    return t;
}

static int upload_tw(mm_ctx *ctx, double2 **dst, int N) {
    std::vector<double2> t = twiddle_table(N);
    int rc = mm_alloc(ctx, (void **)dst, sizeof(double2) * t.size());
    if (rc) return rc;
    MM_CUDA(ctx, cudaMemcpy(*dst, t.data(), sizeof(double2) * t.size(), cudaMemcpyHostToDevice));
    return MM_OK;
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int mm_abi_version(void) { return MM_ABI_VERSION; }

int64_t mm_struct_size(int which) {
    switch (which) {
        case MM_STRUCT_LOCAL_STATS: return (int64_t)sizeof(mm_local_stats);
        case MM_STRUCT_UPDATE_STATS: return (int64_t)sizeof(mm_update_stats);
        case MM_STRUCT_STEP_PARAMS: return (int64_t)sizeof(mm_step_params);
        case MM_STRUCT_STEP_RESULT: return (int64_t)sizeof(mm_step_result);
        case MM_STRUCT_PROFILE: return (int64_t)sizeof(mm_profile);
        case MM_STRUCT_LCE_PARAMS: return (int64_t)sizeof(mm_lce_params);
        case MM_STRUCT_SOLVE_PARAMS: return (int64_t)sizeof(mm_solve_params);
        case MM_STRUCT_SOLVE_RESULT: return (int64_t)sizeof(mm_solve_result);
        default: return -1;
    }
}

const char *mm_last_error(const mm_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t mm_device_bytes(const mm_ctx *ctx) { return ctx ? ctx->bytes : 0; }

int mm_create(int dim, int n, double length, int device, mm_ctx **out) {
    if (!out) return MM_ERR_PARAM;
    *out = nullptr;
    if (dim != 2 && dim != 3) return MM_ERR_CONFIG;
    if (n < 4) return MM_ERR_CONFIG;
    if (!(length > 0.0)) return MM_ERR_CONFIG;
    mm_ctx *ctx = new mm_ctx();
    ctx->dim = dim;
    ctx->n = n;
    ctx->L = length;
    ctx->h = 2.0 * length / n;  // grid.py:84-86
    ctx->M = 1;
    for (int i = 0; i < dim; ++i) ctx->M *= n;
    ctx->D = dim * dim;
    ctx->nh = n / 2 + 1;
    ctx->P = (ctx->nh + 7) / 8 * 8;
    ctx->nrows = ctx->M / n;
    ctx->uM = ctx->dM = ctx->M;
    ctx->device = device;
    *out = ctx;
    int rc;
#define TRY(x)                 \
    do {                       \
        rc = (x);              \
        if (rc) return rc;     \
    } while (0)
    MM_CUDA(ctx, cudaSetDevice(device));
    if (!take_recycled(ctx))
        MM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    MM_CUDA(ctx, cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    const int64_t M = ctx->M;
    TRY(mm_alloc(ctx, (void **)&ctx->F, sizeof(double) * ctx->D * M));
    TRY(mm_alloc(ctx, (void **)&ctx->G, sizeof(double) * ctx->D * M));
    TRY(mm_alloc(ctx, (void **)&ctx->Lam, sizeof(double) * ctx->D * M));
    TRY(mm_alloc(ctx, (void **)&ctx->Ut, sizeof(double) * dim * M));
    TRY(mm_alloc(ctx, (void **)&ctx->spec, sizeof(double2) * dim * ctx->nrows * ctx->P));
    TRY(mm_alloc(ctx, (void **)&ctx->sym, sizeof(double) * dim * n));
    TRY(alloc_red_out(ctx));
    TRY(mm_alloc(ctx, (void **)&ctx->red_count, sizeof(unsigned int) * 4));
    MM_CUDA(ctx, cudaMemset(ctx->red_count, 0, sizeof(unsigned int) * 4));
    MM_CUDA(ctx, cudaMemsetAsync(ctx->F, 0, sizeof(double) * ctx->D * M, ctx->stream));
    MM_CUDA(ctx, cudaMemsetAsync(ctx->G, 0, sizeof(double) * ctx->D * M, ctx->stream));
    MM_CUDA(ctx, cudaMemsetAsync(ctx->Lam, 0, sizeof(double) * ctx->D * M, ctx->stream));
    MM_CUDA(ctx, cudaMemsetAsync(ctx->Ut, 0, sizeof(double) * dim * M, ctx->stream));
    MM_CUDA(ctx, cudaMemsetAsync(ctx->spec, 0, sizeof(double2) * dim * ctx->nrows * ctx->P,
                                 ctx->stream));
    TRY(upload_tw(ctx, &ctx->tw_full, n));
    TRY(upload_tw(ctx, &ctx->tw_half, n / 2));
    TRY(upload_tw(ctx, &ctx->tw_r2c, n));
    TRY(mm_ensure_partials(ctx, 4096));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
#undef TRY
    return MM_OK;
}

int mm_create_slab(int n, double length, int nranks, int rank, int device, mm_ctx **out) {
    if (!out) return MM_ERR_PARAM;
    *out = nullptr;
    if (n < 4 || n % 2 || nranks < 1 || n % nranks || rank < 0 || rank >= nranks ||
        !(length > 0.0))
        return MM_ERR_CONFIG;
    mm_ctx *ctx = new mm_ctx();
    const int dim = 3;
    ctx->dim = dim;
    ctx->n = n;
    ctx->L = length;
    ctx->h = 2.0 * length / n;
    ctx->slab_mode = true;
    ctx->slab_P = nranks;
    ctx->slab_rank = rank;
    ctx->slab_nl = n / nranks;
    ctx->M = (int64_t)ctx->slab_nl * n * n;
    ctx->D = 9;
    ctx->nh = n / 2 + 1;
    ctx->P = (ctx->nh + 7) / 8 * 8;
    ctx->nrows = (int64_t)ctx->slab_nl * n;
    ctx->device = device;
    *out = ctx;
    int rc;
#define TRY(x)             \
    do {                   \
        rc = (x);          \
        if (rc) return rc; \
    } while (0)
    MM_CUDA(ctx, cudaSetDevice(device));
    MM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    MM_CUDA(ctx, cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
    const int64_t M = ctx->M;
    const int64_t nn = (int64_t)n * n;
    const int64_t nl = ctx->slab_nl;
    TRY(mm_alloc(ctx, (void **)&ctx->F, sizeof(double) * 9 * M));
    TRY(mm_alloc(ctx, (void **)&ctx->G, sizeof(double) * 9 * M));
    TRY(mm_alloc(ctx, (void **)&ctx->Lam, sizeof(double) * 9 * M));
    // u_tilde double buffer with one ghost plane on each slab face
    ctx->uM = M + 2 * nn;
    ctx->dM = M + 4 * nn;
    TRY(mm_alloc(ctx, (void **)&ctx->Ut_base, sizeof(double) * 3 * ctx->uM));
    TRY(mm_alloc(ctx, (void **)&ctx->Ut2_base, sizeof(double) * 3 * ctx->uM));
    ctx->Ut = ctx->Ut_base + nn;
    ctx->Ut2 = ctx->Ut2_base + nn;
    TRY(mm_alloc(ctx, (void **)&ctx->spec, sizeof(double2) * 3 * ctx->nrows * ctx->P));
    const int64_t bufc = (int64_t)nranks * 3 * nl * nl * ctx->P;
    // exchange buffers by plain cudaMalloc: CUDA IPC exports need it
    MM_CUDA(ctx, cudaMalloc((void **)&ctx->sendbuf, sizeof(double2) * bufc));
    MM_CUDA(ctx, cudaMalloc((void **)&ctx->recvbuf, sizeof(double2) * bufc));
    ctx->bytes += 2 * (int64_t)sizeof(double2) * bufc;
    TRY(mm_alloc(ctx, (void **)&ctx->halo_in_lo, sizeof(double) * 3 * nn));
    TRY(mm_alloc(ctx, (void **)&ctx->halo_in_hi, sizeof(double) * 3 * nn));
    TRY(mm_alloc(ctx, (void **)&ctx->halo_out_lo, sizeof(double) * 3 * nn));
    TRY(mm_alloc(ctx, (void **)&ctx->halo_out_hi, sizeof(double) * 3 * nn));
    TRY(mm_alloc(ctx, (void **)&ctx->sym, sizeof(double) * dim * n));
    TRY(mm_alloc(ctx, (void **)&ctx->red_out, sizeof(double) * MM_MAX_PARTIALS));
    TRY(mm_alloc(ctx, (void **)&ctx->red_count, sizeof(unsigned int) * 4));
    MM_CUDA(ctx, cudaMemset(ctx->red_count, 0, sizeof(unsigned int) * 4));
    MM_CUDA(ctx, cudaMallocHost((void **)&ctx->host_out, sizeof(double) * MM_MAX_PARTIALS));
    MM_CUDA(ctx, cudaMemset(ctx->F, 0, sizeof(double) * 9 * M));
    MM_CUDA(ctx, cudaMemset(ctx->G, 0, sizeof(double) * 9 * M));
    MM_CUDA(ctx, cudaMemset(ctx->Lam, 0, sizeof(double) * 9 * M));
    MM_CUDA(ctx, cudaMemset(ctx->Ut_base, 0, sizeof(double) * 3 * ctx->uM));
    MM_CUDA(ctx, cudaMemset(ctx->Ut2_base, 0, sizeof(double) * 3 * ctx->uM));
    MM_CUDA(ctx, cudaMemset(ctx->spec, 0, sizeof(double2) * 3 * ctx->nrows * ctx->P));
    MM_CUDA(ctx, cudaMemset(ctx->sendbuf, 0, sizeof(double2) * bufc));
    MM_CUDA(ctx, cudaMemset(ctx->recvbuf, 0, sizeof(double2) * bufc));
    TRY(upload_tw(ctx, &ctx->tw_full, n));
    TRY(upload_tw(ctx, &ctx->tw_half, n / 2));
    TRY(upload_tw(ctx, &ctx->tw_r2c, n));
    TRY(mm_ensure_partials(ctx, 4096));
#undef TRY
    return MM_OK;
}

int mm_slab_buffer(mm_ctx *ctx, int which, void **dev_ptr, int64_t *nbytes) {
    if (!ctx || !dev_ptr || !nbytes) return MM_ERR_PARAM;
    if (!ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "not a slab context");
    const int64_t nn = (int64_t)ctx->n * ctx->n;
    const int64_t nl = ctx->slab_nl;
    const int64_t bufb = (int64_t)ctx->slab_P * 3 * nl * nl * ctx->P * (int64_t)sizeof(double2);
    switch (which) {
        case MM_SLAB_BUF_SEND: *dev_ptr = ctx->sendbuf; *nbytes = bufb; break;
        case MM_SLAB_BUF_RECV: *dev_ptr = ctx->recvbuf; *nbytes = bufb; break;
        case MM_SLAB_BUF_HALO_OUT_LO: *dev_ptr = ctx->halo_out_lo; *nbytes = 3 * nn * 8; break;
        case MM_SLAB_BUF_HALO_OUT_HI: *dev_ptr = ctx->halo_out_hi; *nbytes = 3 * nn * 8; break;
        case MM_SLAB_BUF_HALO_IN_LO: *dev_ptr = ctx->halo_in_lo; *nbytes = 3 * nn * 8; break;
        case MM_SLAB_BUF_HALO_IN_HI: *dev_ptr = ctx->halo_in_hi; *nbytes = 3 * nn * 8; break;
        default: return mm_fail(ctx, MM_ERR_PARAM, "unknown slab buffer %d", which);
    }
    return MM_OK;
}

int mm_slab_step(mm_ctx *ctx, int step, double rho, const double *u_mean, double *sums) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (!ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "not a slab context");
    if (!(rho > 0.0) || !isfinite(rho))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho);
    if (!ctx->have_sym) return mm_fail(ctx, MM_ERR_CONFIG, "symbols were never set");
    if (step == MM_SLAB_RES && (!u_mean || !sums)) return MM_ERR_PARAM;
    if (step >= 4 && step <= 6) return mm_fail(ctx, MM_ERR_PARAM, "slab step %d was retired", step);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    // the projection reads F and lam (or T): a deferred ascent lands first
    if (step == MM_SLAB_HALO_T || step == MM_SLAB_DIRECTOR) {
        int rc = mm_flush_pending(ctx);
        if (rc) return rc;
    }
    if (step == MM_SLAB_DIRECTOR || step == MM_SLAB_FRANK) return mm_run_slab_lce(ctx, step);
    return mm_run_slab_step(ctx, step, rho, u_mean, sums);
}

int mm_slab_field(mm_ctx *ctx, int which, void **base, int64_t *cstride, int *ncomp,
                  int *ghost) {
    if (!ctx || !base || !cstride || !ncomp || !ghost) return MM_ERR_PARAM;
    if (!ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "not a slab context");
    *ncomp = 3;
    switch (which) {
        case MM_SLAB_FIELD_U_NEW: *base = ctx->Ut2; *cstride = ctx->uM; *ghost = 1; break;
        case MM_SLAB_FIELD_U: *base = ctx->Ut; *cstride = ctx->uM; *ghost = 1; break;
        case MM_SLAB_FIELD_DIRECTOR: {
            int rc = mm_slab_alloc_director(ctx);
            if (rc) return rc;
            *base = ctx->dirbuf; *cstride = ctx->dM; *ghost = 2; break;
        }
        default: return mm_fail(ctx, MM_ERR_PARAM, "unknown slab field %d", which);
    }
    return MM_OK;
}

int mm_slab_stream(mm_ctx *ctx, void **stream) {
    if (!ctx || !stream) return MM_ERR_PARAM;
    *stream = (void *)ctx->stream;
    return MM_OK;
}

static int peer_table(mm_ctx *ctx, int which, double2 ****slot) {
    if (!ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "not a slab context");
    if (which == MM_SLAB_BUF_RECV) *slot = &ctx->peer_recv;
    else if (which == MM_SLAB_BUF_SEND) *slot = &ctx->peer_send;
    else return mm_fail(ctx, MM_ERR_PARAM, "peer buffers are SEND or RECV, got %d", which);
    if (!**slot) {
        int rc = mm_alloc(ctx, (void **)*slot, sizeof(double2 *) * ctx->slab_P);
        if (rc) return rc;
    }
    return MM_OK;
}

int mm_slab_set_peers(mm_ctx *ctx, int which, void *const *ptrs, int P) {
    if (!ctx || !ptrs) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (P != ctx->slab_P) return mm_fail(ctx, MM_ERR_CONFIG, "expected %d peers, got %d", ctx->slab_P, P);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    double2 ***slot;
    int rc = peer_table(ctx, which, &slot);
    if (rc) return rc;
    MM_CUDA(ctx, cudaMemcpy(*slot, ptrs, sizeof(void *) * P, cudaMemcpyHostToDevice));
    return MM_OK;
}

int mm_slab_ipc_handle(mm_ctx *ctx, int which, void *handle_out) {
    if (!ctx || !handle_out) return MM_ERR_PARAM;
    if (!ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "not a slab context");
    void *buf = which == MM_SLAB_BUF_RECV ? (void *)ctx->recvbuf
              : which == MM_SLAB_BUF_SEND ? (void *)ctx->sendbuf : nullptr;
    if (!buf) return mm_fail(ctx, MM_ERR_PARAM, "peer buffers are SEND or RECV, got %d", which);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    MM_CUDA(ctx, cudaIpcGetMemHandle(&h, buf));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(handle_out, &h, 64);
    return MM_OK;
}

int mm_slab_open_peers(mm_ctx *ctx, int which, const void *handles, int P) {
    if (!ctx || !handles) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (P != ctx->slab_P) return mm_fail(ctx, MM_ERR_CONFIG, "expected %d peers, got %d", ctx->slab_P, P);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    std::vector<void *> ptrs(P);
    for (int q = 0; q < P; ++q) {
        if (q == ctx->slab_rank) {
            ptrs[q] = which == MM_SLAB_BUF_RECV ? (void *)ctx->recvbuf : (void *)ctx->sendbuf;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, (const char *)handles + 64 * q, 64);
        void *p = nullptr;
        MM_CUDA(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        ctx->ipc_opened.push_back(p);
        ptrs[q] = p;
    }
    return mm_slab_set_peers(ctx, which, ptrs.data(), P);
}

int mm_create_points(int dim, int64_t npts, int device, mm_ctx **out) {
    if (!out) return MM_ERR_PARAM;
    *out = nullptr;
    if (dim != 2 && dim != 3) return MM_ERR_CONFIG;
    if (npts < 0) return MM_ERR_CONFIG;
    mm_ctx *ctx = new mm_ctx();
    ctx->dim = dim;
    ctx->n = 0;
    ctx->M = npts;
    ctx->uM = ctx->dM = npts;
    ctx->D = dim * dim;
    ctx->device = device;
    ctx->points_only = true;
    *out = ctx;
    int rc;
    MM_CUDA(ctx, cudaSetDevice(device));
    if (!take_recycled(ctx))
        MM_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    const int64_t M = npts > 0 ? npts : 1;
    if ((rc = mm_alloc(ctx, (void **)&ctx->F, sizeof(double) * ctx->D * M))) return rc;
    if ((rc = mm_alloc(ctx, (void **)&ctx->G, sizeof(double) * ctx->D * M))) return rc;
    if ((rc = mm_alloc(ctx, (void **)&ctx->Lam, sizeof(double) * ctx->D * M))) return rc;
    if ((rc = alloc_red_out(ctx))) return rc;
    if ((rc = mm_alloc(ctx, (void **)&ctx->red_count, sizeof(unsigned int) * 4))) return rc;
    MM_CUDA(ctx, cudaMemset(ctx->red_count, 0, sizeof(unsigned int) * 4));
    if ((rc = mm_ensure_partials(ctx, 4096))) return rc;
    return MM_OK;
}

void mm_destroy(mm_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    mm_drain_timings(ctx);
    for (cudaEvent_t e : ctx->event_pool) cudaEventDestroy(e);
    mm_bloch_free(ctx);
    if (ctx->Ut_base) ctx->Ut = ctx->Ut_base;
    if (ctx->Ut2_base) ctx->Ut2 = ctx->Ut2_base;
    if (ctx->dir_base) ctx->dirbuf = ctx->dir_base;
    if (ctx->red_mapped) ctx->red_out = nullptr;  // host_out's device alias
    double *ptrs[] = {ctx->F, ctx->G, ctx->Lam, ctx->Ut, ctx->prevF, ctx->modA, ctx->modB,
                      ctx->ang, ctx->chart, ctx->pinc, ctx->n0, ctx->ff, ctx->prevAng,
                      ctx->prevChart, ctx->prevPinc, ctx->dirbuf, ctx->Ut2, ctx->halo_in_lo,
                      ctx->halo_in_hi, ctx->halo_out_lo, ctx->halo_out_hi, ctx->sym, ctx->partials, ctx->red_out,
                      ctx->res, ctx->tstate, ctx->stage, ctx->Pbuf, ctx->Tbuf};
    for (double *p : ptrs) mm_free(ctx, p);
    void *lce_bufs[] = {ctx->lce_fsq0, ctx->lce_list[0], ctx->lce_list[1], ctx->lce_cnt,
                        ctx->dstep};
    for (void *p : lce_bufs) mm_free(ctx, p);
    void *others[] = {ctx->spec, ctx->tw_full, ctx->tw_half, ctx->tw_r2c, ctx->red_count,
                      ctx->nsw, ctx->ok, ctx->freestate, ctx->peer_recv, ctx->peer_send};
    for (void *p : others) mm_free(ctx, p);
    for (void *p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
    if (ctx->sendbuf) cudaFree(ctx->sendbuf);
    if (ctx->recvbuf) cudaFree(ctx->recvbuf);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->ev_red) cudaEventDestroy(ctx->ev_red);
    if (ctx->ev_k1) cudaEventDestroy(ctx->ev_k1);
    if (ctx->xfer_ev[0]) cudaEventDestroy(ctx->xfer_ev[0]);
    if (ctx->xfer_ev[1]) cudaEventDestroy(ctx->xfer_ev[1]);
    if (park_recycled(ctx)) {
        ctx->stream = nullptr;
        ctx->host_out = nullptr;
    }
    if (ctx->host_out) cudaFreeHost(ctx->host_out);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int mm_synchronize(mm_ctx *ctx) {
    if (!ctx) return MM_ERR_PARAM;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_drain_timings(ctx);
    return MM_OK;
}

int mm_profile_enable(mm_ctx *ctx, int on) {
    if (!ctx) return MM_ERR_PARAM;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_drain_timings(ctx);
    ctx->prof_on = on != 0;
    return MM_OK;
}

int mm_profile_read(mm_ctx *ctx, mm_profile *out, int reset) {
    if (!ctx || !out) return MM_ERR_PARAM;
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_drain_timings(ctx);
    for (int i = 0; i < MM_NSTAGE; ++i) {
        out->ms[i] = ctx->prof_ms[i];
        out->launches[i] = ctx->launches[i];
        if (reset) {
            ctx->prof_ms[i] = 0.0;
            ctx->launches[i] = 0;
            ctx->prof_launches[i] = 0;
        }
    }
    return MM_OK;
}

int mm_upload(mm_ctx *ctx, int field, const double *host, int64_t count) {
    if (!ctx || !host) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    double **slot;
    int ncomp;
    int rc = field_info(ctx, field, &slot, &ncomp);
    if (rc) return rc;
    if (count != ctx->M * ncomp)
        return mm_fail(ctx, MM_ERR_CONFIG, "field %d: got %lld doubles, expected %lld", field,
                       (long long)count, (long long)(ctx->M * ncomp));
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    rc = ensure_field(ctx, slot, ncomp);
    if (rc) return rc;
    if (field == MM_FIELD_F) ctx->F_checked = false;
    if (field == MM_FIELD_F || field == MM_FIELD_LAM) ctx->T_valid = false;
    if (field == MM_FIELD_PREV_F) ctx->have_prev_F = true;
    if (field == MM_FIELD_PREV_ANG) ctx->have_prev_int = true;
    if (field == MM_FIELD_UT && ctx->g_implicit) {
        // grad_u was held as ubar + D u_tilde: pin it before u_tilde changes
        if ((rc = mm_materialize_G(ctx))) return rc;
        ctx->g_implicit = false;
    }
    if (field == MM_FIELD_G) {
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    }
    return transfer(ctx, *slot, ncomp, host, nullptr, false, field_cs(ctx, field));
}

int mm_add_field(mm_ctx *ctx, int field, const double *host, int64_t count) {
    if (!ctx || !host) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    if (field != MM_FIELD_F && field != MM_FIELD_LAM && field != MM_FIELD_PREV_F)
        return mm_fail(ctx, MM_ERR_PARAM, "mm_add_field: field %d is not F, LAM or PREV_F", field);
    double **slot;
    int ncomp;
    int rc = field_info(ctx, field, &slot, &ncomp);
    if (rc) return rc;
    if (count != ctx->M * ncomp)
        return mm_fail(ctx, MM_ERR_CONFIG, "field %d: got %lld doubles, expected %lld", field,
                       (long long)count, (long long)(ctx->M * ncomp));
    if (!*slot) return mm_fail(ctx, MM_ERR_CONFIG, "field %d was never set", field);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    if (field == MM_FIELD_F) ctx->F_checked = false;
    if (field == MM_FIELD_F || field == MM_FIELD_LAM) ctx->T_valid = false;
    return transfer(ctx, *slot, ncomp, host, nullptr, true);
}

int mm_equilibrium_residual(mm_ctx *ctx, int material, double dt, double *out) {
    if (!ctx || !out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (ctx->slab_mode)
        return mm_fail(ctx, MM_ERR_CONFIG, "equilibrium_residual is single-context only");
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    if (!ctx->F) return mm_fail(ctx, MM_ERR_CONFIG, "F was never set");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc;
    if (!ctx->Pbuf && (rc = mm_alloc(ctx, (void **)&ctx->Pbuf, sizeof(double) * ctx->D * ctx->M)))
        return rc;
    switch (material) {
        case MM_MAT_MR:
        case MM_MAT_MR_DESCENT: {
            int bad = 0;  // MaterialModel._check_det (base.py:116-121) in stress()
            if ((rc = mm_check_det(ctx, &bad))) return rc;
            if (bad) return mm_fail(ctx, MM_ERR_INADMISSIBLE, "det F <= 0 at %d point(s)", bad);
            rc = mm_run_stress(ctx, material, ctx->Pbuf);
            break;
        }
        case MM_MAT_QUADRATIC: rc = mm_run_stress(ctx, material, ctx->Pbuf); break;
        case MM_MAT_LCE: rc = mm_run_lce_stress(ctx, dt, ctx->Pbuf); break;
        default: return mm_fail(ctx, MM_ERR_PARAM, "unknown material %d", material);
    }
    if (rc) return rc;
    return mm_run_eq_residual(ctx, ctx->Pbuf, out);
}

int mm_download(mm_ctx *ctx, int field, double *host, int64_t count) {
    if (!ctx || !host) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    double **slot;
    int ncomp;
    int rc = field_info(ctx, field, &slot, &ncomp);
    if (rc) return rc;
    if (count != ctx->M * ncomp)
        return mm_fail(ctx, MM_ERR_CONFIG, "field %d: got %lld doubles, expected %lld", field,
                       (long long)count, (long long)(ctx->M * ncomp));
    if (!*slot) return mm_fail(ctx, MM_ERR_CONFIG, "field %d was never set", field);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    if (field == MM_FIELD_G && (rc = mm_materialize_G(ctx))) return rc;
    return transfer(ctx, *slot, ncomp, nullptr, host, false, field_cs(ctx, field));
}

int mm_copy_field(mm_ctx *ctx, int dst_field, int src_field) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    double **ds, **ss;
    int nd, ns;
    int rc = field_info(ctx, dst_field, &ds, &nd);
    if (rc) return rc;
    rc = field_info(ctx, src_field, &ss, &ns);
    if (rc) return rc;
    if (nd != ns) return mm_fail(ctx, MM_ERR_CONFIG, "field shapes differ");
    if (!*ss) return mm_fail(ctx, MM_ERR_CONFIG, "source field %d was never set", src_field);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    if ((src_field == MM_FIELD_G || dst_field == MM_FIELD_UT) && (rc = mm_materialize_G(ctx)))
        return rc;
    if (dst_field == MM_FIELD_UT) ctx->g_implicit = false;
    if (dst_field == MM_FIELD_F || dst_field == MM_FIELD_LAM) ctx->T_valid = false;
    if (dst_field == MM_FIELD_G) {
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    }
    rc = ensure_field(ctx, ds, nd);
    if (rc) return rc;
    const int64_t dcs = field_cs(ctx, dst_field), scs = field_cs(ctx, src_field);
    if (dcs == ctx->M && scs == ctx->M)
        MM_CUDA(ctx, cudaMemcpyAsync(*ds, *ss, sizeof(double) * nd * ctx->M,
                                     cudaMemcpyDeviceToDevice, ctx->stream));
    else
        for (int c = 0; c < nd; ++c)
            MM_CUDA(ctx, cudaMemcpyAsync(*ds + c * dcs, *ss + c * scs, sizeof(double) * ctx->M,
                                         cudaMemcpyDeviceToDevice, ctx->stream));
    if (dst_field == MM_FIELD_PREV_F) ctx->have_prev_F = true;
    if (dst_field == MM_FIELD_PREV_ANG) ctx->have_prev_int = true;
    if (dst_field == MM_FIELD_F) ctx->F_checked = false;
    return MM_OK;
}

int mm_field_sums(mm_ctx *ctx, int field, double *out) {
    if (!ctx || !out) return MM_ERR_PARAM;
    {
        int prc = mm_flush_pending(ctx);
        if (prc) return prc;
    }
    double **slot;
    int ncomp;
    int rc = field_info(ctx, field, &slot, &ncomp);
    if (rc) return rc;
    if (!*slot) return mm_fail(ctx, MM_ERR_CONFIG, "field %d was never set", field);
    if (field_cs(ctx, field) != ctx->M)
        return mm_fail(ctx, MM_ERR_CONFIG, "field sums of u_tilde on a slab are not supported");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    return mm_run_field_sums(ctx, *slot, ncomp, out);
}

int mm_set_symbols(mm_ctx *ctx, const double *axis_tab, double threshold) {
    if (!ctx || !axis_tab) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    MM_CUDA(ctx, cudaMemcpy(ctx->sym, axis_tab, sizeof(double) * ctx->dim * ctx->n,
                            cudaMemcpyHostToDevice));
    ctx->sym_thresh = threshold;
    ctx->have_sym = true;
    return MM_OK;
}

int mm_set_lce(mm_ctx *ctx, const mm_lce_params *p) {
    if (!ctx || !p) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    ctx->lce = *p;
    ctx->have_lce = true;
    return MM_OK;
}

int mm_local_sweeps(mm_ctx *ctx, int material, double rho, double tol, int64_t max_sweeps,
                    double phi_scale, int want_points, mm_local_stats *out) {
    if (!ctx || !out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (!(rho > 0.0) || !isfinite(rho))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho);
    if (max_sweeps < 0) return mm_fail(ctx, MM_ERR_PARAM, "max_sweeps must be >= 0");
    if ((material == MM_MAT_MR || material == MM_MAT_QUADRATIC) && !ctx->modA)
        return mm_fail(ctx, MM_ERR_CONFIG, "material moduli were never uploaded");
    if (material == MM_MAT_MR && !ctx->modB)
        return mm_fail(ctx, MM_ERR_CONFIG, "kappa was never uploaded");
    if (material == MM_MAT_LCE && !ctx->have_lce)
        return mm_fail(ctx, MM_ERR_CONFIG, "LCE parameters were never set");
    if (material < 0 || material > 3) return mm_fail(ctx, MM_ERR_CONFIG, "unknown material");
    if (material == MM_MAT_MR_DESCENT && (!ctx->modA || !ctx->modB))
        return mm_fail(ctx, MM_ERR_CONFIG, "material moduli were never uploaded");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    return mm_run_local(ctx, material, rho, tol, max_sweeps, phi_scale, want_points, out);
}

int mm_download_points(mm_ctx *ctx, double *res, int64_t *nsw, uint8_t *ok, int64_t npts) {
    if (!ctx) return MM_ERR_PARAM;
    if (npts != ctx->M) return mm_fail(ctx, MM_ERR_CONFIG, "npts mismatch");
    if (!ctx->res) return mm_fail(ctx, MM_ERR_CONFIG, "no per-point results kept");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    if (res)
        MM_CUDA(ctx, cudaMemcpyAsync(res, ctx->res, sizeof(double) * npts, cudaMemcpyDeviceToHost,
                                     ctx->stream));
    std::vector<int32_t> tmp;
    if (nsw) {
        tmp.resize(npts);
        MM_CUDA(ctx, cudaMemcpyAsync(tmp.data(), ctx->nsw, sizeof(int32_t) * npts,
                                     cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (ok)
        MM_CUDA(ctx, cudaMemcpyAsync(ok, ctx->ok, npts, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    if (nsw)
        for (int64_t i = 0; i < npts; ++i) nsw[i] = tmp[i];
    return MM_OK;
}

int mm_prepare_frozen(mm_ctx *ctx) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (!ctx->have_lce) return mm_fail(ctx, MM_ERR_CONFIG, "LCE parameters were never set");
    if (ctx->slab_mode)
        return mm_fail(ctx, MM_ERR_CONFIG,
                       "slab context: run MM_SLAB_DIRECTOR, the ghost exchange, MM_SLAB_FRANK");
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    return mm_run_frozen(ctx);
}

int mm_project(mm_ctx *ctx, double rho, const double *u_mean) {
    if (!ctx || !u_mean) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "slab context: use mm_slab_step");
    if (!(rho > 0.0) || !isfinite(rho))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho);
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (!ctx->have_sym) return mm_fail(ctx, MM_ERR_CONFIG, "symbols were never set");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    return mm_run_project(ctx, rho, u_mean, 0, nullptr);
}

int mm_project_residuals(mm_ctx *ctx, double rho, const double *u_mean, mm_update_stats *out) {
    if (!ctx || !u_mean || !out) return MM_ERR_PARAM;
    if (ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "slab context: use mm_slab_step");
    if (!(rho > 0.0) || !isfinite(rho))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho);
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (!ctx->have_sym) return mm_fail(ctx, MM_ERR_CONFIG, "symbols were never set");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    return mm_run_project(ctx, rho, u_mean, 2, out);
}

int mm_update_multiplier(mm_ctx *ctx, mm_update_stats *out) {
    if (!ctx || !out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    return mm_run_update(ctx, 0, 0.0, 0.0, 0, 0.0, 0, nullptr, out);
}

int mm_update_and_sweep(mm_ctx *ctx, int material, double rho_next, double tol,
                        int64_t max_sweeps, double phi_scale, int want_points,
                        mm_local_stats *ls, mm_update_stats *us) {
    if (!ctx || !ls || !us) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (!(rho_next > 0.0) || !isfinite(rho_next))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho_next);
    if (max_sweeps < 0) return mm_fail(ctx, MM_ERR_PARAM, "max_sweeps must be >= 0");
    if ((material == MM_MAT_MR || material == MM_MAT_MR_DESCENT || material == MM_MAT_QUADRATIC) &&
        !ctx->modA)
        return mm_fail(ctx, MM_ERR_CONFIG, "material moduli were never uploaded");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    memset(ls, 0, sizeof *ls);
    return mm_run_update(ctx, material, rho_next, tol, max_sweeps, phi_scale, want_points, ls, us);
}

// One pipelined step: K1 (whose last block also takes the decision,
// decide_step), the fused pass (parameters from the device) and the
// speculative front are queued back to back; the host then
// reads K1's sums, takes the same decision, checks it against the device's
// and finishes.  The GPU never waits for the host between K1 and the fused
// pass.
static int residuals_and_step_pipelined(mm_ctx *ctx, const mm_step_params *p,
                                        mm_step_result *out, mm_local_stats *ls) {
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    if (!ctx->dstep && (rc = mm_alloc(ctx, (void **)&ctx->dstep, sizeof(DevStep)))) return rc;
    if (!ctx->ev_k1) MM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_k1, cudaEventDisableTiming));
    double *k1 = ctx->red_out + MM_MAX_PARTIALS;
    double *dcopy = ctx->red_out + 2 * MM_MAX_PARTIALS;
    ctx->k1_dst = k1;
    ctx->k1_decide.on = 1;
    ctx->k1_decide.p = *p;
    ctx->k1_decide.ds = ctx->dstep;
    ctx->k1_decide.copy = dcopy;
    rc = mm_run_project(ctx, p->rho, p->u_mean, 2, nullptr);
    ctx->k1_dst = nullptr;
    ctx->k1_decide.on = 0;
    if (rc) return rc;
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_k1, ctx->stream));
    ctx->gen++;  // (mm_update_and_sweep's) the front below is this call's
    if ((rc = mm_run_update_pipe(ctx, p->material, p->rho, p->chunk, p->phi_scale))) return rc;
    MM_CUDA(ctx, cudaEventSynchronize(ctx->ev_k1));
    const double *hk1 = ctx->host_out + MM_MAX_PARTIALS;
    const double r_d = p->rho * sqrt(hk1[0] / p->npts) / p->mu_rep;
    const double r_p = sqrt(hk1[1] / p->npts);
    out->r_d = r_d;
    out->r_p = r_p;
    double rho = p->rho;
    bool swept = false;
    double tol = 0.0;
    if (!isfinite(r_p) || r_p > p->divergence_limit) {
        out->diverged = 1;
    } else {
        if (p->adapt && p->outer_iter > 1) {
            if (r_p > p->tau_adapt * r_d) {
                rho *= p->kappa_adapt;
            } else if (r_d > p->tau_adapt * r_p) {
                const double a = rho / p->kappa_adapt;
                rho = (p->rho_floor > a) ? p->rho_floor : a;
            }
        }
        out->done = (r_p <= p->r_p_tol && r_d <= p->r_d_tol && p->r_l <= p->r_l_tol) ? 1 : 0;
        if (!out->done) {
            tol = p->point_tol;
            if (p->ratio_policy) {
                if (!isfinite(r_d)) tol = 1.0;
                else {
                    const double b = p->ratio * r_d;
                    tol = (b > p->point_tol) ? b : p->point_tol;
                }
            }
            tol *= p->mu_rep;
            swept = true;
        }
    }
    out->rho_next = out->diverged ? p->rho : rho;
    mm_update_stats us;
    memset(&us, 0, sizeof us);
    if ((rc = mm_run_update_pipe_finish(ctx, swept, rho, ls, &us))) return rc;
    // the fused pass ran with the device's decision: it must be this one
    const double *hc = ctx->host_out + 2 * MM_MAX_PARTIALS;
    const bool same = (hc[0] != 0.0) == !swept &&
                      (!swept || (hc[1] == rho && hc[2] == tol)) &&
                      (out->diverged || hc[1] == rho);
    if (!same)
        return mm_fail(ctx, MM_ERR_CONFIG,
                       "pipelined step: device decision (skip %g, rho %.17g, tol %.17g) differs "
                       "from the host's (skip %d, rho %.17g, tol %.17g)",
                       hc[0], hc[1], hc[2], swept ? 0 : 1, rho, tol);
    if (swept) {
        out->swept = 1;
    } else if ((rc = mm_update_multiplier(ctx, &us))) {
        return rc;
    }
    memcpy(out->sum_lam, us.sum_lam, sizeof us.sum_lam);
    return MM_OK;
}

// the decisions of solver.py's fused loop, in the Python loop's float order
int mm_residuals_and_step(mm_ctx *ctx, const mm_step_params *p, mm_step_result *out,
                          mm_local_stats *ls) {
    if (!ctx || !p || !out || !ls) return MM_ERR_PARAM;
    if (ctx->opt_pipeline && ctx->red_mapped && !ctx->slab_mode && !ctx->points_only &&
        !p->last_allowed && ctx->have_sym && ctx->modA && p->chunk <= 64 &&
        (p->material == MM_MAT_MR || p->material == MM_MAT_MR_DESCENT ||
         p->material == MM_MAT_QUADRATIC) &&
        p->rho > 0.0 && isfinite(p->rho)) {
        memset(out, 0, sizeof *out);
        memset(ls, 0, sizeof *ls);
        MM_CUDA(ctx, cudaSetDevice(ctx->device));
        return residuals_and_step_pipelined(ctx, p, out, ls);
    }
    int rc = mm_project_residuals(ctx, p->rho, p->u_mean, &ctx->step_us);
    if (rc) return rc;
    const mm_update_stats &up = ctx->step_us;
    memset(out, 0, sizeof *out);
    memset(ls, 0, sizeof *ls);
    const double r_d = p->rho * sqrt(up.sum_dG2 / p->npts) / p->mu_rep;
    const double r_p = sqrt(up.sum_mis2 / p->npts);
    out->r_d = r_d;
    out->r_p = r_p;
    double rho = p->rho;
    mm_update_stats us;
    if (!isfinite(r_p) || r_p > p->divergence_limit) {
        out->diverged = 1;
        out->rho_next = rho;
        if ((rc = mm_update_multiplier(ctx, &us))) return rc;
        memcpy(out->sum_lam, us.sum_lam, sizeof us.sum_lam);
        return MM_OK;
    }
    if (p->adapt && p->outer_iter > 1) {
        if (r_p > p->tau_adapt * r_d) {
            rho *= p->kappa_adapt;
        } else if (r_d > p->tau_adapt * r_p) {
            const double a = rho / p->kappa_adapt;  // Python max(a, b): a unless b > a
            rho = (p->rho_floor > a) ? p->rho_floor : a;
        }
    }
    out->rho_next = rho;
    out->done = (r_p <= p->r_p_tol && r_d <= p->r_d_tol && p->r_l <= p->r_l_tol) ? 1 : 0;
    if (out->done || p->last_allowed) {
        if ((rc = mm_update_multiplier(ctx, &us))) return rc;
    } else {
        double tol = p->point_tol;
        if (p->ratio_policy) {
            if (!isfinite(r_d)) tol = 1.0;
            else {
                const double b = p->ratio * r_d;
                tol = (b > p->point_tol) ? b : p->point_tol;
            }
        }
        if ((rc = mm_update_and_sweep(ctx, p->material, rho, tol * p->mu_rep, p->chunk,
                                      p->phi_scale, 0, ls, &us)))
            return rc;
        out->swept = 1;
    }
    memcpy(out->sum_lam, us.sum_lam, sizeof us.sum_lam);
    return MM_OK;
}

// solve()'s fused loop (solver.py _solve_fused, device-decided branch),
// statement for statement in the Python loop's float order
int mm_solve_fused(mm_ctx *ctx, const mm_solve_params *p, mm_solve_result *r, double *hist) {
    if (!ctx || !p || !r || !hist) return MM_ERR_PARAM;
    if (ctx->slab_mode || ctx->points_only)
        return mm_fail(ctx, MM_ERR_CONFIG, "mm_solve_fused runs on a single-grid context");
    memset(r, 0, sizeof *r);
    const int d = ctx->dim, D = ctx->D;
    const double npts = p->step.npts;
    mm_step_params prm = p->step;
    double rho = p->rho, r_d_prev = p->r_d_prev;
    double lam_sum[9];
    memcpy(lam_sum, p->lam_sum, sizeof lam_sum);
    int64_t outer_iter = p->outer_iter, total_sweeps = 0;
    double point_sweeps = 0.0;
    bool have_pending = false;
    mm_local_stats pending{}, stats{};
    double u_mean[9] = {0};
    int rc = MM_OK;
    const int64_t pchunk = p->policy_chunk;
    for (int64_t it = 0; it < p->max_outer; ++it) {
        // LocalPolicy.target_tol (solver.py:128-199)
        double tol_pt = prm.point_tol;
        if (p->policy == MM_POLICY_RATIO) {
            if (!isfinite(r_d_prev)) tol_pt = 1.0;
            else {
                const double b = p->step.ratio * r_d_prev;
                tol_pt = (b > prm.point_tol) ? b : prm.point_tol;  // Python max(a, b)
            }
        }
        int64_t sweeps_total = 0;
        for (;;) {
            const int64_t chunk = std::min(pchunk, p->max_local - sweeps_total);
            if (have_pending) {
                stats = pending;
                have_pending = false;
            } else {
                // MooneyRivlin/_quadratic _device_local: tol = point_tol * mu_rep
                if ((rc = mm_local_sweeps(ctx, prm.material, rho, tol_pt * prm.mu_rep, chunk,
                                          prm.phi_scale, 0, &stats)))
                    return rc;
            }
            sweeps_total += stats.sweeps;
            point_sweeps += stats.sum_nsw;
            const double frac = npts ? (double)stats.n_conv / npts : 1.0;
            const bool pol_done = p->policy == MM_POLICY_FRACTION ? frac >= p->fraction
                                                                  : frac >= 1.0;
            if (pol_done || stats.sweeps < chunk || sweeps_total >= p->max_local) break;
        }
        total_sweeps += sweeps_total;
        const double r_l = sqrt(stats.sum_res2 / npts) / prm.mu_rep;
        // macro_gradient (projection.py:125-129)
        for (int i = 0; i < 9; ++i) u_mean[i] = 0.0;
        for (int i = 0; i < D; ++i) {
            const double Fm = stats.sum_F[i] / npts;
            const double Lm = lam_sum[i] / npts;
            const double su = Fm - (Lm - p->bc_value[i]) / rho;
            u_mean[i] = p->bc_mask[i] != 0.0 ? p->bc_value[i] : su;
        }
        memcpy(prm.u_mean, u_mean, sizeof u_mean);
        prm.rho = rho;
        prm.r_l = r_l;
        prm.outer_iter = outer_iter + 1;
        prm.last_allowed = it == p->max_outer - 1 ? 1 : 0;
        mm_step_result res;
        mm_local_stats ls;
        if ((rc = mm_residuals_and_step(ctx, &prm, &res, &ls))) return rc;
        outer_iter += 1;
        r_d_prev = res.r_d;
        memcpy(lam_sum, res.sum_lam, sizeof lam_sum);
        r->iterations = it + 1;
        if (res.diverged) {
            r->diverged = 1;
            rc = MM_ERR_DIVERGED;
            mm_fail(ctx, MM_ERR_DIVERGED, "primal residual %.3e at outer iteration %lld",
                    res.r_p, (long long)outer_iter);
            break;
        }
        rho = res.rho_next;
        if (res.swept) {
            pending = ls;
            have_pending = true;
        }
        hist[4 * it + 0] = res.r_p;
        hist[4 * it + 1] = res.r_d;
        hist[4 * it + 2] = r_l;
        hist[4 * it + 3] = rho;
        if (res.done) {
            r->converged = 1;
            break;
        }
    }
    r->outer_iter = outer_iter;
    r->total_sweeps = total_sweeps;
    r->rho = rho;
    r->r_d_prev = r_d_prev;
    r->point_sweeps = point_sweeps;
    memcpy(r->lam_sum, lam_sum, sizeof lam_sum);
    memcpy(r->u_mean, u_mean, sizeof u_mean);
    (void)d;
    return rc;
}

int mm_project_update(mm_ctx *ctx, double rho, const double *u_mean, mm_update_stats *out) {
    if (!ctx || !u_mean || !out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->slab_mode) return mm_fail(ctx, MM_ERR_CONFIG, "slab context: use mm_slab_step");
    if (!(rho > 0.0) || !isfinite(rho))
        return mm_fail(ctx, MM_ERR_PARAM, "rho must be positive and finite, got %g", rho);
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (!ctx->have_sym) return mm_fail(ctx, MM_ERR_CONFIG, "symbols were never set");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = mm_flush_pending(ctx);
    if (rc) return rc;
    return mm_run_project(ctx, rho, u_mean, 1, out);
}

int mm_set_option(mm_ctx *ctx, int option, int64_t value) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    switch (option) {
        case MM_OPT_IMPLICIT_GRAD: {
            const bool on = value != 0;
            if (!on && ctx->g_implicit) {
                int rc = mm_materialize_G(ctx);
                if (rc) return rc;
                ctx->g_implicit = false;
            }
            ctx->opt_implicit_g = on;
            return MM_OK;
        }
        case MM_OPT_STENCIL_MARCH: ctx->opt_march = value != 0; return MM_OK;
        case MM_OPT_T_FIELD:
            ctx->opt_tfield = value != 0;
            if (!ctx->opt_tfield) ctx->T_valid = false;
            return MM_OK;
        case MM_OPT_PLANE_FFT: ctx->opt_plane = value != 0; return MM_OK;
        case MM_OPT_ROWINV_PIPE: ctx->opt_rowinv_p = value != 0; return MM_OK;
        case MM_OPT_SPECULATE: ctx->opt_speculate = value != 0; return MM_OK;
        case MM_OPT_ROWFWD_WARP: ctx->opt_rowfwd_w = value != 0; return MM_OK;
        case MM_OPT_PIPELINE: ctx->opt_pipeline = value != 0; return MM_OK;
        default: return mm_fail(ctx, MM_ERR_PARAM, "unknown option %d", option);
    }
}

int mm_frank_stencil(mm_ctx *ctx) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (!ctx->have_lce) return mm_fail(ctx, MM_ERR_CONFIG, "LCE parameters were never set");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    return mm_run_frank_of_ff(ctx);
}

int mm_stencil(mm_ctx *ctx, int op) {
    if (!ctx) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->points_only) return mm_fail(ctx, MM_ERR_CONFIG, "point-set context has no grid");
    if (op != 0 && op != 1) return mm_fail(ctx, MM_ERR_PARAM, "unknown stencil op %d", op);
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    return mm_run_stencil(ctx, op);
}

}  // extern "C"
