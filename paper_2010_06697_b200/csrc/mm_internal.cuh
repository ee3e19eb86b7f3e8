// Internal definitions shared by the CUDA translation units of libmm_admm.
#pragma once

#include <cuda.h>          // CUtensorMap (TMA descriptors; encoded through the runtime's driver entry point)
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/mm_admm.h"

#define MM_MAX_PARTIALS 24  // doubles reduced per block by any kernel

struct mm_bloch_state;

// the next fused pass's parameters as the device decided them (k_decide)
struct DevStep {
    int skip;  // converged / diverged: the fused pass returns at once
    int pad;
    double rho_next, tol, tol_gs;
};

// mm_residuals_and_step's decision (a pipelined step), taken by the thread
// that finalises K1's sums (decide_step below)
struct DecideArgs {
    int on;
    mm_step_params p;
    DevStep *ds;   // the next fused pass's parameters
    double *copy;  // mapped: skip, rho_next, tol for the host's check
};

struct mm_ctx {
    int dim = 0, n = 0;
    double L = 0.0, h = 0.0;
    int64_t M = 0;       // grid points n^dim
    int D = 0;           // tensor components dim*dim
    int nh = 0;          // n/2 + 1 (half-spectrum length, last axis)
    int P = 0;           // spectral row pitch (complex), multiple of 8
    int64_t nrows = 0;   // M / n rows along the contiguous axis
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;

    // device fields, SoA (component-major): comp c of point p at c*M + p
    double *F = nullptr, *G = nullptr, *Lam = nullptr, *Ut = nullptr, *prevF = nullptr;
    double *modA = nullptr, *modB = nullptr;
    // LCE internal / frozen
    double *ang = nullptr, *chart = nullptr, *pinc = nullptr, *n0 = nullptr, *ff = nullptr;
    double *prevAng = nullptr, *prevChart = nullptr, *prevPinc = nullptr, *dirbuf = nullptr;
    bool have_prev_F = false, have_prev_int = false;
    mm_lce_params lce{};
    bool have_lce = false;
    // spectral workspace: dim comps x nrows x P complex
    double2 *spec = nullptr;
    // symbols
    double *sym = nullptr;   // dim * n
    double sym_thresh = 0.0;
    bool have_sym = false;
    // twiddles: tw_half (N = n/2 complex FFT of the packed real rows),
    // tw_full (N = n), tw_r2c (W_n^k, k < n/2 + 1)
    double2 *tw_full = nullptr, *tw_half = nullptr, *tw_r2c = nullptr;
    // reductions
    double *partials = nullptr;  // [max_blocks][MM_MAX_PARTIALS]
    int64_t partials_cap = 0;
    double *red_out = nullptr;   // MM_MAX_PARTIALS results
    unsigned int *red_count = nullptr;
    double *host_out = nullptr;  // pinned MM_MAX_PARTIALS
    // per-point local outputs / persistent descent state
    double *res = nullptr;
    int32_t *nsw = nullptr;
    uint8_t *ok = nullptr;
    double *tstate = nullptr;
    uint8_t *freestate = nullptr;
    // staging for AoS <-> SoA
    double *stage = nullptr;
    int64_t stage_cap = 0;     // doubles
    cudaEvent_t xfer_ev[2] = {nullptr, nullptr};  // pinned-half reuse (transfers)
    // stage profiling (CUDA events on ctx->stream) and launch counting
    bool prof_on = false;
    double prof_ms[MM_NSTAGE] = {0};
    int64_t prof_launches[MM_NSTAGE] = {0};
    int64_t launches[MM_NSTAGE] = {0};
    struct PendingTiming {
        int stage;
        cudaEvent_t a, b;
    };
    std::vector<PendingTiming> pending;
    std::vector<cudaEvent_t> event_pool;
    // grad_u bookkeeping: after a fused projection grad_u is held implicitly
    // as ubar + D u_tilde (the gradient field is not stored); G is then a
    // cache filled on demand (downloads, LCE local step).
    bool opt_implicit_g = false;  // MM_OPT_IMPLICIT_GRAD
    bool opt_march = true;        // MM_OPT_STENCIL_MARCH
    bool opt_tfield = true;       // MM_OPT_T_FIELD
    bool opt_plane = true;        // MM_OPT_PLANE_FFT
    bool opt_rowinv_p = true;     // MM_OPT_ROWINV_PIPE
    bool opt_rowfwd_w = true;     // MM_OPT_ROWFWD_WARP
    bool red_mapped = false;      // red_out is host_out's device alias (mapped pinned memory)
    // pipelined loop step (mm_residuals_and_step): K1 sums into a second
    // mapped slot, the decision taken on the device (k_decide -> dstep) so the
    // fused pass is queued behind K1 without a host round trip
    bool opt_pipeline = true;     // MM_OPT_PIPELINE
    double *k1_dst = nullptr;     // where K1's sums go (nullptr: red_out)
    struct DevStep *dstep = nullptr;
    struct DecideArgs k1_decide{};  // passed to K1 (on = 0: no decision)
    cudaEvent_t ev_k1 = nullptr;
    bool opt_speculate = true;    // MM_OPT_SPECULATE
    // speculative projection front (A, column passes, E of the next
    // iteration launched by mm_update_and_sweep behind the fused pass): valid
    // for front_rho while no other entry point ran since (gen unchanged)
    uint64_t gen = 0;
    bool front_valid = false;
    double front_rho = 0.0;
    uint64_t front_gen = 0;
    cudaEvent_t ev_red = nullptr;
    mm_update_stats step_us{};  // residual sums of the last mm_residuals_and_step
    bool lam_pending = false;     // multiplier ascent deferred by mm_project_residuals
    double pending_rho = 0.0;
    bool g_implicit = false;
    bool g_buf_valid = true;
    double ubar[9] = {0};
    double *Ut2 = nullptr;  // second u_tilde buffer (new u during a projection)
    double *Pbuf = nullptr; // stress field scratch (equilibrium_residual)
    // T = F - lam / T_rho, written by the fused update + local pass so that
    // the next projection's divergence reads 9 words instead of 18
    double *Tbuf = nullptr;
    bool T_valid = false;
    double T_rho = 0.0;
    mm_bloch_state *bloch = nullptr;  // Bloch stability workspace (mm_bloch.cu)
    bool F_checked = false;
    bool points_only = false;
    // slab decomposition (3D, split along axis 0)
    bool slab_mode = false;
    int slab_P = 1, slab_rank = 0, slab_nl = 0;
    // component strides of the stencil inputs: u_tilde (Ut, Ut2) and the LCE
    // director (dirbuf).  M on a single context; a slab keeps ghost planes
    // on both faces (1 for u, 2 for the director: the radius-2 Frank stencil)
    // so that axis-0 neighbours are plain offsets and the halo exchange
    // writes straight into them.  Ut / Ut2 / dirbuf point at plane 0.
    int64_t uM = 0, dM = 0;
    // Newton-compacted 3D LCE schedule (mm_lce.cu): |F|^2 at call start,
    // two deferred-point lists and three rotating counters
    // TMA descriptor of the plane-layout spectrum (mm_project.cu plane_col_tma)
    CUtensorMap tmap{}, rmap{};
    bool tmap_ok = false, rmap_ok = false;
    const void *tmap_src = nullptr;
    int tmap_n = 0;
    double *lce_fsq0 = nullptr;
    int *lce_list[2] = {nullptr, nullptr};
    int *lce_cnt = nullptr;
    double *Ut_base = nullptr, *Ut2_base = nullptr, *dir_base = nullptr;
    // peer-memory transposes: device tables of every rank's RECV / SEND buffer
    double2 **peer_recv = nullptr, **peer_send = nullptr;
    std::vector<void *> ipc_opened;  // closed at destroy
    double2 *sendbuf = nullptr, *recvbuf = nullptr;
    double *halo_in_lo = nullptr, *halo_in_hi = nullptr, *halo_out_lo = nullptr,
           *halo_out_hi = nullptr;    // F verified admissible since the last upload
    int64_t bytes = 0;
    std::string err;
};

// set error + return code
int mm_fail(mm_ctx *ctx, int code, const char *fmt, ...);

#define MM_CUDA(ctx, call)                                                                 \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return mm_fail((ctx), MM_ERR_CUDA, "%s failed: %s (%s:%d)", #call,             \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                    \
    } while (0)

#define MM_LAUNCH_CHECK(ctx)                                                               \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess)                                                             \
            return mm_fail((ctx), MM_ERR_CUDA, "kernel launch failed: %s (%s:%d)",         \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                    \
    } while (0)

int mm_alloc(mm_ctx *ctx, void **ptr, size_t bytes);
int mm_ensure_partials(mm_ctx *ctx, int64_t nblocks);
void mm_free(mm_ctx *ctx, void *p);
void mm_bloch_free(mm_ctx *ctx);
// copy the finalized reduction results (K doubles) back to host
int mm_fetch_reduction(mm_ctx *ctx, int K, double *out);

// ---------------------------------------------------------------------------
// deterministic block reductions
// ---------------------------------------------------------------------------
// Kinds of per-slot combination.
enum { RED_SUM = 0, RED_MAX = 1 };

__device__ __forceinline__ double red_op(int op, double a, double b) {
    return op == RED_MAX ? fmax(a, b) : a + b;
}

// Reduce K per-thread values over the block in a fixed order (xor-shuffle
// tree inside warps, then warps in index order); thread 0 gets the result.
// smem: >= 32 * K doubles.
template <int K>
__device__ __forceinline__ void block_reduce(double (&vals)[K], const int (&ops)[K],
                                             double *smem) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double v = vals[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = red_op(ops[k], v, __shfl_xor_sync(0xffffffffu, v, o));
        vals[k] = v;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) smem[warp * K + k] = vals[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = smem[k];
            for (int w = 1; w < nw; ++w) s = red_op(ops[k], s, smem[w * K + k]);
            vals[k] = s;
        }
    }
    __syncthreads();
}

// Write this block's partial (thread 0's vals, already block-reduced) and let
// the last block to finish reduce all partials.  Each thread of the last block
// folds a contiguous range of blocks in order, then block_reduce combines the
// threads in a fixed order => deterministic run to run.
template <int K>
__device__ bool grid_finalize(const double (&vals)[K], const int (&ops)[K], double *partials,
                              double *out, unsigned int *count, double *smem,
                              double *final_vals = nullptr) {
    __shared__ bool is_last;
    const int nb = gridDim.x * gridDim.y * gridDim.z;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) partials[(int64_t)bid * K + k] = vals[k];
        __threadfence();
        unsigned int t = atomicAdd(count, 1u);
        is_last = (t == (unsigned int)(nb - 1));
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
    const int nt = blockDim.x;
    const int per = (nb + nt - 1) / nt;
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = ops[k] == RED_MAX ? -1e308 : 0.0;
    const int b0 = threadIdx.x * per;
    const int b1 = min(nb, b0 + per);
    for (int b = b0; b < b1; ++b) {
#pragma unroll
        for (int k = 0; k < K; ++k)
            acc[k] = red_op(ops[k], acc[k], ((volatile double *)partials)[(int64_t)b * K + k]);
    }
    block_reduce<K>(acc, ops, smem);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = acc[k];
        *count = 0u;
        if (final_vals) {
#pragma unroll
            for (int k = 0; k < K; ++k) final_vals[k] = acc[k];
        }
        return true;
    }
    return false;
}

// decide_step: statement for statement the host's code, with no sums of
// products, so no contraction can make the two differ
__device__ inline double gs_threshold_dev(double tol) {  // gs_threshold (mm_local.cu)
    if (tol != tol) return tol;
    if (tol < 0.0) return -INFINITY;
    if (tol == 0.0 || isinf(tol)) return tol;
    double x = tol * tol;
    while (x > 0.0 && sqrt(x) > tol) x = nextafter(x, 0.0);
    while (sqrt(nextafter(x, INFINITY)) <= tol) x = nextafter(x, INFINITY);
    return x;
}

__device__ inline void decide_step(double sum_dG2, double sum_mis2, const DecideArgs &a) {
    const mm_step_params &p = a.p;
    const double r_d = p.rho * sqrt(sum_dG2 / p.npts) / p.mu_rep;
    const double r_p = sqrt(sum_mis2 / p.npts);
    DevStep d{};
    double rho = p.rho;
    if (!isfinite(r_p) || r_p > p.divergence_limit) {
        d.skip = 1;
    } else {
        if (p.adapt && p.outer_iter > 1) {
            if (r_p > p.tau_adapt * r_d) {
                rho *= p.kappa_adapt;
            } else if (r_d > p.tau_adapt * r_p) {
                const double q = rho / p.kappa_adapt;
                rho = (p.rho_floor > q) ? p.rho_floor : q;
            }
        }
        const bool done = r_p <= p.r_p_tol && r_d <= p.r_d_tol && p.r_l <= p.r_l_tol;
        if (done) {
            d.skip = 1;
        } else {
            double tol = p.point_tol;
            if (p.ratio_policy) {
                if (!isfinite(r_d)) tol = 1.0;
                else {
                    const double b = p.ratio * r_d;
                    tol = (b > p.point_tol) ? b : p.point_tol;
                }
            }
            d.tol = tol * p.mu_rep;
            d.tol_gs = gs_threshold_dev(d.tol);
        }
    }
    d.rho_next = rho;
    *a.ds = d;
    a.copy[0] = d.skip;
    a.copy[1] = d.rho_next;
    a.copy[2] = d.tol;
}

// periodic neighbour offsets of point p (< 2^31) along each axis; lgn = log2 n
// when n is a power of two (shift/mask), else -1 (32-bit division)
template <int DIM>
__device__ __forceinline__ void nbr_offsets(int64_t p64, int n, int lgn, int (&off_p)[DIM],
                                            int (&off_m)[DIM], bool wrap0 = true) {
    const unsigned p = (unsigned)p64;
    unsigned c[DIM];
    if (lgn >= 0) {
        const unsigned mask = (unsigned)n - 1u;
#pragma unroll
        for (int j = DIM - 1; j >= 0; --j) c[j] = (p >> (lgn * (DIM - 1 - j))) & mask;
    } else {
        unsigned q = p;
#pragma unroll
        for (int j = DIM - 1; j >= 0; --j) {
            const unsigned nq = q / (unsigned)n;
            c[j] = q - nq * (unsigned)n;
            q = nq;
        }
    }
    int stride = 1;
#pragma unroll
    for (int j = DIM - 1; j >= 0; --j) {
        off_p[j] = (c[j] + 1 == (unsigned)n) ? -(n - 1) * stride : stride;
        off_m[j] = (c[j] == 0) ? (n - 1) * stride : -stride;
        stride *= n;
    }
    if (!wrap0) {  // slab: the planes beyond the slab faces are ghost planes
        stride /= n;
        off_p[0] = stride;
        off_m[0] = -stride;
    }
}

// Source of grad_u for the local step: the explicit field, or (implicit
// mode, after a fused projection) u_mean + central difference of u_tilde,
// evaluated with exactly the expression the projection's gradient pass uses.
struct GSrc {
    const double *G;  // explicit field (nullptr: implicit)
    const double *U;  // u_tilde for the implicit form
    double ubar[9];
    int n, lgn;
    double inv2h;
    int64_t M;
    int64_t uM;       // component stride of U (M; slab: M + 2 ghost planes)
    int wrap0;        // 0 (slab): axis-0 neighbours across the faces are U's ghost planes
};

template <int DIM>
__device__ __forceinline__ void gsrc_load(const GSrc &s, int64_t p, double (&g)[DIM * DIM]) {
    constexpr int D = DIM * DIM;
    if (s.G) {
#pragma unroll
        for (int c = 0; c < D; ++c) g[c] = s.G[c * s.M + p];
        return;
    }
    int op[DIM], om[DIM];
    nbr_offsets<DIM>(p, s.n, s.lgn, op, om, s.wrap0 != 0);
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
        const double *u = s.U + (int64_t)i * s.uM + p;
#pragma unroll
        for (int j = 0; j < DIM; ++j)
            g[i * DIM + j] = (__ldg(u + op[j]) - __ldg(u + om[j])) * s.inv2h + s.ubar[i * DIM + j];
    }
}

// L2 prefetch of everything a local-step point reads (the u stencil or the
// explicit grad_u, F, lam, moduli): issued for the thread's NEXT grid-stride
// point before the current point's sweeps, so that point's loads hit L2
// instead of waiting on DRAM (the first use of the stencil loads was 13 % of
// the fused pass's stall samples).  No registers are held across the sweeps.
__device__ __forceinline__ void pf_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int DIM>
__device__ __forceinline__ void prefetch_point(const GSrc &s, const double *F, const double *L,
                                               const double *mA, const double *mB, int64_t p) {
    constexpr int D = DIM * DIM;
    if (p >= s.M) return;
    if (s.G) {
#pragma unroll
        for (int c = 0; c < D; ++c) pf_l2(s.G + c * s.M + p);
    } else {
        int op[DIM], om[DIM];
        nbr_offsets<DIM>(p, s.n, s.lgn, op, om, s.wrap0 != 0);
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            const double *u = s.U + (int64_t)i * s.uM + p;
            pf_l2(u);
#pragma unroll
            for (int j = 0; j < DIM - 1; ++j) {  // the contiguous axis shares u's lines
                pf_l2(u + op[j]);
                pf_l2(u + om[j]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {
        pf_l2(F + c * s.M + p);
        pf_l2(L + c * s.M + p);
    }
    pf_l2(mA + p);
    if (mB) pf_l2(mB + p);
}

// stage timing: brackets the kernel launches of one pipeline stage with CUDA
// events on the context stream when profiling is on, and counts launches.
void mm_stage_begin(mm_ctx *ctx, int stage, cudaEvent_t *ev);
void mm_stage_end(mm_ctx *ctx, int stage, cudaEvent_t ev, int nlaunch);
void mm_drain_timings(mm_ctx *ctx);
struct StageScope {
    mm_ctx *ctx;
    int stage;
    int nlaunch;
    cudaEvent_t ev = nullptr;
    StageScope(mm_ctx *c, int s, int n = 1) : ctx(c), stage(s), nlaunch(n) {
        mm_stage_begin(ctx, stage, &ev);
    }
    ~StageScope() { mm_stage_end(ctx, stage, ev, nlaunch); }
};

// launch helpers implemented per translation unit
int mm_run_local(mm_ctx *ctx, int material, double rho, double tol, int64_t max_sweeps,
                 double phi_scale, int want_points, mm_local_stats *out);
int mm_run_project(mm_ctx *ctx, double rho, const double *u_mean, int update,
                   mm_update_stats *out);
int mm_run_project_front(mm_ctx *ctx, double rho, int update, double **u_new_out);
int mm_run_frozen(mm_ctx *ctx);
int mm_run_field_sums(mm_ctx *ctx, const double *field, int ncomp, double *out);
int mm_run_stress(mm_ctx *ctx, int material, double *P);
int mm_run_lce_stress(mm_ctx *ctx, double dt, double *P);
int mm_run_eq_residual(mm_ctx *ctx, const double *P, double *out);
int mm_check_det(mm_ctx *ctx, int *bad);
int mm_run_stencil(mm_ctx *ctx, int op);
int mm_run_frank_of_ff(mm_ctx *ctx);
int mm_ilog2(int n);
int mm_run_slab_step(mm_ctx *ctx, int step, double rho, const double *u_mean, double *sums);
GSrc mm_gsrc(mm_ctx *ctx);
int mm_slab_res(mm_ctx *ctx, double rho, const double *u_mean, double *sums);
int mm_run_slab_lce(mm_ctx *ctx, int step);
int mm_slab_alloc_director(mm_ctx *ctx);
int mm_materialize_G(mm_ctx *ctx);
int mm_ensure_points(mm_ctx *ctx);
int mm_flush_pending(mm_ctx *ctx);
int mm_run_update_pipe(mm_ctx *ctx, int material, double rho_placeholder, int64_t max_sweeps,
                       double phi_scale);
int mm_run_update_pipe_finish(mm_ctx *ctx, bool swept, double rho_next, mm_local_stats *ls,
                              mm_update_stats *us);
int mm_run_update(mm_ctx *ctx, int material, double rho_next, double tol, int64_t max_sweeps,
                  double phi_scale, int want_points, mm_local_stats *ls, mm_update_stats *us);
