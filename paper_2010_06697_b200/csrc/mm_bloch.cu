// Bloch-wave stability on the device (the reference's
// stability.py:171-289, bloch_min_eigen): smallest eigenvalue of the
// shifted acoustic operator by the splitting iteration
//
//   G      = (L + rho I)^-1 (g + rho B p)           pointwise, per voxel
//   p_hat  = sphere-constrained projection of FFT(rho G - g) . conj(b)
//   beta   = <B p, L B p>,   g += rho (B p - G)
//
// with B p = IFFT(p_hat_i b_j), b = i (xi + omega).  Fields are complex,
// component-major ([c][point], double2).  Full-spectrum complex transforms
// run one line per CTA (radix-2 in shared memory for power-of-two n, exact
// DFT otherwise); the secular equation of the sphere projection is solved
// by one CTA with deterministic block reductions, in the reference's
// bisection order (stability.py:120-168).  The host supplies the per-point
// (L + rho I)^-1 and L (d^2 x d^2, computed once per solve as the reference
// does with numpy), the shifted frequencies and the live mask.
#include <math.h>

#include <algorithm>
#include <vector>

#include "mm_internal.cuh"

struct mm_bloch_state {
    int D = 0;                 // d*d
    int64_t npts = 0;
    double rho = 0.0, target = 0.0;
    double *Minv = nullptr;    // [a*D + b][point]
    double *L = nullptr;       // [a*D + b][point]
    double *shift = nullptr;   // [j][point] xi_j + omega_j
    double *rbsq = nullptr;    // rho |b|^2
    uint8_t *live = nullptr;
    double2 *phat = nullptr;   // [i][point]
    double2 *num = nullptr;    // [i][point]
    double2 *Gp = nullptr;     // [a][point]  (B p, real space)
    double2 *G = nullptr;      // [a][point]
    double2 *g = nullptr;      // [a][point]  multiplier
    double2 *X = nullptr;      // [a][point]  rho G - g, then its transform
    double *w2 = nullptr;      // |num|^2 per mode
    double *scal = nullptr;    // secular outputs: eta, scale, hard flag, deficit index
    double beta_prev = INFINITY;
    bool have_gp = false;
};

namespace {

__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// ---------------------------------------------------------------------------
// complex line transforms along one axis of a d-dimensional n^d field
// ---------------------------------------------------------------------------
__global__ void k_fft_axis(double2 *__restrict__ data, int n, int lgn, int64_t stride,
                           int64_t npts, int64_t lines_per_comp, const double2 *__restrict__ tw,
                           int inv) {
    extern __shared__ double2 ln[];
    double2 *tmp = ln + n;
    const int64_t line = blockIdx.x;
    const int64_t comp = line / lines_per_comp;
    const int64_t l = line - comp * lines_per_comp;
    // line l: index of the point with axis coordinate 0
    const int64_t outer = l / stride, inner = l - outer * stride;
    double2 *base = data + comp * npts + outer * stride * n + inner;
    if (lgn >= 0) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int r = (int)(__brev((unsigned)i) >> (32 - lgn));
            ln[r] = base[(int64_t)i * stride];
        }
        __syncthreads();
        for (int half = 1; half < n; half <<= 1) {
            const int tstep = n / (2 * half);
            for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
                const int grp = b / half, j = b - grp * half;
                const int i0 = grp * 2 * half + j, i1 = i0 + half;
                double2 w = tw[j * tstep];
                if (inv) w.y = -w.y;
                const double2 t = c_mul(w, ln[i1]);
                const double2 u = ln[i0];
                ln[i0] = make_double2(u.x + t.x, u.y + t.y);
                ln[i1] = make_double2(u.x - t.x, u.y - t.y);
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) base[(int64_t)i * stride] = ln[i];
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) ln[i] = base[(int64_t)i * stride];
        __syncthreads();
        for (int k = threadIdx.x; k < n; k += blockDim.x) {
            double2 s = make_double2(0.0, 0.0);
            int idx = 0;
            for (int j = 0; j < n; ++j) {
                double2 w = tw[idx];
                if (inv) w.y = -w.y;
                const double2 t = c_mul(ln[j], w);
                s.x += t.x;
                s.y += t.y;
                idx += k;
                if (idx >= n) idx -= n;
            }
            tmp[k] = s;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) base[(int64_t)i * stride] = tmp[i];
    }
}

// B p in spectral space: out[i*d + j] = phat_i * b_j, b_j = i * shift_j
__global__ void k_form_grad(const double2 *__restrict__ phat, const double *__restrict__ shift,
                            double2 *__restrict__ out, int d, int64_t npts) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        for (int i = 0; i < d; ++i) {
            const double2 a = phat[i * npts + p];
            for (int j = 0; j < d; ++j) {
                const double s = shift[j * npts + p];
                out[(i * d + j) * npts + p] = make_double2(-a.y * s, a.x * s);
            }
        }
    }
}

// 1/npts of the inverse transform, then G = Minv (g + rho Gp), X = rho G - g
__global__ void k_local_apply(double2 *__restrict__ Gp, const double2 *__restrict__ g,
                              const double *__restrict__ Minv, double2 *__restrict__ G,
                              double2 *__restrict__ X, int D, int64_t npts, double rho,
                              double inv_n, int scale_gp) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        double2 rhs[9];
        for (int a = 0; a < D; ++a) {
            double2 v = Gp[a * npts + p];
            if (scale_gp) {
                v = make_double2(v.x * inv_n, v.y * inv_n);
                Gp[a * npts + p] = v;
            }
            const double2 ga = g[a * npts + p];
            rhs[a] = make_double2(ga.x + rho * v.x, ga.y + rho * v.y);
        }
        for (int a = 0; a < D; ++a) {
            double2 s = make_double2(0.0, 0.0);
            for (int b = 0; b < D; ++b) {
                const double m = Minv[(a * D + b) * npts + p];
                s.x += m * rhs[b].x;
                s.y += m * rhs[b].y;
            }
            G[a * npts + p] = s;
            const double2 ga = g[a * npts + p];
            X[a * npts + p] = make_double2(rho * s.x - ga.x, rho * s.y - ga.y);
        }
    }
}

// num_i = sum_j Chat_ij conj(b_j), w2 = sum_i |num_i|^2
__global__ void k_num(const double2 *__restrict__ Chat, const double *__restrict__ shift,
                      double2 *__restrict__ num, double *__restrict__ w2, int d, int64_t npts) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        double w = 0.0;
        for (int i = 0; i < d; ++i) {
            double2 s = make_double2(0.0, 0.0);
            for (int j = 0; j < d; ++j) {
                const double2 c = Chat[(i * d + j) * npts + p];
                const double sh = shift[j * npts + p];  // conj(i sh) = -i sh
                s.x += c.y * sh;
                s.y += -c.x * sh;
            }
            num[i * npts + p] = s;
            w += s.x * s.x + s.y * s.y;
        }
        w2[p] = w;
    }
}

// deterministic block sum (fixed thread order)
__device__ double block_sum(double v, double *sh) {
    double a[1] = {v};
    const int ops[1] = {RED_SUM};
    block_reduce<1>(a, ops, sh);
    __shared__ double res;
    if (threadIdx.x == 0) res = a[0];
    __syncthreads();
    const double r = res;
    __syncthreads();
    return r;
}

__device__ double psi_eval(const double *__restrict__ w2, const double *__restrict__ rbsq,
                           const uint8_t *__restrict__ live, int64_t npts, double eta,
                           double *sh) {
    double s = 0.0;
    for (int64_t p = threadIdx.x; p < npts; p += blockDim.x) {
        if (live[p]) {
            const double den = rbsq[p] - eta;
            s += w2[p] / (den * den);
        }
    }
    return block_sum(s, sh);
}

// the secular equation of the sphere projection (stability.py:120-168);
// out: [0] eta, [1] hard case (0/1), [2] index of the smallest live pole
__global__ void k_secular(const double *__restrict__ w2, const double *__restrict__ rbsq,
                          const uint8_t *__restrict__ live, int64_t npts, double target,
                          double *out) {
    __shared__ double sh[32];
    __shared__ double smin[32];
    __shared__ long long sidx[32];
    // smallest live pole, first index on ties (np.argmin order)
    double best = INFINITY;
    long long bi = -1;
    for (int64_t p = threadIdx.x; p < npts; p += blockDim.x) {
        const double v = live[p] ? rbsq[p] : INFINITY;
        if (v < best || (v == best && bi < 0)) {
            best = v;
            bi = p;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob < best || (ob == best && oi >= 0 && (bi < 0 || oi < bi))) {
            best = ob;
            bi = oi;
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) {
        smin[warp] = best;
        sidx[warp] = bi;
    }
    __syncthreads();
    __shared__ double pole_min;
    __shared__ long long pole_idx;
    if (threadIdx.x == 0) {
        double b = smin[0];
        long long ix = sidx[0];
        for (int w = 1; w < (int)((blockDim.x + 31) / 32); ++w) {
            if (smin[w] < b || (smin[w] == b && sidx[w] >= 0 && (ix < 0 || sidx[w] < ix))) {
                b = smin[w];
                ix = sidx[w];
            }
        }
        pole_min = b;
        pole_idx = ix;
    }
    __syncthreads();
    const double pm = pole_min;
    const double span = fmax(isfinite(pm) ? pm : 1.0, 1.0);
    double hi = pm - 1e-13 * span;
    double eta;
    int hard = 0;
    if (psi_eval(w2, rbsq, live, npts, hi, sh) < target) {
        eta = hi;
        hard = 1;
    } else {
        double lo = hi - span;
        while (psi_eval(w2, rbsq, live, npts, lo, sh) > target) lo -= 2.0 * (hi - lo);
        for (int it = 0; it < 200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (mid == lo || mid == hi) break;
            if (psi_eval(w2, rbsq, live, npts, mid, sh) > target) hi = mid;
            else lo = mid;
        }
        eta = 0.5 * (lo + hi);
    }
    if (threadIdx.x == 0) {
        out[0] = eta;
        out[1] = hard;
        out[2] = (double)pole_idx;
    }
}

// phat = live ? num / (rho bsq - eta) : 0, and its squared norm (block partials)
__global__ void k_phat(const double2 *__restrict__ num, const double *__restrict__ rbsq,
                       const uint8_t *__restrict__ live, const double *__restrict__ sec,
                       double2 *__restrict__ phat, int d, int64_t npts, double *partials,
                       double *red_out, unsigned int *count) {
    __shared__ double sh[32];
    const double eta = sec[0];
    double acc[1] = {0.0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        const bool lv = live[p] != 0;
        const double den = rbsq[p] - eta;
        for (int i = 0; i < d; ++i) {
            double2 v = make_double2(0.0, 0.0);
            if (lv) {
                const double2 a = num[i * npts + p];
                v = make_double2(a.x / den, a.y / den);
            }
            phat[i * npts + p] = v;
            acc[0] += v.x * v.x + v.y * v.y;
        }
    }
    const int ops[1] = {RED_SUM};
    block_reduce<1>(acc, ops, sh);
    grid_finalize<1>(acc, ops, partials, red_out, count, sh);
}

// phat[~live] = 0 and |phat|^2 (block partials)
__global__ void k_mask_norm(double2 *__restrict__ phat, const uint8_t *__restrict__ live, int d,
                            int64_t npts, double *partials, double *red_out, unsigned int *count) {
    __shared__ double sh[32];
    double acc[1] = {0.0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        for (int i = 0; i < d; ++i) {
            double2 v = phat[i * npts + p];
            if (!live[p]) {
                v = make_double2(0.0, 0.0);
                phat[i * npts + p] = v;
            }
            acc[0] += v.x * v.x + v.y * v.y;
        }
    }
    const int ops[1] = {RED_SUM};
    block_reduce<1>(acc, ops, sh);
    grid_finalize<1>(acc, ops, partials, red_out, count, sh);
}

__global__ void k_scale_c(double2 *__restrict__ a, int64_t n, double s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        a[i] = make_double2(a[i].x * s, a[i].y * s);
}

// Rayleigh quotient part, multiplier ascent, primal residual:
// sums [0] Re conj(Gp) . L Gp, [1] |Gp - G|^2
__global__ void k_rayleigh(const double2 *__restrict__ Gp, const double2 *__restrict__ G,
                           double2 *__restrict__ g, const double *__restrict__ L, int D,
                           int64_t npts, double rho, double *partials, double *red_out,
                           unsigned int *count) {
    __shared__ double sh[64];
    double acc[2] = {0.0, 0.0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        double2 v[9];
        for (int a = 0; a < D; ++a) v[a] = Gp[a * npts + p];
        for (int a = 0; a < D; ++a) {
            double2 s = make_double2(0.0, 0.0);
            for (int b = 0; b < D; ++b) {
                const double m = L[(a * D + b) * npts + p];
                s.x += m * v[b].x;
                s.y += m * v[b].y;
            }
            acc[0] += v[a].x * s.x + v[a].y * s.y;  // Re(conj(v_a) s_a)
            const double2 ga = G[a * npts + p];
            const double dx = v[a].x - ga.x, dy = v[a].y - ga.y;
            acc[1] += dx * dx + dy * dy;
            double2 gg = g[a * npts + p];
            gg.x += rho * dx;
            gg.y += rho * dy;
            g[a * npts + p] = gg;
        }
    }
    const int ops[2] = {RED_SUM, RED_SUM};
    block_reduce<2>(acc, ops, sh);
    grid_finalize<2>(acc, ops, partials, red_out, count, sh);
}

__global__ void k_aos_complex_to_soa(const double *__restrict__ src, double2 *__restrict__ dst,
                                     int nc, int64_t npts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts * nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / nc;
        const int c = (int)(i - p * nc);
        dst[c * npts + p] = make_double2(src[2 * i], src[2 * i + 1]);
    }
}

__global__ void k_soa_complex_to_aos(const double2 *__restrict__ src, double *__restrict__ dst,
                                     int nc, int64_t npts, double s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts * nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / nc;
        const int c = (int)(i - p * nc);
        const double2 v = src[c * npts + p];
        dst[2 * i] = v.x * s;
        dst[2 * i + 1] = v.y * s;
    }
}

__global__ void k_aos_mat_to_soa(const double *__restrict__ src, double *__restrict__ dst,
                                 int nc, int64_t npts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npts * nc;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i / nc;
        const int c = (int)(i - p * nc);
        dst[c * npts + p] = src[i];
    }
}

int grid_blocks(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 8); }

// full-spectrum complex transform of `ncomp` fields (unnormalised both ways)
int fft_fields(mm_ctx *ctx, double2 *data, int ncomp, bool inv) {
    const int n = ctx->n, d = ctx->dim;
    const int64_t npts = ctx->M;
    int lgn = -1;
    if ((n & (n - 1)) == 0) {
        lgn = 0;
        while ((1 << lgn) < n) ++lgn;
    }
    const int threads = std::max(32, std::min(512, lgn >= 0 ? n / 2 : n));
    const size_t smem = sizeof(double2) * 2 * n;
    int64_t stride = 1;
    for (int ax = d - 1; ax >= 0; --ax) {
        const int64_t lines = npts / n;
        k_fft_axis<<<(unsigned)(lines * ncomp), threads, smem, ctx->stream>>>(
            data, n, lgn, stride, npts, lines, ctx->tw_full, inv ? 1 : 0);
        MM_LAUNCH_CHECK(ctx);
        stride *= n;
    }
    return MM_OK;
}

}  // namespace

void mm_bloch_free(mm_ctx *ctx) {
    mm_bloch_state *b = ctx->bloch;
    if (!b) return;
    void *ptrs[] = {b->Minv, b->L, b->shift, b->rbsq, b->live, b->phat, b->num, b->Gp,
                    b->G, b->g, b->X, b->w2, b->scal};
    for (void *p : ptrs) mm_free(ctx, p);
    delete b;
    ctx->bloch = nullptr;
}

extern "C" {

int mm_bloch_setup(mm_ctx *ctx, const double *Minv, const double *Lmat, const double *shift,
                   const double *bsq, const uint8_t *live, double rho, double target) {
    if (!ctx || !Minv || !Lmat || !shift || !bsq || !live) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    if (ctx->points_only || ctx->slab_mode)
        return mm_fail(ctx, MM_ERR_CONFIG, "Bloch analysis needs a full-grid context");
    if (ctx->n > 2048) return mm_fail(ctx, MM_ERR_CONFIG, "Bloch lines limited to n <= 2048");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    mm_bloch_free(ctx);
    mm_bloch_state *b = new mm_bloch_state();
    ctx->bloch = b;
    const int d = ctx->dim, D = d * d;
    const int64_t npts = ctx->M;
    b->D = D;
    b->npts = npts;
    b->rho = rho;
    b->target = target;
    int rc;
#define ALLOC(p, bytes) \
    if ((rc = mm_alloc(ctx, (void **)&(p), (bytes)))) return rc
    ALLOC(b->Minv, sizeof(double) * D * D * npts);
    ALLOC(b->L, sizeof(double) * D * D * npts);
    ALLOC(b->shift, sizeof(double) * d * npts);
    ALLOC(b->rbsq, sizeof(double) * npts);
    ALLOC(b->live, npts);
    ALLOC(b->phat, sizeof(double2) * d * npts);
    ALLOC(b->num, sizeof(double2) * d * npts);
    ALLOC(b->Gp, sizeof(double2) * D * npts);
    ALLOC(b->G, sizeof(double2) * D * npts);
    ALLOC(b->g, sizeof(double2) * D * npts);
    ALLOC(b->X, sizeof(double2) * D * npts);
    ALLOC(b->w2, sizeof(double) * npts);
    ALLOC(b->scal, sizeof(double) * 8);
#undef ALLOC
    // stage the AoS host arrays through a scratch device buffer
    double *tmp = nullptr;
    const size_t big = sizeof(double) * (size_t)D * D * npts;
    if ((rc = mm_alloc(ctx, (void **)&tmp, big))) return rc;
    const int blocks = grid_blocks(npts * D * D);
    MM_CUDA(ctx, cudaMemcpyAsync(tmp, Minv, big, cudaMemcpyHostToDevice, ctx->stream));
    k_aos_mat_to_soa<<<blocks, 256, 0, ctx->stream>>>(tmp, b->Minv, D * D, npts);
    MM_CUDA(ctx, cudaMemcpyAsync(tmp, Lmat, big, cudaMemcpyHostToDevice, ctx->stream));
    k_aos_mat_to_soa<<<blocks, 256, 0, ctx->stream>>>(tmp, b->L, D * D, npts);
    MM_CUDA(ctx, cudaMemcpyAsync(tmp, shift, sizeof(double) * d * npts, cudaMemcpyHostToDevice,
                                 ctx->stream));
    k_aos_mat_to_soa<<<grid_blocks(npts * d), 256, 0, ctx->stream>>>(tmp, b->shift, d, npts);
    std::vector<double> rb(npts);
    for (int64_t p = 0; p < npts; ++p) rb[p] = rho * bsq[p];  // rho_bsq = rho * bsq
    MM_CUDA(ctx, cudaMemcpyAsync(b->rbsq, rb.data(), sizeof(double) * npts, cudaMemcpyHostToDevice,
                                 ctx->stream));
    MM_CUDA(ctx, cudaMemcpyAsync(b->live, live, npts, cudaMemcpyHostToDevice, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_free(ctx, tmp);
    ctx->bytes -= (int64_t)big;
    return MM_OK;
}

// p: complex AoS (npts x d, re/im interleaved).  phat = FFT(p), masked to live
// modes and scaled to the target norm (stability.py:236-242); g = 0.
int mm_bloch_start(mm_ctx *ctx, const double *p) {
    if (!ctx || !p) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    mm_bloch_state *b = ctx->bloch;
    if (!b) return mm_fail(ctx, MM_ERR_CONFIG, "mm_bloch_setup was not called");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    const int d = ctx->dim;
    const int64_t npts = b->npts;
    int rc;
    double *tmp = nullptr;
    if ((rc = mm_alloc(ctx, (void **)&tmp, sizeof(double) * 2 * d * npts))) return rc;
    MM_CUDA(ctx, cudaMemcpyAsync(tmp, p, sizeof(double) * 2 * d * npts, cudaMemcpyHostToDevice,
                                 ctx->stream));
    k_aos_complex_to_soa<<<grid_blocks(npts * d), 256, 0, ctx->stream>>>(tmp, b->phat, d, npts);
    MM_LAUNCH_CHECK(ctx);
    if ((rc = fft_fields(ctx, b->phat, d, false))) return rc;
    MM_CUDA(ctx, cudaMemsetAsync(b->g, 0, sizeof(double2) * b->D * npts, ctx->stream));
    const int blocks = grid_blocks(npts);
    if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
    k_mask_norm<<<blocks, 256, 0, ctx->stream>>>(b->phat, b->live, d, npts, ctx->partials,
                                                 ctx->red_out, ctx->red_count);
    MM_LAUNCH_CHECK(ctx);
    double nrm;
    if ((rc = mm_fetch_reduction(ctx, 1, &nrm))) return rc;
    if (!(nrm > 0.0)) {
        mm_free(ctx, tmp);
        return mm_fail(ctx, MM_ERR_PARAM, "starting mode has no live Bloch content");
    }
    k_scale_c<<<grid_blocks(npts * d), 256, 0, ctx->stream>>>(b->phat, npts * d,
                                                             sqrt(b->target / nrm));
    MM_LAUNCH_CHECK(ctx);
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_free(ctx, tmp);
    ctx->bytes -= (int64_t)(sizeof(double) * 2 * d * npts);
    b->beta_prev = INFINITY;
    b->have_gp = false;
    return MM_OK;
}

// Up to max_iter iterations (stability.py:244-283).  out[0] beta, [1] primal,
// [2] iterations run, [3] converged, [4] diverged.
int mm_bloch_iterate(mm_ctx *ctx, int max_iter, double tol_beta, double tol_primal,
                     double floor_, double mu_rep, double *out) {
    if (!ctx || !out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    mm_bloch_state *b = ctx->bloch;
    if (!b) return mm_fail(ctx, MM_ERR_CONFIG, "mm_bloch_setup was not called");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    const int d = ctx->dim, D = b->D;
    const int64_t npts = b->npts;
    const double rho = b->rho, inv_n = 1.0 / (double)npts;
    const int blocks = grid_blocks(npts);
    int rc = mm_ensure_partials(ctx, blocks);
    if (rc) return rc;
    double beta = INFINITY, primal = INFINITY;
    int it = 0;
    bool converged = false, diverged = false;
    for (it = 1; it <= max_iter; ++it) {
        // step 1: G = (L + rho I)^-1 (g + rho B p)
        const bool fresh = !b->have_gp;
        if (fresh) {
            k_form_grad<<<blocks, 256, 0, ctx->stream>>>(b->phat, b->shift, b->Gp, d, npts);
            MM_LAUNCH_CHECK(ctx);
            if ((rc = fft_fields(ctx, b->Gp, D, true))) return rc;
        }
        k_local_apply<<<blocks, 256, 0, ctx->stream>>>(b->Gp, b->g, b->Minv, b->G, b->X, D, npts,
                                                       rho, inv_n, fresh ? 1 : 0);
        MM_LAUNCH_CHECK(ctx);
        // step 2: sphere-constrained projection onto Bloch gradients
        if ((rc = fft_fields(ctx, b->X, D, false))) return rc;
        k_num<<<blocks, 256, 0, ctx->stream>>>(b->X, b->shift, b->num, b->w2, d, npts);
        MM_LAUNCH_CHECK(ctx);
        k_secular<<<1, 1024, 0, ctx->stream>>>(b->w2, b->rbsq, b->live, npts, b->target, b->scal);
        MM_LAUNCH_CHECK(ctx);
        double sec[3];
        MM_CUDA(ctx, cudaMemcpyAsync(sec, b->scal, sizeof sec, cudaMemcpyDeviceToHost, ctx->stream));
        k_phat<<<blocks, 256, 0, ctx->stream>>>(b->num, b->rbsq, b->live, b->scal, b->phat, d,
                                                npts, ctx->partials, ctx->red_out, ctx->red_count);
        MM_LAUNCH_CHECK(ctx);
        double nrm;
        if ((rc = mm_fetch_reduction(ctx, 1, &nrm))) return rc;  // synchronises: sec is valid
        if (sec[1] != 0.0) {
            // hard case: the deficit goes to component 0 of the smallest pole
            const double deficit = b->target - nrm;
            if (deficit > 0.0) {
                const int64_t at = (int64_t)sec[2];
                double2 v;
                MM_CUDA(ctx, cudaMemcpy(&v, b->phat + at, sizeof v, cudaMemcpyDeviceToHost));
                v.x += sqrt(deficit);
                MM_CUDA(ctx, cudaMemcpy(b->phat + at, &v, sizeof v, cudaMemcpyHostToDevice));
            }
        } else {
            k_scale_c<<<grid_blocks(npts * d), 256, 0, ctx->stream>>>(b->phat, npts * d,
                                                                     sqrt(b->target / nrm));
            MM_LAUNCH_CHECK(ctx);
        }
        // Rayleigh quotient, multiplier ascent, primal residual
        k_form_grad<<<blocks, 256, 0, ctx->stream>>>(b->phat, b->shift, b->Gp, d, npts);
        MM_LAUNCH_CHECK(ctx);
        if ((rc = fft_fields(ctx, b->Gp, D, true))) return rc;
        k_scale_c<<<grid_blocks(npts * D), 256, 0, ctx->stream>>>(b->Gp, npts * D, inv_n);
        MM_LAUNCH_CHECK(ctx);
        b->have_gp = true;
        k_rayleigh<<<blocks, 256, 0, ctx->stream>>>(b->Gp, b->G, b->g, b->L, D, npts, rho,
                                                    ctx->partials, ctx->red_out, ctx->red_count);
        MM_LAUNCH_CHECK(ctx);
        double r[2];
        if ((rc = mm_fetch_reduction(ctx, 2, r))) return rc;
        beta = r[0] / (double)npts;
        primal = sqrt(r[1] / (double)npts);
        if (!isfinite(beta) || !isfinite(primal) || beta < 4.0 * floor_ - mu_rep) {
            diverged = true;
            break;
        }
        const double dbeta = fabs(beta - b->beta_prev) / fmax(fabs(beta), mu_rep * 1e-12);
        b->beta_prev = beta;
        if (dbeta < tol_beta && primal < tol_primal * fmax(1.0, fabs(beta))) {
            converged = true;
            break;
        }
    }
    out[0] = beta;
    out[1] = primal;
    out[2] = (double)std::min(it, max_iter);
    out[3] = converged ? 1.0 : 0.0;
    out[4] = diverged ? 1.0 : 0.0;
    return MM_OK;
}

// p = IFFT(phat) (1/npts), complex AoS
int mm_bloch_mode(mm_ctx *ctx, double *p_out) {
    if (!ctx || !p_out) return MM_ERR_PARAM;
    ctx->gen++;  // invalidates a speculative projection front
    mm_bloch_state *b = ctx->bloch;
    if (!b) return mm_fail(ctx, MM_ERR_CONFIG, "mm_bloch_setup was not called");
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    const int d = ctx->dim;
    const int64_t npts = b->npts;
    MM_CUDA(ctx, cudaMemcpyAsync(b->num, b->phat, sizeof(double2) * d * npts,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    int rc = fft_fields(ctx, b->num, d, true);
    if (rc) return rc;
    double *tmp = nullptr;
    if ((rc = mm_alloc(ctx, (void **)&tmp, sizeof(double) * 2 * d * npts))) return rc;
    k_soa_complex_to_aos<<<grid_blocks(npts * d), 256, 0, ctx->stream>>>(b->num, tmp, d, npts,
                                                                         1.0 / (double)npts);
    MM_LAUNCH_CHECK(ctx);
    MM_CUDA(ctx, cudaMemcpyAsync(p_out, tmp, sizeof(double) * 2 * d * npts,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_free(ctx, tmp);
    ctx->bytes -= (int64_t)(sizeof(double) * 2 * d * npts);
    return MM_OK;
}

}  // extern "C"
