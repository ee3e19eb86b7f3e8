// Local (per-voxel) constitutive step for the Mooney-Rivlin and quadratic
// materials: ADMM step 1 of solver.py:252-265.
//
// One thread per voxel, fields SoA in HBM (coalesced 8-byte loads per
// component), all per-point state in registers.  Two algorithms, each a
// faithful restatement of the reference's:
//   * k_mr2d      — the compiled 2D kernel, mooney_rivlin.py:169-255
//   * k_descent   — the vectorised numpy descent used by 3D Mooney-Rivlin
//                   (mooney_rivlin.py:126-162) and the quadratic material
//                   (quadratic.py:46-69), base.py:124-230.  Its only
//                   cross-point coupling (the stall guard every 32 sweeps,
//                   base.py:224-229) is honoured by running the sweep loop in
//                   32-sweep segments with a host check in between, and only
//                   when the call may exceed 64 sweeps (below that the guard
//                   cannot fire).
// Each launch ends with a deterministic block + grid reduction of the batch
// statistics (sum res^2, converged count, max sweeps, guard sum, sum F).
#include <math.h>

#include <algorithm>
#include <stdint.h>
#include <string.h>

#include "mm_internal.cuh"

namespace {

constexpr double BT_DECREASE = 1e-4;  // base.py:37
constexpr double BT_SHRINK = 0.5;     // base.py:38
constexpr int MAX_BT = 60;            // base.py:39
constexpr double MEAS_EPS = 64.0 * 2.220446049250313e-16;  // base.py:41

#ifndef MM_LOCAL_THREADS
#define MM_LOCAL_THREADS 128
#endif
constexpr int LOCAL_THREADS = MM_LOCAL_THREADS;
#ifndef LOCAL_MIN_BLOCKS
#define LOCAL_MIN_BLOCKS 4
#endif
#ifndef MM_B_SMEM  // fused pass: B and lam_{k+1} in shared memory instead of registers:
#define MM_B_SMEM 0  // measured 2.05 -> 2.27 ms (4 blocks/SM), 2.70 ms (5 blocks): off
#endif
#ifndef MM_PREFETCH  // L2 prefetch of the next grid-stride point (prefetch_point):
#define MM_PREFETCH 0  // measured 2.05 -> 2.13 ms in the fused pass at 256^3, off
#endif

// ---------------------------------------------------------------------------
// log(J) of the Mooney-Rivlin objective, table-driven.  x = 2^k z with z in
// [0.6875, 1.375) split into 128 subintervals (7 leading bits of the
// biased representation); log x = k ln2 + log(c) + log1p(r), r = z/c - 1,
// |r| < 0.0039, log1p(r) as its degree-7 Taylor polynomial (truncation
// < 1e-20), log(c) in double-double from a host long-double table.  Absolute
// error is ~1e-19 for x near 1 (where the objective evaluates it: J = det F
// ~ 1) -- far below one ulp of the objective -- at ~25 instructions instead
// of the ~45 of the libdevice routine, which took 28 % of the local step's
// instructions (ncu source view).  Non-normal or non-positive x fall back to
// log().
// ---------------------------------------------------------------------------
constexpr int LOGTAB_N = 128;
#ifndef MM_LOGK_CONST  // 1: log_pos constants from the constant bank (c_logk)
#define MM_LOGK_CONST 1
#endif
#if MM_LOGK_CONST
#define MM_LOGK(i) c_logk[i]
#else
#define MM_LOGK(i) (((const double[8]){1.0 / 7.0, -1.0 / 6.0, 0.2, -0.25, 1.0 / 3.0, -0.5, \
                                       0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45})[i])
#endif
__device__ double g_logtab[3 * LOGTAB_N];  // invc | log c (hi) | log c (lo)
static bool g_logtab_ready[64];

// polynomial / ln 2 constants as constant-bank operands of the DFMAs (as
// double immediates each use was rematerialised by two UMOVs per evaluation)
__constant__ double c_logk[8] = {1.0 / 7.0, -1.0 / 6.0, 0.2, -0.25, 1.0 / 3.0, -0.5,
                                 0x1.62e42fefa3800p-1, 0x1.ef35793c76730p-45};

__device__ __forceinline__ double log_pos(double x, const double *__restrict__ T) {
    const uint64_t ix = (uint64_t)__double_as_longlong(x);
    if (ix - 0x0010000000000000ULL >= 0x7fe0000000000000ULL) return log(x);
    const uint64_t tmp = ix - 0x3fe6000000000000ULL;
    const int i = (int)((tmp >> 45) & (LOGTAB_N - 1));
    const double kd = (double)((int64_t)tmp >> 52);
    const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ULL)));
    const double r = fma(z, T[i], -1.0);
    const double w = fma(kd, MM_LOGK(6), T[LOGTAB_N + i]);
    const double hi = w + r;
    const double lo = (w - hi) + r;
    const double r2 = r * r;
    double p = fma(r, MM_LOGK(0), MM_LOGK(1));
    p = fma(r, p, MM_LOGK(2));
    p = fma(r, p, MM_LOGK(3));
    p = fma(r, p, MM_LOGK(4));
    p = fma(r, p, MM_LOGK(5));
    return hi + (fma(kd, MM_LOGK(7), T[2 * LOGTAB_N + i]) + fma(r2, p, lo));
}

static int ensure_logtab(mm_ctx *ctx) {
    const int dev = ctx->device;
    if (dev >= 0 && dev < 64 && g_logtab_ready[dev]) return MM_OK;
    double h[3 * LOGTAB_N];
    for (int i = 0; i < LOGTAB_N; ++i) {
        const uint64_t lo = 0x3fe6000000000000ULL + ((uint64_t)i << 45);
        const uint64_t hi = 0x3fe6000000000000ULL + ((uint64_t)(i + 1) << 45);
        double zl, zh;
        memcpy(&zl, &lo, 8);
        memcpy(&zh, &hi, 8);
        const long double c = 0.5L * ((long double)zl + (long double)zh);
        const double invc = (double)(1.0L / c);
        const long double lc = -logl((long double)invc);  // log c' with c' = 1/invc exactly
        h[i] = invc;
        h[LOGTAB_N + i] = (double)lc;
        h[2 * LOGTAB_N + i] = (double)(lc - (long double)(double)lc);
    }
    MM_CUDA(ctx, cudaMemcpyToSymbol(g_logtab, h, sizeof h));
    if (dev >= 0 && dev < 64) g_logtab_ready[dev] = true;
    return MM_OK;
}

// Largest double T with sqrt_rn(T) <= tol, so that sqrt(gs) > tol <=> gs > T
// exactly (sqrt is correctly rounded and monotone): the sweep loop tests the
// squared gradient norm and takes square roots only where the reference's
// residual value itself is needed.
static double gs_threshold(double tol) {
    if (tol != tol) return tol;
    if (tol < 0.0) return -INFINITY;
    if (tol == 0.0 || isinf(tol)) return tol;
    double x = tol * tol;
    while (x > 0.0 && sqrt(x) > tol) x = nextafter(x, 0.0);
    while (sqrt(nextafter(x, INFINITY)) <= tol) x = nextafter(x, INFINITY);
    return x;
}

#ifndef MM_LOCAL_GRID
#define MM_LOCAL_GRID 16  // grid-stride blocks per SM (x 128 / LOCAL_THREADS)
#endif
inline int local_blocks(int64_t M) {
    int64_t b = (M + LOCAL_THREADS - 1) / LOCAL_THREADS;
    return (int)std::min<int64_t>(b, 148 * MM_LOCAL_GRID * 128 / LOCAL_THREADS);
}

// One point of the compiled 2D kernel (mooney_rivlin.py:169-255).
__device__ __forceinline__ void mr2d_point(double &a, double &b, double &c, double &d,
                                           const double (&gv)[4], double l00, double l01,
                                           double l10, double l11, double m, double k,
                                           double rho, double tol, int64_t max_sweeps,
                                           double phi_scale, double &res, int64_t &nsw) {
    const double g00 = gv[0], g01 = gv[1], g10 = gv[2], g11 = gv[3];
    double t = 1.0 / (rho + m + 4.0 * k);
    const double tmax = 16.0 * t;
    bool freemode = false;
    double res_prev = 1e300;
    res = 0.0;
    nsw = 0;
    for (int64_t it = 0; it < max_sweeps + 1; ++it) {
        const double J = a * d - b * c;
        const double iJ = 1.0 / J;
        const double jm1 = J - 1.0;
        const double s00 = m * (a - d * iJ) + k * jm1 * d;
        const double s01 = m * (b + c * iJ) - k * jm1 * c;
        const double s10 = m * (c + b * iJ) - k * jm1 * b;
        const double s11 = m * (d - a * iJ) + k * jm1 * a;
        const double r00 = s00 - l00 - rho * (g00 - a);
        const double r01 = s01 - l01 - rho * (g01 - b);
        const double r10 = s10 - l10 - rho * (g10 - c);
        const double r11 = s11 - l11 - rho * (g11 - d);
        const double gsq = r00 * r00 + r01 * r01 + r10 * r10 + r11 * r11;
        res = sqrt(gsq);
        if (freemode) {
            if (res > res_prev) t *= BT_SHRINK;
            else t = fmin(t * 1.3, tmax);
            res_prev = res;
        }
        if (res < tol || nsw >= max_sweeps) break;
        nsw += 1;
        bool did = false;
        if (!freemode) {
            const double W = 0.5 * m * (a * a + b * b + c * c + d * d - 2.0 * log(J) - 2.0) +
                             0.5 * k * jm1 * jm1;
            const double phi0 =
                W - (l00 * a + l01 * b + l10 * c + l11 * d) +
                0.5 * rho * ((g00 - a) * (g00 - a) + (g01 - b) * (g01 - b) +
                             (g10 - c) * (g10 - c) + (g11 - d) * (g11 - d));
            if (BT_DECREASE * t * gsq <= MEAS_EPS * (fabs(phi0) + phi_scale)) {
                freemode = true;
                res_prev = res;
            } else {
                const double t_in = t;
                for (int bt = 0; bt < MAX_BT; ++bt) {
                    const double a2 = a - t * r00, b2 = b - t * r01;
                    const double c2 = c - t * r10, d2 = d - t * r11;
                    const double J2 = a2 * d2 - b2 * c2;
                    if (J2 > 1e-12) {
                        const double jm2 = J2 - 1.0;
                        const double W2 =
                            0.5 * m * (a2 * a2 + b2 * b2 + c2 * c2 + d2 * d2 - 2.0 * log(J2) - 2.0) +
                            0.5 * k * jm2 * jm2;
                        const double phi2 =
                            W2 - (l00 * a2 + l01 * b2 + l10 * c2 + l11 * d2) +
                            0.5 * rho * ((g00 - a2) * (g00 - a2) + (g01 - b2) * (g01 - b2) +
                                         (g10 - c2) * (g10 - c2) + (g11 - d2) * (g11 - d2));
                        if (phi2 <= phi0 - BT_DECREASE * t * gsq) {
                            a = a2; b = b2; c = c2; d = d2;
                            did = true;
                            break;
                        }
                    }
                    t *= BT_SHRINK;
                }
                if (did) {
                    t = fmin(t * 1.6, tmax);
                } else {
                    freemode = true;
                    t = t_in;
                    res_prev = res;
                }
            }
        }
        if (freemode && !did) {
            for (int bt = 0; bt < 12; ++bt) {
                const double a2 = a - t * r00, b2 = b - t * r01;
                const double c2 = c - t * r10, d2 = d - t * r11;
                if (a2 * d2 - b2 * c2 > 1e-12) {
                    a = a2; b = b2; c = c2; d = d2;
                    break;
                }
                t *= BT_SHRINK;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// 2D compiled kernel (mooney_rivlin.py:169-255)
// slots: 0 sum res^2, 1 n_conv, 2 max nsw, 3..6 sum F
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(LOCAL_THREADS)
k_mr2d(double *__restrict__ F, const GSrc gs, const double *__restrict__ Lam,
       const double *__restrict__ mu, const double *__restrict__ kap, int64_t M, double rho,
       double tol, int64_t max_sweeps, double phi_scale, double *__restrict__ res_out,
       int32_t *__restrict__ nsw_out, double *partials, double *red_out, unsigned int *count) {
    __shared__ double smem[32 * 8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double a = F[p], b = F[M + p], c = F[2 * M + p], d = F[3 * M + p];
        double gv[4];
        gsrc_load<2>(gs, p, gv);
        const double l00 = Lam[p], l01 = Lam[M + p], l10 = Lam[2 * M + p], l11 = Lam[3 * M + p];
        const double m = mu[p], k = kap[p];
        double res;
        int64_t nsw;
        mr2d_point(a, b, c, d, gv, l00, l01, l10, l11, m, k, rho, tol, max_sweeps, phi_scale, res,
                   nsw);
        F[p] = a; F[M + p] = b; F[2 * M + p] = c; F[3 * M + p] = d;
        if (res_out) res_out[p] = res;
        if (nsw_out) nsw_out[p] = (int32_t)nsw;
        acc[0] += res * res;
        acc[1] += (res < tol) ? 1.0 : 0.0;
        acc[2] = fmax(acc[2], (double)nsw);
        acc[3] += a; acc[4] += b; acc[5] += c; acc[6] += d;
        acc[7] += (double)nsw;
    }
    const int ops[8] = {RED_SUM, RED_SUM, RED_MAX, RED_SUM, RED_SUM, RED_SUM, RED_SUM, RED_SUM};
    block_reduce<8>(acc, ops, smem);
    grid_finalize<8>(acc, ops, partials, red_out, count, smem);
}

// Per-thread batch accumulators kept in shared memory ([slot][thread]) so
// they do not occupy registers across the sweep loop; touched once per point.
template <int K>
struct SmemAcc {
    double *p;
    __device__ __forceinline__ void init(double *base) {
        p = base + threadIdx.x;
#pragma unroll
        for (int q = 0; q < K; ++q) p[q * LOCAL_THREADS] = 0.0;
    }
    __device__ __forceinline__ void add(int q, double v) { p[q * LOCAL_THREADS] += v; }
    __device__ __forceinline__ void max(int q, double v) {
        p[q * LOCAL_THREADS] = fmax(p[q * LOCAL_THREADS], v);
    }
    __device__ __forceinline__ void load(double (&acc)[K]) const {
#pragma unroll
        for (int q = 0; q < K; ++q) acc[q] = p[q * LOCAL_THREADS];
    }
};

// ---------------------------------------------------------------------------
// vectorised descent restated per point (base.py:124-230)
// ---------------------------------------------------------------------------
enum { MAT_MR = 0, MAT_QUAD = 1 };

template <int D>
__device__ __forceinline__ double det_t(const double (&X)[D]) {
    if constexpr (D == 4) return X[0] * X[3] - X[1] * X[2];
    else
    return X[0] * (X[4] * X[8] - X[5] * X[7]) - X[1] * (X[3] * X[8] - X[5] * X[6]) +
           X[2] * (X[3] * X[7] - X[4] * X[6]);
}

template <int D>
__device__ __forceinline__ void cof_t(const double (&X)[D], double (&C)[D]) {
    if constexpr (D == 4) {
        C[0] = X[3]; C[1] = -X[2]; C[2] = -X[1]; C[3] = X[0];
    } else {
        C[0] = X[4] * X[8] - X[5] * X[7];
        C[1] = X[5] * X[6] - X[3] * X[8];
        C[2] = X[3] * X[7] - X[4] * X[6];
        C[3] = X[2] * X[7] - X[1] * X[8];
        C[4] = X[0] * X[8] - X[2] * X[6];
        C[5] = X[1] * X[6] - X[0] * X[7];
        C[6] = X[1] * X[5] - X[2] * X[4];
        C[7] = X[2] * X[3] - X[0] * X[5];
        C[8] = X[0] * X[4] - X[1] * X[3];
    }
}

// Per-thread column in shared memory ([i][thread], conflict-free): the fused
// pass keeps B = lam + rho G (read-only across the sweeps) there instead of
// in 18 registers, so more warps fit an SM (MM_B_SMEM).
struct SmemCol {
    const double *p;
    // volatile: a plain load is loop-invariant in the sweep loop and the
    // compiler would hoist all nine back into registers
    __device__ __forceinline__ double operator[](int i) const {
        return *(const volatile double *)(p + i * LOCAL_THREADS);
    }
};

// The per-point coupling  -lam:X + rho/2 |G - X|^2  is carried as
//   rho/2 |X|^2 - B:X + cG,   B = lam + rho G,  cG = rho/2 |G|^2,
// (identical up to roundoff) so only 9 + 1 doubles of (G, lam) stay live in
// registers across the sweep loop instead of 18.

// objective (mooney_rivlin.py:132-141 / quadratic.py:52-55); +inf if det <= 0
template <int MAT, int D, typename BT>
__device__ __forceinline__ double objective(const double (&X)[D], const BT &B,
                                            double cG, double m, double k, double rho,
                                            const double *__restrict__ LT) {
    double bx = 0.0, I1 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        bx += B[i] * X[i];
        I1 += X[i] * X[i];
    }
    const double coupling = 0.5 * rho * I1 - bx + cG;
    if constexpr (MAT == MAT_QUAD) return 0.5 * m * I1 + coupling;
    const double J = det_t<D>(X);
    if (J <= 0.0) return INFINITY;
    const double dd = (D == 4) ? 2.0 : 3.0;
    return 0.5 * m * (I1 - 2.0 * log_pos(J, LT) - dd) + 0.5 * k * (J - 1.0) * (J - 1.0) + coupling;
}

// objective given det X (>0) already computed by the admissibility test
template <int MAT, int D, typename BT>
__device__ __forceinline__ double objective_J(const double (&X)[D], double J, const BT &B,
                                              double cG, double m, double k, double rho,
                                              const double *__restrict__ LT) {
    double bx = 0.0, I1 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        bx += B[i] * X[i];
        I1 += X[i] * X[i];
    }
    const double coupling = 0.5 * rho * I1 - bx + cG;
    if constexpr (MAT == MAT_QUAD) return 0.5 * m * I1 + coupling;
    const double dd = (D == 4) ? 2.0 : 3.0;
    return 0.5 * m * (I1 - 2.0 * log_pos(J, LT) - dd) + 0.5 * k * (J - 1.0) * (J - 1.0) + coupling;
}

// gradient S(X) - lam - rho (G - X) = S(X) + rho X - B
// (mooney_rivlin.py:143-151 / quadratic.py:57-58)
template <int MAT, int D, typename BT>
__device__ __forceinline__ void gradient(const double (&X)[D], const BT &B, double m,
                                         double k, double rho, double (&g)[D]) {
    if constexpr (MAT == MAT_QUAD) {
#pragma unroll
        for (int i = 0; i < D; ++i) g[i] = (m + rho) * X[i] - B[i];
    } else {
        const double J = det_t<D>(X);
        double C[D];
        cof_t<D>(X, C);
        const double iJ = 1.0 / J;
        // S + rho X - B with S = m (X - F^{-T}) + k (J^2 - J) F^{-T}, F^{-T} = C / J
        const double cf = (k * (J * J - J) - m) * iJ;
        const double mr = m + rho;
#pragma unroll
        for (int i = 0; i < D; ++i) g[i] = fma(mr, X[i], fma(cf, C[i], -B[i]));
    }
}

// gradient at X with det X = J already known (the accepted trial's det)
template <int MAT, int D, typename BT>
__device__ __forceinline__ void gradient_J(const double (&X)[D], double J, const BT &B,
                                           double m, double k, double rho, double (&g)[D]) {
    if constexpr (MAT == MAT_QUAD) {
#pragma unroll
        for (int i = 0; i < D; ++i) g[i] = (m + rho) * X[i] - B[i];
    } else {
        double C[D];
        cof_t<D>(X, C);
        const double iJ = 1.0 / J;
        const double cf = (k * (J * J - J) - m) * iJ;
        const double mr = m + rho;
#pragma unroll
        for (int i = 0; i < D; ++i) g[i] = fma(mr, X[i], fma(cf, C[i], -B[i]));
    }
}

template <int MAT, int D>
__device__ __forceinline__ bool admissible(const double (&X)[D]) {
    if (MAT == MAT_QUAD) return true;
    return det_t<D>(X) > 0.0;
}

// One point of the vectorised descent (base.py:124-230) for global sweeps
// [s0, s1): X updated in place; t, freem, nsw persist across segments.
// tol_gs = gs_threshold(tol): the activity test res > tol is evaluated as
// |g|^2 > tol_gs (exactly equivalent); res = sqrt(|g|^2) is formed only for
// the free-mode trend test and on return.
template <int MAT, int D, typename BT>
__device__ __forceinline__ void descent_point(double (&X)[D], const BT &B, double cG,
                                              double m, double k, double rho, double tol_gs,
                                              double phi_scale, int s0, int s1, double tmax,
                                              double &t, bool &freem, int &nsw, double &res,
                                              bool &moved, const double *__restrict__ LT) {
    double g[D], Xt[D];
    gradient<MAT, D>(X, B, m, k, rho, g);
    double gs = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) gs += g[i] * g[i];
    moved = false;
    bool have_phi = false;
    double phi_cur = 0.0;
    // a point is active at global sweep s iff it was active at every
    // earlier sweep (nsw == s) and res > tol; once inactive it stays so
    for (int s = s0; s < s1; ++s) {
        if (nsw != s || !(gs > tol_gs)) break;
        nsw += 1;
        moved = true;
        bool in_free = freem, in_arm = false;
        double phi0 = 0.0, gsq = 0.0;
        double Jacc = 0.0;      // det of the accepted trial point (reused by the gradient)
        bool armijo_step = false, x_changed = false;
        if (!freem) {
            // phi at the current X is known when the previous sweep ended on
            // an accepted Armijo step or took no step (same X, same bits)
            phi0 = have_phi ? phi_cur : objective<MAT, D>(X, B, cG, m, k, rho, LT);
            phi_cur = phi0;
            have_phi = true;
            gsq = gs;  // same g, same summation order as res (base.py:167 vs :156)
            // base.py:168-171: unmeasurable decrease -> free mode, and the
            // point takes this sweep's free step
            const bool meas = BT_DECREASE * t * gsq > MEAS_EPS * (fabs(phi0) + phi_scale);
            if (!meas) {
                freem = true;
                in_free = true;
            } else {
                in_arm = true;
            }
        }
        const double gs_before = gs;
        if (in_arm) {
            const double t_in = t;
            bool accepted = false;
            for (int bt = 0; bt < MAX_BT; ++bt) {
#pragma unroll
                for (int i = 0; i < D; ++i) Xt[i] = X[i] - t * g[i];
                double phi_try = INFINITY;
                double Jt = 0.0;
                if constexpr (MAT == MAT_QUAD) {
                    phi_try = objective<MAT, D>(Xt, B, cG, m, k, rho, LT);
                } else {
                    Jt = det_t<D>(Xt);  // admissibility and objective share J
                    if (Jt > 0.0) phi_try = objective_J<MAT, D>(Xt, Jt, B, cG, m, k, rho, LT);
                }
                if (phi_try <= phi0 - BT_DECREASE * t * gsq) {
#pragma unroll
                    for (int i = 0; i < D; ++i) X[i] = Xt[i];
                    Jacc = Jt;
                    armijo_step = x_changed = true;
                    phi_cur = phi_try;
                    accepted = true;
                    break;
                }
                t *= BT_SHRINK;
            }
            if (accepted) {
                t = fmin(t * 1.6, tmax);
            } else {
                freem = true;
                t = t_in;
            }
        }
        if (in_free) {
#pragma unroll
            for (int i = 0; i < D; ++i) Xt[i] = X[i] - t * g[i];
            bool took = admissible<MAT, D>(Xt);
            for (int bt = 0; bt < 12 && !took; ++bt) {
                t *= BT_SHRINK;
#pragma unroll
                for (int i = 0; i < D; ++i) Xt[i] = X[i] - t * g[i];
                took = admissible<MAT, D>(Xt);
            }
            if (took) {
#pragma unroll
                for (int i = 0; i < D; ++i) X[i] = Xt[i];
                have_phi = false;
                x_changed = true;
            }
        }
        // an unchanged X keeps its gradient, |g|^2 and residual bit for bit
        if (x_changed) {
            if (armijo_step) gradient_J<MAT, D>(X, Jacc, B, m, k, rho, g);
            else gradient<MAT, D>(X, B, m, k, rho, g);
            gs = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) gs += g[i] * g[i];
        }
        if (in_free) {  // residual trend (base.py:218-223) on the residual values
            if (sqrt(gs) > sqrt(gs_before)) t *= BT_SHRINK;
            else t = fmin(t * 1.3, tmax);
        }
    }
    res = sqrt(gs);
}

// stage the log table into shared memory (every thread of the block calls)
__device__ __forceinline__ void load_logtab(double *sh) {
    for (int i = threadIdx.x; i < 3 * LOGTAB_N; i += blockDim.x) sh[i] = g_logtab[i];
    __syncthreads();
}

// slots: 0 sum res^2, 1 n_conv (res < tol), 2 max nsw (cumulative),
//        3 guard sum (sum res where res > tol), 4..4+D sum F
template <int MAT, int D>
__global__ void __launch_bounds__(LOCAL_THREADS, LOCAL_MIN_BLOCKS)
k_descent(double *__restrict__ F, const GSrc gs, const double *__restrict__ Lam,
          const double *__restrict__ modA, const double *__restrict__ modB, int64_t M,
          double rho, double tol, double tol_gs, double phi_scale, int s0, int s1,
          double *__restrict__ tstate, uint8_t *__restrict__ freestate, double *__restrict__ res_out,
          int32_t *__restrict__ nsw_io, double *__restrict__ Tout, double *partials,
          double *red_out, unsigned int *count) {
    constexpr int K = 5 + D;  // ..., last slot: sum of per-point sweeps
    __shared__ double smem[32 * K];
    __shared__ double sacc[K * LOCAL_THREADS];
    __shared__ double ltab[3 * LOGTAB_N];
    load_logtab(ltab);
    SmemAcc<K> A;
    A.init(sacc);
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double X[D], B[D];
        double cG = 0.0;
        gsrc_load<(D == 4 ? 2 : 3)>(gs, p, B);  // B holds grad_u until the next line
        if (MM_PREFETCH) prefetch_point<(D == 4 ? 2 : 3)>(gs, F, Lam, modA, modB,
                                                          p + (int64_t)gridDim.x * blockDim.x);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            X[i] = F[i * M + p];
            const double gi = B[i];
            B[i] = Lam[i * M + p] + rho * gi;
            cG += gi * gi;
        }
        cG *= 0.5 * rho;
        const double m = modA[p];
        const double k = (MAT == MAT_MR) ? modB[p] : 0.0;
        // t0 ~ inverse local curvature (mooney_rivlin.py:388-390, quadratic.py:63)
        const double t0 = (MAT == MAT_MR) ? 1.0 / (rho + m + 4.0 * k) : 1.0 / (rho + m);
        const double tmax = t0 * 16.0;
        double t = t0;
        bool freem = false;
        int nsw = 0;
        int nsw_start = 0;
        if (s0 > 0) {
            t = tstate[p];
            freem = freestate[p] != 0;
            nsw = nsw_io[p];
            nsw_start = nsw;
        }
        double res = 0.0;
        bool moved = false;
        descent_point<MAT, D>(X, B, cG, m, k, rho, tol_gs, phi_scale, s0, s1, tmax, t, freem, nsw,
                              res, moved, ltab);
        if (moved) {
#pragma unroll
            for (int i = 0; i < D; ++i) F[i * M + p] = X[i];
            if (Tout) {  // keep T = F - lam / rho current for the projection
                const double irho = 1.0 / rho;
#pragma unroll
                for (int i = 0; i < D; ++i) Tout[i * M + p] = fma(-Lam[i * M + p], irho, X[i]);
            }
        }
        if (tstate) {
            tstate[p] = t;
            freestate[p] = freem ? 1 : 0;
        }
        if (nsw_io) nsw_io[p] = nsw;
        if (res_out) res_out[p] = res;
        A.add(0, res * res);
        A.add(1, (res < tol) ? 1.0 : 0.0);
        A.max(2, (double)nsw);
        A.add(3, (res > tol) ? res : 0.0);
#pragma unroll
        for (int i = 0; i < D; ++i) A.add(4 + i, X[i]);
        A.add(K - 1, (double)(nsw - (s0 > 0 ? nsw_start : 0)));
    }
    double acc[K];
    A.load(acc);
    int ops[K];
#pragma unroll
    for (int k = 0; k < K; ++k) ops[k] = RED_SUM;
    ops[2] = RED_MAX;
    block_reduce<K>(acc, ops, smem);
    grid_finalize<K>(acc, ops, partials, red_out, count, smem);
}



// ---------------------------------------------------------------------------
// Multiplier ascent of outer iteration k fused with the first local chunk of
// iteration k+1 (solver.py:279, then :255-264 of the next call).  The
// projection already left u_{k+1} current and ubar = <grad u>_{k+1}, so
// grad_u_{k+1} = ubar + D u is rebuilt in registers; lam_{k+1} =
// lam_k + rho_k (grad_u - F) is stored; then (SWEEP) the point runs the
// local sweeps with rho_{k+1} and the policy tolerance, exactly as a
// standalone first chunk would.  One pass over (u, F, lam, mu, kappa)
// instead of a gradient pass plus a local pass, and the FP64-heavy sweeps
// overlap the memory traffic of the update.
// slots: 0 sum res^2, 1 n_conv, 2 max nsw, 3 guard sum, 4.. sum F (D), then sum lam (D)
// ALGO: 0 = descent (3D MR, quadratic), 1 = compiled 2D MR kernel
// ---------------------------------------------------------------------------
template <int MAT, int D, int ALGO, bool SWEEP>
__global__ void __launch_bounds__(LOCAL_THREADS, LOCAL_MIN_BLOCKS)
k_update_local(double *__restrict__ F, double *__restrict__ Lam, double *__restrict__ Gout,
               double *__restrict__ Tout, const GSrc gs,
               const double *__restrict__ modA, const double *__restrict__ modB, int64_t M,
               double rho_k, double rho, double tol, double tol_gs, double phi_scale, int chunk,
               double *__restrict__ res_out, int32_t *__restrict__ nsw_out, double *partials,
               double *red_out, unsigned int *count, const DevStep *__restrict__ ds) {
    constexpr int K = 5 + 2 * D;  // ..., last slot: sum of per-point sweeps
    if (ds) {  // pipelined step: parameters decided on the device
        if (ds->skip) return;  // every block, before any side effect
        rho = ds->rho_next;
        tol = ds->tol;
        tol_gs = ds->tol_gs;
    }
    // MM_B_SMEM: B = lam + rho G and lam_{k+1} (for the T store) live in
    // per-thread shared-memory columns across the sweeps; the block
    // reduction's scratch reuses that space after the loop
    constexpr bool BSM = MM_B_SMEM && SWEEP && ALGO == 0;
    __shared__ double sBL[BSM ? 2 * D * LOCAL_THREADS : 32 * K];
    double *smem = sBL;
    static_assert(!BSM || 2 * D * LOCAL_THREADS >= 32 * K, "reduction scratch fits");
    __shared__ double sacc[K * LOCAL_THREADS];
    __shared__ double ltab[(SWEEP && ALGO == 0) ? 3 * LOGTAB_N : 1];
    if constexpr (SWEEP && ALGO == 0) load_logtab(ltab);
    SmemAcc<K> A;
    A.init(sacc);
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double G[D], X[D], L[D];
        gsrc_load<(D == 4 ? 2 : 3)>(gs, p, G);
        if (MM_PREFETCH && SWEEP) prefetch_point<(D == 4 ? 2 : 3)>(gs, F, Lam, modA, modB,
                                                                   p + (int64_t)gridDim.x * blockDim.x);
#pragma unroll
        for (int i = 0; i < D; ++i) {
            X[i] = F[i * M + p];
            L[i] = Lam[i * M + p];
        }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            L[i] = L[i] + rho_k * (G[i] - X[i]);  // solver.py:277-279
            Lam[i * M + p] = L[i];
            if (Gout) Gout[i * M + p] = G[i];     // keep grad_u explicit for the next pass
            A.add(4 + D + i, L[i]);
        }
        if (SWEEP) {
            const double m = modA[p];
            const double k = (MAT == MAT_MR) ? modB[p] : 0.0;
            double res = 0.0;
            int nsw = 0;
            bool moved = false;
            if constexpr (ALGO == 1) {
                int64_t nsw64 = 0;
                double a = X[0], b = X[1], c = X[2], d = X[3];
                const double gv[4] = {G[0], G[1], G[2], G[3]};
                mr2d_point(a, b, c, d, gv, L[0], L[1], L[2], L[3], m, k, rho, tol, chunk,
                           phi_scale, res, nsw64);
                nsw = (int)nsw64;
                moved = nsw > 0;
                X[0] = a; X[1] = b; X[2] = c; X[3] = d;
            } else if constexpr (BSM) {
                double *Bs = sBL + threadIdx.x, *Ls = sBL + D * LOCAL_THREADS + threadIdx.x;
                double cG = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    Bs[i * LOCAL_THREADS] = L[i] + rho * G[i];
                    Ls[i * LOCAL_THREADS] = L[i];
                    cG += G[i] * G[i];
                }
                cG *= 0.5 * rho;
                const double t0 = (MAT == MAT_MR) ? 1.0 / (rho + m + 4.0 * k) : 1.0 / (rho + m);
                double t = t0;
                bool freem = false;
                descent_point<MAT, D>(X, SmemCol{Bs}, cG, m, k, rho, tol_gs, phi_scale, 0, chunk,
                                      t0 * 16.0, t, freem, nsw, res, moved, ltab);
            } else {
                double B[D];
                double cG = 0.0;
#pragma unroll
                for (int i = 0; i < D; ++i) {
                    B[i] = L[i] + rho * G[i];
                    cG += G[i] * G[i];
                }
                cG *= 0.5 * rho;
                const double t0 = (MAT == MAT_MR) ? 1.0 / (rho + m + 4.0 * k) : 1.0 / (rho + m);
                double t = t0;
                bool freem = false;
                descent_point<MAT, D>(X, B, cG, m, k, rho, tol_gs, phi_scale, 0, chunk, t0 * 16.0,
                                      t, freem, nsw, res, moved, ltab);
            }
            if (moved) {
#pragma unroll
                for (int i = 0; i < D; ++i) F[i * M + p] = X[i];
            }
            if (Tout) {  // T = F - lam / rho for the next projection (row_fwd's expression)
                const double irho = 1.0 / rho;
                if constexpr (BSM) {
                    const double *Ls = sBL + D * LOCAL_THREADS + threadIdx.x;
#pragma unroll
                    for (int i = 0; i < D; ++i)
                        Tout[i * M + p] = fma(-Ls[i * LOCAL_THREADS], irho, X[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < D; ++i) Tout[i * M + p] = fma(-L[i], irho, X[i]);
                }
            }
            if (res_out) {
                res_out[p] = res;
                nsw_out[p] = nsw;
            }
            A.add(0, res * res);
            A.add(1, (res < tol) ? 1.0 : 0.0);
            A.max(2, (double)nsw);
            A.add(3, (res > tol) ? res : 0.0);
#pragma unroll
            for (int i = 0; i < D; ++i) A.add(4 + i, X[i]);
            A.add(K - 1, (double)nsw);
        }
    }
    double acc[K];
    A.load(acc);
    int ops[K];
#pragma unroll
    for (int q = 0; q < K; ++q) ops[q] = RED_SUM;
    ops[2] = RED_MAX;
    if constexpr (BSM) __syncthreads();  // every thread is done with its sBL column
    block_reduce<K>(acc, ops, smem);
    grid_finalize<K>(acc, ops, partials, red_out, count, smem);
}

// ---------------------------------------------------------------------------
// det F > 0 pre-check (base.py:116-121), run once after F is uploaded
// ---------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256)
k_count_bad_det(const double *__restrict__ F, int64_t M, double *partials, double *red_out,
                unsigned int *count) {
    __shared__ double smem[32];
    double acc[1] = {0.0};
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double X[D];
#pragma unroll
        for (int i = 0; i < D; ++i) X[i] = F[i * M + p];
        acc[0] += (det_t<D>(X) <= 0.0) ? 1.0 : 0.0;
    }
    const int ops[1] = {RED_SUM};
    block_reduce<1>(acc, ops, smem);
    grid_finalize<1>(acc, ops, partials, red_out, count, smem);
}

// per-component sums over points
template <int NC>
__global__ void __launch_bounds__(256)
k_field_sums(const double *__restrict__ f, int64_t M, double *partials, double *red_out,
             unsigned int *count) {
    __shared__ double smem[32 * NC];
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += f[c * M + p];
    }
    int ops[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) ops[c] = RED_SUM;
    block_reduce<NC>(acc, ops, smem);
    grid_finalize<NC>(acc, ops, partials, red_out, count, smem);
}

// first Piola stress of the hyperelastic models into P (SoA), the input of
// equilibrium_residual: Mooney-Rivlin mu (F - F^-T) + kappa (J^2 - J) F^-T
// (mooney_rivlin.py:78-85), quadratic c F (quadratic.py:34-36)
template <int MAT, int D>
__global__ void __launch_bounds__(256)
k_stress(const double *__restrict__ F, const double *__restrict__ modA,
         const double *__restrict__ modB, double *__restrict__ P, int64_t M) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double X[D];
#pragma unroll
        for (int i = 0; i < D; ++i) X[i] = F[i * M + p];
        const double m = modA[p];
        if constexpr (MAT == MAT_QUAD) {
#pragma unroll
            for (int i = 0; i < D; ++i) P[i * M + p] = m * X[i];
        } else {
            const double k = modB[p];
            const double J = det_t<D>(X);
            double C[D];
            cof_t<D>(X, C);
            const double kj = k * (J * J - J);
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const double finvt = C[i] / J;
                P[i * M + p] = m * (X[i] - finvt) + kj * finvt;
            }
        }
    }
}

}  // namespace

int mm_run_stress(mm_ctx *ctx, int material, double *P) {
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((ctx->M + threads - 1) / threads, 148 * 16);
    StageScope ss(ctx, MM_STAGE_OTHER);
    const bool quad = material == MM_MAT_QUADRATIC;
    const double *kap = quad ? ctx->modA : ctx->modB;
    if (!ctx->modA || !kap) return mm_fail(ctx, MM_ERR_CONFIG, "material moduli were never set");
    if (ctx->dim == 2) {
        if (quad) k_stress<MAT_QUAD, 4><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->modA, kap, P, ctx->M);
        else k_stress<MAT_MR, 4><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->modA, kap, P, ctx->M);
    } else {
        if (quad) k_stress<MAT_QUAD, 9><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->modA, kap, P, ctx->M);
        else k_stress<MAT_MR, 9><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->modA, kap, P, ctx->M);
    }
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

static int reduce_blocks(mm_ctx *ctx, int threads) {
    int64_t b = (ctx->M + threads - 1) / threads;
    return (int)std::min<int64_t>(b, 148 * 8);
}

int mm_run_field_sums(mm_ctx *ctx, const double *field, int ncomp, double *out) {
    const int blocks = reduce_blocks(ctx, 256);
    int rc = mm_ensure_partials(ctx, blocks);
    if (rc) return rc;
    {
        StageScope ss(ctx, MM_STAGE_OTHER);
        switch (ncomp) {
#define CASE(N)                                                                               \
    case N:                                                                                   \
        k_field_sums<N><<<blocks, 256, 0, ctx->stream>>>(field, ctx->M, ctx->partials,        \
                                                         ctx->red_out, ctx->red_count);       \
        break;
            CASE(1) CASE(2) CASE(3) CASE(4) CASE(9)
#undef CASE
            default: return mm_fail(ctx, MM_ERR_CONFIG, "field_sums: unsupported ncomp %d", ncomp);
        }
    }
    MM_LAUNCH_CHECK(ctx);
    return mm_fetch_reduction(ctx, ncomp, out);
}

int mm_check_det(mm_ctx *ctx, int *bad) {
    const int blocks = reduce_blocks(ctx, 256);
    int rc = mm_ensure_partials(ctx, blocks);
    if (rc) return rc;
    {
        StageScope ss(ctx, MM_STAGE_OTHER);
        if (ctx->dim == 2)
            k_count_bad_det<4><<<blocks, 256, 0, ctx->stream>>>(ctx->F, ctx->M, ctx->partials,
                                                                ctx->red_out, ctx->red_count);
        else
            k_count_bad_det<9><<<blocks, 256, 0, ctx->stream>>>(ctx->F, ctx->M, ctx->partials,
                                                                ctx->red_out, ctx->red_count);
    }
    MM_LAUNCH_CHECK(ctx);
    double v;
    rc = mm_fetch_reduction(ctx, 1, &v);
    if (rc) return rc;
    *bad = (int)v;
    return MM_OK;
}

int mm_ensure_points(mm_ctx *ctx) {
    int rc;
    if (!ctx->res && (rc = mm_alloc(ctx, (void **)&ctx->res, sizeof(double) * ctx->M))) return rc;
    if (!ctx->nsw && (rc = mm_alloc(ctx, (void **)&ctx->nsw, sizeof(int32_t) * ctx->M))) return rc;
    if (!ctx->ok && (rc = mm_alloc(ctx, (void **)&ctx->ok, ctx->M))) return rc;
    return MM_OK;
}

template <int MAT, int D>
static int launch_descent(mm_ctx *ctx, double rho, double tol, double phi_scale, int s0, int s1,
                          bool persist, bool want_points) {
    const int blocks = local_blocks(ctx->M);
    int rc = mm_ensure_partials(ctx, blocks);
    if (rc) return rc;
    StageScope ss(ctx, MM_STAGE_LOCAL);
    if ((rc = ensure_logtab(ctx))) return rc;
    // a later chunk keeps the fused pass's T field current for moved points
    const bool keepT = ctx->T_valid && ctx->Tbuf && ctx->T_rho == rho;
    if (!keepT) ctx->T_valid = false;
    k_descent<MAT, D><<<blocks, LOCAL_THREADS, 0, ctx->stream>>>(
        ctx->F, mm_gsrc(ctx), ctx->Lam, ctx->modA, MAT == MAT_MR ? ctx->modB : ctx->modA, ctx->M, rho,
        tol, gs_threshold(tol), phi_scale, s0, s1, persist ? ctx->tstate : nullptr,
        persist ? ctx->freestate : nullptr, want_points ? ctx->res : nullptr,
        (persist || want_points) ? ctx->nsw : nullptr, keepT ? ctx->Tbuf : nullptr,
        ctx->partials, ctx->red_out, ctx->red_count);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

static int launch_descent_any(mm_ctx *ctx, int material, double rho, double tol,
                              double phi_scale, int s0, int s1, bool persist, bool want_points) {
    const bool mr = material == MM_MAT_MR || material == MM_MAT_MR_DESCENT;
    if (ctx->dim == 2)
        return mr ? launch_descent<MAT_MR, 4>(ctx, rho, tol, phi_scale, s0, s1, persist, want_points)
                  : launch_descent<MAT_QUAD, 4>(ctx, rho, tol, phi_scale, s0, s1, persist,
                                                want_points);
    return mr ? launch_descent<MAT_MR, 9>(ctx, rho, tol, phi_scale, s0, s1, persist, want_points)
              : launch_descent<MAT_QUAD, 9>(ctx, rho, tol, phi_scale, s0, s1, persist,
                                            want_points);
}

int mm_run_lce(mm_ctx *ctx, double rho, double tol, int64_t max_sweeps, int want_points,
               mm_local_stats *out);

int mm_run_local(mm_ctx *ctx, int material, double rho, double tol, int64_t max_sweeps,
                 double phi_scale, int want_points, mm_local_stats *out) {
    int rc;
    const int D = ctx->D;
    memset(out, 0, sizeof *out);
    if (want_points && (rc = mm_ensure_points(ctx))) return rc;
    if (material == MM_MAT_LCE || (material == MM_MAT_MR && ctx->dim == 2))
        ctx->T_valid = false;  // these kernels do not maintain the T field
    if (material == MM_MAT_LCE) return mm_run_lce(ctx, rho, tol, max_sweeps, want_points, out);
    if (material == MM_MAT_MR && ctx->dim == 2) {
        // compiled 2D kernel (mooney_rivlin.py:169-255)
        const int blocks = local_blocks(ctx->M);
        if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
        {
            StageScope ss(ctx, MM_STAGE_LOCAL);
            k_mr2d<<<blocks, LOCAL_THREADS, 0, ctx->stream>>>(
                ctx->F, mm_gsrc(ctx), ctx->Lam, ctx->modA, ctx->modB, ctx->M, rho, tol, max_sweeps,
                phi_scale, want_points ? ctx->res : nullptr, want_points ? ctx->nsw : nullptr,
                ctx->partials, ctx->red_out, ctx->red_count);
        }
        MM_LAUNCH_CHECK(ctx);
        double r[7];
        if ((rc = mm_fetch_reduction(ctx, 8, r))) return rc;
        out->sum_nsw = r[7];
        out->sum_res2 = r[0];
        out->n_conv = (int64_t)r[1];
        out->sweeps = ctx->M ? (int64_t)r[2] : 0;
        for (int i = 0; i < 4; ++i) out->sum_F[i] = r[3 + i];
        if (want_points) MM_CUDA(ctx, cudaMemsetAsync(ctx->ok, 0, ctx->M, ctx->stream));
        return MM_OK;
    }
    // vectorised-descent semantics (base.py:124-230)
    if (material == MM_MAT_MR_DESCENT) material = MM_MAT_MR;
    if (material == MM_MAT_MR && !ctx->F_checked) {
        int bad = 0;
        if ((rc = mm_check_det(ctx, &bad))) return rc;
        if (bad) return mm_fail(ctx, MM_ERR_INADMISSIBLE, "det F <= 0 at %d point(s)", bad);
        ctx->F_checked = true;
    }
    const int K = 5 + D;
    double sum_nsw = 0.0;
    double r[MM_MAX_PARTIALS];
    const bool segmented = max_sweeps > 64;
    if (segmented) {
        if (!ctx->tstate && (rc = mm_alloc(ctx, (void **)&ctx->tstate, sizeof(double) * ctx->M)))
            return rc;
        if (!ctx->freestate && (rc = mm_alloc(ctx, (void **)&ctx->freestate, ctx->M))) return rc;
        if (!ctx->nsw && (rc = mm_alloc(ctx, (void **)&ctx->nsw, sizeof(int32_t) * ctx->M)))
            return rc;
    }
    int64_t sweeps = 0;
    if (!segmented) {
        rc = launch_descent_any(ctx, material, rho, tol, phi_scale, 0, (int)max_sweeps, false,
                                want_points);
        if (rc) return rc;
        if ((rc = mm_fetch_reduction(ctx, K, r))) return rc;
        sweeps = (int64_t)r[2];
        sum_nsw = r[K - 1];
    } else {
        double ref = INFINITY;
        while (sweeps < max_sweeps) {
            const int64_t s1 = std::min<int64_t>((sweeps / 32 + 1) * 32, max_sweeps);
            rc = launch_descent_any(ctx, material, rho, tol, phi_scale, (int)sweeps, (int)s1, true,
                                    want_points);
            if (rc) return rc;
            if ((rc = mm_fetch_reduction(ctx, K, r))) return rc;
            sum_nsw += r[K - 1];
            const int64_t mx = (int64_t)r[2];
            if (mx < s1) {  // every point stopped before s1
                sweeps = mx;
                break;
            }
            sweeps = s1;
            if (sweeps % 32 == 0) {  // stall guard, base.py:224-229
                const double cur = r[3];
                if (cur > 0.995 * ref) break;
                ref = cur;
            }
        }
    }
    out->sum_res2 = r[0];
    out->n_conv = (int64_t)r[1];
    out->sweeps = ctx->M ? sweeps : 0;
    for (int i = 0; i < D; ++i) out->sum_F[i] = r[4 + i];
    out->sum_nsw = sum_nsw;
    if (want_points) MM_CUDA(ctx, cudaMemsetAsync(ctx->ok, 0, ctx->M, ctx->stream));
    return MM_OK;
}

// ---------------------------------------------------------------------------
// fused multiplier ascent (+ first local chunk of the next iteration)
// ---------------------------------------------------------------------------
// Whether the fused pass also stores grad_u.  Measured on B200 at 256^3: not
// storing it (the next residual pass rebuilds grad_u_old from u_old by the
// same stencil) is 0.1 ms/iteration faster, so grad_u stays implicit.
constexpr bool kFusedStoresG = false;

template <int MAT, int D, int ALGO, bool SWEEP>
static int launch_update_local(mm_ctx *ctx, double rho_next, double tol, double phi_scale,
                               int chunk, bool want_points, const DevStep *ds = nullptr) {
    const int blocks = local_blocks(ctx->M);
    int rc = mm_ensure_partials(ctx, blocks);
    if (rc) return rc;
    StageScope ss(ctx, SWEEP ? MM_STAGE_FUSED : MM_STAGE_GRAD);
    if ((rc = ensure_logtab(ctx))) return rc;
    // T = F - lam / rho_next for the next projection (single-context grids
    // with packed even-length rows, where row_fwd uses this expression)
    double *Tout = nullptr;
    if (SWEEP && !ctx->points_only && ctx->n % 2 == 0 && ctx->opt_tfield) {
        if (!ctx->Tbuf && (rc = mm_alloc(ctx, (void **)&ctx->Tbuf, sizeof(double) * D * ctx->M)))
            return rc;
        Tout = ctx->Tbuf;
    }
    ctx->T_valid = false;
    k_update_local<MAT, D, ALGO, SWEEP><<<blocks, LOCAL_THREADS, 0, ctx->stream>>>(
        ctx->F, ctx->Lam, kFusedStoresG ? ctx->G : nullptr, Tout, mm_gsrc(ctx), ctx->modA, MAT == MAT_MR ? ctx->modB : ctx->modA, ctx->M,
        ctx->pending_rho, rho_next, tol, gs_threshold(tol), phi_scale, chunk, want_points ? ctx->res : nullptr,
        want_points ? ctx->nsw : nullptr, ctx->partials, ctx->red_out, ctx->red_count, ds);
    MM_LAUNCH_CHECK(ctx);
    if (Tout) {
        ctx->T_valid = true;
        ctx->T_rho = rho_next;  // pipelined: a placeholder until the decision is read
    }
    return MM_OK;
}

int mm_run_update(mm_ctx *ctx, int material, double rho_next, double tol, int64_t max_sweeps,
                  double phi_scale, int want_points, mm_local_stats *ls, mm_update_stats *us) {
    int rc;
    const int D = ctx->D;
    const bool sweep = ls != nullptr;
    if (!ctx->lam_pending)
        return mm_fail(ctx, MM_ERR_CONFIG, "no multiplier update pending (call mm_project_residuals)");
    if (want_points && (rc = mm_ensure_points(ctx))) return rc;
    if (!sweep) {
        // update only; the material does not matter
        rc = ctx->dim == 2 ? launch_update_local<MAT_QUAD, 4, 0, false>(ctx, 0, 0, 0, 0, false)
                           : launch_update_local<MAT_QUAD, 9, 0, false>(ctx, 0, 0, 0, 0, false);
    } else {
        if (max_sweeps > 64)
            return mm_fail(ctx, MM_ERR_CONFIG, "fused local chunk limited to 64 sweeps");
        if (material == MM_MAT_MR_DESCENT || (material == MM_MAT_MR && ctx->dim == 3))
            rc = ctx->dim == 2 ? launch_update_local<MAT_MR, 4, 0, true>(ctx, rho_next, tol, phi_scale, (int)max_sweeps, want_points)
                               : launch_update_local<MAT_MR, 9, 0, true>(ctx, rho_next, tol, phi_scale, (int)max_sweeps, want_points);
        else if (material == MM_MAT_MR)
            rc = launch_update_local<MAT_MR, 4, 1, true>(ctx, rho_next, tol, phi_scale, (int)max_sweeps, want_points);
        else if (material == MM_MAT_QUADRATIC)
            rc = ctx->dim == 2 ? launch_update_local<MAT_QUAD, 4, 0, true>(ctx, rho_next, tol, phi_scale, (int)max_sweeps, want_points)
                               : launch_update_local<MAT_QUAD, 9, 0, true>(ctx, rho_next, tol, phi_scale, (int)max_sweeps, want_points);
        else
            return mm_fail(ctx, MM_ERR_CONFIG, "material %d has no fused local chunk", material);
    }
    if (rc) return rc;
    ctx->lam_pending = false;
    if (kFusedStoresG) {  // the pass stored grad_u
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    }
    double r[MM_MAX_PARTIALS];
    const int K = 5 + 2 * D;
    // Speculative front: the next projection's A / column passes / E depend
    // only on the T field this pass writes (for rho_next), so they are queued
    // right behind it and run while the host waits for this pass's sums and
    // takes its decisions; mm_project_residuals uses them when nothing else
    // ran in between (generation count) and rho is rho_next, else recomputes.
    const bool spec = sweep && ctx->opt_speculate && !ctx->slab_mode && !ctx->points_only &&
                      ctx->have_sym && ctx->T_valid && ctx->T_rho == rho_next;
    ctx->front_valid = false;
    if (spec) {
        if (!ctx->ev_red) MM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_red, cudaEventDisableTiming));
        if (!ctx->red_mapped)
            MM_CUDA(ctx, cudaMemcpyAsync(ctx->host_out, ctx->red_out, sizeof(double) * K,
                                         cudaMemcpyDeviceToHost, ctx->stream));
        MM_CUDA(ctx, cudaEventRecord(ctx->ev_red, ctx->stream));
        double *u_new = nullptr;
        if ((rc = mm_run_project_front(ctx, rho_next, 2, &u_new))) return rc;
        ctx->front_valid = true;
        ctx->front_rho = rho_next;
        ctx->front_gen = ctx->gen;
        MM_CUDA(ctx, cudaEventSynchronize(ctx->ev_red));
        memcpy(r, ctx->host_out, sizeof(double) * K);
    } else if ((rc = mm_fetch_reduction(ctx, K, r))) {
        return rc;
    }
    for (int i = 0; i < 9; ++i) us->sum_lam[i] = i < D ? r[4 + D + i] : 0.0;
    if (sweep) {
        ls->sum_res2 = r[0];
        ls->n_conv = (int64_t)r[1];
        ls->sweeps = ctx->M ? (int64_t)r[2] : 0;
        for (int i = 0; i < 9; ++i) ls->sum_F[i] = i < D ? r[4 + i] : 0.0;
        ls->sum_nsw = r[K - 1];
        if (want_points) MM_CUDA(ctx, cudaMemsetAsync(ctx->ok, 0, ctx->M, ctx->stream));
    }
    return MM_OK;
}

// Pipelined step (mm_residuals_and_step): the pending ascent fused with the
// next first local chunk, with rho_next / tol read from ctx->dstep (k_decide,
// queued behind K1), then the speculative projection front; nothing waits.
// mm_run_update_pipe_finish takes the host's (identical) decision: swept ->
// the pass ran (its sums are read), else it returned at once, the ascent is
// still pending and the front is void.
int mm_run_update_pipe(mm_ctx *ctx, int material, double rho_placeholder, int64_t max_sweeps,
                       double phi_scale) {
    int rc;
    if (!ctx->lam_pending)
        return mm_fail(ctx, MM_ERR_CONFIG, "no multiplier update pending (call mm_project_residuals)");
    if (max_sweeps > 64) return mm_fail(ctx, MM_ERR_CONFIG, "fused local chunk limited to 64 sweeps");
    const DevStep *ds = ctx->dstep;
    const double r = rho_placeholder;
    if (material == MM_MAT_MR_DESCENT || (material == MM_MAT_MR && ctx->dim == 3))
        rc = ctx->dim == 2 ? launch_update_local<MAT_MR, 4, 0, true>(ctx, r, 0.0, phi_scale, (int)max_sweeps, false, ds)
                           : launch_update_local<MAT_MR, 9, 0, true>(ctx, r, 0.0, phi_scale, (int)max_sweeps, false, ds);
    else if (material == MM_MAT_MR)
        rc = launch_update_local<MAT_MR, 4, 1, true>(ctx, r, 0.0, phi_scale, (int)max_sweeps, false, ds);
    else if (material == MM_MAT_QUADRATIC)
        rc = ctx->dim == 2 ? launch_update_local<MAT_QUAD, 4, 0, true>(ctx, r, 0.0, phi_scale, (int)max_sweeps, false, ds)
                           : launch_update_local<MAT_QUAD, 9, 0, true>(ctx, r, 0.0, phi_scale, (int)max_sweeps, false, ds);
    else
        return mm_fail(ctx, MM_ERR_CONFIG, "material %d has no fused local chunk", material);
    if (rc) return rc;
    if (!ctx->ev_red) MM_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_red, cudaEventDisableTiming));
    MM_CUDA(ctx, cudaEventRecord(ctx->ev_red, ctx->stream));
    ctx->front_valid = false;
    if (ctx->opt_speculate && ctx->have_sym && ctx->T_valid && ctx->T_rho == rho_placeholder) {
        double *u_new = nullptr;
        if ((rc = mm_run_project_front(ctx, rho_placeholder, 2, &u_new))) return rc;
        ctx->front_valid = true;  // confirmed (or voided) by the finish
    }
    return MM_OK;
}

int mm_run_update_pipe_finish(mm_ctx *ctx, bool swept, double rho_next, mm_local_stats *ls,
                              mm_update_stats *us) {
    MM_CUDA(ctx, cudaEventSynchronize(ctx->ev_red));
    if (!swept) {
        ctx->T_valid = false;
        ctx->front_valid = false;
        return MM_OK;
    }
    const int D = ctx->D;
    ctx->lam_pending = false;
    if (kFusedStoresG) {
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    }
    if (ctx->T_valid) ctx->T_rho = rho_next;
    if (ctx->front_valid) {
        ctx->front_rho = rho_next;
        ctx->front_gen = ctx->gen;
    }
    const int K = 5 + 2 * D;
    double r[MM_MAX_PARTIALS];
    memcpy(r, ctx->host_out, sizeof(double) * K);
    for (int i = 0; i < 9; ++i) us->sum_lam[i] = i < D ? r[4 + D + i] : 0.0;
    ls->sum_res2 = r[0];
    ls->n_conv = (int64_t)r[1];
    ls->sweeps = ctx->M ? (int64_t)r[2] : 0;
    for (int i = 0; i < 9; ++i) ls->sum_F[i] = i < D ? r[4 + i] : 0.0;
    ls->sum_nsw = r[K - 1];
    mm_drain_timings(ctx);
    return MM_OK;
}

int mm_flush_pending(mm_ctx *ctx) {
    if (!ctx->lam_pending) return MM_OK;
    mm_update_stats us;
    return mm_run_update(ctx, 0, 0.0, 0.0, 0, 0.0, 0, nullptr, &us);
}

// ---------------------------------------------------------------------------
// test hook: the device log of the objective on caller-supplied arguments
// ---------------------------------------------------------------------------
namespace {
__global__ void k_selftest_log(const double *__restrict__ x, double *__restrict__ y, int64_t n) {
    __shared__ double ltab[3 * LOGTAB_N];
    load_logtab(ltab);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = log_pos(x[i], ltab);
}
}  // namespace

extern "C" int mm_selftest_log(mm_ctx *ctx, const double *x, double *y, int64_t n) {
    if (ctx) ctx->gen++;
    if (!ctx || !x || !y || n < 0) return MM_ERR_PARAM;
    MM_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = ensure_logtab(ctx);
    if (rc) return rc;
    double *d = nullptr;
    if ((rc = mm_alloc(ctx, (void **)&d, sizeof(double) * 2 * (n ? n : 1)))) return rc;
    MM_CUDA(ctx, cudaMemcpyAsync(d, x, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    const int blocks = (int)std::min<int64_t>((n + 255) / 256 + 1, 148 * 8);
    k_selftest_log<<<blocks, 256, 0, ctx->stream>>>(d, d + n, n);
    MM_LAUNCH_CHECK(ctx);
    MM_CUDA(ctx, cudaMemcpyAsync(y, d + n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    MM_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    mm_free(ctx, d);
    ctx->bytes -= (int64_t)(sizeof(double) * 2 * (n ? n : 1));
    return MM_OK;
}
