// Liquid-crystal-elastomer local step and frozen Frank force
// (ADMM step 1 for micromech/materials/lce.py).
//
//   k_lce2d   joint damped Newton on (F 2x2, theta), 5x5 system in registers
//             (lce.py:371-584)
//   k_lce3d   joint damped Newton on (F 3x3, phi, theta) with per-point chart,
//             11x11 system; the elimination matrix lives in shared memory in
//             a [entry][thread] layout (conflict-free, 968 B per thread)
//             (lce.py:676-995)
//   k_director / k_frank   director from the stored angles (lce.py:126-134)
//             and 2 kappa (D^T D) n as the exact radius-2 real-space stencil
//             sum_j (2n - n(x+2h e_j) - n(x-2h e_j)) / (4h^2), which equals the
//             reference's spectral form |g|^2 n_hat (lce.py:213-221).
//
// Both Newton kernels follow the reference's operation order (Levenberg
// inflation x10 up to 4 tries, Armijo on the exact objective, 12-step det
// guard when the decrement is unmeasurable, scaled-gradient fallback, nested
// multiplier p += gamma (J - 1)); Gaussian elimination keeps the reference's
// partial-pivot order (lce.py:315-349).
#include <math.h>

#include <algorithm>

#include "mm_internal.cuh"

namespace {

constexpr double BT_DECREASE = 1e-4;
constexpr double MEAS_EPS = 64.0 * 2.220446049250313e-16;
constexpr int NEWTON_BT = 60;
constexpr double DET_FLOOR = 1e-12;

struct LcePar {
    double mu, r1d, rr, al, gam, rho, visF, visn, tol, det_tol;
    double mur, mual, q, scale;
    int64_t max_sweeps;
};

inline LcePar make_par(const mm_lce_params &p, double rho, double tol, int64_t max_sweeps) {
    LcePar P;
    P.mu = p.mu;
    P.r1d = p.r1d;
    P.rr = p.rr;
    P.al = p.alpha;
    P.gam = p.gamma_inc;
    P.rho = rho;
    P.visF = p.vis_F;
    P.visn = p.vis_n;
    P.tol = tol;
    P.det_tol = p.det_tol;
    P.mur = p.mu * p.r1d;
    P.mual = p.mu * p.alpha;
    P.q = P.mual - P.mur * p.rr;
    P.scale = p.phiF_scale + p.phin_scale;
    P.max_sweeps = max_sweeps;
    return P;
}

// ---------------------------------------------------------------------------
// Gaussian elimination with partial pivoting (lce.py:315-349), fully unrolled
// so the 5x5 system stays in registers; row swaps are predicated moves.
// ---------------------------------------------------------------------------
template <int m>
__device__ __forceinline__ bool gauss_reg(double (&A)[m][m], double (&b)[m], double (&x)[m]) {
#pragma unroll
    for (int col = 0; col < m; ++col) {
        int piv = col;
        double best = fabs(A[col][col]);
#pragma unroll
        for (int r = col + 1; r < m; ++r) {
            const double v = fabs(A[r][col]);
            if (v > best) {
                best = v;
                piv = r;
            }
        }
        if (best < 1e-250) return false;
#pragma unroll
        for (int r = col + 1; r < m; ++r) {
            if (piv == r) {
#pragma unroll
                for (int c = 0; c < m; ++c) {
                    const double t = A[col][c];
                    A[col][c] = A[r][c];
                    A[r][c] = t;
                }
                const double t = b[col];
                b[col] = b[r];
                b[r] = t;
            }
        }
        const double inv = 1.0 / A[col][col];
#pragma unroll
        for (int r = col + 1; r < m; ++r) {
            const double f = A[r][col] * inv;
            if (f != 0.0) {
#pragma unroll
                for (int c = col; c < m; ++c) A[r][c] -= f * A[col][c];
                b[r] -= f * b[col];
            }
        }
    }
#pragma unroll
    for (int r = m - 1; r >= 0; --r) {
        double s = b[r];
#pragma unroll
        for (int c = r + 1; c < m; ++c) s -= A[r][c] * x[c];
        x[r] = s / A[r][r];
    }
    return true;
}

// 2D augmented point objective (lce.py:352-368) plus director terms
__device__ __forceinline__ double phiJ2(const double (&f)[4], double p1, double p2, double m01,
                                       double m02, const LcePar &P, double pp,
                                       const double (&L)[4], const double (&Gv)[4],
                                       const double (&K)[4], double ff1, double ff2, double nk1,
                                       double nk2) {
    const double u1 = f[0] * p1 + f[2] * p2;
    const double u2 = f[1] * p1 + f[3] * p2;
    const double cc = u1 * m01 + u2 * m02;
    const double dJ = f[0] * f[3] - f[1] * f[2] - 1.0;
    const double e0 = Gv[0] - f[0], e1 = Gv[1] - f[1], e2 = Gv[2] - f[2], e3 = Gv[3] - f[3];
    const double v0 = f[0] - K[0], v1 = f[1] - K[1], v2 = f[2] - K[2], v3 = f[3] - K[3];
    const double phiF =
        0.5 * P.mur * (f[0] * f[0] + f[1] * f[1] + f[2] * f[2] + f[3] * f[3]) -
        0.5 * P.mur * P.rr * (u1 * u1 + u2 * u2) + 0.5 * P.mual * (u1 * u1 + u2 * u2 - cc * cc) +
        pp * dJ + 0.5 * P.gam * dJ * dJ - (L[0] * f[0] + L[1] * f[1] + L[2] * f[2] + L[3] * f[3]) +
        0.5 * P.rho * (e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3) +
        0.5 * P.visF * (v0 * v0 + v1 * v1 + v2 * v2 + v3 * v3);
    const double a = p1 - nk1, b = p2 - nk2;
    return phiF + ff1 * p1 + ff2 * p2 + 0.5 * P.visn * (a * a + b * b);
}

// slots: 0 sum res^2, 1 n_ok, 2 max nsw, 3..6 sum F
__global__ void __launch_bounds__(128)
k_lce2d(double *__restrict__ Fg, double *__restrict__ ang, double *__restrict__ pinc,
        const double *__restrict__ Gg, const double *__restrict__ Lg,
        const double *__restrict__ n0, const double *__restrict__ ffg,
        const double *__restrict__ Fk, const double *__restrict__ angk, int64_t M, LcePar P,
        double *__restrict__ res_out, int32_t *__restrict__ nsw_out, uint8_t *__restrict__ ok_out,
        double *partials, double *red_out, unsigned int *count) {
    __shared__ double smem[32 * 8];
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const double q = P.q, mur = P.mur, mual = P.mual, rho = P.rho, gam = P.gam;
    const double visF = P.visF, visn = P.visn;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double f[4], L[4], Gv[4], K[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[i] = Fg[i * M + p];
            L[i] = Lg[i * M + p];
            Gv[i] = Gg[i * M + p];
            K[i] = Fk ? Fk[i * M + p] : 0.0;
        }
        double th = ang[p], pp = pinc[p];
        const double m01 = n0[p], m02 = n0[M + p];
        const double ff1 = ffg[p], ff2 = ffg[M + p];
        double nk1 = 0.0, nk2 = 0.0;
        if (angk) sincos(angk[p], &nk2, &nk1);
        const double fsq0 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2] + f[3] * f[3];
        const double tF0 = 1.0 / (rho + 2.0 * mur + 2.0 * mual + 2.0 * gam + visF);
        const double tN0 = 1.0 / (P.mu * (2.0 * P.r1d + 2.0 * P.al) * fmax(fsq0, 1.0) + visn + 1e-30);
        const double base = mur + rho + visF;
        int64_t nsw = 0;
        double res = 0.0;
        bool converged = false;
        for (int64_t it = 0; it < P.max_sweeps + 1; ++it) {
            double n1, n2;
            sincos(th, &n2, &n1);
            const double u1 = f[0] * n1 + f[2] * n2, u2 = f[1] * n1 + f[3] * n2;
            const double cc = u1 * m01 + u2 * m02;
            const double v1 = f[0] * m01 + f[1] * m02, v2 = f[2] * m01 + f[3] * m02;
            const double h1 = f[0] * u1 + f[1] * u2, h2 = f[2] * u1 + f[3] * u2;
            const double J = f[0] * f[3] - f[1] * f[2];
            const double dJ = J - 1.0;
            const double pr = pp + gam * dJ;
            double rF[4];
            rF[0] = mur * f[0] + q * n1 * u1 - mual * cc * n1 * m01 + pr * f[3] - L[0] -
                    rho * (Gv[0] - f[0]) + visF * (f[0] - K[0]);
            rF[1] = mur * f[1] + q * n1 * u2 - mual * cc * n1 * m02 - pr * f[2] - L[1] -
                    rho * (Gv[1] - f[1]) + visF * (f[1] - K[1]);
            rF[2] = mur * f[2] + q * n2 * u1 - mual * cc * n2 * m01 - pr * f[1] - L[2] -
                    rho * (Gv[2] - f[2]) + visF * (f[2] - K[2]);
            rF[3] = mur * f[3] + q * n2 * u2 - mual * cc * n2 * m02 + pr * f[0] - L[3] -
                    rho * (Gv[3] - f[3]) + visF * (f[3] - K[3]);
            const double gF2 = rF[0] * rF[0] + rF[1] * rF[1] + rF[2] * rF[2] + rF[3] * rF[3];
            const double gn1 = q * h1 - mual * cc * v1 + ff1 + visn * (n1 - nk1);
            const double gn2 = q * h2 - mual * cc * v2 + ff2 + visn * (n2 - nk2);
            const double gth = -gn1 * n2 + gn2 * n1;
            res = sqrt(gF2 + gth * gth);
            if (res < P.tol && fabs(dJ) <= P.det_tol) {
                converged = true;
                break;
            }
            if (nsw >= P.max_sweeps) break;
            nsw += 1;
            // nested multiplier ascent on det F = 1 (lce.py:444-447)
            if (fabs(dJ) > P.det_tol && res <= fmax(P.tol, 0.25 * gam * fabs(dJ))) {
                pp += gam * dJ;
                continue;
            }
            const double phi0 = phiJ2(f, n1, n2, m01, m02, P, pp, L, Gv, K, ff1, ff2, nk1, nk2);
            // joint Hessian on (F, theta) (lce.py:456-486)
            double H[5][5];
#pragma unroll
            for (int a = 0; a < 5; ++a)
#pragma unroll
                for (int b = 0; b < 5; ++b) H[a][b] = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a) H[a][a] = base;
            const double n11 = q * n1 * n1, n12 = q * n1 * n2, n22 = q * n2 * n2;
            H[0][0] += n11; H[0][2] += n12; H[2][0] += n12; H[2][2] += n22;
            H[1][1] += n11; H[1][3] += n12; H[3][1] += n12; H[3][3] += n22;
            const double wv[4] = {n1 * m01, n1 * m02, n2 * m01, n2 * m02};
            const double cv[4] = {f[3], -f[2], -f[1], f[0]};
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) H[a][b] += gam * cv[a] * cv[b] - mual * wv[a] * wv[b];
            H[0][3] += pr; H[3][0] += pr;
            H[1][2] -= pr; H[2][1] -= pr;
            const double up1 = -f[0] * n2 + f[2] * n1, up2 = -f[1] * n2 + f[3] * n1;
            const double ccp = up1 * m01 + up2 * m02;
            H[0][4] = q * (-n2 * u1 + n1 * up1) - mual * (ccp * n1 - cc * n2) * m01;
            H[1][4] = q * (-n2 * u2 + n1 * up2) - mual * (ccp * n1 - cc * n2) * m02;
            H[2][4] = q * (n1 * u1 + n2 * up1) - mual * (ccp * n2 + cc * n1) * m01;
            H[3][4] = q * (n1 * u2 + n2 * up2) - mual * (ccp * n2 + cc * n1) * m02;
#pragma unroll
            for (int a = 0; a < 4; ++a) H[4][a] = H[a][4];
            H[4][4] = q * (up1 * up1 + up2 * up2) - mual * ccp * ccp + visn - (gn1 * n1 + gn2 * n2);
            const double rhs[5] = {-rF[0], -rF[1], -rF[2], -rF[3], -gth};
            // Newton direction, Levenberg inflation if indefinite (lce.py:489-505)
            double lam = 0.0, gd = 0.0;
            double dv[5];
            bool found = false;
            for (int lm = 0; lm < 4; ++lm) {
                double A[5][5], bw[5];
#pragma unroll
                for (int a = 0; a < 5; ++a) {
#pragma unroll
                    for (int b = 0; b < 5; ++b) A[a][b] = H[a][b];
                    A[a][a] += lam;
                    bw[a] = rhs[a];
                }
                if (gauss_reg<5>(A, bw, dv)) {
                    gd = -(rhs[0] * dv[0] + rhs[1] * dv[1] + rhs[2] * dv[2] + rhs[3] * dv[3] +
                           rhs[4] * dv[4]);
                    if (gd < 0.0) {
                        found = true;
                        break;
                    }
                }
                lam = (lam == 0.0) ? base : lam * 10.0;
            }
            bool did = false;
            for (int pass = 0; pass < 2 && !did; ++pass) {
                double decr;
                if (pass == 0) {
                    if (!found) continue;
                    decr = -0.5 * gd;
                } else {  // scaled-gradient fallback (lce.py:541-576)
                    dv[0] = -tF0 * rF[0]; dv[1] = -tF0 * rF[1];
                    dv[2] = -tF0 * rF[2]; dv[3] = -tF0 * rF[3];
                    dv[4] = -tN0 * gth;
                    gd = -(tF0 * gF2 + tN0 * gth * gth);
                    decr = -BT_DECREASE * gd;
                }
                double t = 1.0;
                if (decr <= MEAS_EPS * (fabs(phi0) + P.scale)) {
                    for (int bt = 0; bt < 12; ++bt) {
                        const double a2 = f[0] + t * dv[0], b2 = f[1] + t * dv[1];
                        const double c2 = f[2] + t * dv[2], d2 = f[3] + t * dv[3];
                        if (a2 * d2 - b2 * c2 > DET_FLOOR) {
                            f[0] = a2; f[1] = b2; f[2] = c2; f[3] = d2;
                            th = th + t * dv[4];
                            did = true;
                            break;
                        }
                        t *= 0.5;
                    }
                } else {
                    for (int bt = 0; bt < NEWTON_BT; ++bt) {
                        const double ft[4] = {f[0] + t * dv[0], f[1] + t * dv[1], f[2] + t * dv[2],
                                              f[3] + t * dv[3]};
                        if (ft[0] * ft[3] - ft[1] * ft[2] > DET_FLOOR) {
                            const double th2 = th + t * dv[4];
                            double p1, p2;
                            sincos(th2, &p2, &p1);
                            const double phi2 =
                                phiJ2(ft, p1, p2, m01, m02, P, pp, L, Gv, K, ff1, ff2, nk1, nk2);
                            if (phi2 <= phi0 + BT_DECREASE * t * gd) {
#pragma unroll
                                for (int i = 0; i < 4; ++i) f[i] = ft[i];
                                th = th2;
                                did = true;
                                break;
                            }
                        }
                        t *= 0.5;
                    }
                }
                if (pass == 1) did = true;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) Fg[i * M + p] = f[i];
        ang[p] = th;
        pinc[p] = pp;
        if (res_out) {
            res_out[p] = res;
            nsw_out[p] = (int32_t)nsw;
            ok_out[p] = converged ? 1 : 0;
        }
        acc[0] += res * res;
        acc[1] += converged ? 1.0 : 0.0;
        acc[2] = fmax(acc[2], (double)nsw);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[3 + i] += f[i];
        acc[7] += (double)nsw;
    }
    const int ops[8] = {RED_SUM, RED_SUM, RED_MAX, RED_SUM, RED_SUM, RED_SUM, RED_SUM, RED_SUM};
    block_reduce<8>(acc, ops, smem);
    grid_finalize<8>(acc, ops, partials, red_out, count, smem);
}

// ---------------------------------------------------------------------------
// 3D
// ---------------------------------------------------------------------------
constexpr int LCE3_THREADS = 64;

__device__ __forceinline__ double det3(const double (&A)[9]) {
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

__device__ __forceinline__ void n_from_chart(double ph, double th, const double (&E)[9],
                                             double (&out)[3]) {
    double sp, cp, st, ct;
    sincos(ph, &sp, &cp);
    sincos(th, &st, &ct);
    const double a = sp * ct, b = sp * st, c = cp;
#pragma unroll
    for (int i = 0; i < 3; ++i) out[i] = a * E[3 * i + 0] + b * E[3 * i + 1] + c * E[3 * i + 2];
}

struct PointData3 {
    const double *G, *L, *K;  // strided pointers (stride M) into SoA arrays at point p
    int64_t M;
    __device__ __forceinline__ double g(int i) const { return G[i * M]; }
    __device__ __forceinline__ double l(int i) const { return L[i * M]; }
    __device__ __forceinline__ double k(int i) const { return K ? K[i * M] : 0.0; }
};

// lce.py:620-650 (_phiF_3 + _phiJ_3)
__device__ __forceinline__ double phiJ3(const double (&Fl)[9], const double (&n)[3],
                                       const double (&n0l)[3], const LcePar &P, double pp,
                                       const PointData3 &D, const double (&ffl)[3],
                                       const double (&nkl)[3]) {
    double fsq = 0.0, coup = 0.0;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
        const double fij = Fl[i];
        fsq += fij * fij;
        const double e = D.g(i) - fij, v = fij - D.k(i);
        coup += (-D.l(i) * fij + 0.5 * P.rho * (e * e) + 0.5 * P.visF * (v * v));
    }
    double usq = 0.0, cc = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double ui = Fl[0 * 3 + i] * n[0] + Fl[1 * 3 + i] * n[1] + Fl[2 * 3 + i] * n[2];
        usq += ui * ui;
        cc += ui * n0l[i];
    }
    const double dJ = det3(Fl) - 1.0;
    const double phiF = 0.5 * P.mur * (fsq - P.rr * usq) + 0.5 * P.mual * (usq - cc * cc) +
                        pp * dJ + 0.5 * P.gam * dJ * dJ + coup;
    double extra = 0.0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double e = n[i] - nkl[i];
        extra += ffl[i] * n[i] + 0.5 * P.visn * (e * e);
    }
    return phiF + extra;
}

// Gaussian elimination on the 11x11 system held in shared memory: entry
// (r, c) at S[(r*11 + c) * T], right-hand side r at S[(121 + r) * T]
// (T = threads per block; each thread owns one column of the buffer).
template <int T>
__device__ __forceinline__ bool gauss_smem11(double *S, double (&x)[11]) {
    // fully unrolled: every (r, c) offset is an immediate; the pivot row is
    // held in registers while the rows below it are updated (same
    // operations in the same order as the loop form, lce.py:315-349)
#define AS(r, c) S[((r) * 11 + (c)) * T]
#define BS(r) S[(121 + (r)) * T]
#pragma unroll
    for (int col = 0; col < 11; ++col) {
        int piv = col;
        double best = fabs(AS(col, col));
#pragma unroll
        for (int r = col + 1; r < 11; ++r) {
            const double v = fabs(AS(r, col));
            if (v > best) {
                best = v;
                piv = r;
            }
        }
        if (best < 1e-250) return false;
        double prow[11];
        double bcol;
        if (piv != col) {
            // columns < col of both rows are never read again: not swapped
#pragma unroll
            for (int c = col; c < 11; ++c) {
                prow[c] = S[(piv * 11 + c) * T];
                S[(piv * 11 + c) * T] = AS(col, c);
            }
#pragma unroll
            for (int c = col; c < 11; ++c) AS(col, c) = prow[c];
            bcol = S[(121 + piv) * T];
            S[(121 + piv) * T] = BS(col);
            BS(col) = bcol;
        } else {
#pragma unroll
            for (int c = col; c < 11; ++c) prow[c] = AS(col, c);
            bcol = BS(col);
        }
        const double inv = 1.0 / prow[col];
#pragma unroll
        for (int r = col + 1; r < 11; ++r) {
            const double f = AS(r, col) * inv;
            if (f != 0.0) {
#pragma unroll
                for (int c = col; c < 11; ++c) AS(r, c) -= f * prow[c];
                BS(r) -= f * bcol;
            }
        }
    }
#pragma unroll
    for (int r = 10; r >= 0; --r) {
        double s = BS(r);
#pragma unroll
        for (int c = r + 1; c < 11; ++c) s -= AS(r, c) * x[c];
        x[r] = s / AS(r, r);
    }
#undef AS
#undef BS
    return true;
}

// Work counters of the 3D Newton kernel (diagnostics build, -DMM_LCE_STATS=1):
// 0 multiplier-only sweeps, 1 Newton steps, 2 eliminations (Levenberg tries),
// 3 Armijo objective evaluations, 4 det-guard trials, 5 gradient-fallback
// passes, 6 fallback objective evaluations, 7 warp Newton iterations x 32
#ifndef MM_LCE_STATS
#define MM_LCE_STATS 0
#endif
__device__ unsigned long long g_lce_cnt[8];
#if MM_LCE_STATS
#define LCE_CNT(i) (++cnt[i])
#else
#define LCE_CNT(i) ((void)0)
#endif

// Newton-compacted schedule (LceSplit.mode != 0).  A policy chunk runs as
// rounds: round 0 (mode 1) walks every point through its cheap multiplier-
// only sweeps and stops it at its first Newton step, which it defers
// (state stored, sweep count one back, index appended to list_out); round
// k >= 1 (mode 2) takes the deferred points, re-evaluates the deferring
// sweep (same state, same bits, same decision), performs that Newton step,
// continues with cheap sweeps and defers again at the next Newton step.
// Every lane of a warp therefore executes exactly one Newton step per
// round, instead of the warp running the Newton code whenever any of its
// points needs it (8 of 32 lanes active per instruction on polydomain
// inputs).  The per-point sequence of sweeps is the plain loop's; the batch
// sums come from k_lce3_reduce over the per-point results.
struct LceSplit {
    int mode;                      // 0: plain loop; 1: round 0; 2: round >= 1
    const int *list_in;            // mode 2: points of this round
    const int *count_in;
    int *list_out, *count_out;     // deferred points (appended)
    int *count_clear;              // the counter the next round appends to
    int32_t *nsw_io;               // sweeps of this call so far (split: always)
    int budget;                    // Newton steps a round-k >= 1 point takes (1)
    double *fsq0_io;               // |F|^2 at the start of the call (tN0)
};

// resident 64-thread blocks per SM asked of the lean round-0 kernel (no
// elimination workspace, so only registers bound its occupancy)
#ifndef MM_LCE_LEAN_MINB
#define MM_LCE_LEAN_MINB 8
#endif

// slots: 0 sum res^2, 1 n_ok, 2 max nsw, 3..11 sum F
template <int MODE>  // == LceSplit.mode, a compile-time constant
__global__ void __launch_bounds__(LCE3_THREADS, (MODE == 1 || MODE == 4) ? MM_LCE_LEAN_MINB : 1)
k_lce3d(double *__restrict__ Fg, double *__restrict__ ang, double *__restrict__ chart,
        double *__restrict__ pinc, const double *__restrict__ Gg, const double *__restrict__ Lg,
        const double *__restrict__ n0, const double *__restrict__ ffg,
        const double *__restrict__ Fk, const double *__restrict__ angk,
        const double *__restrict__ chartk, int64_t M, LcePar P, double *__restrict__ res_out,
        int32_t *__restrict__ nsw_out, uint8_t *__restrict__ ok_out, double *partials,
        double *red_out, unsigned int *count, LceSplit SP) {
    extern __shared__ double smA[];  // 132 * LCE3_THREADS
    __shared__ double smem[32 * 13];
    double *S = smA + threadIdx.x;
    constexpr int T = LCE3_THREADS;
    double acc[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) acc[k] = 0.0;
    const double q = P.q, mur = P.mur, mual = P.mual, rho = P.rho, gam = P.gam;
    const double visF = P.visF, visn = P.visn;
    const double PI = 3.141592653589793;
#if MM_LCE_STATS
    unsigned long long cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    // modes 2, 3, 4 walk a list; 3 (Newton step only) appends nothing
    constexpr bool LIST = MODE >= 2;
    if (MODE && MODE != 3 && blockIdx.x == 0 && threadIdx.x == 0) *SP.count_clear = 0;
    const int64_t npoints = LIST ? (int64_t)*SP.count_in : M;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < npoints;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = LIST ? (int64_t)SP.list_in[idx] : idx;
        double Fl[9], E[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            Fl[i] = Fg[i * M + p];
            E[i] = chart[i * M + p];
        }
        PointData3 D{Gg + p, Lg + p, Fk ? Fk + p : nullptr, M};
        double n0l[3], ffl[3], nkl[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            n0l[i] = n0[i * M + p];
            ffl[i] = ffg[i * M + p];
        }
        if (angk) {
            double Ek[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) Ek[i] = chartk[i * M + p];
            n_from_chart(angk[p], angk[M + p], Ek, nkl);
        }
        double ph = ang[p], th = ang[M + p], pp = pinc[p];
        double fsq0 = 0.0;
        if (LIST) {
            fsq0 = SP.fsq0_io[p];
        } else {
#pragma unroll
            for (int i = 0; i < 9; ++i) fsq0 += Fl[i] * Fl[i];
        }
        const double tF0 = 1.0 / (rho + 2.0 * mur + 2.0 * mual + 3.0 * gam + visF);
        const double tN0 = 1.0 / (P.mu * (2.0 * P.r1d + 2.0 * P.al) * fmax(fsq0, 1.0) + visn + 1e-30);
        const double base = mur + rho + visF;
        int64_t nsw = LIST ? (int64_t)SP.nsw_io[p] : 0;
        double res = 0.0;
        bool converged = false;
        bool deferred = false;
        // a runtime value for round k >= 1 (SP.budget = 1): a compile-time 1
        // lets the compiler peel the first Newton step into a second copy of
        // the step (1.8 KB of spills instead of 0.65)
        int newton_budget = (MODE == 1 || MODE == 4) ? 0
                            : (MODE == 2 || MODE == 3) ? SP.budget : 0x7fffffff;
        // Sweeps that only ascend the nested det multiplier (the polydomain
        // stall regime) are cheap; Newton sweeps are ~20x dearer.  Each lane
        // first runs through its cheap sweeps (inner loop) and the warp then
        // takes the Newton step for every lane that reached one, so Newton
        // steps of different lanes execute together instead of one
        // divergent Newton per sweep in which only the few lanes that need
        // it are active.  Every lane performs exactly the same sequence of
        // sweeps as the plain loop.
        int64_t it = nsw;  // the loop keeps it == nsw at the top of every sweep
        while (it < P.max_sweeps + 1) {
            double n[3], sp, cp, st, ct, u[3], cc, J, dJ, pr, cof[9], gFl[9], gF2, gn[3];
            double m1[3], mth[3], g1, g2, gnn, sp2;
            bool newton = false;
            // A multiplier-only sweep changes p_inc alone: F, the angles and
            // the chart stay, so the director, its angle frame, J, cof F and
            // dW/dn of the next sweep are the values already in registers
            // (same inputs, same bits).  Only pr and the F-gradient, which
            // depend on p_inc, are re-evaluated (82 % of polydomain sweeps).
            bool fresh = true;
            for (; it < P.max_sweeps + 1; ++it) {
              if (fresh) {
                // keep the chart's azimuth well conditioned (lce.py:709-730)
                if (sin(ph) < 0.1) {
                    n_from_chart(ph, th, E, n);
                    int k = 0;
                    if (fabs(n[1]) < fabs(n[k])) k = 1;
                    if (fabs(n[2]) < fabs(n[k])) k = 2;
                    const double dot = (k == 0) ? n[0] : (k == 1 ? n[1] : n[2]);
                    double e3[3], e3n = 0.0;
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const double v = (i == k ? 1.0 : 0.0) - dot * n[i];
                        e3[i] = v;
                        e3n += v * v;
                    }
                    e3n = sqrt(e3n);
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        E[3 * i + 0] = n[i];
                        E[3 * i + 2] = e3[i] / e3n;
                    }
                    E[0 * 3 + 1] = E[1 * 3 + 2] * E[2 * 3 + 0] - E[2 * 3 + 2] * E[1 * 3 + 0];
                    E[1 * 3 + 1] = E[2 * 3 + 2] * E[0 * 3 + 0] - E[0 * 3 + 2] * E[2 * 3 + 0];
                    E[2 * 3 + 1] = E[0 * 3 + 2] * E[1 * 3 + 0] - E[1 * 3 + 2] * E[0 * 3 + 0];
                    ph = 0.5 * PI;
                    th = 0.0;
                }
                n_from_chart(ph, th, E, n);
                sincos(ph, &sp, &cp);
                sincos(th, &st, &ct);
#pragma unroll
                for (int j = 0; j < 3; ++j) u[j] = Fl[0 * 3 + j] * n[0] + Fl[1 * 3 + j] * n[1] + Fl[2 * 3 + j] * n[2];
                cc = u[0] * n0l[0] + u[1] * n0l[1] + u[2] * n0l[2];
                J = det3(Fl);
                dJ = J - 1.0;
                cof[0] = Fl[4] * Fl[8] - Fl[5] * Fl[7];
                cof[1] = Fl[5] * Fl[6] - Fl[3] * Fl[8];
                cof[2] = Fl[3] * Fl[7] - Fl[4] * Fl[6];
                cof[3] = Fl[2] * Fl[7] - Fl[1] * Fl[8];
                cof[4] = Fl[0] * Fl[8] - Fl[2] * Fl[6];
                cof[5] = Fl[1] * Fl[6] - Fl[0] * Fl[7];
                cof[6] = Fl[1] * Fl[5] - Fl[2] * Fl[4];
                cof[7] = Fl[2] * Fl[3] - Fl[0] * Fl[5];
                cof[8] = Fl[0] * Fl[4] - Fl[1] * Fl[3];
                // dW/dn (lce.py:653-663)
                {
                    const double v0 = Fl[0] * n[0] + Fl[3] * n[1] + Fl[6] * n[2];
                    const double v1 = Fl[1] * n[0] + Fl[4] * n[1] + Fl[7] * n[2];
                    const double v2 = Fl[2] * n[0] + Fl[5] * n[1] + Fl[8] * n[2];
                    const double c2 = v0 * n0l[0] + v1 * n0l[1] + v2 * n0l[2];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const double h = Fl[3 * i + 0] * v0 + Fl[3 * i + 1] * v1 + Fl[3 * i + 2] * v2;
                        const double v = Fl[3 * i + 0] * n0l[0] + Fl[3 * i + 1] * n0l[1] + Fl[3 * i + 2] * n0l[2];
                        gn[i] = q * h - mual * c2 * v + ffl[i] + visn * (n[i] - nkl[i]);
                    }
                }
                g1 = 0.0;
                g2 = 0.0;
                gnn = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    m1[i] = cp * ct * E[3 * i + 0] + cp * st * E[3 * i + 1] - sp * E[3 * i + 2];
                    mth[i] = sp * (-st * E[3 * i + 0] + ct * E[3 * i + 1]);
                    g1 += gn[i] * m1[i];
                    g2 += gn[i] * mth[i];
                    gnn += gn[i] * n[i];
                }
                sp2 = fmax(sp * sp, 1e-4);
              }
                pr = pp + gam * dJ;
                gF2 = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const int a = 3 * i + j;
                        const double gg = (mur * Fl[a] + q * n[i] * u[j] - mual * cc * n[i] * n0l[j] +
                                           pr * cof[a] - D.l(a) - rho * (D.g(a) - Fl[a]) +
                                           visF * (Fl[a] - D.k(a)));
                        gFl[a] = gg;
                        gF2 += gg * gg;
                    }
                res = sqrt(gF2 + g1 * g1 + g2 * g2 / sp2);
                if (res < P.tol && fabs(dJ) <= P.det_tol) {
                    converged = true;
                    break;
                }
                if (nsw >= P.max_sweeps) break;
                nsw += 1;
                if (fabs(dJ) > P.det_tol && res <= fmax(P.tol, 0.25 * gam * fabs(dJ))) {
                    pp += gam * dJ;
                    LCE_CNT(0);
                    fresh = false;
                    continue;
                }
                newton = true;
                break;
            }
#if MM_LCE_STATS
            if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) cnt[7] += 32;
#endif
            if (!newton) break;
            if (newton_budget == 0) {
                // defer this Newton step to the next round (split schedule): the
                // sweep is re-evaluated there, so its count is taken back
                deferred = true;
                nsw -= 1;
                break;
            }
            --newton_budget;
            ++it;
            LCE_CNT(1);
            const double phi0 = phiJ3(Fl, n, n0l, P, pp, D, ffl, nkl);
            // angle-block and cross-term ingredients (lce.py:807-882)
            double ua[3], ub[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                ua[j] = Fl[0 * 3 + j] * m1[0] + Fl[1 * 3 + j] * m1[1] + Fl[2 * 3 + j] * m1[2];
                ub[j] = Fl[0 * 3 + j] * mth[0] + Fl[1 * 3 + j] * mth[1] + Fl[2 * 3 + j] * mth[2];
            }
            const double cca = ua[0] * n0l[0] + ua[1] * n0l[1] + ua[2] * n0l[2];
            const double ccb = ub[0] * n0l[0] + ub[1] * n0l[1] + ub[2] * n0l[2];
            double gchd = 0.0, gt2 = 0.0;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                gchd += gn[i] * cp * (-st * E[3 * i + 0] + ct * E[3 * i + 1]);
                gt2 += gn[i] * (-sp) * (ct * E[3 * i + 0] + st * E[3 * i + 1]);
            }
            double Fn0[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                Fn0[i] = Fl[3 * i + 0] * n0l[0] + Fl[3 * i + 1] * n0l[1] + Fl[3 * i + 2] * n0l[2];
            double h11 = -gnn, h12 = gchd, h22 = gt2;
            {
                // _Qdot (lce.py:666-673) applied to m1, then mth
                double qv[3];
#pragma unroll
                for (int pass = 0; pass < 2; ++pass) {
                    const double *v = pass == 0 ? m1 : mth;
                    const double w0 = Fl[0] * v[0] + Fl[3] * v[1] + Fl[6] * v[2];
                    const double w1 = Fl[1] * v[0] + Fl[4] * v[1] + Fl[7] * v[2];
                    const double w2 = Fl[2] * v[0] + Fl[5] * v[1] + Fl[8] * v[2];
                    const double vf = v[0] * Fn0[0] + v[1] * Fn0[1] + v[2] * Fn0[2];
#pragma unroll
                    for (int i = 0; i < 3; ++i) {
                        const double h = Fl[3 * i + 0] * w0 + Fl[3 * i + 1] * w1 + Fl[3 * i + 2] * w2;
                        qv[i] = q * h - mual * vf * Fn0[i] + visn * v[i];
                    }
                    if (pass == 0) {
#pragma unroll
                        for (int i = 0; i < 3; ++i) {
                            h11 += m1[i] * qv[i];
                            h12 += mth[i] * qv[i];
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 3; ++i) h22 += mth[i] * qv[i];
                    }
                }
            }
            double rhs[11];
#pragma unroll
            for (int a = 0; a < 9; ++a) rhs[a] = -gFl[a];
            rhs[9] = -g1;
            rhs[10] = -g2;
            // Newton direction with Levenberg inflation; the Hessian is rebuilt
            // into the shared-memory elimination matrix for each try
            double lam = 0.0, gd = 0.0;
            double dv[11];
            bool found = false;
            for (int lm = 0; lm < 4; ++lm) {
#define AS(r, c) S[((r) * 11 + (c)) * T]
                // F-F block, each entry formed in registers and stored once, with
                // the terms added in the reference's order: base (diagonal),
                // q n_i n_k (j = l), gam cof cof - mual w w, pr d^2 J (Levi-Civita,
                // lce.py:832-845), lam (diagonal)
                {
                    double wv[9];
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 3; ++j) wv[3 * i + j] = n[i] * n0l[j];
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 3; ++j)
#pragma unroll
                            for (int k = 0; k < 3; ++k)
#pragma unroll
                                for (int l = 0; l < 3; ++l) {
                                    const int a = 3 * i + j, b = 3 * k + l;
                                    double v = (a == b) ? base : 0.0;
                                    if (j == l) v += q * n[i] * n[k];
                                    v += gam * cof[a] * cof[b] - mual * wv[a] * wv[b];
                                    if (i != k && j != l) {
                                        const int mm_ = 3 - i - k, nn = 3 - j - l;
                                        const double si = (k == (i + 1) % 3) ? 1.0 : -1.0;
                                        const double sj = (l == (j + 1) % 3) ? 1.0 : -1.0;
                                        v += pr * si * sj * Fl[3 * mm_ + nn];
                                    }
                                    if (a == b) v += lam;
                                    AS(a, b) = v;
                                }
                }
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const int a = 3 * i + j;
                        const double h9 = q * (m1[i] * u[j] + n[i] * ua[j]) -
                                          mual * (cca * n[i] + cc * m1[i]) * n0l[j];
                        const double h10 = q * (mth[i] * u[j] + n[i] * ub[j]) -
                                           mual * (ccb * n[i] + cc * mth[i]) * n0l[j];
                        AS(a, 9) = h9;
                        AS(9, a) = h9;
                        AS(a, 10) = h10;
                        AS(10, a) = h10;
                    }
                AS(9, 9) = h11;
                AS(9, 10) = h12;
                AS(10, 9) = h12;
                AS(10, 10) = h22;
                AS(9, 9) += lam;
                AS(10, 10) += lam;
#undef AS
#pragma unroll
                for (int a = 0; a < 11; ++a) S[(121 + a) * T] = rhs[a];
                LCE_CNT(2);
                if (gauss_smem11<T>(S, dv)) {
                    gd = 0.0;
#pragma unroll
                    for (int a = 0; a < 11; ++a) gd -= rhs[a] * dv[a];
                    if (gd < 0.0) {
                        found = true;
                        break;
                    }
                }
                lam = (lam == 0.0) ? base : lam * 10.0;
            }
            bool did = false;
            for (int pass = 0; pass < 2 && !did; ++pass) {
                double decr;
                if (pass == 0) {
                    if (!found) continue;
                    decr = -0.5 * gd;
                } else {
#pragma unroll
                    for (int a = 0; a < 9; ++a) dv[a] = -tF0 * gFl[a];
                    dv[9] = -tN0 * g1;
                    dv[10] = -tN0 * g2 / sp2;
                    gd = -(tF0 * gF2 + tN0 * (g1 * g1 + g2 * g2 / sp2));
                    decr = -BT_DECREASE * gd;
                }
                double t = 1.0;
                double Ft[9];
                if (pass == 1) LCE_CNT(5);
                if (decr <= MEAS_EPS * (fabs(phi0) + P.scale)) {
                    for (int bt = 0; bt < 12; ++bt) {
                        LCE_CNT(4);
#pragma unroll
                        for (int a = 0; a < 9; ++a) Ft[a] = Fl[a] + t * dv[a];
                        if (det3(Ft) > DET_FLOOR) {
#pragma unroll
                            for (int a = 0; a < 9; ++a) Fl[a] = Ft[a];
                            ph = ph + t * dv[9];
                            th = th + t * dv[10];
                            did = true;
                            break;
                        }
                        t *= 0.5;
                    }
                } else {
                    for (int bt = 0; bt < NEWTON_BT; ++bt) {
#pragma unroll
                        for (int a = 0; a < 9; ++a) Ft[a] = Fl[a] + t * dv[a];
                        if (det3(Ft) > DET_FLOOR) {
                            if (pass == 0) LCE_CNT(3); else LCE_CNT(6);
                            const double ph2 = ph + t * dv[9], th2 = th + t * dv[10];
                            double nt[3];
                            n_from_chart(ph2, th2, E, nt);
                            const double phi2 = phiJ3(Ft, nt, n0l, P, pp, D, ffl, nkl);
                            if (phi2 <= phi0 + BT_DECREASE * t * gd) {
#pragma unroll
                                for (int a = 0; a < 9; ++a) Fl[a] = Ft[a];
                                ph = ph2;
                                th = th2;
                                did = true;
                                break;
                            }
                        }
                        t *= 0.5;
                    }
                }
                if (pass == 1) did = true;
            }
            if constexpr (MODE == 3) break;  // Newton step only: the lean round continues
        }
#pragma unroll
        for (int i = 0; i < 9; ++i) {
            Fg[i * M + p] = Fl[i];
            chart[i * M + p] = E[i];
        }
        ang[p] = ph;
        ang[M + p] = th;
        pinc[p] = pp;
        if (MODE) {
            SP.nsw_io[p] = (int32_t)nsw;
            if (MODE == 1) SP.fsq0_io[p] = fsq0;
            if (MODE == 3) continue;  // mid-chunk state: the lean round (mode 4) takes it on
            if (deferred) {
                // warp-aggregated append of the deferred points
                const unsigned m = __activemask();
                const int lane = threadIdx.x & 31, lead = __ffs(m) - 1;
                int base = 0;
                if (lane == lead) base = atomicAdd(SP.count_out, __popc(m));
                base = __shfl_sync(m, base, lead);
                SP.list_out[base + __popc(m & ((1u << lane) - 1u))] = (int)p;
                continue;
            }
            res_out[p] = res;
            ok_out[p] = converged ? 1 : 0;
            continue;
        }
        if (res_out) {
            res_out[p] = res;
            nsw_out[p] = (int32_t)nsw;
            ok_out[p] = converged ? 1 : 0;
        }
        acc[0] += res * res;
        acc[1] += converged ? 1.0 : 0.0;
        acc[2] = fmax(acc[2], (double)nsw);
#pragma unroll
        for (int i = 0; i < 9; ++i) acc[3 + i] += Fl[i];
        acc[12] += (double)nsw;
    }
#if MM_LCE_STATS
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (cnt[i]) atomicAdd(&g_lce_cnt[i], cnt[i]);
#endif
    if (MODE) return;  // split schedule: k_lce3_reduce sums the per-point results
    int ops[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) ops[k] = RED_SUM;
    ops[2] = RED_MAX;
    block_reduce<13>(acc, ops, smem);
    grid_finalize<13>(acc, ops, partials, red_out, count, smem);
}

// batch sums of a split-schedule chunk from the per-point results (slots as
// k_lce3d's: sum res^2, n_ok, max nsw, sum F (9), sum nsw)
__global__ void __launch_bounds__(256)
k_lce3_reduce(const double *__restrict__ Fg, const double *__restrict__ res,
              const uint8_t *__restrict__ ok, const int32_t *__restrict__ nsw, int64_t M,
              double *partials, double *red_out, unsigned int *count) {
    __shared__ double smem[32 * 13];
    double acc[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) acc[k] = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        const double r = res[p];
        acc[0] += r * r;
        acc[1] += ok[p] ? 1.0 : 0.0;
        acc[2] = fmax(acc[2], (double)nsw[p]);
#pragma unroll
        for (int i = 0; i < 9; ++i) acc[3 + i] += Fg[i * M + p];
        acc[12] += (double)nsw[p];
    }
    int ops[13];
#pragma unroll
    for (int k = 0; k < 13; ++k) ops[k] = RED_SUM;
    ops[2] = RED_MAX;
    block_reduce<13>(acc, ops, smem);
    grid_finalize<13>(acc, ops, partials, red_out, count, smem);
}

// ---------------------------------------------------------------------------
// director and Frank stencil
// ---------------------------------------------------------------------------
template <int DIM>
__global__ void k_director(const double *__restrict__ ang, const double *__restrict__ chart,
                           double *__restrict__ nout, int64_t M, int64_t cs) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        if (DIM == 2) {
            double s, c;
            sincos(ang[p], &s, &c);
            nout[p] = c;
            nout[cs + p] = s;
        } else {
            double E[9], n[3];
#pragma unroll
            for (int i = 0; i < 9; ++i) E[i] = chart[i * M + p];
            n_from_chart(ang[p], ang[M + p], E, n);
#pragma unroll
            for (int i = 0; i < 3; ++i) nout[i * cs + p] = n[i];
        }
    }
}

// ff_i = 2 kappa / (4 h^2) sum_j (2 n_i - n_i(x + 2 e_j) - n_i(x - 2 e_j))
// cs: component stride of nf; wrap0 = 0 (slab): nf keeps two ghost planes
// on each face, so the axis-0 neighbours are plain offsets
template <int DIM>
__global__ void k_frank(const double *__restrict__ nf, double *__restrict__ ff, int n, int64_t M,
                        double coef, int64_t cs, int wrap0) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        unsigned q = (unsigned)p, c[DIM];
#pragma unroll
        for (int j = DIM - 1; j >= 0; --j) {
            const unsigned nq = q / (unsigned)n;
            c[j] = q - nq * (unsigned)n;
            q = nq;
        }
        int op[DIM], om[DIM];
        int stride = 1;
#pragma unroll
        for (int j = DIM - 1; j >= 0; --j) {
            const int cp2 = (int)((c[j] + 2) % (unsigned)n);
            const int cm2 = (int)((c[j] + (unsigned)n - 2) % (unsigned)n);
            op[j] = (cp2 - (int)c[j]) * stride;
            om[j] = (cm2 - (int)c[j]) * stride;
            if (j == 0 && !wrap0) {
                op[0] = 2 * stride;
                om[0] = -2 * stride;
            }
            stride *= n;
        }
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            const double *v = nf + (int64_t)i * cs + p;
            const double c0 = v[0];
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < DIM; ++j) s += (2.0 * c0 - v[op[j]]) - v[om[j]];
            ff[(int64_t)i * M + p] = coef * s;
        }
    }
}

// total mechanical stress (lce.py:166-174, 186-196) into P (SoA d*d):
//   mu r1d (F - rr n (F^T n)) + mu alpha (n (F^T n) - c n n0)
//   + (p_inc + gamma (J - 1)) cof F + (nu_F / dt) (F - F_k)
template <int DIM>
__global__ void __launch_bounds__(256)
k_lce_stress(const double *__restrict__ F, const double *__restrict__ nf,
             const double *__restrict__ n0, const double *__restrict__ pinc,
             const double *__restrict__ Fk, double visc, double mu, double r1d, double rr,
             double alpha, double gamma, double *__restrict__ P, int64_t M) {
    constexpr int D = DIM * DIM;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        double X[D], n[DIM], m0[DIM], Ftn[DIM], C[D];
#pragma unroll
        for (int i = 0; i < D; ++i) X[i] = F[i * M + p];
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            n[i] = nf[i * M + p];
            m0[i] = n0[i * M + p];
        }
        double c = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
            double t = 0.0;
#pragma unroll
            for (int i = 0; i < DIM; ++i) t += X[i * DIM + j] * n[i];
            Ftn[j] = t;
            c += t * m0[j];
        }
        double J;
        if constexpr (DIM == 2) {
            J = X[0] * X[3] - X[1] * X[2];
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
            J = X[0] * C[0] + X[1] * C[1] + X[2] * C[2];
        }
        const double react = pinc[p] + gamma * (J - 1.0);
        const double a = mu * r1d, b = mu * alpha;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
                const int q = i * DIM + j;
                const double nF = n[i] * Ftn[j];
                double v = a * (X[q] - rr * nF) + b * (nF - c * (n[i] * m0[j])) + react * C[q];
                if (Fk) v += visc * (X[q] - Fk[q * M + p]);
                P[q * M + p] = v;
            }
        }
    }
}

int lce_blocks(int64_t M, int threads) {
    return (int)std::min<int64_t>((M + threads - 1) / threads, 148 * 32);
}

}  // namespace

// diagnostics: the 3D Newton kernel's work counters (zeros unless built
// with -DMM_LCE_STATS=1); reset = 1 clears them after the read
extern "C" int mm_debug_lce_counters(double *out, int reset) {
    unsigned long long c[8];
    if (cudaMemcpyFromSymbol(c, g_lce_cnt, sizeof c) != cudaSuccess) return MM_ERR_CUDA;
    for (int i = 0; i < 8; ++i) out[i] = (double)c[i];
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (cudaMemcpyToSymbol(g_lce_cnt, z, sizeof z) != cudaSuccess) return MM_ERR_CUDA;
    }
    return MM_OK;
}

int mm_run_lce(mm_ctx *ctx, double rho, double tol, int64_t max_sweeps, int want_points,
               mm_local_stats *out) {
    int rc;
    const int64_t M = ctx->M;
    const int d = ctx->dim;
    if (!ctx->ang || !ctx->pinc || !ctx->n0 || (d == 3 && !ctx->chart))
        return mm_fail(ctx, MM_ERR_CONFIG, "LCE internal variables were never uploaded");
    if (!ctx->ff) {
        if ((rc = mm_alloc(ctx, (void **)&ctx->ff, sizeof(double) * d * (M ? M : 1)))) return rc;
        MM_CUDA(ctx, cudaMemsetAsync(ctx->ff, 0, sizeof(double) * d * M, ctx->stream));
    }
    const bool viscous = ctx->lce.vis_F > 0.0 || ctx->lce.vis_n > 0.0;
    if (viscous && (!ctx->prevF || !ctx->prevAng || (d == 3 && !ctx->prevChart)))
        return mm_fail(ctx, MM_ERR_PARAM,
                       "viscous update needs the previous step (begin_time_step)");
    // the Newton kernels read grad_u many times per sweep: use the explicit field
    if ((rc = mm_materialize_G(ctx))) return rc;
    LcePar P = make_par(ctx->lce, rho, tol, max_sweeps);
    const double *Fk = viscous ? ctx->prevF : nullptr;
    const double *angk = viscous ? ctx->prevAng : nullptr;
    const int K = 4 + ctx->D;  // + sum of per-point sweeps
    if (d == 2) {
        const int threads = 128;
        const int blocks = lce_blocks(M, threads);
        if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
        StageScope ss(ctx, MM_STAGE_LOCAL);
        k_lce2d<<<blocks, threads, 0, ctx->stream>>>(
            ctx->F, ctx->ang, ctx->pinc, ctx->G, ctx->Lam, ctx->n0, ctx->ff, Fk, angk, M, P,
            want_points ? ctx->res : nullptr, want_points ? ctx->nsw : nullptr,
            want_points ? ctx->ok : nullptr, ctx->partials, ctx->red_out, ctx->red_count);
    } else {
        const int threads = LCE3_THREADS;
        const int blocks = lce_blocks(M, threads);
        if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
        const size_t smem = sizeof(double) * 132 * LCE3_THREADS;
        if (smem > 48 * 1024) {
            for (auto kern : {k_lce3d<0>, k_lce3d<2>, k_lce3d<3>}) {
                cudaError_t e = cudaFuncSetAttribute(
                    kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess)
                    return mm_fail(ctx, MM_ERR_CUDA, "%s", cudaGetErrorString(e));
            }
        }
        const char *split_env = getenv("MM_LCE_SPLIT_MIN");  // per call (tests A/B it)
        const int64_t split_min = split_env ? atoll(split_env) : (int64_t)1 << 18;
        const bool split = M >= split_min && max_sweeps <= 256;
        const double *chk = viscous ? ctx->prevChart : nullptr;
        if (!split) {
            StageScope ss(ctx, MM_STAGE_LOCAL);
            k_lce3d<0><<<blocks, threads, smem, ctx->stream>>>(
                ctx->F, ctx->ang, ctx->chart, ctx->pinc, ctx->G, ctx->Lam, ctx->n0, ctx->ff, Fk,
                angk, chk, M, P, want_points ? ctx->res : nullptr,
                want_points ? ctx->nsw : nullptr, want_points ? ctx->ok : nullptr, ctx->partials,
                ctx->red_out, ctx->red_count, LceSplit{});
        } else {
            if ((rc = mm_ensure_points(ctx))) return rc;
            if (!ctx->lce_fsq0 &&
                (rc = mm_alloc(ctx, (void **)&ctx->lce_fsq0, sizeof(double) * M)))
                return rc;
            for (int b = 0; b < 2; ++b)
                if (!ctx->lce_list[b] &&
                    (rc = mm_alloc(ctx, (void **)&ctx->lce_list[b], sizeof(int) * M)))
                    return rc;
            if (!ctx->lce_cnt && (rc = mm_alloc(ctx, (void **)&ctx->lce_cnt, sizeof(int) * 3)))
                return rc;
            MM_CUDA(ctx, cudaMemsetAsync(ctx->lce_cnt, 0, sizeof(int) * 3, ctx->stream));
            StageScope ss(ctx, MM_STAGE_LOCAL, (int)max_sweeps + 2);
            // round k reads counter k % 3 / list k % 2, appends to counter (k + 1) % 3 /
            // list (k + 1) % 2 and clears counter (k + 2) % 3; a round finds at most
            // one Newton step per point, so max_sweeps rounds after round 0 finish
            // every point (the empty late rounds exit at once)
            const char *kind_env = getenv("MM_LCE_SPLIT_KIND");
            // 2 (default): the Newton step and the next cheap sweeps in one kernel; 3: a
            // Newton-only kernel + a lean one (measured 10.38 vs 10.50 s at 256^3)
            const int kind = kind_env ? atoi(kind_env) : 2;
            for (int64_t k = 0; k <= max_sweeps; ++k) {
                LceSplit sp;
                sp.mode = k == 0 ? 1 : 2;
                sp.list_in = ctx->lce_list[k % 2];
                sp.count_in = ctx->lce_cnt + k % 3;
                sp.list_out = ctx->lce_list[(k + 1) % 2];
                sp.count_out = ctx->lce_cnt + (k + 1) % 3;
                sp.count_clear = ctx->lce_cnt + (k + 2) % 3;
                sp.nsw_io = ctx->nsw;
                sp.fsq0_io = ctx->lce_fsq0;
                sp.budget = 1;
                if (k == 0)  // round 0 has no Newton step: no elimination workspace
                    k_lce3d<1><<<lce_blocks(M, threads), threads, 0, ctx->stream>>>(
                        ctx->F, ctx->ang, ctx->chart, ctx->pinc, ctx->G, ctx->Lam, ctx->n0,
                        ctx->ff, Fk, angk, chk, M, P, ctx->res, ctx->nsw, ctx->ok, ctx->partials,
                        ctx->red_out, ctx->red_count, sp);
                else if (kind == 2)
                    k_lce3d<2><<<blocks, threads, smem, ctx->stream>>>(
                        ctx->F, ctx->ang, ctx->chart, ctx->pinc, ctx->G, ctx->Lam, ctx->n0,
                        ctx->ff, Fk, angk, chk, M, P, ctx->res, ctx->nsw, ctx->ok, ctx->partials,
                        ctx->red_out, ctx->red_count, sp);
                else {
                    // the Newton step of every deferred point at 6 warps/SM (elimination
                    // workspace), then its cheap sweeps without the workspace at 16
                    k_lce3d<3><<<blocks, threads, smem, ctx->stream>>>(
                        ctx->F, ctx->ang, ctx->chart, ctx->pinc, ctx->G, ctx->Lam, ctx->n0,
                        ctx->ff, Fk, angk, chk, M, P, ctx->res, ctx->nsw, ctx->ok, ctx->partials,
                        ctx->red_out, ctx->red_count, sp);
                    MM_LAUNCH_CHECK(ctx);
                    k_lce3d<4><<<lce_blocks(M, threads), threads, 0, ctx->stream>>>(
                        ctx->F, ctx->ang, ctx->chart, ctx->pinc, ctx->G, ctx->Lam, ctx->n0,
                        ctx->ff, Fk, angk, chk, M, P, ctx->res, ctx->nsw, ctx->ok, ctx->partials,
                        ctx->red_out, ctx->red_count, sp);
                }
                MM_LAUNCH_CHECK(ctx);
            }
            const int rb = (int)std::min<int64_t>((M + 255) / 256, 148 * 8);
            if ((rc = mm_ensure_partials(ctx, rb))) return rc;
            k_lce3_reduce<<<rb, 256, 0, ctx->stream>>>(ctx->F, ctx->res, ctx->ok, ctx->nsw, M,
                                                     ctx->partials, ctx->red_out,
                                                     ctx->red_count);
        }
    }
    MM_LAUNCH_CHECK(ctx);
    double r[MM_MAX_PARTIALS];
    if ((rc = mm_fetch_reduction(ctx, K, r))) return rc;
    out->sum_res2 = r[0];
    out->n_conv = (int64_t)r[1];
    out->sweeps = M ? (int64_t)r[2] : 0;
    for (int i = 0; i < ctx->D; ++i) out->sum_F[i] = r[3 + i];
    out->sum_nsw = r[K - 1];
    return MM_OK;
}

// director from the stored angles into `dst` (d components)
static int run_director(mm_ctx *ctx, double *dst, int64_t cs = -1) {
    const int64_t M = ctx->M;
    if (cs < 0) cs = M;
    const int threads = 256;
    const int blocks = lce_blocks(M, threads);
    if (ctx->dim == 2)
        k_director<2><<<blocks, threads, 0, ctx->stream>>>(ctx->ang, nullptr, dst, M, cs);
    else
        k_director<3><<<blocks, threads, 0, ctx->stream>>>(ctx->ang, ctx->chart, dst, M, cs);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

static int run_frank(mm_ctx *ctx, const double *nf, int64_t cs = -1, int wrap0 = 1) {
    const int64_t M = ctx->M;
    if (cs < 0) cs = M;
    const int threads = 256;
    const int blocks = lce_blocks(M, threads);
    const double coef = 2.0 * ctx->lce.frank_kappa / (4.0 * ctx->h * ctx->h);
    if (ctx->dim == 2)
        k_frank<2><<<blocks, threads, 0, ctx->stream>>>(nf, ctx->ff, ctx->n, M, coef, cs, wrap0);
    else
        k_frank<3><<<blocks, threads, 0, ctx->stream>>>(nf, ctx->ff, ctx->n, M, coef, cs, wrap0);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

// slab: the director buffer keeps two ghost planes on each face (the
// radius-2 Frank stencil); dirbuf points at plane 0
int mm_slab_alloc_director(mm_ctx *ctx) {
    if (ctx->dir_base) return MM_OK;
    const int64_t nn = (int64_t)ctx->n * ctx->n;
    int rc = mm_alloc(ctx, (void **)&ctx->dir_base, sizeof(double) * 3 * ctx->dM);
    if (rc) return rc;
    MM_CUDA(ctx, cudaMemsetAsync(ctx->dir_base, 0, sizeof(double) * 3 * ctx->dM, ctx->stream));
    ctx->dirbuf = ctx->dir_base + 2 * nn;
    return MM_OK;
}

// LCE frozen data on a slab (lce.py:223-229): DIRECTOR writes the director
// into the data planes of the ghosted buffer; after the caller's 2-plane
// ghost exchange FRANK applies the radius-2 stencil
int mm_run_slab_lce(mm_ctx *ctx, int step) {
    int rc;
    if (!ctx->have_lce) return mm_fail(ctx, MM_ERR_CONFIG, "LCE parameters were never set");
    if (!ctx->ang || !ctx->chart) return mm_fail(ctx, MM_ERR_CONFIG, "LCE angles were never uploaded");
    if (ctx->slab_nl < 2)
        return mm_fail(ctx, MM_ERR_CONFIG, "the Frank stencil needs >= 2 planes per rank");
    if ((rc = mm_slab_alloc_director(ctx))) return rc;
    if (!ctx->ff) {
        if ((rc = mm_alloc(ctx, (void **)&ctx->ff, sizeof(double) * 3 * ctx->M))) return rc;
    }
    StageScope ss(ctx, MM_STAGE_FROZEN);
    if (!(ctx->lce.frank_kappa > 0.0)) {  // lce.py:225-228
        if (step == MM_SLAB_FRANK)
            MM_CUDA(ctx, cudaMemsetAsync(ctx->ff, 0, sizeof(double) * 3 * ctx->M, ctx->stream));
        return MM_OK;
    }
    if (step == MM_SLAB_DIRECTOR) return run_director(ctx, ctx->dirbuf, ctx->dM);
    return run_frank(ctx, ctx->dirbuf, ctx->dM, 0);
}

int mm_run_frozen(mm_ctx *ctx) {
    int rc;
    const int64_t M = ctx->M;
    const int d = ctx->dim;
    if (!ctx->ang || (d == 3 && !ctx->chart))
        return mm_fail(ctx, MM_ERR_CONFIG, "LCE angles were never uploaded");
    if (!ctx->ff) {
        if ((rc = mm_alloc(ctx, (void **)&ctx->ff, sizeof(double) * d * M))) return rc;
    }
    StageScope ss(ctx, MM_STAGE_FROZEN, 2);
    if (!(ctx->lce.frank_kappa > 0.0)) {  // lce.py:225-228
        MM_CUDA(ctx, cudaMemsetAsync(ctx->ff, 0, sizeof(double) * d * M, ctx->stream));
        return MM_OK;
    }
    if (!ctx->dirbuf && (rc = mm_alloc(ctx, (void **)&ctx->dirbuf, sizeof(double) * d * M)))
        return rc;
    if ((rc = run_director(ctx, ctx->dirbuf))) return rc;
    return run_frank(ctx, ctx->dirbuf);
}

int mm_run_lce_stress(mm_ctx *ctx, double dt, double *P) {
    int rc;
    const int64_t M = ctx->M;
    const int d = ctx->dim;
    if (!ctx->ang || !ctx->pinc || !ctx->n0 || (d == 3 && !ctx->chart))
        return mm_fail(ctx, MM_ERR_CONFIG, "LCE state was never uploaded");
    const bool visc = dt > 0.0 && ctx->lce.vis_F > 0.0;  // lce.py:194-195
    if (visc && !ctx->prevF)
        return mm_fail(ctx, MM_ERR_PARAM, "viscous stress needs prev_F");
    if (!ctx->dirbuf && (rc = mm_alloc(ctx, (void **)&ctx->dirbuf, sizeof(double) * d * M)))
        return rc;
    StageScope ss(ctx, MM_STAGE_OTHER, 2);
    if ((rc = run_director(ctx, ctx->dirbuf))) return rc;
    const int threads = 256;
    const int blocks = lce_blocks(M, threads);
    const mm_lce_params &L = ctx->lce;
    const double vis = visc ? ctx->lce.vis_F : 0.0;  // nu_F / dt, set by mm_set_lce
    const double *Fk = visc ? ctx->prevF : nullptr;
    if (d == 2)
        k_lce_stress<2><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->dirbuf, ctx->n0,
            ctx->pinc, Fk, vis, L.mu, L.r1d, L.rr, L.alpha, L.gamma_inc, P, M);
    else
        k_lce_stress<3><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->dirbuf, ctx->n0,
            ctx->pinc, Fk, vis, L.mu, L.r1d, L.rr, L.alpha, L.gamma_inc, P, M);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

// Frank force of a director field the caller placed in the FF slot
int mm_run_frank_of_ff(mm_ctx *ctx) {
    int rc;
    const int64_t M = ctx->M;
    if (!ctx->ff) return mm_fail(ctx, MM_ERR_CONFIG, "director field (FF slot) was never set");
    if (!ctx->dirbuf &&
        (rc = mm_alloc(ctx, (void **)&ctx->dirbuf, sizeof(double) * ctx->dim * M)))
        return rc;
    StageScope ss(ctx, MM_STAGE_FROZEN);
    MM_CUDA(ctx, cudaMemcpyAsync(ctx->dirbuf, ctx->ff, sizeof(double) * ctx->dim * M,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
    return run_frank(ctx, ctx->dirbuf);
}
