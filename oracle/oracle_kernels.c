/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's per-point local solvers (the
 * numba / vectorised-numpy kernels of `micromech`), used as the parity
 * checker for the CUDA product path and as the CPU baseline ("port") in
 * bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  Nothing in
 * the product package links or calls it.
 *
 * Compiled with -O2 -fno-fast-math -ffp-contract=off so that the
 * arithmetic is plain IEEE double without contraction, like numba's
 * default (no fastmath) code generation.
 *
 * Reference anchors (paths relative to /root/reference/pkg/src/micromech):
 *   orc_mr2d_sweeps       materials/mooney_rivlin.py:169-255 (_mr_sweeps_2d)
 *   orc_descent_sweeps    materials/base.py:124-230 (descent_sweeps_numpy)
 *                         with the objective/gradient closures of
 *                         materials/mooney_rivlin.py:126-162 (MR, any dim)
 *                         and materials/quadratic.py:46-69 (quadratic)
 *   orc_lce2d_sweeps      materials/lce.py:371-584 (_lce_sweeps_2d)
 *   orc_lce3d_sweeps      materials/lce.py:676-995 (_lce_sweeps_3d)
 *   gauss_solve           materials/lce.py:315-349 (_gauss_solve)
 *
 * Layouts are the reference's: F, G, Lam are (npts, d, d) row-major
 * doubles (point-major, AoS), exactly the arrays local_sweeps receives.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* base.py:37-41 */
#define BT_DECREASE 1e-4
#define BT_SHRINK 0.5
#define MAX_BT 60
#define MEAS_EPS (64.0 * 2.220446049250313e-16)
/* lce.py:311-312 */
#define NEWTON_BT 60
#define DET_FLOOR 1e-12

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------------
 * 2D Mooney-Rivlin kernel, mooney_rivlin.py:169-255
 * ------------------------------------------------------------------- */
void orc_mr2d_sweeps(int64_t npts, double *F, const double *G, const double *Lam,
                     const double *mu, const double *kap, double rho, double tol,
                     int64_t max_sweeps, double phi_scale, double *res_out,
                     int64_t *nsw_out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < npts; ++p) {
        double a = F[4 * p + 0], b = F[4 * p + 1], c = F[4 * p + 2], d = F[4 * p + 3];
        const double g00 = G[4 * p + 0], g01 = G[4 * p + 1], g10 = G[4 * p + 2], g11 = G[4 * p + 3];
        const double l00 = Lam[4 * p + 0], l01 = Lam[4 * p + 1], l10 = Lam[4 * p + 2],
                     l11 = Lam[4 * p + 3];
        const double m = mu[p], k = kap[p];
        double t = 1.0 / (rho + m + 4.0 * k);
        const double tmax = 16.0 * t;
        int freemode = 0;
        double res_prev = 1e300, res = 0.0;
        int64_t nsw = 0;
        for (int64_t it = 0; it < max_sweeps + 1; ++it) {
            double J = a * d - b * c;
            double iJ = 1.0 / J;
            double jm1 = J - 1.0;
            double s00 = m * (a - d * iJ) + k * jm1 * d;
            double s01 = m * (b + c * iJ) - k * jm1 * c;
            double s10 = m * (c + b * iJ) - k * jm1 * b;
            double s11 = m * (d - a * iJ) + k * jm1 * a;
            double r00 = s00 - l00 - rho * (g00 - a);
            double r01 = s01 - l01 - rho * (g01 - b);
            double r10 = s10 - l10 - rho * (g10 - c);
            double r11 = s11 - l11 - rho * (g11 - d);
            double gsq = r00 * r00 + r01 * r01 + r10 * r10 + r11 * r11;
            res = sqrt(gsq);
            if (freemode) {
                if (res > res_prev) t *= BT_SHRINK;
                else t = fmin(t * 1.3, tmax);
                res_prev = res;
            }
            if (res < tol || nsw >= max_sweeps) break;
            nsw += 1;
            int did = 0;
            if (!freemode) {
                double W = 0.5 * m * (a * a + b * b + c * c + d * d - 2.0 * log(J) - 2.0) +
                           0.5 * k * jm1 * jm1;
                double phi0 = W - (l00 * a + l01 * b + l10 * c + l11 * d) +
                              0.5 * rho * ((g00 - a) * (g00 - a) + (g01 - b) * (g01 - b) +
                                           (g10 - c) * (g10 - c) + (g11 - d) * (g11 - d));
                if (BT_DECREASE * t * gsq <= MEAS_EPS * (fabs(phi0) + phi_scale)) {
                    freemode = 1;
                    res_prev = res;
                } else {
                    double t_in = t;
                    for (int bt = 0; bt < MAX_BT; ++bt) {
                        double a2 = a - t * r00, b2 = b - t * r01;
                        double c2 = c - t * r10, d2 = d - t * r11;
                        double J2 = a2 * d2 - b2 * c2;
                        if (J2 > 1e-12) {
                            double jm2 = J2 - 1.0;
                            double W2 = 0.5 * m * (a2 * a2 + b2 * b2 + c2 * c2 + d2 * d2 -
                                                   2.0 * log(J2) - 2.0) +
                                        0.5 * k * jm2 * jm2;
                            double phi2 = W2 - (l00 * a2 + l01 * b2 + l10 * c2 + l11 * d2) +
                                          0.5 * rho *
                                              ((g00 - a2) * (g00 - a2) + (g01 - b2) * (g01 - b2) +
                                               (g10 - c2) * (g10 - c2) + (g11 - d2) * (g11 - d2));
                            if (phi2 <= phi0 - BT_DECREASE * t * gsq) {
                                a = a2; b = b2; c = c2; d = d2;
                                did = 1;
                                break;
                            }
                        }
                        t *= BT_SHRINK;
                    }
                    if (did) t = fmin(t * 1.6, tmax);
                    else {
                        freemode = 1;
                        t = t_in;
                        res_prev = res;
                    }
                }
            }
            if (freemode && !did) {
                for (int bt = 0; bt < 12; ++bt) {
                    double a2 = a - t * r00, b2 = b - t * r01;
                    double c2 = c - t * r10, d2 = d - t * r11;
                    if (a2 * d2 - b2 * c2 > 1e-12) {
                        a = a2; b = b2; c = c2; d = d2;
                        break;
                    }
                    t *= BT_SHRINK;
                }
            }
        }
        F[4 * p + 0] = a; F[4 * p + 1] = b; F[4 * p + 2] = c; F[4 * p + 3] = d;
        res_out[p] = res;
        nsw_out[p] = nsw;
    }
}

/* ---------------------------------------------------------------------
 * Vectorised descent (base.py:124-230) restated per point.
 *
 * material 0: Mooney-Rivlin numpy path (mooney_rivlin.py:126-162), any d
 * material 1: quadratic (quadratic.py:46-69); `mu` holds c, `kap` unused
 * ------------------------------------------------------------------- */
enum { MAT_MR = 0, MAT_QUAD = 1 };

static double det_d(const double *X, int d) {
    if (d == 2) return X[0] * X[3] - X[1] * X[2];
    return X[0] * (X[4] * X[8] - X[5] * X[7]) - X[1] * (X[3] * X[8] - X[5] * X[6]) +
           X[2] * (X[3] * X[7] - X[4] * X[6]);
}

/* cofactor matrix (cof = det * inv^T) */
static void cof_d(const double *X, int d, double *C) {
    if (d == 2) {
        C[0] = X[3]; C[1] = -X[2]; C[2] = -X[1]; C[3] = X[0];
        return;
    }
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

/* objective, inf if inadmissible (mooney_rivlin.py:132-141) */
static double objective(int mat, int d, const double *X, const double *Gp, const double *Lp,
                        double m, double k, double rho) {
    int D = d * d;
    double coup_l = 0.0, coup_g = 0.0, I1 = 0.0;
    for (int i = 0; i < D; ++i) {
        coup_l += Lp[i] * X[i];
        double e = Gp[i] - X[i];
        coup_g += e * e;
        I1 += X[i] * X[i];
    }
    double coupling = -coup_l + 0.5 * rho * coup_g;
    if (mat == MAT_QUAD) return 0.5 * m * I1 + coupling;
    double J = det_d(X, d);
    if (J <= 0.0) return INFINITY;
    double W = 0.5 * m * (I1 - 2.0 * log(J) - (double)d) + 0.5 * k * (J - 1.0) * (J - 1.0);
    return W + coupling;
}

/* gradient (mooney_rivlin.py:143-151); returns 0 if det <= 0 */
static int gradient(int mat, int d, const double *X, const double *Gp, const double *Lp,
                    double m, double k, double rho, double *g) {
    int D = d * d;
    if (mat == MAT_QUAD) {
        for (int i = 0; i < D; ++i) g[i] = m * X[i] - Lp[i] - rho * (Gp[i] - X[i]);
        return 1;
    }
    double J = det_d(X, d);
    if (J <= 0.0) return 0;
    double C[9];
    cof_d(X, d, C);
    double c2 = k * (J * J - J);
    for (int i = 0; i < D; ++i) {
        double finvt = C[i] / J;
        double s = m * (X[i] - finvt) + c2 * finvt;
        g[i] = s - Lp[i] - rho * (Gp[i] - X[i]);
    }
    return 1;
}

static int admissible(int mat, int d, const double *X) {
    if (mat == MAT_QUAD) return 1;
    return det_d(X, d) > 0.0;
}

/*
 * Returns the global sweep count (>= 0), or -1 if the gradient met
 * det F <= 0 (InadmissibleStateError, base.py:116-121); X is then left
 * unchanged.  X is updated in place only on success, like the reference
 * which works on a copy and writes back at the end.
 */
int64_t orc_descent_sweeps(int mat, int d, int64_t npts, double *Xio, const double *G,
                           const double *Lam, const double *mu, const double *kap, double rho,
                           double tol, int64_t max_sweeps, double phi_scale, double *res_out) {
    const int D = d * d;
    double *X = (double *)malloc(sizeof(double) * D * npts);
    double *grad = (double *)malloc(sizeof(double) * D * npts);
    double *t = (double *)malloc(sizeof(double) * npts);
    double *tmax = (double *)malloc(sizeof(double) * npts);
    unsigned char *freem = (unsigned char *)calloc(npts, 1);
    double *res = res_out;
    memcpy(X, Xio, sizeof(double) * D * npts);
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (int64_t p = 0; p < npts; ++p) {
        /* t0 = 1/(rho + mu + 4 kappa) for MR, 1/(rho + c) for quadratic */
        t[p] = (mat == MAT_MR) ? 1.0 / (rho + mu[p] + 4.0 * kap[p]) : 1.0 / (rho + mu[p]);
        tmax[p] = t[p] * 16.0;
        double *g = grad + D * p;
        if (!gradient(mat, d, X + D * p, G + D * p, Lam + D * p, mu[p],
                      mat == MAT_MR ? kap[p] : 0.0, rho, g)) {
            bad = 1;
            continue;
        }
        double s = 0.0;
        for (int i = 0; i < D; ++i) s += g[i] * g[i];
        res[p] = sqrt(s);
    }
    int64_t sweeps = 0;
    double ref = INFINITY;
    if (bad) goto fail;
    for (int64_t it = 0; it < max_sweeps; ++it) {
        int64_t nact = 0;
#pragma omp parallel for schedule(static) reduction(+ : nact)
        for (int64_t p = 0; p < npts; ++p) nact += (res[p] > tol);
        if (nact == 0) break;
        sweeps += 1;
#pragma omp parallel for schedule(static) reduction(| : bad)
        for (int64_t p = 0; p < npts; ++p) {
            if (!(res[p] > tol)) continue;
            const double m = mu[p], k = (mat == MAT_MR) ? kap[p] : 0.0;
            double *Xp = X + D * p, *g = grad + D * p;
            const double *Gp = G + D * p, *Lp = Lam + D * p;
            double Xtry[9];
            int in_free = freem[p];
            int in_arm = 0;
            double phi0 = 0.0, gsq = 0.0;
            if (!freem[p]) {
                phi0 = objective(mat, d, Xp, Gp, Lp, m, k, rho);
                for (int i = 0; i < D; ++i) gsq += g[i] * g[i];
                int meas = BT_DECREASE * t[p] * gsq > MEAS_EPS * (fabs(phi0) + phi_scale);
                if (!meas) {
                    freem[p] = 1;
                    in_free = 1; /* joins this sweep's free-step set */
                } else {
                    in_arm = 1;
                }
            }
            double res_before = res[p];
            if (in_arm) {
                double t_in = t[p];
                int accepted = 0;
                for (int bt = 0; bt < MAX_BT; ++bt) {
                    for (int i = 0; i < D; ++i) Xtry[i] = Xp[i] - t[p] * g[i];
                    double phi_try = INFINITY;
                    if (admissible(mat, d, Xtry)) phi_try = objective(mat, d, Xtry, Gp, Lp, m, k, rho);
                    if (phi_try <= phi0 - BT_DECREASE * t[p] * gsq) {
                        memcpy(Xp, Xtry, sizeof(double) * D);
                        accepted = 1;
                        break;
                    }
                    t[p] *= BT_SHRINK;
                }
                if (accepted) {
                    t[p] = fmin(t[p] * 1.6, tmax[p]);
                } else {
                    freem[p] = 1;
                    t[p] = t_in;
                }
            }
            if (in_free) {
                for (int i = 0; i < D; ++i) Xtry[i] = Xp[i] - t[p] * g[i];
                int took = admissible(mat, d, Xtry);
                for (int bt = 0; bt < 12 && !took; ++bt) {
                    t[p] *= BT_SHRINK;
                    for (int i = 0; i < D; ++i) Xtry[i] = Xp[i] - t[p] * g[i];
                    took = admissible(mat, d, Xtry);
                }
                if (took) memcpy(Xp, Xtry, sizeof(double) * D);
            }
            if (!gradient(mat, d, Xp, Gp, Lp, m, k, rho, g)) {
                bad = 1;
                continue;
            }
            double s = 0.0;
            for (int i = 0; i < D; ++i) s += g[i] * g[i];
            res[p] = sqrt(s);
            if (in_free) {
                if (res[p] > res_before) t[p] *= BT_SHRINK;
                else t[p] = fmin(t[p] * 1.3, tmax[p]);
            }
        }
        if (bad) goto fail;
        /* stall guard, base.py:224-229 */
        if (sweeps % 32 == 0) {
            double cur = 0.0;
            for (int64_t p = 0; p < npts; ++p)
                if (res[p] > tol) cur += res[p];
            if (cur > 0.995 * ref) break;
            ref = cur;
        }
    }
    memcpy(Xio, X, sizeof(double) * D * npts);
    free(X); free(grad); free(t); free(tmax); free(freem);
    return sweeps;
fail:
    free(X); free(grad); free(t); free(tmax); free(freem);
    return -1;
}

/* ---------------------------------------------------------------------
 * LCE: Gaussian elimination with partial pivoting, lce.py:315-349
 * ------------------------------------------------------------------- */
static int gauss_solve(int m, double *A, double *b, double *x) {
    for (int col = 0; col < m; ++col) {
        int piv = col;
        double best = fabs(A[col * m + col]);
        for (int r = col + 1; r < m; ++r) {
            if (fabs(A[r * m + col]) > best) {
                best = fabs(A[r * m + col]);
                piv = r;
            }
        }
        if (best < 1e-250) return 0;
        if (piv != col) {
            for (int c = 0; c < m; ++c) {
                double tmp = A[col * m + c];
                A[col * m + c] = A[piv * m + c];
                A[piv * m + c] = tmp;
            }
            double tmp = b[col];
            b[col] = b[piv];
            b[piv] = tmp;
        }
        double inv = 1.0 / A[col * m + col];
        for (int r = col + 1; r < m; ++r) {
            double f = A[r * m + col] * inv;
            if (f != 0.0) {
                for (int c = col; c < m; ++c) A[r * m + c] -= f * A[col * m + c];
                b[r] -= f * b[col];
            }
        }
    }
    for (int r = m - 1; r >= 0; --r) {
        double s = b[r];
        for (int c = r + 1; c < m; ++c) s -= A[r * m + c] * x[c];
        x[r] = s / A[r * m + r];
    }
    return 1;
}

/* scalar objective parameters shared by both LCE kernels */
typedef struct {
    double mur, rr, mual, gam, rho, visF, visn, q;
} lce_par;

/* 2D augmented point objective, lce.py:352-368 */
static double phiF2(const double f[4], double n1, double n2, double m01, double m02,
                    const lce_par *P, double pp, const double L[4], const double Gv[4],
                    const double K[4]) {
    double u1 = f[0] * n1 + f[2] * n2;
    double u2 = f[1] * n1 + f[3] * n2;
    double cc = u1 * m01 + u2 * m02;
    double dJ = f[0] * f[3] - f[1] * f[2] - 1.0;
    double e0 = Gv[0] - f[0], e1 = Gv[1] - f[1], e2 = Gv[2] - f[2], e3 = Gv[3] - f[3];
    double v0 = f[0] - K[0], v1 = f[1] - K[1], v2 = f[2] - K[2], v3 = f[3] - K[3];
    return 0.5 * P->mur * (f[0] * f[0] + f[1] * f[1] + f[2] * f[2] + f[3] * f[3]) -
           0.5 * P->mur * P->rr * (u1 * u1 + u2 * u2) +
           0.5 * P->mual * (u1 * u1 + u2 * u2 - cc * cc) + pp * dJ + 0.5 * P->gam * dJ * dJ -
           (L[0] * f[0] + L[1] * f[1] + L[2] * f[2] + L[3] * f[3]) +
           0.5 * P->rho * (e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3) +
           0.5 * P->visF * (v0 * v0 + v1 * v1 + v2 * v2 + v3 * v3);
}

static double phiJ2(const double f[4], double th, const double n0[2], const lce_par *P, double pp,
                    const double L[4], const double Gv[4], const double K[4], const double ffp[2],
                    const double nkp[2]) {
    double p1 = cos(th), p2 = sin(th);
    double a = p1 - nkp[0], b = p2 - nkp[1];
    return phiF2(f, p1, p2, n0[0], n0[1], P, pp, L, Gv, K) + ffp[0] * p1 + ffp[1] * p2 +
           0.5 * P->visn * (a * a + b * b);
}

/* lce.py:371-584 */
void orc_lce2d_sweeps(int64_t npts, double *F, double *ang, double *p_inc, const double *G,
                      const double *Lam, const double *n0, const double *ff, const double *Fk,
                      const double *nk, double mu, double r1d, double rr, double al, double gam,
                      double rho, double vis_F, double vis_n, double tol, double det_tol,
                      int64_t max_sweeps, double phiF_scale, double phin_scale, double *res_out,
                      int64_t *nsw_out, unsigned char *ok_out) {
    lce_par P;
    P.mur = mu * r1d;
    P.mual = mu * al;
    P.q = P.mual - P.mur * rr;
    P.rr = rr;
    P.gam = gam;
    P.rho = rho;
    P.visF = vis_F;
    P.visn = vis_n;
    const double q = P.q, mur = P.mur, mual = P.mual;
    const double scale = phiF_scale + phin_scale;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t p = 0; p < npts; ++p) {
        double f[4], L[4], Gv[4], K[4];
        for (int i = 0; i < 4; ++i) {
            f[i] = F[4 * p + i];
            L[i] = Lam[4 * p + i];
            Gv[i] = G[4 * p + i];
            K[i] = Fk[4 * p + i];
        }
        double th = ang[p], pp = p_inc[p];
        const double m0[2] = {n0[2 * p], n0[2 * p + 1]};
        const double ffp[2] = {ff[2 * p], ff[2 * p + 1]};
        const double nkp[2] = {nk[2 * p], nk[2 * p + 1]};
        double H[25], A[25], rhs[5], bw[5], dv[5];
        double fsq0 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2] + f[3] * f[3];
        double tF0 = 1.0 / (rho + 2.0 * mur + 2.0 * mual + 2.0 * gam + vis_F);
        double tN0 = 1.0 / (mu * (2.0 * r1d + 2.0 * al) * fmax(fsq0, 1.0) + vis_n + 1e-30);
        double base = mur + rho + vis_F;
        int64_t nsw = 0;
        double res = 0.0;
        int converged = 0;
        for (int64_t it = 0; it < max_sweeps + 1; ++it) {
            double n1 = cos(th), n2 = sin(th);
            double u1 = f[0] * n1 + f[2] * n2, u2 = f[1] * n1 + f[3] * n2;
            double cc = u1 * m0[0] + u2 * m0[1];
            double v1 = f[0] * m0[0] + f[1] * m0[1], v2 = f[2] * m0[0] + f[3] * m0[1];
            double h1 = f[0] * u1 + f[1] * u2, h2 = f[2] * u1 + f[3] * u2;
            double J = f[0] * f[3] - f[1] * f[2];
            double dJ = J - 1.0;
            double pr = pp + gam * dJ;
            double rF[4];
            rF[0] = mur * f[0] + q * n1 * u1 - mual * cc * n1 * m0[0] + pr * f[3] - L[0] -
                    rho * (Gv[0] - f[0]) + vis_F * (f[0] - K[0]);
            rF[1] = mur * f[1] + q * n1 * u2 - mual * cc * n1 * m0[1] - pr * f[2] - L[1] -
                    rho * (Gv[1] - f[1]) + vis_F * (f[1] - K[1]);
            rF[2] = mur * f[2] + q * n2 * u1 - mual * cc * n2 * m0[0] - pr * f[1] - L[2] -
                    rho * (Gv[2] - f[2]) + vis_F * (f[2] - K[2]);
            rF[3] = mur * f[3] + q * n2 * u2 - mual * cc * n2 * m0[1] + pr * f[0] - L[3] -
                    rho * (Gv[3] - f[3]) + vis_F * (f[3] - K[3]);
            double gF2 = rF[0] * rF[0] + rF[1] * rF[1] + rF[2] * rF[2] + rF[3] * rF[3];
            double gn1 = q * h1 - mual * cc * v1 + ffp[0] + vis_n * (n1 - nkp[0]);
            double gn2 = q * h2 - mual * cc * v2 + ffp[1] + vis_n * (n2 - nkp[1]);
            double gth = -gn1 * n2 + gn2 * n1;
            res = sqrt(gF2 + gth * gth);
            if (res < tol && fabs(dJ) <= det_tol) {
                converged = 1;
                break;
            }
            if (nsw >= max_sweeps) break;
            nsw += 1;
            if (fabs(dJ) > det_tol && res <= fmax(tol, 0.25 * gam * fabs(dJ))) {
                pp += gam * dJ;
                continue;
            }
            double phi0 = phiF2(f, n1, n2, m0[0], m0[1], &P, pp, L, Gv, K) + ffp[0] * n1 +
                          ffp[1] * n2 +
                          0.5 * vis_n * ((n1 - nkp[0]) * (n1 - nkp[0]) + (n2 - nkp[1]) * (n2 - nkp[1]));
            /* joint Hessian on (F, theta) */
            for (int i = 0; i < 25; ++i) H[i] = 0.0;
            for (int a = 0; a < 4; ++a) H[a * 5 + a] = base;
            double n11 = q * n1 * n1, n12 = q * n1 * n2, n22 = q * n2 * n2;
            H[0 * 5 + 0] += n11; H[0 * 5 + 2] += n12; H[2 * 5 + 0] += n12; H[2 * 5 + 2] += n22;
            H[1 * 5 + 1] += n11; H[1 * 5 + 3] += n12; H[3 * 5 + 1] += n12; H[3 * 5 + 3] += n22;
            double wv[4] = {n1 * m0[0], n1 * m0[1], n2 * m0[0], n2 * m0[1]};
            double cv[4] = {f[3], -f[2], -f[1], f[0]};
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) H[a * 5 + b] += gam * cv[a] * cv[b] - mual * wv[a] * wv[b];
            H[0 * 5 + 3] += pr; H[3 * 5 + 0] += pr;
            H[1 * 5 + 2] -= pr; H[2 * 5 + 1] -= pr;
            double up1 = -f[0] * n2 + f[2] * n1, up2 = -f[1] * n2 + f[3] * n1;
            double ccp = up1 * m0[0] + up2 * m0[1];
            H[0 * 5 + 4] = q * (-n2 * u1 + n1 * up1) - mual * (ccp * n1 - cc * n2) * m0[0];
            H[1 * 5 + 4] = q * (-n2 * u2 + n1 * up2) - mual * (ccp * n1 - cc * n2) * m0[1];
            H[2 * 5 + 4] = q * (n1 * u1 + n2 * up1) - mual * (ccp * n2 + cc * n1) * m0[0];
            H[3 * 5 + 4] = q * (n1 * u2 + n2 * up2) - mual * (ccp * n2 + cc * n1) * m0[1];
            for (int a = 0; a < 4; ++a) H[4 * 5 + a] = H[a * 5 + 4];
            H[4 * 5 + 4] = q * (up1 * up1 + up2 * up2) - mual * ccp * ccp + vis_n - (gn1 * n1 + gn2 * n2);
            rhs[0] = -rF[0]; rhs[1] = -rF[1]; rhs[2] = -rF[2]; rhs[3] = -rF[3]; rhs[4] = -gth;
            /* Newton direction with Levenberg inflation */
            double lam = 0.0, gd = 0.0;
            int found = 0;
            for (int lm = 0; lm < 4; ++lm) {
                for (int a = 0; a < 5; ++a) {
                    for (int b = 0; b < 5; ++b) A[a * 5 + b] = H[a * 5 + b];
                    A[a * 5 + a] += lam;
                    bw[a] = rhs[a];
                }
                if (gauss_solve(5, A, bw, dv)) {
                    gd = -(rhs[0] * dv[0] + rhs[1] * dv[1] + rhs[2] * dv[2] + rhs[3] * dv[3] +
                           rhs[4] * dv[4]);
                    if (gd < 0.0) {
                        found = 1;
                        break;
                    }
                }
                lam = (lam == 0.0) ? base : lam * 10.0;
            }
            int did = 0;
            for (int pass = 0; pass < 2 && !did; ++pass) {
                /* pass 0: Newton direction (if found); pass 1: scaled gradient */
                double decr;
                if (pass == 0) {
                    if (!found) continue;
                    decr = -0.5 * gd;
                } else {
                    dv[0] = -tF0 * rF[0]; dv[1] = -tF0 * rF[1];
                    dv[2] = -tF0 * rF[2]; dv[3] = -tF0 * rF[3];
                    dv[4] = -tN0 * gth;
                    gd = -(tF0 * gF2 + tN0 * gth * gth);
                    decr = -BT_DECREASE * gd;
                }
                double t = 1.0;
                if (decr <= MEAS_EPS * (fabs(phi0) + scale)) {
                    for (int bt = 0; bt < 12; ++bt) {
                        double a2 = f[0] + t * dv[0], b2 = f[1] + t * dv[1];
                        double c2 = f[2] + t * dv[2], d2 = f[3] + t * dv[3];
                        if (a2 * d2 - b2 * c2 > DET_FLOOR) {
                            f[0] = a2; f[1] = b2; f[2] = c2; f[3] = d2;
                            th = th + t * dv[4];
                            did = 1;
                            break;
                        }
                        t *= 0.5;
                    }
                } else {
                    for (int bt = 0; bt < NEWTON_BT; ++bt) {
                        double ft[4] = {f[0] + t * dv[0], f[1] + t * dv[1], f[2] + t * dv[2],
                                        f[3] + t * dv[3]};
                        if (ft[0] * ft[3] - ft[1] * ft[2] > DET_FLOOR) {
                            double th2 = th + t * dv[4];
                            double phi2 = phiJ2(ft, th2, m0, &P, pp, L, Gv, K, ffp, nkp);
                            if (phi2 <= phi0 + BT_DECREASE * t * gd) {
                                f[0] = ft[0]; f[1] = ft[1]; f[2] = ft[2]; f[3] = ft[3];
                                th = th2;
                                did = 1;
                                break;
                            }
                        }
                        t *= 0.5;
                    }
                }
                if (pass == 1) did = 1; /* fallback never retries */
            }
        }
        for (int i = 0; i < 4; ++i) F[4 * p + i] = f[i];
        ang[p] = th;
        p_inc[p] = pp;
        res_out[p] = res;
        nsw_out[p] = nsw;
        ok_out[p] = (unsigned char)converged;
    }
}

/* ---------------------------------------------------------------------
 * LCE 3D helpers, lce.py:589-673
 * ------------------------------------------------------------------- */
static double det3(const double *A) {
    return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
           A[2] * (A[3] * A[7] - A[4] * A[6]);
}

static void n_from_chart(double ph, double th, const double *E, double *out) {
    double sp = sin(ph);
    double a = sp * cos(th), b = sp * sin(th), c = cos(ph);
    for (int i = 0; i < 3; ++i) out[i] = a * E[3 * i + 0] + b * E[3 * i + 1] + c * E[3 * i + 2];
}

static double phiF3(const double *Fl, const double *n, const double *n0l, const lce_par *P,
                    double pp, const double *Ll, const double *Gl, const double *Kl) {
    double fsq = 0.0, coup = 0.0;
    for (int i = 0; i < 9; ++i) {
        double fij = Fl[i];
        fsq += fij * fij;
        double e = Gl[i] - fij, v = fij - Kl[i];
        coup += (-Ll[i] * fij + 0.5 * P->rho * (e * e) + 0.5 * P->visF * (v * v));
    }
    double usq = 0.0, cc = 0.0;
    for (int i = 0; i < 3; ++i) {
        double ui = Fl[0 * 3 + i] * n[0] + Fl[1 * 3 + i] * n[1] + Fl[2 * 3 + i] * n[2];
        usq += ui * ui;
        cc += ui * n0l[i];
    }
    double dJ = det3(Fl) - 1.0;
    return (0.5 * P->mur * (fsq - P->rr * usq) + 0.5 * P->mual * (usq - cc * cc) + pp * dJ +
            0.5 * P->gam * dJ * dJ + coup);
}

static double phiJ3(const double *Fl, const double *n, const double *n0l, const lce_par *P,
                    double pp, const double *Ll, const double *Gl, const double *Kl,
                    const double *ffl, const double *nkl) {
    double extra = 0.0;
    for (int i = 0; i < 3; ++i) {
        double e = n[i] - nkl[i];
        extra += ffl[i] * n[i] + 0.5 * P->visn * (e * e);
    }
    return phiF3(Fl, n, n0l, P, pp, Ll, Gl, Kl) + extra;
}

static void gradN3(const double *n, const double *Fl, const double *n0l, const lce_par *P,
                   const double *ffl, const double *nkl, double *out) {
    double u0 = Fl[0] * n[0] + Fl[3] * n[1] + Fl[6] * n[2];
    double u1 = Fl[1] * n[0] + Fl[4] * n[1] + Fl[7] * n[2];
    double u2 = Fl[2] * n[0] + Fl[5] * n[1] + Fl[8] * n[2];
    double cc = u0 * n0l[0] + u1 * n0l[1] + u2 * n0l[2];
    double q = P->mual - P->mur * P->rr;
    for (int i = 0; i < 3; ++i) {
        double h = Fl[3 * i + 0] * u0 + Fl[3 * i + 1] * u1 + Fl[3 * i + 2] * u2;
        double v = Fl[3 * i + 0] * n0l[0] + Fl[3 * i + 1] * n0l[1] + Fl[3 * i + 2] * n0l[2];
        out[i] = q * h - P->mual * cc * v + ffl[i] + P->visn * (n[i] - nkl[i]);
    }
}

static void Qdot(const double *Fl, const double *Fn0, double q, double mual, double visn,
                 const double *v, double *out) {
    double u0 = Fl[0] * v[0] + Fl[3] * v[1] + Fl[6] * v[2];
    double u1 = Fl[1] * v[0] + Fl[4] * v[1] + Fl[7] * v[2];
    double u2 = Fl[2] * v[0] + Fl[5] * v[1] + Fl[8] * v[2];
    double vf = v[0] * Fn0[0] + v[1] * Fn0[1] + v[2] * Fn0[2];
    for (int i = 0; i < 3; ++i) {
        double h = Fl[3 * i + 0] * u0 + Fl[3 * i + 1] * u1 + Fl[3 * i + 2] * u2;
        out[i] = q * h - mual * vf * Fn0[i] + visn * v[i];
    }
}

/* lce.py:676-995 */
void orc_lce3d_sweeps(int64_t npts, double *F, double *ang, double *chart, double *p_inc,
                      const double *G, const double *Lam, const double *n0, const double *ff,
                      const double *Fk, const double *nk, double mu, double r1d, double rr,
                      double al, double gam, double rho, double vis_F, double vis_n, double tol,
                      double det_tol, int64_t max_sweeps, double phiF_scale, double phin_scale,
                      double *res_out, int64_t *nsw_out, unsigned char *ok_out) {
    lce_par P;
    P.mur = mu * r1d;
    P.mual = mu * al;
    P.q = P.mual - P.mur * rr;
    P.rr = rr;
    P.gam = gam;
    P.rho = rho;
    P.visF = vis_F;
    P.visn = vis_n;
    const double q = P.q, mur = P.mur, mual = P.mual;
    const double scale = phiF_scale + phin_scale;
    const double PI = 3.141592653589793;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t p = 0; p < npts; ++p) {
        double Fl[9], E[9];
        memcpy(Fl, F + 9 * p, sizeof Fl);
        memcpy(E, chart + 9 * p, sizeof E);
        const double *Gl = G + 9 * p, *Ll = Lam + 9 * p, *Kl = Fk + 9 * p;
        const double *n0l = n0 + 3 * p, *ffl = ff + 3 * p, *nkl = nk + 3 * p;
        double ph = ang[2 * p + 0], th = ang[2 * p + 1], pp = p_inc[p];
        double n[3], u[3], gFl[9], cof[9], Ftry[9], gn[3], ntry[3], Fn0[3], m1[3], mth[3];
        double ua[3], ub[3], qv[3];
        double H[121], A[121], rhs[11], bw[11], dv[11], wv[9], cv[9];
        double fsq0 = 0.0;
        for (int i = 0; i < 9; ++i) fsq0 += Fl[i] * Fl[i];
        double tF0 = 1.0 / (rho + 2.0 * mur + 2.0 * mual + 3.0 * gam + vis_F);
        double tN0 = 1.0 / (mu * (2.0 * r1d + 2.0 * al) * fmax(fsq0, 1.0) + vis_n + 1e-30);
        double base = mur + rho + vis_F;
        int64_t nsw = 0;
        double res = 0.0;
        int converged = 0;
        for (int64_t it = 0; it < max_sweeps + 1; ++it) {
            /* re-chart when the azimuth degenerates (lce.py:709-730) */
            if (sin(ph) < 0.1) {
                n_from_chart(ph, th, E, n);
                int k = 0;
                if (fabs(n[1]) < fabs(n[k])) k = 1;
                if (fabs(n[2]) < fabs(n[k])) k = 2;
                double dot = n[k], e3n = 0.0;
                for (int i = 0; i < 3; ++i) {
                    double v = (i == k ? 1.0 : 0.0) - dot * n[i];
                    gn[i] = v;
                    e3n += v * v;
                }
                e3n = sqrt(e3n);
                for (int i = 0; i < 3; ++i) {
                    E[3 * i + 0] = n[i];
                    E[3 * i + 2] = gn[i] / e3n;
                }
                E[0 * 3 + 1] = E[1 * 3 + 2] * E[2 * 3 + 0] - E[2 * 3 + 2] * E[1 * 3 + 0];
                E[1 * 3 + 1] = E[2 * 3 + 2] * E[0 * 3 + 0] - E[0 * 3 + 2] * E[2 * 3 + 0];
                E[2 * 3 + 1] = E[0 * 3 + 2] * E[1 * 3 + 0] - E[1 * 3 + 2] * E[0 * 3 + 0];
                ph = 0.5 * PI;
                th = 0.0;
            }
            n_from_chart(ph, th, E, n);
            double sp = sin(ph), cp = cos(ph), ct = cos(th), st = sin(th);
            for (int j = 0; j < 3; ++j) u[j] = Fl[0 * 3 + j] * n[0] + Fl[1 * 3 + j] * n[1] + Fl[2 * 3 + j] * n[2];
            double cc = u[0] * n0l[0] + u[1] * n0l[1] + u[2] * n0l[2];
            double J = det3(Fl);
            double dJ = J - 1.0;
            double pr = pp + gam * dJ;
            cof_d(Fl, 3, cof);
            double gF2 = 0.0;
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double g = (mur * Fl[3 * i + j] + q * n[i] * u[j] - mual * cc * n[i] * n0l[j] +
                                pr * cof[3 * i + j] - Ll[3 * i + j] - rho * (Gl[3 * i + j] - Fl[3 * i + j]) +
                                vis_F * (Fl[3 * i + j] - Kl[3 * i + j]));
                    gFl[3 * i + j] = g;
                    gF2 += g * g;
                }
            gradN3(n, Fl, n0l, &P, ffl, nkl, gn);
            double g1 = 0.0, g2 = 0.0, gnn = 0.0;
            for (int i = 0; i < 3; ++i) {
                m1[i] = cp * ct * E[3 * i + 0] + cp * st * E[3 * i + 1] - sp * E[3 * i + 2];
                mth[i] = sp * (-st * E[3 * i + 0] + ct * E[3 * i + 1]);
                g1 += gn[i] * m1[i];
                g2 += gn[i] * mth[i];
                gnn += gn[i] * n[i];
            }
            double sp2 = fmax(sp * sp, 1e-4);
            res = sqrt(gF2 + g1 * g1 + g2 * g2 / sp2);
            if (res < tol && fabs(dJ) <= det_tol) {
                converged = 1;
                break;
            }
            if (nsw >= max_sweeps) break;
            nsw += 1;
            if (fabs(dJ) > det_tol && res <= fmax(tol, 0.25 * gam * fabs(dJ))) {
                pp += gam * dJ;
                continue;
            }
            double phi0 = phiJ3(Fl, n, n0l, &P, pp, Ll, Gl, Kl, ffl, nkl);
            for (int a = 0; a < 121; ++a) H[a] = 0.0;
            for (int a = 0; a < 9; ++a) H[a * 11 + a] = base;
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k) {
                    double qnn = q * n[i] * n[k];
                    for (int j = 0; j < 3; ++j) H[(3 * i + j) * 11 + 3 * k + j] += qnn;
                }
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    wv[3 * i + j] = n[i] * n0l[j];
                    cv[3 * i + j] = cof[3 * i + j];
                }
            for (int a = 0; a < 9; ++a)
                for (int b = 0; b < 9; ++b) H[a * 11 + b] += gam * cv[a] * cv[b] - mual * wv[a] * wv[b];
            /* pr * d2J/dF2 via the Levi-Civita contraction */
            for (int i = 0; i < 3; ++i)
                for (int k = 0; k < 3; ++k) {
                    if (k == i) continue;
                    int m = 3 - i - k;
                    double si = (k == (i + 1) % 3) ? 1.0 : -1.0;
                    for (int j = 0; j < 3; ++j)
                        for (int l = 0; l < 3; ++l) {
                            if (l == j) continue;
                            int nn = 3 - j - l;
                            double sj = (l == (j + 1) % 3) ? 1.0 : -1.0;
                            H[(3 * i + j) * 11 + 3 * k + l] += pr * si * sj * Fl[3 * m + nn];
                        }
                }
            for (int j = 0; j < 3; ++j) {
                ua[j] = Fl[0 * 3 + j] * m1[0] + Fl[1 * 3 + j] * m1[1] + Fl[2 * 3 + j] * m1[2];
                ub[j] = Fl[0 * 3 + j] * mth[0] + Fl[1 * 3 + j] * mth[1] + Fl[2 * 3 + j] * mth[2];
            }
            double cca = ua[0] * n0l[0] + ua[1] * n0l[1] + ua[2] * n0l[2];
            double ccb = ub[0] * n0l[0] + ub[1] * n0l[1] + ub[2] * n0l[2];
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    int a = 3 * i + j;
                    H[a * 11 + 9] = q * (m1[i] * u[j] + n[i] * ua[j]) - mual * (cca * n[i] + cc * m1[i]) * n0l[j];
                    H[9 * 11 + a] = H[a * 11 + 9];
                    H[a * 11 + 10] = q * (mth[i] * u[j] + n[i] * ub[j]) - mual * (ccb * n[i] + cc * mth[i]) * n0l[j];
                    H[10 * 11 + a] = H[a * 11 + 10];
                }
            double gchd = 0.0, gt2 = 0.0;
            for (int i = 0; i < 3; ++i) {
                gchd += gn[i] * cp * (-st * E[3 * i + 0] + ct * E[3 * i + 1]);
                gt2 += gn[i] * (-sp) * (ct * E[3 * i + 0] + st * E[3 * i + 1]);
            }
            for (int i = 0; i < 3; ++i) Fn0[i] = Fl[3 * i + 0] * n0l[0] + Fl[3 * i + 1] * n0l[1] + Fl[3 * i + 2] * n0l[2];
            Qdot(Fl, Fn0, q, mual, vis_n, m1, qv);
            double h11 = -gnn, h12 = gchd;
            for (int i = 0; i < 3; ++i) {
                h11 += m1[i] * qv[i];
                h12 += mth[i] * qv[i];
            }
            Qdot(Fl, Fn0, q, mual, vis_n, mth, qv);
            double h22 = gt2;
            for (int i = 0; i < 3; ++i) h22 += mth[i] * qv[i];
            H[9 * 11 + 9] = h11;
            H[9 * 11 + 10] = h12;
            H[10 * 11 + 9] = h12;
            H[10 * 11 + 10] = h22;
            for (int a = 0; a < 9; ++a) rhs[a] = -gFl[a];
            rhs[9] = -g1;
            rhs[10] = -g2;
            double lam = 0.0, gd = 0.0;
            int found = 0;
            for (int lm = 0; lm < 4; ++lm) {
                for (int a = 0; a < 11; ++a) {
                    for (int b = 0; b < 11; ++b) A[a * 11 + b] = H[a * 11 + b];
                    A[a * 11 + a] += lam;
                    bw[a] = rhs[a];
                }
                if (gauss_solve(11, A, bw, dv)) {
                    gd = 0.0;
                    for (int a = 0; a < 11; ++a) gd -= rhs[a] * dv[a];
                    if (gd < 0.0) {
                        found = 1;
                        break;
                    }
                }
                lam = (lam == 0.0) ? base : lam * 10.0;
            }
            int did = 0;
            for (int pass = 0; pass < 2 && !did; ++pass) {
                double decr;
                if (pass == 0) {
                    if (!found) continue;
                    decr = -0.5 * gd;
                } else {
                    for (int a = 0; a < 9; ++a) dv[a] = -tF0 * gFl[a];
                    dv[9] = -tN0 * g1;
                    dv[10] = -tN0 * g2 / sp2;
                    gd = -(tF0 * gF2 + tN0 * (g1 * g1 + g2 * g2 / sp2));
                    decr = -BT_DECREASE * gd;
                }
                double t = 1.0;
                if (decr <= MEAS_EPS * (fabs(phi0) + scale)) {
                    for (int bt = 0; bt < 12; ++bt) {
                        for (int a = 0; a < 9; ++a) Ftry[a] = Fl[a] + t * dv[a];
                        if (det3(Ftry) > DET_FLOOR) {
                            memcpy(Fl, Ftry, sizeof Fl);
                            ph = ph + t * dv[9];
                            th = th + t * dv[10];
                            did = 1;
                            break;
                        }
                        t *= 0.5;
                    }
                } else {
                    for (int bt = 0; bt < NEWTON_BT; ++bt) {
                        for (int a = 0; a < 9; ++a) Ftry[a] = Fl[a] + t * dv[a];
                        if (det3(Ftry) > DET_FLOOR) {
                            double ph2 = ph + t * dv[9], th2 = th + t * dv[10];
                            n_from_chart(ph2, th2, E, ntry);
                            double phi2 = phiJ3(Ftry, ntry, n0l, &P, pp, Ll, Gl, Kl, ffl, nkl);
                            if (phi2 <= phi0 + BT_DECREASE * t * gd) {
                                memcpy(Fl, Ftry, sizeof Fl);
                                ph = ph2;
                                th = th2;
                                did = 1;
                                break;
                            }
                        }
                        t *= 0.5;
                    }
                }
                if (pass == 1) did = 1;
            }
        }
        memcpy(F + 9 * p, Fl, sizeof Fl);
        memcpy(chart + 9 * p, E, sizeof E);
        ang[2 * p + 0] = ph;
        ang[2 * p + 1] = th;
        p_inc[p] = pp;
        res_out[p] = res;
        nsw_out[p] = nsw;
        ok_out[p] = (unsigned char)converged;
    }
}
