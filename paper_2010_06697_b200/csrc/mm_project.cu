// Global step of the ADMM iteration: Helmholtz projection (projection.py:132-168)
// fused with the multiplier ascent and residuals (solver.py:268-279).
//
// The reference transforms 9 tensor components forward and 3 + 9 inverse.
// Here the same result (exact in exact arithmetic) is obtained with d
// components each way:
//   A  k_row_fwd   stencil divergence d_i = sum_j T_ij(x+e_j) - T_ij(x-e_j),
//                  T = F - lam/rho, fused with the real-to-complex FFT along
//                  the contiguous axis (two reals packed per complex, one
//                  N/2-point complex FFT per row + split)
//   B  k_col       complex FFT along axis 1 (3D only)
//   C  k_col<SOLVE> complex FFT along axis 0, the per-wavevector solve
//                  u_hat = -d_hat / |g|^2 (masked modes -> 0, projection.py:
//                  155-157), and the inverse FFT along axis 0, in one pass
//   D  k_col       inverse FFT along axis 1 (3D only)
//   E  k_row_inv   complex-to-real inverse along the contiguous axis -> u_tilde
//   F  k_grad      grad_u = u_mean + central difference of u_tilde, and (solver
//                  path) |dG|^2, lam += rho (grad_u - F), |misfit|^2, sum lam
// Every FFT keeps a tile of lines in shared memory; power-of-two lengths use a
// register four-step (N = N1 x N2, one N1-point FFT per thread, twiddle, one
// shared-memory exchange, one N2-point FFT per thread); other lengths use an
// exact O(N^2) DFT over the same tile (small grids only).
#include <math.h>

#include <algorithm>

#include "mm_internal.cuh"

namespace {

// build-time kernel variants (A/B with tools/gpu_ab.sh)
#ifndef MM_ROWINV_BAL
#define MM_ROWINV_BAL 0
#endif
#ifndef MM_TW_PROD
#define MM_TW_PROD 1  // plane pass 0.713 -> 0.695 ms at 256^3
#endif
#ifndef MM_ROWINV_REGS
#define MM_ROWINV_REGS 128  // row_inv_p: 80 spilled 364 B; 164 registers, 0.321 -> 0.220 ms
#endif
#ifndef MM_COL32_MINB
#define MM_COL32_MINB 2
#endif
#ifndef MM_ROWINV_P_ROWS
#define MM_ROWINV_P_ROWS 1
#endif
#ifndef MM_ROWINV_P_MAXN
#define MM_ROWINV_P_MAXN 256
#endif
#ifndef MM_ROWFWD_REGS
#define MM_ROWFWD_REGS 96
#endif
#ifndef MM_RFW_TWP
#define MM_RFW_TWP 1  // k_row_fwd_w: twiddles from 4 loads + products (0.375 -> 0.353 ms; 0: bitwise = k_row_fwd)
#endif
#ifndef MM_LM_TWP
#define MM_LM_TWP 1  // plane row passes: twiddles from 4 loads + products (tile_fft_lm256): 0.475 -> 0.457 ms
#endif
#ifndef MM_PLANE_COLSWZ
// 1: n = 256 column pass on 128-byte swizzled tiles (plane_col_swz): measured
// 0.51 vs 0.485 ms and it costs the default kernel registers, so not built
#define MM_PLANE_COLSWZ 0
#endif
#ifndef MM_ROWFWD_W
#define MM_ROWFWD_W 1  // n = 256: the warp-per-task R2C rows (k_row_fwd_w)
#endif
#ifndef MM_ROWFWD_W_MINB
#define MM_ROWFWD_W_MINB 4  // 128 registers: 0.369 ms at 256^3 (5: 0.399, 6: 0.574, tiled kernel 0.459)
#endif
__constant__ double2 c_w32[32];  // exp(-2 pi i k / 32)

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

template <int R>
__host__ __device__ constexpr int brev(int i) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

// In-register radix-2 DIT FFT of R <= 32 points, natural-order output.
template <int R, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&v)[R]) {
    if constexpr (R > 1) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int j = brev<R>(i);
            if (j > i) {
                double2 t = v[i];
                v[i] = v[j];
                v[j] = t;
            }
        }
#pragma unroll
        for (int half = 1; half < R; half <<= 1) {
#pragma unroll
            for (int i = 0; i < R; i += 2 * half) {
#pragma unroll
                for (int k = 0; k < half; ++k) {
                    const double2 a = v[i + k];
                    double2 b = v[i + k + half];
                    if (k != 0) {
                        if (2 * k == half) {  // W_{2 half}^{half/2} = -i (fwd) / +i (inv)
                            b = INV ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
                        } else {
                            double2 w = c_w32[k * (16 / half)];
                            if (INV) w.y = -w.y;
                            b = cmul(b, w);
                        }
                    }
                    v[i + k] = cadd(a, b);
                    v[i + k + half] = csub(a, b);
                }
            }
        }
    }
}

// FFT of TK lines of length N = N1*N2 held in shared memory, element n of
// line c at buf[n*LD + c], LD = TK + 1.  Requires blockDim >= TK*max(N1,N2).
// tw: exp(-2 pi i k / N), k < N.
template <int N1, int N2, int TK, bool INV, int NTH = TK * (N1 > N2 ? N1 : N2)>
__device__ __forceinline__ void tile_fft(double2 *buf, const double2 *__restrict__ tw) {
    constexpr int LD = TK + 1;
    static_assert(N2 == 1 || NTH >= TK * N2, "step 1 needs TK * N2 threads");
    const int tid = threadIdx.x;
    const int c = tid % TK;
    if constexpr (N2 == 1) {
        if (tid < TK) {
            double2 v[N1];
#pragma unroll
            for (int i = 0; i < N1; ++i) v[i] = buf[i * LD + c];
            fft_reg<N1, INV>(v);
#pragma unroll
            for (int i = 0; i < N1; ++i) buf[i * LD + c] = v[i];
        }
        __syncthreads();
    } else {
        double2 v[N1];
        const int n2 = tid / TK;
        const bool act1 = tid < TK * N2;
        if (act1) {
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) v[n1] = buf[(N2 * n1 + n2) * LD + c];
            fft_reg<N1, INV>(v);
#pragma unroll
            for (int k1 = 1; k1 < N1; ++k1) {
                if (n2 != 0) {
                    double2 w = __ldg(&tw[n2 * k1]);
                    if (INV) w.y = -w.y;
                    v[k1] = cmul(v[k1], w);
                }
            }
        }
        __syncthreads();
        if (act1) {
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) buf[(k1 * N2 + n2) * LD + c] = v[k1];
        }
        __syncthreads();
        // step 2: N1 columns of N2 points per line; with NTH < TK * N1
        // threads a thread takes columns k1, k1 + STR, ... (all read before
        // the barrier, written after it)
        constexpr int STR = NTH / TK;
        constexpr int NIT = (N1 + STR - 1) / STR;
        double2 u[NIT][N2];
        const int k1 = tid / TK;
        const bool act2 = tid < TK * STR;
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int kk = k1 + it * STR;
            if (act2 && kk < N1) {
#pragma unroll
                for (int j = 0; j < N2; ++j) u[it][j] = buf[(kk * N2 + j) * LD + c];
                fft_reg<N2, INV>(u[it]);
            }
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int kk = k1 + it * STR;
            if (act2 && kk < N1) {
#pragma unroll
                for (int k2 = 0; k2 < N2; ++k2) buf[(kk + N1 * k2) * LD + c] = u[it][k2];
            }
        }
        __syncthreads();
    }
}

// In-register radix-2 FFT with the direction a runtime argument (twiddle
// imaginary parts and the +-i rotations selected): one instantiation serves
// both directions, so the forward and inverse transforms of the plane pass's
// solve step share one register allocation (inlined compile-time pairs kept
// values of the first live into the second and spilled).
template <int R>
__device__ __forceinline__ void fft_reg_rt(double2 (&v)[R], bool inv) {
    if constexpr (R > 1) {
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int j = brev<R>(i);
            if (j > i) {
                double2 t = v[i];
                v[i] = v[j];
                v[j] = t;
            }
        }
#pragma unroll
        for (int half = 1; half < R; half <<= 1) {
#pragma unroll
            for (int i = 0; i < R; i += 2 * half) {
#pragma unroll
                for (int k = 0; k < half; ++k) {
                    const double2 a = v[i + k];
                    double2 b = v[i + k + half];
                    if (k != 0) {
                        if (2 * k == half) {
                            b = inv ? make_double2(-b.y, b.x) : make_double2(b.y, -b.x);
                        } else {
                            double2 w = c_w32[k * (16 / half)];
                            if (inv) w.y = -w.y;
                            b = cmul(b, w);
                        }
                    }
                    v[i + k] = cadd(a, b);
                    v[i + k + half] = csub(a, b);
                }
            }
        }
    }
}

// Stockham autosort FFT of TK lines held in shared memory (element n of
// line c at buf[n*LD + c]) with PPT points per thread: thread t serves line
// t % TK and butterfly column q = t / TK < N/PPT.  A pass of radix R
// (<= PPT) with NS = product of the earlier radices takes butterflies
// j = q + b*N/PPT (b < PPT/R): reads x[j + r N/R], multiplies by
// W_{NS R}^{(j mod NS) r}, transforms in registers and writes
// y[(j / NS) NS R + (j mod NS) + r NS]; the last pass leaves natural order.
// PPT = 8 (three passes at N = 256, 80 registers) or 16 (two passes: one
// shared-memory round trip and two barriers fewer per transform, 168
// registers, half the threads per tile; the plane pass default: 0.805 ->
// 0.714 ms at 256^3).
template <int N, int TK, int R, int NS, int PPT = 8, int LDX = TK + 1>
__device__ __forceinline__ void stockham_pass(double2 *buf, const double2 *__restrict__ tw, bool inv) {
    constexpr int LD = LDX, NB = PPT / R, JS = N / PPT;
    const int c = threadIdx.x % TK, q = threadIdx.x / TK;
    double2 v[NB][R];
    // MM_TW_PROD (R = 16, one butterfly per thread): the twiddles W^{jm r}
    // come from four table loads (r = 1, 2, 4, 8), issued before the
    // shared-memory reads, and at most three products (r = 3 .. 15) instead
    // of fifteen dependent-latency loads after the barrier
    constexpr bool TWP = MM_TW_PROD && R == 16 && NB == 1 && NS > 1;
    double2 wb[4];
    if constexpr (TWP) {
        const int jm = q & (NS - 1);
        constexpr int ST = N / (NS * R);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            wb[e] = __ldg(&tw[jm * (1 << e) * ST]);
            if (inv) wb[e].y = -wb[e].y;
        }
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[b][r] = buf[(q + b * JS + r * (N / R)) * LD + c];
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
        const int j = q + b * JS;
        const int jm = j & (NS - 1);
        if constexpr (TWP) {
            double2 w[16];
            w[1] = wb[0]; w[2] = wb[1]; w[4] = wb[2]; w[8] = wb[3];
            w[3] = cmul(w[1], w[2]);
            w[5] = cmul(w[1], w[4]);
            w[6] = cmul(w[2], w[4]);
            w[7] = cmul(w[3], w[4]);
#pragma unroll
            for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
#pragma unroll
            for (int r = 1; r < 16; ++r) v[b][r] = cmul(v[b][r], w[r]);
        } else if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = __ldg(&tw[jm * r * (N / (NS * R))]);
                if (inv) w.y = -w.y;
                v[b][r] = cmul(v[b][r], w);
            }
        }
        fft_reg_rt<R>(v[b], inv);
        const int base = (j - jm) * R + jm;
#pragma unroll
        for (int r = 0; r < R; ++r) buf[(base + r * NS) * LD + c] = v[b][r];
    }
    __syncthreads();
}

// radix plan: N = 8 * 8 * 4 (256), 8 * 4 * 4 (128), 8 * 8 (64), 8 * 4 (32), 4 * 4 (16)
template <int N, int TK, int PPT = 8, int LDX = TK + 1>
__device__ __forceinline__ void tile_fft_s(double2 *buf, const double2 *__restrict__ tw, bool inv) {
    static_assert(N >= 16 && N <= 256 && (N & (N - 1)) == 0, "N in 16..256, power of two");
    static_assert(PPT == 16 || LDX == TK + 1, "a dense (TMA) tile layout needs PPT = 16");
    if constexpr (PPT == 16) {
        // 16 points per thread: radix-16 first pass, then the remaining factor
        stockham_pass<N, TK, 16, 1, 16, LDX>(buf, tw, inv);
        if constexpr (N > 16) stockham_pass<N, TK, N / 16, 16, 16, LDX>(buf, tw, inv);
    } else if constexpr (N == 256) {
        stockham_pass<N, TK, 8, 1>(buf, tw, inv);
        stockham_pass<N, TK, 8, 8>(buf, tw, inv);
        stockham_pass<N, TK, 4, 64>(buf, tw, inv);
    } else if constexpr (N == 128) {
        stockham_pass<N, TK, 8, 1>(buf, tw, inv);
        stockham_pass<N, TK, 4, 8>(buf, tw, inv);
        stockham_pass<N, TK, 4, 32>(buf, tw, inv);
    } else if constexpr (N == 64) {
        stockham_pass<N, TK, 8, 1>(buf, tw, inv);
        stockham_pass<N, TK, 8, 8>(buf, tw, inv);
    } else if constexpr (N == 32) {
        stockham_pass<N, TK, 8, 1>(buf, tw, inv);
        stockham_pass<N, TK, 4, 8>(buf, tw, inv);
    } else {
        stockham_pass<N, TK, 4, 1>(buf, tw, inv);
        stockham_pass<N, TK, 4, 4>(buf, tw, inv);
    }
}

#ifndef MM_DFT_FALLBACK  // 1: the O(N^2) direct DFT for non-power-of-two lines (A/B)
#define MM_DFT_FALLBACK 0
#endif
// Exact DFT of TK lines of runtime length N (any N), via a scratch tile.
template <int TK, bool INV>
__device__ __forceinline__ void tile_dft(double2 *buf, double2 *scr, int N,
                                         const double2 *__restrict__ tw) {
    constexpr int LD = TK + 1;
    for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
        const int k = w / TK, c = w % TK;
        double2 s = make_double2(0.0, 0.0);
        int idx = 0;
        for (int n = 0; n < N; ++n) {
            double2 t = tw[idx];
            if (INV) t.y = -t.y;
            s = cadd(s, cmul(buf[n * LD + c], t));
            idx += k;
            if (idx >= N) idx -= N;
        }
        scr[k * LD + c] = s;
    }
    __syncthreads();
    for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
        const int k = w / TK, c = w % TK;
        buf[k * LD + c] = scr[k * LD + c];
    }
    __syncthreads();
}

// Mixed-radix Stockham FFT of TK lines of runtime length N (any N): one pass
// per factor of N (4, 2, 3, 5, then any remaining prime), ping-pong between
// buf and scr, result in buf.  Pass with radix R after the radices NS:
// butterfly j < N/R of line c reads x[j + r N/R], twiddles by
// W_{NS R}^{(j mod NS) r} (the length-N table: index (j mod NS) r N/(NS R)),
// takes the R-point DFT and writes y[(j - j mod NS) R + j mod NS + r NS].
// O(N sum of factors) instead of the O(N^2) direct DFT for the grids
// pocketfft serves in the reference (grid.py:195-220: any n, e.g. the
// 640 / 800 weak-scaling sizes of SURVEY 8(d) config 5).
__device__ __forceinline__ int next_radix(int rem) {
    if (rem % 4 == 0) return 4;
    if (rem % 2 == 0) return 2;
    if (rem % 3 == 0) return 3;
    if (rem % 5 == 0) return 5;
    for (int p = 7; p * p <= rem; p += 2)
        if (rem % p == 0) return p;
    return rem;
}

template <int TK, bool INV>
__device__ __noinline__ void tile_fft_mixed(double2 *buf, double2 *scr, int N,
                                            const double2 *__restrict__ tw) {
    constexpr int LD = TK + 1;
    double2 *src = buf, *dst = scr;
    int NS = 1;
    for (int rem = N; rem > 1;) {
        const int R = next_radix(rem);
        const int nb = N / R, tws = N / (NS * R), rs = N / R;
        for (int w = threadIdx.x; w < nb * TK; w += blockDim.x) {
            const int j = w / TK, c = w - j * TK;
            const int jm = j % NS;
            const int base = (j - jm) * R + jm;
            if (R == 2 || R == 4) {
                double2 v[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    if (r >= R) break;
                    v[r] = src[(j + r * nb) * LD + c];
                    if (r > 0 && NS > 1) {
                        double2 t = __ldg(&tw[jm * r * tws]);
                        if (INV) t.y = -t.y;
                        v[r] = cmul(v[r], t);
                    }
                }
                if (R == 2) {
                    dst[base * LD + c] = cadd(v[0], v[1]);
                    dst[(base + NS) * LD + c] = csub(v[0], v[1]);
                } else {
                    const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
                    const double2 b0 = cadd(v[1], v[3]), b1 = csub(v[1], v[3]);
                    // forward: x (-i); inverse: x (+i)
                    const double2 b1r = INV ? make_double2(-b1.y, b1.x) : make_double2(b1.y, -b1.x);
                    dst[base * LD + c] = cadd(a0, b0);
                    dst[(base + NS) * LD + c] = cadd(a1, b1r);
                    dst[(base + 2 * NS) * LD + c] = csub(a0, b0);
                    dst[(base + 3 * NS) * LD + c] = csub(a1, b1r);
                }
            } else {
                // generic R-point DFT (R odd prime); W_R^k = tw[k N / R]
                for (int sidx = 0; sidx < R; ++sidx) {
                    double2 acc = make_double2(0.0, 0.0);
                    int k = 0;  // (r * sidx) mod R
                    for (int r = 0; r < R; ++r) {
                        double2 v = src[(j + r * nb) * LD + c];
                        if (r > 0 && NS > 1) {
                            double2 t = __ldg(&tw[jm * r * tws]);
                            if (INV) t.y = -t.y;
                            v = cmul(v, t);
                        }
                        double2 wr = __ldg(&tw[k * rs]);
                        if (INV) wr.y = -wr.y;
                        acc = cadd(acc, cmul(v, wr));
                        k += sidx;
                        if (k >= R) k -= R;
                    }
                    dst[(base + sidx * NS) * LD + c] = acc;
                }
            }
        }
        __syncthreads();
        double2 *t = src;
        src = dst;
        dst = t;
        NS *= R;
        rem /= R;
    }
    if (src != buf) {
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int k = w / TK, c = w % TK;
            buf[k * LD + c] = src[k * LD + c];
        }
        __syncthreads();
    }
}

template <int N1, int N2, int TK, bool INV, int NTH = TK * (N1 > N2 ? N1 : N2)>
__device__ __forceinline__ void line_transform(double2 *buf, double2 *scr, int N,
                                               const double2 *__restrict__ tw) {
    if constexpr (N1 == 0) {
        if (MM_DFT_FALLBACK)
            tile_dft<TK, INV>(buf, scr, N, tw);
        else
            tile_fft_mixed<TK, INV>(buf, scr, N, tw);
    } else {
        tile_fft<N1, N2, TK, INV, NTH>(buf, tw);
    }
}

struct RowGeom {
    int n;          // points per axis
    int dim;
    int64_t M;      // points
    int64_t nrows;  // M / n
    int P;          // spectral pitch
    int N;          // complex line length (n/2 packed, or n when odd)
    int packed;     // 1: two reals per complex (even n)
    // slab mode (3D): nl local planes; T_c0 of the plane below the first /
    // above the last local plane come from neighbour ranks ([c][i1*n + x]).
    int nl;
    const double *hlo, *hhi;
    int64_t uM;     // component stride of the real rows written by the inverse pass
    // spectrum layout: 0 = rows ((c*nrows + row)*P + k); 1 = planes
    // ((c*nh + k)*nrows + row), every (c, k) an n x n plane [i0][i1] (k_plane)
    int plane;
};

// ---------------------------------------------------------------------------
// A: divergence of T = F - lam/rho fused with the R2C transform of each row
// ---------------------------------------------------------------------------
__device__ __forceinline__ double tval(const double *__restrict__ F, const double *__restrict__ L,
                                       int64_t off, double rho) {
    if (!L) return __ldg(&F[off]);                  // F holds T already
    return __ldg(&F[off]) - __ldg(&L[off]) / rho;  // projection.py:154 (F - lam / rho)
}

// start offsets (row * n) of a row and of its neighbour rows along axes 0, 1
struct RowNbr {
    int64_t self, zp, zm, yp, ym;
    bool zp_h, zm_h;  // axis-0 neighbour lives in the halo plane (slab mode)
    int hoff;         // offset of this row inside a halo plane
};

__device__ __forceinline__ RowNbr row_nbrs(const RowGeom &g, int row) {
    const int n = g.n;
    RowNbr r;
    r.zp_h = r.zm_h = false;
    r.hoff = 0;
    if (g.dim == 3) {
        const int i0 = row / n, i1 = row - i0 * n;
        const int nl = g.nl;
        int i0p = (i0 + 1 == nl) ? 0 : i0 + 1, i0m = (i0 == 0) ? nl - 1 : i0 - 1;
        if (g.hhi) {  // slab: neighbours across the slab faces come from halos
            r.zp_h = (i0 + 1 == nl);
            r.zm_h = (i0 == 0);
            if (r.zp_h) i0p = i0;
            if (r.zm_h) i0m = i0;
            r.hoff = i1 * n;
        }
        const int i1p = (i1 + 1 == n) ? 0 : i1 + 1, i1m = (i1 == 0) ? n - 1 : i1 - 1;
        r.zp = (int64_t)(i0p * n + i1) * n;
        r.zm = (int64_t)(i0m * n + i1) * n;
        r.yp = (int64_t)(i0 * n + i1p) * n;
        r.ym = (int64_t)(i0 * n + i1m) * n;
    } else {
        const int rp = (row + 1 == n) ? 0 : row + 1, rm = (row == 0) ? n - 1 : row - 1;
        r.zp = (int64_t)rp * n;
        r.zm = (int64_t)rm * n;
        r.yp = r.ym = 0;
    }
    r.self = (int64_t)row * n;
    return r;
}

// unscaled divergence sum_j [T_cj(x+e_j) - T_cj(x-e_j)] at point x of a row
__device__ __forceinline__ double div_at(const double *__restrict__ F, const double *__restrict__ L,
                                         double rho, const RowGeom &g, int c, const RowNbr &nb,
                                         int x) {
    const int n = g.n;
    const int64_t M = g.M;
    const int d = g.dim;
    double s;
    {  // axis 0 (slowest)
        const int64_t comp = (int64_t)(c * d + 0) * M + x;
        s = tval(F, L, comp + nb.zp, rho) - tval(F, L, comp + nb.zm, rho);
    }
    if (d == 3) {  // axis 1
        const int64_t comp = (int64_t)(c * d + 1) * M + x;
        s += tval(F, L, comp + nb.yp, rho) - tval(F, L, comp + nb.ym, rho);
    }
    {  // contiguous axis
        const int64_t comp = (int64_t)(c * d + d - 1) * M + nb.self;
        const int xp = (x + 1 == n) ? 0 : x + 1, xm = (x == 0) ? n - 1 : x - 1;
        s += tval(F, L, comp + xp, rho) - tval(F, L, comp + xm, rho);
    }
    return s;
}

template <int N1, int N2, int DIM, int ROWS>
struct RowCfg {
    static constexpr int TK = DIM * ROWS;  // lines per tile (component x row)
    static constexpr int NT0 = N1 ? TK * (N1 > N2 ? N1 : N2) : 256;
    static constexpr int NT = NT0 < 64 ? 64 : NT0;
    // inverse (C2R) kernels with MM_ROWINV_BAL: TK * N2 threads, every thread
    // busy in both steps of the four-step (two step-2 columns each)
    static constexpr int NTI0 = (N1 && MM_ROWINV_BAL && N2 > 1) ? TK * N2 : NT0;
    static constexpr int NTI = NTI0 < 64 ? 64 : NTI0;
    static constexpr int MINB0 = 65536 / (NT * MM_ROWFWD_REGS);
    static constexpr int MINB = MINB0 < 1 ? 1 : MINB0;  // aim at <= 96 registers
    // the C2R pass: a register budget of 80 (4 tiles per SM) spilled 364 B
    // per thread in the persistent kernel; 128 (2 tiles, 164 registers used,
    // no spills) runs it in 0.22 instead of 0.32 ms
    static constexpr int MINB_INV0 = 65536 / (NTI * MM_ROWINV_REGS);
    static constexpr int MINB_INV = MINB_INV0 < 1 ? 1 : MINB_INV0;
    static constexpr int NC = N1 * N2;                  // compile-time line length (0: runtime)
};

// A tile holds ROWS consecutive rows x DIM components; line = c * ROWS + r.
// HAS_L = false: F already holds T = F - lam/rho (written by the fused
// update + local pass) and is differentiated as is; half the loads.
template <int N1, int N2, int DIM, int ROWS, bool HAS_L = true>
__global__ void __launch_bounds__(RowCfg<N1, N2, DIM, ROWS>::NT, RowCfg<N1, N2, DIM, ROWS>::MINB)
k_row_fwd(const double *__restrict__ F, const double *__restrict__ L, double rho,
          double2 *__restrict__ spec, RowGeom g, const double2 *__restrict__ tw_line,
          const double2 *__restrict__ tw_r2c) {
    using C = RowCfg<N1, N2, DIM, ROWS>;
    constexpr int TK = C::TK, LD = TK + 1;
    extern __shared__ double2 smem_c[];
    double2 *buf = smem_c;
    const int N = C::NC ? C::NC : g.N;  // compile-time for power-of-two lines
    const bool packed = C::NC ? true : (g.packed != 0);
    double2 *scr = smem_c + (size_t)(N + 1) * LD;
    const int64_t row0 = (int64_t)blockIdx.x * ROWS;
    const int64_t M = g.M;
    const double irho = 1.0 / rho;
    // pack: a work item (row r, complex slot m) produces the slot of every
    // component; all loads of a component are issued before its arithmetic
    if (packed) {
        for (int w = threadIdx.x; w < ROWS * N; w += C::NT) {
            const int r = w / N, m = w - r * N;
            const int64_t row = row0 + r;
            if (row >= g.nrows) {
#pragma unroll
                for (int c = 0; c < DIM; ++c) buf[m * LD + c * ROWS + r] = make_double2(0.0, 0.0);
                continue;
            }
            const RowNbr nb = row_nbrs(g, (int)row);
            const int n = g.n;
            const int x0 = 2 * m, x1 = 2 * m + 1;
            const int xm = (x0 == 0) ? n - 1 : x0 - 1;
            const int xp = (x1 + 1 == n) ? 0 : x1 + 1;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                const int64_t cz = (int64_t)(c * DIM) * M;                  // T_c0 (axis 0)
                const int64_t cy = (int64_t)(c * DIM + 1) * M;              // T_c1 (axis 1, 3D)
                const int64_t cx = (int64_t)(c * DIM + DIM - 1) * M + nb.self;  // contiguous
                const double fxm = __ldg(&F[cx + xm]), lxm = HAS_L ? __ldg(&L[cx + xm]) : 0.0;
                const double fx0 = __ldg(&F[cx + x0]), lx0 = HAS_L ? __ldg(&L[cx + x0]) : 0.0;
                const double fx1 = __ldg(&F[cx + x1]), lx1 = HAS_L ? __ldg(&L[cx + x1]) : 0.0;
                const double fxp = __ldg(&F[cx + xp]), lxp = HAS_L ? __ldg(&L[cx + xp]) : 0.0;
                const double fzp0 = __ldg(&F[cz + nb.zp + x0]), lzp0 = HAS_L ? __ldg(&L[cz + nb.zp + x0]) : 0.0;
                const double fzp1 = __ldg(&F[cz + nb.zp + x1]), lzp1 = HAS_L ? __ldg(&L[cz + nb.zp + x1]) : 0.0;
                const double fzm0 = __ldg(&F[cz + nb.zm + x0]), lzm0 = HAS_L ? __ldg(&L[cz + nb.zm + x0]) : 0.0;
                const double fzm1 = __ldg(&F[cz + nb.zm + x1]), lzm1 = HAS_L ? __ldg(&L[cz + nb.zm + x1]) : 0.0;
                double y0 = 0.0, y1 = 0.0;
                if (DIM == 3) {
                    const double fyp0 = __ldg(&F[cy + nb.yp + x0]), lyp0 = HAS_L ? __ldg(&L[cy + nb.yp + x0]) : 0.0;
                    const double fyp1 = __ldg(&F[cy + nb.yp + x1]), lyp1 = HAS_L ? __ldg(&L[cy + nb.yp + x1]) : 0.0;
                    const double fym0 = __ldg(&F[cy + nb.ym + x0]), lym0 = HAS_L ? __ldg(&L[cy + nb.ym + x0]) : 0.0;
                    const double fym1 = __ldg(&F[cy + nb.ym + x1]), lym1 = HAS_L ? __ldg(&L[cy + nb.ym + x1]) : 0.0;
                    y0 = (fyp0 - lyp0 * irho) - (fym0 - lym0 * irho);
                    y1 = (fyp1 - lyp1 * irho) - (fym1 - lym1 * irho);
                }
                // T = F - lam/rho (projection.py:154), as F - lam * (1/rho)
                double tzp0 = fzp0 - lzp0 * irho, tzp1 = fzp1 - lzp1 * irho;
                double tzm0 = fzm0 - lzm0 * irho, tzm1 = fzm1 - lzm1 * irho;
                if (DIM == 3 && (nb.zp_h || nb.zm_h)) {
                    const int64_t hp = (int64_t)c * n * n + nb.hoff;
                    if (nb.zp_h) {
                        tzp0 = g.hhi[hp + x0];
                        tzp1 = g.hhi[hp + x1];
                    }
                    if (nb.zm_h) {
                        tzm0 = g.hlo[hp + x0];
                        tzm1 = g.hlo[hp + x1];
                    }
                }
                double2 z;
                z.x = (tzp0 - tzm0) + y0 + ((fx1 - lx1 * irho) - (fxm - lxm * irho));
                z.y = (tzp1 - tzm1) + y1 + ((fxp - lxp * irho) - (fx0 - lx0 * irho));
                buf[m * LD + c * ROWS + r] = z;
            }
        }
    } else {
        for (int w = threadIdx.x; w < TK * N; w += C::NT) {
            const int line = w / N, m = w - line * N;
            const int c = line / ROWS, r = line - c * ROWS;
            const int64_t row = row0 + r;
            double2 z = make_double2(0.0, 0.0);
            if (row < g.nrows)
                z.x = div_at(F, HAS_L ? L : nullptr, rho, g, c, row_nbrs(g, (int)row), m);
            buf[m * LD + line] = z;
        }
    }
    __syncthreads();
    line_transform<N1, N2, TK, false, C::NT>(buf, scr, N, tw_line);
    // split (packed) and store k = 0 .. n/2
    const int nh = packed ? N + 1 : g.n / 2 + 1;
    for (int w = threadIdx.x; w < TK * nh; w += C::NT) {
        // plane layout: consecutive threads take consecutive rows of one
        // (c, k) (ROWS x 16 B runs); row layout: consecutive k of one row
        int line, k;
        if (g.plane) {
            const int r0 = w % ROWS, t = w / ROWS;
            k = t % nh;
            line = (t / nh) * ROWS + r0;
        } else {
            line = w / nh;
            k = w - line * nh;
        }
        const int c = line / ROWS, r = line - c * ROWS;
        const int64_t row = row0 + r;
        if (row >= g.nrows) continue;
        double2 X;
        if (packed) {
            const double2 Zk = buf[(k == N ? 0 : k) * LD + line];
            const double2 Zc = cconj(buf[(k == 0 ? 0 : N - k) * LD + line]);
            const double2 E = cscale(cadd(Zk, Zc), 0.5);
            const double2 Od = csub(Zk, Zc);  // 2i * O
            // X = E + W^k * Od / (2i) = E - 0.5 i W^k Od
            const double2 WO = cmul(__ldg(&tw_r2c[k]), Od);
            X = make_double2(E.x + 0.5 * WO.y, E.y - 0.5 * WO.x);
        } else {
            X = buf[k * LD + line];
        }
        if (g.plane)
            spec[((int64_t)c * nh + k) * g.nrows + row] = X;
        else
            spec[((int64_t)c * g.nrows + row) * g.P + k] = X;
    }
}

__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc, int src_bytes) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gsrc),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND));
}

// A for n = 256 (3D, T field, single GPU): one warp per task of 4
// consecutive rows x one component, 8 lanes per row, no block barrier.  Lane
// q of a row holds slots m = q + 8 s (s < 16) of the packed row
// z[m] = d[2m] + i d[2m+1]: its loads are 128-byte row segments (T_c2 of the
// row, T_c0 of the axis-0 neighbour rows, T_c1 of the axis-1 neighbour
// rows), the stencil arithmetic is k_row_fwd's, and the 128-point transform
// is tile_fft<16, 8>'s four-step in the same order (16-point FFTs over s,
// twiddles W^{q k1}, an XOR-swizzled exchange through the warp's own shared
// memory, 8-point FFTs), so the spectrum is k_row_fwd's.  The split and the
// stores read the natural-order row back from shared memory: 64-byte runs
// (4 rows of one (c, k)) in the plane layout, 128-byte runs in the row
// layout.
constexpr int RFW_WARPS = 4;
__global__ void __launch_bounds__(32 * RFW_WARPS, MM_ROWFWD_W_MINB)
k_row_fwd_w(const double *__restrict__ T, double2 *__restrict__ spec, RowGeom g,
            const double2 *__restrict__ tw, const double2 *__restrict__ tw_r2c) {
    constexpr int n = 256, N = 128, nh = 129;
    __shared__ double2 sm[RFW_WARPS][4][N];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t task = (int64_t)blockIdx.x * RFW_WARPS + warp;
    if (task >= 3 * (g.nrows / 4)) return;
    const int c = (int)(task % 3);
    const int64_t row0 = (task / 3) * 4;
    const int j = lane >> 3, q = lane & 7;
    const int64_t row = row0 + j;
    const int64_t M = g.M;
    const RowNbr nb = row_nbrs(g, (int)row);
    const double *Tz = T + (int64_t)(c * 3) * M;
    const double *Ty = T + (int64_t)(c * 3 + 1) * M;
    const double *Tx = T + (int64_t)(c * 3 + 2) * M + nb.self;
    double2 v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int m = q + 8 * s;
        const int x0 = 2 * m;
        const int xm = (x0 == 0) ? n - 1 : x0 - 1;
        const int xp = (x0 + 2 == n) ? 0 : x0 + 2;
        const double2 fx = __ldg(reinterpret_cast<const double2 *>(Tx + x0));
        const double fxm = __ldg(Tx + xm), fxp = __ldg(Tx + xp);
        const double2 zp = __ldg(reinterpret_cast<const double2 *>(Tz + nb.zp + x0));
        const double2 zm = __ldg(reinterpret_cast<const double2 *>(Tz + nb.zm + x0));
        const double2 yp = __ldg(reinterpret_cast<const double2 *>(Ty + nb.yp + x0));
        const double2 ym = __ldg(reinterpret_cast<const double2 *>(Ty + nb.ym + x0));
        const double y0 = yp.x - ym.x, y1 = yp.y - ym.y;
        v[s].x = (zp.x - zm.x) + y0 + (fx.y - fxm);
        v[s].y = (zp.y - zm.y) + y1 + (fxp - fx.x);
        if ((s & 3) == 3) asm volatile("" ::: "memory");  // loads in batches of 4 slots
    }
    // step 1 (tile_fft<16, 8>): n2 = q, 16 points x[8 n1 + q]
    fft_reg<16, false>(v);
    if (q != 0) {
#if MM_RFW_TWP
        double2 w[16];  // W^{q k1} from four loads and products (MM_TW_PROD's scheme)
        w[1] = __ldg(&tw[q]);
        w[2] = __ldg(&tw[2 * q]);
        w[4] = __ldg(&tw[4 * q]);
        w[8] = __ldg(&tw[8 * q]);
        w[3] = cmul(w[1], w[2]);
        w[5] = cmul(w[1], w[4]);
        w[6] = cmul(w[2], w[4]);
        w[7] = cmul(w[3], w[4]);
#pragma unroll
        for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
#pragma unroll
        for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], w[k1]);
#else
#pragma unroll
        for (int k1 = 1; k1 < 16; ++k1) v[k1] = cmul(v[k1], __ldg(&tw[q * k1]));
#endif
    }
    double2 *L = sm[warp][j];
    // element (k1, n2) of the exchange at k1 * 8 + (n2 ^ (k1 & 7))
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) L[k1 * 8 + (q ^ (k1 & 7))] = v[k1];
    __syncwarp();
    // step 2: columns k1 = q and q + 8, 8 points each -> X[k1 + 16 k2]
    double2 u[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int k1 = q + 8 * h;
#pragma unroll
        for (int t = 0; t < 8; ++t) u[h][t] = L[k1 * 8 + (t ^ (k1 & 7))];
        fft_reg<8, false>(u[h]);
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) L[q + 8 * h + 16 * k2] = u[h][k2];
    __syncwarp();
    // split (k_row_fwd's expression) and store
    const double2 *W = sm[warp][0];
    const int rj = g.plane ? (lane & 3) : (lane >> 3);
    const int kk = g.plane ? (lane >> 2) : (lane & 7);
    const int kst = g.plane ? 8 : 8;
    const double2 *Lr = W + rj * N;
    const int64_t orow = row0 + rj;
#pragma unroll 3
    for (int k = kk; k < nh; k += kst) {
        const double2 Zk = Lr[k == N ? 0 : k];
        const double2 Zc = cconj(Lr[k == 0 ? 0 : N - k]);
        const double2 E = cscale(cadd(Zk, Zc), 0.5);
        const double2 Od = csub(Zk, Zc);
        const double2 WO = cmul(__ldg(&tw_r2c[k]), Od);
        const double2 X = make_double2(E.x + 0.5 * WO.y, E.y - 0.5 * WO.x);
        if (g.plane)
            spec[((int64_t)c * nh + k) * g.nrows + orow] = X;
        else
            spec[((int64_t)c * g.nrows + orow) * g.P + k] = X;
    }
}

// ---------------------------------------------------------------------------
// E: inverse C2R along rows -> u_tilde (unnormalised; 1/n^d folded into C)
// ---------------------------------------------------------------------------
// everything after a tile's spectrum is in buf: Hermitian pair packing,
// inverse line transform, real rows out (k_row_inv and k_row_inv_p)
template <int N1, int N2, int DIM, int ROWS>
__device__ __forceinline__ void row_inv_tile(double2 *buf, double2 *scr, double *__restrict__ Ut,
                                             const RowGeom &g, int64_t row0, int N, bool packed,
                                             const double2 *__restrict__ tw_line,
                                             const double2 *__restrict__ tw_r2c) {
    using C = RowCfg<N1, N2, DIM, ROWS>;
    constexpr int TK = C::TK, LD = TK + 1;
    const int nh = packed ? N + 1 : g.n / 2 + 1;
    if (packed) {
        // Z[k] = A[k] + i B[k], A = X[k] + conj X[N-k], B = (X[k] - conj X[N-k]) conj(W^k)
        const int npair = N / 2 + 1;
        for (int w = threadIdx.x; w < TK * npair; w += C::NTI) {
            const int line = w / npair, k = w - line * npair;
            const int kc = N - k;
            const double2 Xk = buf[k * LD + line];
            const double2 Xc = buf[kc * LD + line];
            const double2 A1 = cadd(Xk, cconj(Xc));
            const double2 B1 = cmul(csub(Xk, cconj(Xc)), cconj(__ldg(&tw_r2c[k])));
            const double2 Z1 = make_double2(A1.x - B1.y, A1.y + B1.x);
            if (kc != k && kc != N) {
                const double2 A2 = cadd(Xc, cconj(Xk));
                const double2 B2 = cmul(csub(Xc, cconj(Xk)), cconj(__ldg(&tw_r2c[kc])));
                buf[kc * LD + line] = make_double2(A2.x - B2.y, A2.y + B2.x);
            }
            buf[k * LD + line] = Z1;  // k == 0 also overwrites slot 0; slot N unused
        }
    } else {
        // odd n: full Hermitian spectrum
        for (int w = threadIdx.x; w < TK * (N - nh); w += C::NTI) {
            const int line = w / (N - nh), k = nh + (w - line * (N - nh));
            buf[k * LD + line] = cconj(buf[(N - k) * LD + line]);
        }
    }
    __syncthreads();
    line_transform<N1, N2, TK, true, C::NTI>(buf, scr, N, tw_line);
    // store: a work item (row r, slot m) writes every component of the slot
    for (int w = threadIdx.x; w < ROWS * N; w += C::NTI) {
        const int r = w / N, m = w - r * N;
        const int64_t row = row0 + r;
        if (row >= g.nrows) continue;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const double2 z = buf[m * LD + c * ROWS + r];
            double *dst = Ut + (int64_t)c * g.uM + row * g.n;
            if (packed) {
                *reinterpret_cast<double2 *>(dst + 2 * m) = z;
            } else {
                dst[m] = z.x;
            }
        }
    }
}

template <int N1, int N2, int DIM, int ROWS>
__global__ void __launch_bounds__(RowCfg<N1, N2, DIM, ROWS>::NTI, RowCfg<N1, N2, DIM, ROWS>::MINB_INV)
k_row_inv(const double2 *__restrict__ spec, double *__restrict__ Ut, RowGeom g,
          const double2 *__restrict__ tw_line, const double2 *__restrict__ tw_r2c) {
    using C = RowCfg<N1, N2, DIM, ROWS>;
    constexpr int TK = C::TK, LD = TK + 1;
    extern __shared__ double2 smem_c[];
    double2 *buf = smem_c;
    const int N = C::NC ? C::NC : g.N;
    const bool packed = C::NC ? true : (g.packed != 0);
    double2 *scr = smem_c + (size_t)(N + 1) * LD;
    const int64_t row0 = (int64_t)blockIdx.x * ROWS;
    const int nh = packed ? N + 1 : g.n / 2 + 1;
    for (int w = threadIdx.x; w < TK * nh; w += C::NTI) {
        int line, k;
        if (g.plane) {
            const int r0 = w % ROWS, t = w / ROWS;
            k = t % nh;
            line = (t / nh) * ROWS + r0;
        } else {
            line = w / nh;
            k = w - line * nh;
        }
        const int c = line / ROWS, r = line - c * ROWS;
        const int64_t row = row0 + r;
        double2 X = make_double2(0.0, 0.0);
        if (row < g.nrows)
            X = g.plane ? spec[((int64_t)c * nh + k) * g.nrows + row]
                        : spec[((int64_t)c * g.nrows + row) * g.P + k];
        buf[k * LD + line] = X;
    }
    __syncthreads();
    row_inv_tile<N1, N2, DIM, ROWS>(buf, scr, Ut, g, row0, N, packed, tw_line, tw_r2c);
}

// ---------------------------------------------------------------------------
// B/C/D: column transforms on the half spectrum (TK contiguous columns / tile)
// ---------------------------------------------------------------------------
struct ColGeom {
    int N;             // line length (= n)
    int ncol;          // valid columns (n/2 + 1)
    int64_t es;        // element stride along the line (complex units)
    int64_t os;        // outer stride
    int64_t cs;        // component stride
    // solve (MODE 2) and norm (MODE 3)
    int n, dim;
    const double *sym;
    double thresh, scale;
    // norm (MODE 3): deterministic block partials
    double *partials, *red_out;
    unsigned int *count;
};

// COL_NORM: forward FFT along the line, then sum over the tile of
// m(k2) |X|^2 / |g|^2 on live modes, m = 1 on the k2 = 0 and Nyquist columns
// of the half spectrum and 2 elsewhere (the full-spectrum sum of a real
// field's transform; equilibrium_residual, solver.py:364-371)
enum { COL_FWD = 0, COL_INV = 1, COL_SOLVE = 2, COL_NORM = 3 };

// resident CTAs of the persistent column kernel (TK + 1 = 9 column pitch)
// that shared memory admits, at most 3
constexpr int colp_minb(int smem_bytes) {
    return (227 * 1024) / (smem_bytes + 1024) >= 3 ? 3
           : (227 * 1024) / (smem_bytes + 1024) < 1 ? 1
                                                     : (227 * 1024) / (smem_bytes + 1024);
}
template <int N1, int N2>
struct ColCfg {
    static constexpr int TK = 8;
    static constexpr int NT = N1 ? (TK * (N1 > N2 ? N1 : N2) < 64 ? 64 : TK * (N1 > N2 ? N1 : N2))
                                 : 256;
    // resident blocks per SM requested from the register allocator
    static constexpr int MINB = N1 ? (NT <= 128 ? 5 : (N1 >= 32 ? MM_COL32_MINB : 2)) : 1;
};

#ifndef COL_SOLVE_MINB
#define COL_SOLVE_MINB 6
#endif
template <int N1, int N2, int MODE>
__global__ void __launch_bounds__(ColCfg<N1, N2>::NT,
                                  (MODE == COL_SOLVE && N1 == 16 && N2 == 16) ? COL_SOLVE_MINB
                                                                              : ColCfg<N1, N2>::MINB)
k_col(double2 *__restrict__ spec, ColGeom g, const double2 *__restrict__ tw) {
    constexpr int TK = ColCfg<N1, N2>::TK, LD = TK + 1, NT = ColCfg<N1, N2>::NT;
    extern __shared__ double2 smem_c[];
    double2 *buf = smem_c;
    double2 *scr = smem_c + (size_t)g.N * LD;
    const int k0 = blockIdx.x * TK;
    const int outer = blockIdx.y;
    const int comp = blockIdx.z;
    double2 *base = spec + comp * g.cs + outer * g.os + k0;
    const int N = g.N;
    const bool full = k0 + TK <= g.ncol;
    if constexpr (N1 != 0) {
        // compile-time trip count: all loads of the tile are in flight at once
        constexpr int NN = N1 * N2;
        constexpr int IT = (NN * TK + NT - 1) / NT;
        double2 v[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + threadIdx.x;
            const int n = w / TK, c = w % TK;
            v[it] = (w < NN * TK && (full || k0 + c < g.ncol)) ? base[n * g.es + c]
                                                               : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + threadIdx.x;
            if (w < NN * TK) buf[(w / TK) * LD + (w % TK)] = v[it];
        }
    } else {
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int n = w / TK, c = w - n * TK;
            double2 v = make_double2(0.0, 0.0);
            if (k0 + c < g.ncol) v = base[n * g.es + c];
            buf[n * LD + c] = v;
        }
    }
    __syncthreads();
    if constexpr (MODE == COL_FWD || MODE == COL_SOLVE || MODE == COL_NORM)
        line_transform<N1, N2, TK, false>(buf, scr, N, tw);
    else
        line_transform<N1, N2, TK, true>(buf, scr, N, tw);
    if constexpr (MODE == COL_NORM) {
        __shared__ double red_sm[32];
        const double *s0 = g.sym;
        const double *slast = g.sym + (int64_t)(g.dim - 1) * g.n;
        const double s1 = (g.dim == 3) ? g.sym[g.n + outer] : 0.0;
        const int nyq = (g.n % 2 == 0) ? g.n / 2 : -1;
        double acc[1] = {0.0};
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int kl = w / TK, c = w - kl * TK;
            const int k2 = k0 + c;
            if (k2 >= g.ncol) continue;
            double gsq = s0[kl];
            if (g.dim == 3) gsq = gsq + s1;
            gsq = gsq + slast[k2];
            if (!(gsq > g.thresh)) continue;
            const double2 X = buf[kl * LD + c];
            const double m = (k2 == 0 || k2 == nyq) ? 1.0 : 2.0;
            acc[0] += m * (X.x * X.x + X.y * X.y) / gsq;
        }
        const int ops[1] = {RED_SUM};
        block_reduce<1>(acc, ops, red_sm);
        grid_finalize<1>(acc, ops, g.partials, g.red_out, g.count, red_sm);
        return;
    }
    if constexpr (MODE == COL_SOLVE) {
        // u_hat = -d_hat / |g|^2 on live modes (projection.py:150-158); the
        // column is the last-axis frequency, `outer` the axis-1 one in 3D
        const double *s0 = g.sym;
        const double *slast = g.sym + (int64_t)(g.dim - 1) * g.n;
        const double s1 = (g.dim == 3) ? g.sym[g.n + outer] : 0.0;
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int kl = w / TK, c = w - kl * TK;
            double gsq = s0[kl];
            if (g.dim == 3) gsq = gsq + s1;
            gsq = gsq + slast[min(k0 + c, g.n - 1)];
            const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
            buf[kl * LD + c] = cscale(buf[kl * LD + c], -inv * g.scale);
        }
        __syncthreads();
        line_transform<N1, N2, TK, true>(buf, scr, N, tw);
    }
    if constexpr (N1 != 0) {
        constexpr int NN = N1 * N2;
        constexpr int IT = (NN * TK + NT - 1) / NT;
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + threadIdx.x;
            const int n = w / TK, c = w % TK;
            if (w < NN * TK && (full || k0 + c < g.ncol)) base[n * g.es + c] = buf[n * LD + c];
        }
    } else {
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int n = w / TK, c = w - n * TK;
            if (k0 + c < g.ncol) base[n * g.es + c] = buf[n * LD + c];
        }
    }
}

// Persistent, software-pipelined variant for power-of-two lines: each block
// walks tiles t = blockIdx.x, +gridDim.x, ...; while it transforms tile t in
// one shared buffer, the cp.async (LDGSTS) copies of tile t+gridDim.x land in
// the other, so global loads are always in flight (the plain variant above is
// load-latency bound: ncu long_scoreboard stalls dominate).

struct TileMap {
    int ntk, n_outer;  // column tiles per line set, outer lines
};

template <int N1, int N2, int MODE>
// persistent column kernel: two tile buffers; the register allocator is asked
// for no more resident CTAs than shared memory admits (at N = 512 one: a
// request for 3 capped it at 80 registers and spilled 1.8 KB per thread;
// col_fwd / col_inv at 512^3 5.2 / 5.0 -> 2.8 / 2.6 ms)
__global__ void __launch_bounds__(ColCfg<N1, N2>::NT, colp_minb(2 * N1 * N2 * 9 * 16))
k_colp(double2 *__restrict__ spec, ColGeom g, const double2 *__restrict__ tw, TileMap tm,
       int ntiles) {
    using C = ColCfg<N1, N2>;
    constexpr int TK = C::TK, LD = TK + 1, NT = C::NT, N = N1 * N2;
    constexpr int IT = (N * TK + NT - 1) / NT;
    extern __shared__ double2 smem_c[];
    auto tile_base = [&](int t, int &k0, int &outer) -> double2 * {
        const int tk = t % tm.ntk;
        const int rest = t / tm.ntk;
        outer = rest % tm.n_outer;
        const int comp = rest / tm.n_outer;
        k0 = tk * TK;
        return spec + comp * g.cs + outer * g.os + k0;
    };
    auto issue = [&](int t, double2 *dst) {
        int k0, outer;
        const double2 *base = tile_base(t, k0, outer);
#pragma unroll 2
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + threadIdx.x;
            if (w < N * TK) {
                const int n = w / TK, c = w % TK;
                const bool ok = k0 + c < g.ncol;
                cp_async16(&dst[n * LD + c], ok ? (const void *)&base[n * g.es + c] : (const void *)base,
                           ok ? 16 : 0);
            }
        }
        cp_async_commit();
    };
    int t = blockIdx.x;
    if (t < ntiles) issue(t, smem_c);
    for (int iter = 0; t < ntiles; t += gridDim.x, ++iter) {
        double2 *buf = smem_c + (iter & 1) * (N * LD);  // offsets keep LDS/STS (not generic)
        const int tn = t + gridDim.x;
        if (tn < ntiles) issue(tn, smem_c + ((iter + 1) & 1) * (N * LD));
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        int k0, outer;
        double2 *base = tile_base(t, k0, outer);
        if constexpr (MODE == COL_FWD || MODE == COL_SOLVE)
            tile_fft<N1, N2, TK, false>(buf, tw);
        else
            tile_fft<N1, N2, TK, true>(buf, tw);
        if constexpr (MODE == COL_SOLVE) {
            const double *s0 = g.sym;
            const double *slast = g.sym + (int64_t)(g.dim - 1) * g.n;
            const double s1 = (g.dim == 3) ? g.sym[g.n + outer] : 0.0;
#pragma unroll 2
            for (int it = 0; it < IT; ++it) {
                const int w = it * NT + threadIdx.x;
                if (w < N * TK) {
                    const int kl = w / TK, c = w % TK;
                    double gsq = s0[kl];
                    if (g.dim == 3) gsq = gsq + s1;
                    gsq = gsq + slast[min(k0 + c, g.n - 1)];
                    const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
                    buf[kl * LD + c] = cscale(buf[kl * LD + c], -inv * g.scale);
                }
            }
            __syncthreads();
            tile_fft<N1, N2, TK, true>(buf, tw);
        }
        const bool full = k0 + TK <= g.ncol;
#pragma unroll 4
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + threadIdx.x;
            const int n = w / TK, c = w % TK;
            if (w < N * TK && (full || k0 + c < g.ncol)) base[n * g.es + c] = buf[n * LD + c];
        }
        __syncthreads();  // this buffer is refilled two tiles later
    }
    cp_async_wait<0>();
}

// E on the plane layout, persistent and software-pipelined: each block walks
// tiles t = blockIdx.x, +gridDim.x, ...; the cp.async copies of the next
// tile's spectrum (ROWS x 16 B runs per (c, k2)) land in the second shared
// buffer while the current tile is transformed, so loads stay in flight (the
// one-tile kernel is global-load-latency bound: ncu long_scoreboard).
template <int N1, int N2, int DIM, int ROWS>
__global__ void __launch_bounds__(RowCfg<N1, N2, DIM, ROWS>::NTI, RowCfg<N1, N2, DIM, ROWS>::MINB_INV)
k_row_inv_p(const double2 *__restrict__ spec, double *__restrict__ Ut, RowGeom g,
            const double2 *__restrict__ tw_line, const double2 *__restrict__ tw_r2c, int ntiles) {
    using C = RowCfg<N1, N2, DIM, ROWS>;
    constexpr int TK = C::TK, LD = TK + 1, N = N1 * N2, NH = N + 1;
    extern __shared__ double2 smem_c[];
    auto issue = [&](int t, double2 *dst) {
        const int64_t row0 = (int64_t)t * ROWS;
        for (int w = threadIdx.x; w < TK * NH; w += C::NTI) {
            int k, line, r0;
            if (g.plane) {  // ROWS x 16 B runs per (c, k2)
                r0 = w % ROWS;
                const int tt = w / ROWS;
                k = tt % NH;
                line = (tt / NH) * ROWS + r0;
            } else {        // row layout: consecutive k of one row
                line = w / NH;
                k = w - line * NH;
                r0 = line % ROWS;
            }
            const int c = line / ROWS;
            const int64_t row = row0 + r0;
            const bool ok = row < g.nrows;
            const double2 *src =
                g.plane ? spec + ((int64_t)c * NH + k) * g.nrows + (ok ? row : 0)
                        : spec + ((int64_t)c * g.nrows + (ok ? row : 0)) * g.P + k;
            cp_async16(&dst[k * LD + line], src, ok ? 16 : 0);
        }
        cp_async_commit();
    };
    int t = blockIdx.x;
    if (t < ntiles) issue(t, smem_c);
    for (int iter = 0; t < ntiles; t += gridDim.x, ++iter) {
        double2 *buf = smem_c + (iter & 1) * ((N + 1) * LD);
        const int tn = t + gridDim.x;
        if (tn < ntiles) issue(tn, smem_c + ((iter + 1) & 1) * ((N + 1) * LD));
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        asm volatile("" : "+l"(tw_line), "+l"(tw_r2c));  // twiddle loads stay per tile
        row_inv_tile<N1, N2, DIM, ROWS>(buf, nullptr, Ut, g, (int64_t)t * ROWS, N, true, tw_line,
                                        tw_r2c);
        __syncthreads();  // this buffer is refilled two tiles on
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// B + C + D in one launch on the plane layout (RowGeom::plane): a cluster of
// CS CTAs owns one (component, k2) plane [i0][i1] of the half spectrum
// (n x n complex, 1 MB at 256^3) and runs
//   pass 1  FFT along axis 1 (contiguous lines of the plane)
//   pass 2  FFT along axis 0, u_hat = -d_hat / |g|^2 on live modes, inverse
//   pass 3  inverse FFT along axis 1
// with cluster barriers (release / acquire at cluster scope) between the
// passes.  CTA r of the cluster takes tiles r*NTILE/CS .. of every pass.  The
// plane stays in L2 from pass 1 to pass 3, so the spectrum crosses HBM once
// each way instead of three times (B, C, D of the row layout each read and
// write it).  The per-line arithmetic (tile_fft, the solve expression and its
// summation order) is that of k_colp / k_col: results are bitwise identical.
// ---------------------------------------------------------------------------
#ifndef MM_PLANE_PPT
#define MM_PLANE_PPT 16
#endif
struct PlaneGeom {
    int n, nh;
    const double *sym;
    double thresh, scale;
};

template <int N1, int N2, int TK>
struct PlaneCfg {
    static constexpr int N = N1 * N2;
    static constexpr int PPT = MM_PLANE_PPT;  // points per thread (tile_fft_s)
    static constexpr int NT = TK * N / PPT;
    static constexpr int IT = (N * TK + NT - 1) / NT;
    // resident CTAs per SM the two tile buffers allow (<= 227 KB of shared
    // memory), requested from the register allocator
    static constexpr int SMEM = 2 * N * (TK + 1) * 16;
    static constexpr int MINB0 = (227 * 1024) / (SMEM + 1024);
    static constexpr int MINB1 = MINB0 > 8 ? 8 : (MINB0 < 1 ? 1 : MINB0);
    // ... but not below 64 registers per thread
    static constexpr int MINB = MINB1 * NT * 64 > 65536 ? 65536 / (NT * 64) : MINB1;
};

__device__ __forceinline__ void cluster_barrier() {
    asm volatile(
        "barrier.cluster.arrive.release.aligned;\n"
        "barrier.cluster.wait.acquire.aligned;\n" ::
            : "memory");
}

// One pass over tiles [t0, t1) of a plane, double-buffered: while tile t is
// transformed in one shared buffer, the cp.async copies of tile t+1 land in
// the other (global -> shared without registers; .cg bypasses L1, so data
// another CTA of the cluster wrote before the barrier is read from L2).
// KIND 0 / 1: forward / inverse FFT of TK consecutive lines along axis 1
// (contiguous); KIND 2: forward FFT of TK consecutive columns along axis 0,
// solve, inverse (k_col<COL_SOLVE>'s arithmetic).
enum { PL_ROW_FWD = 0, PL_ROW_INV = 1, PL_COL_SOLVE = 2 };

template <int N1, int N2, int TK, int KIND>
__device__ __forceinline__ void plane_pass(double2 *__restrict__ pl, double2 *smem, int t0, int t1,
                                           const PlaneGeom &g, int k2,
                                           const double2 *__restrict__ tw) {
    using C = PlaneCfg<N1, N2, TK>;
    constexpr int N = C::N, NT = C::NT, IT = C::IT, LD = TK + 1;
    // buffer b at smem + b * N * LD (plain offsets from the shared base keep
    // the accesses LDS/STS; an array of two pointers made them generic)
    // element w of tile t: global offset and shared slot
    auto goff = [&](int t, int w) -> int64_t {
        if constexpr (KIND == PL_COL_SOLVE) return (int64_t)(w / TK) * N + t * TK + w % TK;
        else return (int64_t)t * TK * N + w;
    };
    auto slot = [&](int w) -> int {
        if constexpr (KIND == PL_COL_SOLVE) return (w / TK) * LD + (w % TK);
        else return (w % N) * LD + w / N;
    };
    auto issue = [&](int t, double2 *dst) {
        int tx = threadIdx.x;
        asm volatile("" : "+r"(tx));  // addresses are recomputed per tile, not kept live
#pragma unroll 4
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + tx;
            if (w < N * TK) cp_async16(&dst[slot(w)], &pl[goff(t, w)], 16);
        }
        cp_async_commit();
    };
    if (t0 < t1) issue(t0, smem);
#pragma unroll 1
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
        // keep loop-invariant loads (twiddles, symbols) and addresses inside
        // the loop instead of hoisted into registers for all tiles
        int tx = threadIdx.x;
        const double *sym = g.sym;
        asm volatile("" : "+l"(tw), "+l"(sym), "+r"(tx));
        double2 *buf = smem + (i & 1) * (N * LD);
        if (t + 1 < t1) issue(t + 1, smem + ((i + 1) & 1) * (N * LD));
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        // COL_SOLVE: the symbols of this thread's elements are loaded before
        // the forward transform (their latency hides behind it)
        double s0v[KIND == PL_COL_SOLVE ? IT : 1], s1v = 0.0;
        if constexpr (KIND == PL_COL_SOLVE) {
#pragma unroll
            for (int it = 0; it < IT; ++it) {
                const int w = it * NT + tx;
                s0v[it] = w < N * TK ? __ldg(&sym[w / TK]) : 0.0;
            }
            s1v = __ldg(&sym[N + t * TK + tx % TK]);  // NT is a multiple of TK
        }
        // COL_SOLVE: forward, solve, inverse as two trips of one loop body
        constexpr int NPH = KIND == PL_COL_SOLVE ? 2 : 1;
#pragma unroll 1
        for (int ph = 0; ph < NPH; ++ph) {
            asm volatile("" : "+l"(tw));
            tile_fft_s<N, TK, C::PPT>(buf, tw, KIND == PL_ROW_INV || ph == 1);
            if (KIND == PL_COL_SOLVE && ph == 0) {
                const double sl = __ldg(&sym[2 * N + k2]);
#pragma unroll
                for (int it = 0; it < IT; ++it) {
                    const int w = it * NT + tx;
                    if (w < N * TK) {
                        const int kl = w / TK, c = w % TK;
                        double gsq = s0v[it];
                        gsq = gsq + s1v;
                        gsq = gsq + sl;
                        const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
                        buf[kl * LD + c] = cscale(buf[kl * LD + c], -inv * g.scale);
                    }
                }
                __syncthreads();
            }
        }
#pragma unroll 4
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + tx;
            if (w < N * TK) pl[goff(t, w)] = buf[slot(w)];
        }
        __syncthreads();  // this buffer is refilled by the issue two tiles on
    }
    cp_async_wait<0>();
}

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers -------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// bounded wait on an mbarrier phase: a descriptor error would otherwise hang
// the GPU; 2^24 probes is ~a second, far beyond any tile
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    for (uint32_t it = 0; !ok; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (it > (1u << 24)) __trap();
    }
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int x, int y,
                                             int z) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map),
                 "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int x, int y, int z, int w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, const void *src, int x, int y,
                                             int z, int w) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(map),
                 "r"(x), "r"(y), "r"(z), "r"(w), "r"(smem_u32(src))
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Column tiles (pass 2, n = 256) through TMA with the hardware 128-byte
// swizzle: element n of column c of an 8-column tile sits at complex slot
// n * 8 + (c ^ (n & 7)).  16 lanes own one column; the in-warp radix-16 x 16
// FFT keeps its intermediate at row rho(i) = i ^ ((i >> 4) & 7), which makes
// both the transposed write (y[16 q + r]) and the strided read (x[q + 16 r])
// hit eight distinct 16-byte bank groups.  The forward transform's output is
// in natural order in registers, so the solve and the first stage of the
// inverse run without a shared-memory round trip.
__device__ __forceinline__ int csw(int row, int c) { return row * 8 + (c ^ (row & 7)); }
__device__ __forceinline__ int crho(int i) { return i ^ ((i >> 4) & 7); }

__device__ __forceinline__ void col_fft_solve_256(double2 *buf, const double2 *__restrict__ tw,
                                                  const PlaneGeom &g, int col, int k2) {
    const int c = threadIdx.x >> 4, q = threadIdx.x & 15;
    double2 v[16];
    const double s1 = __ldg(&g.sym[256 + col]);
    const double sl = __ldg(&g.sym[2 * 256 + k2]);
    // forward, stage 1: x[q + 16 r] -> y[16 q + r]
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[csw(q + 16 * r, c)];
    __syncwarp();
    fft_reg_rt<16>(v, false);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[csw(crho(16 * q + r), c)] = v[r];
    __syncwarp();
    // forward, stage 2: twiddle W^{q r}, natural order out (element q + 16 r)
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[csw(crho(q + 16 * r), c)];
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], __ldg(&tw[q * r]));
    fft_reg_rt<16>(v, false);
    // solve (k_col<COL_SOLVE>'s expression and summation order) on element q + 16 r
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        double gsq = __ldg(&g.sym[q + 16 * r]);
        gsq = gsq + s1;
        gsq = gsq + sl;
        const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
        v[r] = cscale(v[r], -inv * g.scale);
    }
    // inverse, stage 1 straight from registers: x[q + 16 r] = v[r]
    fft_reg_rt<16>(v, true);
    __syncwarp();  // every lane is done reading the forward intermediate
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[csw(crho(16 * q + r), c)] = v[r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[csw(crho(q + 16 * r), c)];
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        const double2 w = __ldg(&tw[q * r]);
        v[r] = cmul(v[r], make_double2(w.x, -w.y));
    }
    fft_reg_rt<16>(v, true);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[csw(q + 16 * r, c)] = v[r];
    __syncwarp();
}

// Pass 2 of the plane (FFT along axis 0, solve, inverse) with TMA: a tile of
// TK columns x N rows is one cp.async.bulk.tensor load into a dense
// [row][column] shared-memory tile (the line-interleaved layout the Stockham
// FFT wants, no padding needed: 8 consecutive 16-byte elements fill the 32
// banks), completion on an mbarrier (expect_tx); the result goes back with a
// TMA store.  Double-buffered: thread 0 issues tile t+1's load while the
// CTA transforms tile t, after the previous store from that buffer has read
// its shared memory.
// plane_col_tma's double-buffered TMA loop around col_fft_solve_256
__device__ __forceinline__ void plane_col_swz(const CUtensorMap *map, int plane, double2 *smem,
                                              uint64_t *bars, uint32_t (&phase)[2], int t0,
                                              int t1, const PlaneGeom &g, int k2,
                                              const double2 *__restrict__ tw) {
    constexpr int N = 256, TK = 8;
    constexpr uint32_t BYTES = (uint32_t)(N * TK * sizeof(double2));
    const int tx = threadIdx.x;
    double2 *buf[2] = {smem, smem + N * (TK + 1)};  // 1024-byte aligned offsets
    if (tx == 0 && t0 < t1) {
        bulk_wait_read0();
        mbar_expect_tx(&bars[0], BYTES);
        tma_load_3d(buf[0], map, &bars[0], 2 * t0 * TK, 0, plane);
    }
#pragma unroll 1
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int b = i & 1;
        if (tx == 0 && t + 1 < t1) {
            bulk_wait_read0();
            mbar_expect_tx(&bars[1 - b], BYTES);
            tma_load_3d(buf[1 - b], map, &bars[1 - b], 2 * (t + 1) * TK, 0, plane);
        }
        mbar_wait(&bars[b], phase[b]);
        phase[b] ^= 1u;
        col_fft_solve_256(buf[b], tw, g, t * TK + (tx >> 4), k2);
        fence_proxy_async();
        __syncthreads();
        if (tx == 0) {
            tma_store_3d(map, buf[b], 2 * t * TK, 0, plane);
            bulk_commit();
        }
    }
    if (tx == 0) bulk_wait0();
    __syncthreads();
}

template <int N1, int N2, int TK>
__device__ __forceinline__ void plane_col_tma(const CUtensorMap *map, int plane, double2 *smem,
                                              uint64_t *bars, uint32_t (&phase)[2], int t0,
                                              int t1, const PlaneGeom &g, int k2,
                                              const double2 *__restrict__ tw, bool swz) {
    using C = PlaneCfg<N1, N2, TK>;
    constexpr int N = C::N, NT = C::NT, IT = C::IT, LD = TK;
    if constexpr (MM_PLANE_COLSWZ && N == 256 && TK == 8 && NT == 128) {
        if (swz) {  // 16 lanes per column on the swizzled tile, no block barrier
            plane_col_swz(map, plane, smem, bars, phase, t0, t1, g, k2, tw);
            return;
        }
    }
    constexpr uint32_t BYTES = (uint32_t)(N * TK * sizeof(double2));
    const int tx = threadIdx.x;
    double2 *buf[2] = {smem, smem + N * (TK + 1)};  // 128-byte aligned offsets
    if (tx == 0 && t0 < t1) {
        bulk_wait_read0();
        mbar_expect_tx(&bars[0], BYTES);
        tma_load_3d(buf[0], map, &bars[0], 2 * t0 * TK, 0, plane);
    }
#pragma unroll 1
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int b = i & 1;
        if (tx == 0 && t + 1 < t1) {
            bulk_wait_read0();  // the store of tile t-1 has read buffer 1-b
            mbar_expect_tx(&bars[1 - b], BYTES);
            tma_load_3d(buf[1 - b], map, &bars[1 - b], 2 * (t + 1) * TK, 0, plane);
        }
        double s0v[IT];
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + tx;
            s0v[it] = w < N * TK ? __ldg(&g.sym[w / TK]) : 0.0;
        }
        const double s1v = __ldg(&g.sym[N + t * TK + tx % TK]);
        mbar_wait(&bars[b], phase[b]);
        phase[b] ^= 1u;
        double2 *bf = buf[b];
        tile_fft_s<N, TK, C::PPT, LD>(bf, tw, false);
        const double sl = __ldg(&g.sym[2 * N + k2]);
#pragma unroll
        for (int it = 0; it < IT; ++it) {
            const int w = it * NT + tx;
            if (w < N * TK) {
                const int kl = w / TK, c = w % TK;
                double gsq = s0v[it];
                gsq = gsq + s1v;
                gsq = gsq + sl;
                const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
                bf[kl * LD + c] = cscale(bf[kl * LD + c], -inv * g.scale);
            }
        }
        __syncthreads();
        tile_fft_s<N, TK, C::PPT, LD>(bf, tw, true);
        fence_proxy_async();  // this thread's shared-memory writes -> the async proxy
        __syncthreads();
        if (tx == 0) {
            tma_store_3d(map, bf, 2 * t * TK, 0, plane);
            bulk_commit();
        }
    }
    if (tx == 0) bulk_wait0();  // the stores are performed before the cluster barrier
    __syncthreads();
}

// 256-point FFT of the lines of a dense line-major tile (element n of line c
// at buf[c * 256 + n], the TMA layout of a row tile): 16 lanes per line, two
// radix-16 stages in registers; stage 1 writes an XOR-swizzled transpose
// (slot 16 a + (b ^ a)), stage 2 reads it and writes natural order back, so
// every exchange is conflict-free and synchronised within the warp only.
__device__ __forceinline__ int lm_swz(int a, int b) { return 16 * a + (b ^ a); }

__device__ __forceinline__ void tile_fft_lm256(double2 *buf, const double2 *__restrict__ tw,
                                               bool inv) {
    const int c = threadIdx.x >> 4, q = threadIdx.x & 15;
    double2 *L = buf + c * 256;
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = L[q + 16 * r];
    __syncwarp();
    fft_reg_rt<16>(v, inv);
#pragma unroll
    for (int r = 0; r < 16; ++r) L[lm_swz(q, r)] = v[r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = L[lm_swz(r, q)];
    __syncwarp();
#if MM_LM_TWP
    // W^{q r}: four table loads (r = 1, 2, 4, 8) and products, as
    // stockham_pass's MM_TW_PROD (fewer dependent loads in the LSU queue)
    {
        double2 w[16];
        w[1] = __ldg(&tw[q]);
        w[2] = __ldg(&tw[2 * q]);
        w[4] = __ldg(&tw[4 * q]);
        w[8] = __ldg(&tw[8 * q]);
        if (inv) {
            w[1].y = -w[1].y;
            w[2].y = -w[2].y;
            w[4].y = -w[4].y;
            w[8].y = -w[8].y;
        }
        w[3] = cmul(w[1], w[2]);
        w[5] = cmul(w[1], w[4]);
        w[6] = cmul(w[2], w[4]);
        w[7] = cmul(w[3], w[4]);
#pragma unroll
        for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], w[r]);
    }
#else
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        double2 w = __ldg(&tw[q * r]);
        if (inv) w.y = -w.y;
        v[r] = cmul(v[r], w);
    }
#endif
    fft_reg_rt<16>(v, inv);
#pragma unroll
    for (int r = 0; r < 16; ++r) L[q + 16 * r] = v[r];
    __syncwarp();
}

// Passes 1 and 3 of the plane (FFT along axis 1) with TMA, n = 256: a tile
// of TK rows is one 4D cp.async.bulk.tensor load (rows are contiguous: box
// {256 doubles, 2 halves, TK rows, 1 plane}) into a dense line-major tile,
// transformed by tile_fft_lm256, stored back by TMA; double-buffered as
// plane_col_tma.
template <int TK>
__device__ __forceinline__ void plane_row_tma(const CUtensorMap *map, int plane, double2 *smem,
                                              uint64_t *bars, uint32_t (&phase)[2], int t0,
                                              int t1, const double2 *__restrict__ tw, bool inv) {
    constexpr int N = 256;
    constexpr uint32_t BYTES = (uint32_t)(N * TK * sizeof(double2));
    const int tx = threadIdx.x;
    double2 *buf[2] = {smem, smem + N * (TK + 1)};
    if (tx == 0 && t0 < t1) {
        bulk_wait_read0();
        mbar_expect_tx(&bars[0], BYTES);
        tma_load_4d(buf[0], map, &bars[0], 0, 0, t0 * TK, plane);
    }
#pragma unroll 1
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
        const int b = i & 1;
        if (tx == 0 && t + 1 < t1) {
            bulk_wait_read0();
            mbar_expect_tx(&bars[1 - b], BYTES);
            tma_load_4d(buf[1 - b], map, &bars[1 - b], 0, 0, (t + 1) * TK, plane);
        }
        mbar_wait(&bars[b], phase[b]);
        phase[b] ^= 1u;
        tile_fft_lm256(buf[b], tw, inv);
        fence_proxy_async();
        __syncthreads();
        if (tx == 0) {
            tma_store_4d(map, buf[b], 0, 0, t * TK, plane);
            bulk_commit();
        }
    }
    if (tx == 0) bulk_wait0();
    __syncthreads();
}

template <int N1, int N2, int TK, int CS>
__global__ void __cluster_dims__(CS, 1, 1)
    __launch_bounds__(PlaneCfg<N1, N2, TK>::NT, PlaneCfg<N1, N2, TK>::MINB)
k_plane(double2 *__restrict__ spec, PlaneGeom g, const double2 *__restrict__ tw,
        const __grid_constant__ CUtensorMap tmap, int use_tma,
        const __grid_constant__ CUtensorMap rmap) {
    constexpr int N = N1 * N2;
    constexpr int PER = N / TK / CS;  // tiles per CTA per pass
    extern __shared__ __align__(1024) double2 smem_c[];  // 128-byte swizzled TMA tiles
    const int plane = blockIdx.x / CS;  // c * nh + k2
    const int r = blockIdx.x % CS;      // rank in the cluster
    const int k2 = plane % g.nh;
    double2 *pl = spec + (int64_t)plane * N * N;
    // use_tma: 1 = the column pass through TMA, 2 = the row passes too,
    // 3 = and the column pass on swizzled tiles
    // (n = 256, 8-row tiles, 128 threads: 16 lanes per row)
    constexpr bool ROWTMA = N1 * N2 == 256 && TK == 8 && PlaneCfg<N1, N2, TK>::NT == 128;
    constexpr bool COLTMA = PlaneCfg<N1, N2, TK>::PPT == 16;
    __shared__ __align__(8) uint64_t bars[2];
    uint32_t phase[2] = {0u, 0u};
    if ((COLTMA || ROWTMA) && use_tma) {
        if (threadIdx.x == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncthreads();
    }
    if (ROWTMA && use_tma >= 2)
        plane_row_tma<TK>(&rmap, plane, smem_c, bars, phase, r * PER, (r + 1) * PER, tw, false);
    else
        plane_pass<N1, N2, TK, PL_ROW_FWD>(pl, smem_c, r * PER, (r + 1) * PER, g, k2, tw);
    cluster_barrier();
    if constexpr (COLTMA) {
        if (use_tma) {
            plane_col_tma<N1, N2, TK>(&tmap, plane, smem_c, bars, phase, r * PER, (r + 1) * PER,
                                      g, k2, tw, use_tma == 3);
        } else {
            plane_pass<N1, N2, TK, PL_COL_SOLVE>(pl, smem_c, r * PER, (r + 1) * PER, g, k2, tw);
        }
    } else {
        plane_pass<N1, N2, TK, PL_COL_SOLVE>(pl, smem_c, r * PER, (r + 1) * PER, g, k2, tw);
    }
    cluster_barrier();
    if (ROWTMA && use_tma >= 2)
        plane_row_tma<TK>(&rmap, plane, smem_c, bars, phase, r * PER, (r + 1) * PER, tw, true);
    else
        plane_pass<N1, N2, TK, PL_ROW_INV>(pl, smem_c, r * PER, (r + 1) * PER, g, k2, tw);
}

// ---------------------------------------------------------------------------
// Plane pass, half-warp per line (n = 256, MM_PLANE_HW).  The same three
// passes per (c, k2) plane and cluster barriers as k_plane, but each line is
// owned by 16 consecutive lanes that load it (cp.async, double-buffered per
// line slot), transform it (256 = 16 x 16: two radix-16 Stockham stages in
// registers, exchanged through the slot's shared buffer) and store it with
// warp-level synchronisation only: no block-wide barrier inside a pass, so
// every half-warp streams its lines independently (k_plane's tile FFT was
// bound by __syncthreads and shared-memory latency: 12 warps/SM, barrier
// stalls 24 %).  Element i = 16 a + b of a line sits at slot 16 a + (b ^ a):
// the stage-1 transpose (y[16 q + r] for fixed r across lanes q) and the
// natural-order reads / writes (x[q + 16 r]) are both conflict-free.
// ---------------------------------------------------------------------------
#ifndef MM_PLANE_HW  // measured 0.697 (k_plane) -> 0.743 ms at 256^3: the column pass loses
#define MM_PLANE_HW 0  // coalescing with one line per half-warp; off
#endif
#ifndef MM_PLANE_HW_NT
#define MM_PLANE_HW_NT 128
#endif
#ifndef MM_PLANE_HW_MINB
#define MM_PLANE_HW_MINB 3
#endif

__device__ __forceinline__ int hw_slot(int a, int b) { return 16 * a + (b ^ a); }

// 256-point FFT of the line in `buf` (this half-warp's slot), lane q of 16
__device__ __forceinline__ void hw_fft256(double2 *buf, int q, const double2 *__restrict__ tw,
                                          bool inv) {
    double2 v[16];
    // stage 1 (radix 16, NS = 1): x[q + 16 r] -> y[16 q + r]
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[hw_slot(r, q)];
    __syncwarp();
    fft_reg_rt<16>(v, inv);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[hw_slot(q, r)] = v[r];
    __syncwarp();
    // stage 2 (radix 16, NS = 16): twiddle W_256^{q r}, x[q + 16 r] -> y[q + 16 r]
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = buf[hw_slot(r, q)];
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        double2 w = __ldg(&tw[q * r]);
        if (inv) w.y = -w.y;
        v[r] = cmul(v[r], w);
    }
    fft_reg_rt<16>(v, inv);
#pragma unroll
    for (int r = 0; r < 16; ++r) buf[hw_slot(r, q)] = v[r];
    __syncwarp();
}

template <int KIND, int NSLOT, int LPC>
__device__ __forceinline__ void hw_pass(double2 *__restrict__ pl, double2 *bufs, int r0, int slot,
                                        int q, const PlaneGeom &g, int k2,
                                        const double2 *__restrict__ tw) {
    constexpr int N = 256, NL = LPC / NSLOT;  // lines per slot in this pass
    auto elem = [&](int t, int n) -> int64_t {
        if constexpr (KIND == PL_COL_SOLVE) return (int64_t)n * N + t;
        else return (int64_t)t * N + n;
    };
    auto issue = [&](int t, double2 *dst) {
#pragma unroll
        for (int k = 0; k < 16; ++k) cp_async16(&dst[hw_slot(k, q)], &pl[elem(t, 16 * k + q)], 16);
        cp_async_commit();
    };
    issue(r0 + slot, bufs);
#pragma unroll 1
    for (int i = 0; i < NL; ++i) {
        const int t = r0 + slot + i * NSLOT;
        double2 *buf = bufs + (i & 1) * N;
        if (i + 1 < NL) issue(t + NSLOT, bufs + ((i + 1) & 1) * N);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncwarp();
        hw_fft256(buf, q, tw, KIND == PL_ROW_INV);
        if constexpr (KIND == PL_COL_SOLVE) {
            // u_hat = -d_hat / |g|^2 on live modes (k_col<COL_SOLVE>'s expression
            // and summation order); the line is column i1 = t of plane k2
            const double s1 = __ldg(&g.sym[N + t]);
            const double sl = __ldg(&g.sym[2 * N + k2]);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const int n = 16 * k + q;
                double gsq = __ldg(&g.sym[n]);
                gsq = gsq + s1;
                gsq = gsq + sl;
                const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
                const int sidx = hw_slot(k, q);
                buf[sidx] = cscale(buf[sidx], -inv * g.scale);
            }
            __syncwarp();
            hw_fft256(buf, q, tw, true);
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) pl[elem(t, 16 * k + q)] = buf[hw_slot(k, q)];
        __syncwarp();  // the buffer is refilled by the issue two lines on
    }
    cp_async_wait<0>();
}

template <int NTH, int CS>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NTH, MM_PLANE_HW_MINB)
k_plane_hw(double2 *__restrict__ spec, PlaneGeom g, const double2 *__restrict__ tw) {
    constexpr int N = 256, NSLOT = NTH / 16, LPC = N / CS;
    static_assert(LPC % NSLOT == 0, "lines per CTA divide among the slots");
    extern __shared__ __align__(1024) double2 smem_c[];  // 128-byte swizzled TMA tiles
    const int plane = blockIdx.x / CS;  // c * nh + k2
    const int r = blockIdx.x % CS;      // rank in the cluster
    const int k2 = plane % g.nh;
    const int slot = threadIdx.x >> 4, q = threadIdx.x & 15;
    double2 *bufs = smem_c + slot * 2 * N;
    double2 *pl = spec + (int64_t)plane * N * N;
    hw_pass<PL_ROW_FWD, NSLOT, LPC>(pl, bufs, r * LPC, slot, q, g, k2, tw);
    cluster_barrier();
    hw_pass<PL_COL_SOLVE, NSLOT, LPC>(pl, bufs, r * LPC, slot, q, g, k2, tw);
    cluster_barrier();
    hw_pass<PL_ROW_INV, NSLOT, LPC>(pl, bufs, r * LPC, slot, q, g, k2, tw);
}

// ---------------------------------------------------------------------------
// F: gradient of u_tilde, multiplier ascent and residual sums
// slots: 0 sum dG^2, 1 sum misfit^2, 2.. sum lam (D)
// ---------------------------------------------------------------------------
struct Mean9 {
    double v[9];
};

// MODE: GRAD_WRITE  grad_u = u_mean + D u (projection API; writes G)
//       GRAD_EXPL   solver tail with an explicit previous grad_u (reads G)
//       GRAD_IMPL   solver tail with grad_u_old = ubar_old + D u_old implicit
// The solver modes do not write G: afterwards grad_u is implicit.
//       GRAD_EXPLW  solver tail, explicit grad_u in and out (reads and writes G)
//       GRAD_RES_EXPL / GRAD_RES_IMPL  residual sums only (r_d, r_p); the ascent is
//                   deferred to the fused update + local pass (mm_local.cu)
enum { GRAD_WRITE = 0, GRAD_EXPL = 1, GRAD_IMPL = 2, GRAD_EXPLW = 3, GRAD_RES_EXPL = 4,
       GRAD_RES_IMPL = 5 };

template <int DIM, int MODE>
__global__ void __launch_bounds__(256)
k_grad(const double *__restrict__ Ut, const double *__restrict__ Uold, double *__restrict__ G,
       const double *__restrict__ F, double *__restrict__ Lam, int n, int lgn, int64_t M,
       double inv2h, double rho, Mean9 um, Mean9 um_old, double *partials, double *red_out,
       unsigned int *count, int64_t uM, int wrap0, const DecideArgs dec) {
    constexpr int D = DIM * DIM;
    constexpr int K = 2 + D;
    __shared__ double smem[32 * K];
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        int off_p[DIM], off_m[DIM];
        nbr_offsets<DIM>(p, n, lgn, off_p, off_m, wrap0 != 0);
        // issue every load before any store
        double up[D], dn[D];
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            const double *u = Ut + (int64_t)i * uM + p;
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
                up[i * DIM + j] = __ldg(u + off_p[j]);
                dn[i * DIM + j] = __ldg(u + off_m[j]);
            }
        }
        double gold[D], fv[D], lv[D];
        constexpr bool RES = MODE == GRAD_RES_EXPL || MODE == GRAD_RES_IMPL;
        if (MODE == GRAD_IMPL || MODE == GRAD_RES_IMPL) {
#pragma unroll
            for (int i = 0; i < DIM; ++i) {
                const double *u = Uold + (int64_t)i * uM + p;
#pragma unroll
                for (int j = 0; j < DIM; ++j)
                    gold[i * DIM + j] = (__ldg(u + off_p[j]) - __ldg(u + off_m[j])) * inv2h +
                                        um_old.v[i * DIM + j];
            }
        }
        if (MODE != GRAD_WRITE) {
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const int64_t o = (int64_t)c * M + p;
                if (MODE == GRAD_EXPL || MODE == GRAD_EXPLW || MODE == GRAD_RES_EXPL) gold[c] = G[o];
                fv[c] = __ldg(&F[o]);
                if (!RES) lv[c] = Lam[o];
            }
        }
#pragma unroll
        for (int c = 0; c < D; ++c) {
            const double gnew = (up[c] - dn[c]) * inv2h + um.v[c];  // projection.py:168
            const int64_t o = (int64_t)c * M + p;
            if (RES) {
                const double dg = gnew - gold[c];          // solver.py:271
                const double mis = gnew - fv[c];           // solver.py:277
                acc[0] += dg * dg;
                acc[1] += mis * mis;
            } else if (MODE != GRAD_WRITE) {
                const double dg = gnew - gold[c];          // solver.py:271
                const double mis = gnew - fv[c];           // solver.py:277
                const double lnew = lv[c] + rho * mis;     // solver.py:279
                Lam[o] = lnew;
                if (MODE == GRAD_EXPLW) G[o] = gnew;
                acc[0] += dg * dg;
                acc[1] += mis * mis;
                acc[2 + c] += lnew;
            } else {
                G[o] = gnew;
            }
        }
    }
    if (MODE != GRAD_WRITE) {
        int ops[K];
#pragma unroll
        for (int k = 0; k < K; ++k) ops[k] = RED_SUM;
        block_reduce<K>(acc, ops, smem);
        double fin[K];
        if (grid_finalize<K>(acc, ops, partials, red_out, count, smem, fin) && dec.on)
            decide_step(fin[0], fin[1], dec);
    }
}

// K1 residual pass (GRAD_RES_IMPL, 3D) with explicit stencil reuse: a CTA
// owns a 32 (axis 2) x 8 (axis 1) tile of columns and marches along axis 0
// over a chunk of planes.  Each thread keeps its column's u values at planes
// i-1, i, i+1 in registers (axis-0 differences); plane i of u_new / u_old
// with a one-cell ring is staged in shared memory for the axis-1 / axis-2
// differences.  Every u element is loaded from global memory once per chunk
// (plus the ring), instead of seven times through L1/L2 as in k_grad, whose
// axis-0 neighbours miss in L2 (ncu: 1.5x the algorithmic DRAM bytes).
// The per-voxel arithmetic is k_grad's, in the same order.
#ifndef MM_RES_ZC
#define MM_RES_ZC 32
#endif
#ifndef MM_RES_MINB
#define MM_RES_MINB 2
#endif
constexpr int RT_X = 32, RT_Y = 8, RT_ZC = MM_RES_ZC;
constexpr int RT_RING = 2 * RT_X + 2 * RT_Y;  // ring cells per plane (no corners needed)

// ring cell r of the tile at plane offset `pl`: rows y0-1 / y0+RT_Y, then
// columns x0-1 / x0+RT_X; returns the in-plane offset and the smem slot
__device__ __forceinline__ void ring_cell(int r, int x0, int y0, int n, int &off, int &sy,
                                          int &sx) {
    if (r < 2 * RT_X) {
        const int side = r / RT_X, xx = r % RT_X;
        const int y = side ? (y0 + RT_Y == n ? 0 : y0 + RT_Y) : (y0 == 0 ? n - 1 : y0 - 1);
        off = y * n + x0 + xx;
        sy = side ? RT_Y + 1 : 0;
        sx = xx + 1;
    } else {
        const int rr = r - 2 * RT_X;
        const int side = rr / RT_Y, yy = rr % RT_Y;
        const int x = side ? (x0 + RT_X == n ? 0 : x0 + RT_X) : (x0 == 0 ? n - 1 : x0 - 1);
        off = (y0 + yy) * n + x;
        sy = yy + 1;
        sx = side ? RT_X + 1 : 0;
    }
}

__global__ void __launch_bounds__(RT_X * RT_Y, MM_RES_MINB)
k_res_march(const double *__restrict__ Un, const double *__restrict__ Uo,
            const double *__restrict__ F, int n, int64_t M, double inv2h, Mean9 um, Mean9 umo,
            double *partials, double *red_out, unsigned int *count, int64_t uM, int wrap0,
            const DecideArgs dec) {
    __shared__ double sm[2][3][RT_Y + 2][RT_X + 2];
    __shared__ double red_sm[32 * 2];
    // 1D block (block_reduce / grid_finalize index threads by threadIdx.x)
    const int tx = threadIdx.x % RT_X, ty = threadIdx.x / RT_X;
    const int x0 = blockIdx.x * RT_X, y0 = blockIdx.y * RT_Y;
    const int x = x0 + tx, y = y0 + ty;
    const int z0 = blockIdx.z * RT_ZC;
    const int nn = n * n;
    const int col = y * n + x;
    const bool ringer = threadIdx.x < RT_RING;
    int roff = 0, rsy = 0, rsx = 0;
    if (ringer) ring_cell(threadIdx.x, x0, y0, n, roff, rsy, rsx);
    auto uval = [&](int f, int c, int z, int off) {
        return __ldg((f ? Uo : Un) + (int64_t)c * uM + (int64_t)z * nn + off);
    };
    // software pipeline: everything plane z needs is in registers before
    // the iteration for z starts; the loads for z + 1 are issued before the
    // arithmetic of z
    double prv[2][3], cur[2][3], nxt[2][3], ring[2][3], fv[9];
    {
        // slab (wrap0 = 0): planes -1 and nl are the ghost planes of u
        const int zm = (z0 == 0 && wrap0) ? n - 1 : z0 - 1;
        const int zn = (z0 + 1 == n && wrap0) ? 0 : z0 + 1;
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                prv[f][c] = uval(f, c, zm, col);
                cur[f][c] = uval(f, c, z0, col);
                nxt[f][c] = uval(f, c, zn, col);
                ring[f][c] = ringer ? uval(f, c, z0, roff) : 0.0;
            }
#pragma unroll
        for (int q = 0; q < 9; ++q) fv[q] = __ldg(&F[(int64_t)q * M + (int64_t)z0 * nn + col]);
    }
    double acc[2] = {0.0, 0.0};
    for (int z = z0; z < z0 + RT_ZC; ++z) {
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                sm[f][c][ty + 1][tx + 1] = cur[f][c];
                if (ringer) sm[f][c][rsy][rsx] = ring[f][c];
            }
        __syncthreads();
        // prefetch plane z + 1 (ring, F) and z + 2 (column)
        const bool more = z + 1 < z0 + RT_ZC;
        const int z1 = wrap0 ? (z + 1) % n : z + 1, z2 = wrap0 ? (z + 2) % n : z + 2;
        double nn2[2][3], ring1[2][3], fv1[9];
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                nn2[f][c] = more ? uval(f, c, z2, col) : 0.0;
                ring1[f][c] = (more && ringer) ? uval(f, c, z1, roff) : 0.0;
            }
#pragma unroll
        for (int q = 0; q < 9; ++q)
            fv1[q] = more ? __ldg(&F[(int64_t)q * M + (int64_t)z1 * nn + col]) : 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            double up_n[3], dn_n[3], up_o[3], dn_o[3];
            up_n[0] = nxt[0][i]; dn_n[0] = prv[0][i];
            up_o[0] = nxt[1][i]; dn_o[0] = prv[1][i];
            up_n[1] = sm[0][i][ty + 2][tx + 1]; dn_n[1] = sm[0][i][ty][tx + 1];
            up_o[1] = sm[1][i][ty + 2][tx + 1]; dn_o[1] = sm[1][i][ty][tx + 1];
            up_n[2] = sm[0][i][ty + 1][tx + 2]; dn_n[2] = sm[0][i][ty + 1][tx];
            up_o[2] = sm[1][i][ty + 1][tx + 2]; dn_o[2] = sm[1][i][ty + 1][tx];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const int q = i * 3 + j;
                const double gold = (up_o[j] - dn_o[j]) * inv2h + umo.v[q];
                const double gnew = (up_n[j] - dn_n[j]) * inv2h + um.v[q];  // projection.py:168
                const double dg = gnew - gold;                              // solver.py:271
                const double mis = gnew - fv[q];                            // solver.py:277
                acc[0] += dg * dg;
                acc[1] += mis * mis;
            }
        }
        __syncthreads();
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                prv[f][c] = cur[f][c];
                cur[f][c] = nxt[f][c];
                nxt[f][c] = nn2[f][c];
                ring[f][c] = ring1[f][c];
            }
#pragma unroll
        for (int q = 0; q < 9; ++q) fv[q] = fv1[q];
    }
    const int ops[2] = {RED_SUM, RED_SUM};
    block_reduce<2>(acc, ops, red_sm);
    double fin[2];
    if (grid_finalize<2>(acc, ops, partials, red_out, count, red_sm, fin) && dec.on)
        decide_step(fin[0], fin[1], dec);
}

// stencil divergence of F into Ut: (div F)_i = sum_j (F_ij(x+e_j) - F_ij(x-e_j)) / (2h)
template <int DIM>
__global__ void __launch_bounds__(256)
k_div(const double *__restrict__ F, double *__restrict__ Ut, int n, int lgn, int64_t M,
      double inv2h) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M;
         p += (int64_t)gridDim.x * blockDim.x) {
        int off_p[DIM], off_m[DIM];
        nbr_offsets<DIM>(p, n, lgn, off_p, off_m);
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < DIM; ++j) {
                const double *f = F + (int64_t)(i * DIM + j) * M + p;
                s += (__ldg(f + off_p[j]) - __ldg(f + off_m[j])) * inv2h;
            }
            Ut[(int64_t)i * M + p] = s;
        }
    }
}

// ---------------------------------------------------------------------------
// host-side dispatch
// ---------------------------------------------------------------------------
bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

int ilog2_(int n) {
    if (!is_pow2(n)) return -1;
    int l = 0;
    while ((1 << l) < n) ++l;
    return l;
}

// (N1, N2) factorisation for the register four-step; (0,0) = exact DFT path
void factor(int N, int &N1, int &N2) {
    N1 = N2 = 0;
    if (!is_pow2(N) || N > 1024) return;
    switch (N) {
        case 1: N1 = 1; N2 = 1; break;
        case 2: N1 = 2; N2 = 1; break;
        case 4: N1 = 4; N2 = 1; break;
        case 8: N1 = 8; N2 = 1; break;
        case 16: N1 = 4; N2 = 4; break;
        case 32: N1 = 8; N2 = 4; break;
        case 64: N1 = 8; N2 = 8; break;
        case 128: N1 = 16; N2 = 8; break;
        case 256: N1 = 16; N2 = 16; break;
        case 512: N1 = 32; N2 = 16; break;
        case 1024: N1 = 32; N2 = 32; break;
    }
}

template <typename Kern>
int launch_smem(mm_ctx *ctx, Kern kern, dim3 grid, int threads, size_t smem) {
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess)
            return mm_fail(ctx, MM_ERR_CUDA, "smem attribute (%zu B): %s", smem,
                           cudaGetErrorString(e));
    }
    return MM_OK;
}

template <int N1, int N2, int DIM, int ROWS>
int run_rows_t(mm_ctx *ctx, bool fwd, double rho, const RowGeom &g, const double2 *tw_line,
               double *u_out, const double *fsrc) {
    using C = RowCfg<N1, N2, DIM, ROWS>;
    const int threads = C::NT;
    const size_t smem = sizeof(double2) * (size_t)(g.N + 1) * (C::TK + 1) * (N1 ? 1 : 2);
    dim3 grid((unsigned)((g.nrows + ROWS - 1) / ROWS));
    if (fwd) {
        if constexpr (N1 == 16 && N2 == 8 && DIM == 3) {
            if (fsrc && MM_ROWFWD_W && g.packed && !g.hhi && !ctx->slab_mode && g.nrows % 4 == 0 &&
                ctx->opt_rowfwd_w) {
                const int64_t tasks = 3 * (g.nrows / 4);
                const unsigned blocks = (unsigned)((tasks + RFW_WARPS - 1) / RFW_WARPS);
                k_row_fwd_w<<<blocks, 32 * RFW_WARPS, 0, ctx->stream>>>(fsrc, ctx->spec, g, tw_line,
                                                                       ctx->tw_r2c);
                MM_LAUNCH_CHECK(ctx);
                return MM_OK;
            }
        }
        if (fsrc) {
            // divergence of the given field alone (T supplied, or a stress field)
            auto kern = k_row_fwd<N1, N2, DIM, ROWS, false>;
            int rc = launch_smem(ctx, kern, grid, threads, smem);
            if (rc) return rc;
            kern<<<grid, threads, smem, ctx->stream>>>(fsrc, nullptr, rho, ctx->spec, g, tw_line,
                                                       ctx->tw_r2c);
        } else {
            auto kern = k_row_fwd<N1, N2, DIM, ROWS, true>;
            int rc = launch_smem(ctx, kern, grid, threads, smem);
            if (rc) return rc;
            kern<<<grid, threads, smem, ctx->stream>>>(ctx->F, ctx->Lam, rho, ctx->spec, g,
                                                       tw_line, ctx->tw_r2c);
        }
    } else if (DIM == 3 && N1 * N2 >= 16 && N1 * N2 <= MM_ROWINV_P_MAXN && g.packed &&
               (g.plane || (MM_ROWINV_P_ROWS && !ctx->slab_mode)) && ctx->opt_rowinv_p) {
        // persistent, double-buffered (plane layout, and the row layout of
        // single-GPU grids up to n = 2 * MM_ROWINV_P_MAXN)
        auto kern = k_row_inv_p<N1 * N2 >= 16 ? N1 : 4, N1 * N2 >= 16 ? N2 : 4, 3, ROWS>;
        const size_t smem2 = sizeof(double2) * (size_t)(g.N + 1) * (C::TK + 1) * 2;
        int rc = launch_smem(ctx, kern, dim3(1), threads, smem2);
        if (rc) return rc;
        using CI = RowCfg<N1 * N2 >= 16 ? N1 : 4, N1 * N2 >= 16 ? N2 : 4, 3, ROWS>;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, CI::NTI, smem2);
        if (per_sm < 1) per_sm = 1;
        const int ntiles = (int)grid.x;
        const int blocks = std::min(ntiles, per_sm * ctx->num_sms);
        kern<<<blocks, CI::NTI, smem2, ctx->stream>>>(ctx->spec, u_out, g, tw_line, ctx->tw_r2c,
                                                      ntiles);
    } else {
        auto kern = k_row_inv<N1, N2, DIM, ROWS>;
        int rc = launch_smem(ctx, kern, grid, C::NTI, smem);
        if (rc) return rc;
        kern<<<grid, C::NTI, smem, ctx->stream>>>(ctx->spec, u_out, g, tw_line, ctx->tw_r2c);
    }
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

template <int N1, int N2>
int run_rows_n(mm_ctx *ctx, bool fwd, double rho, const RowGeom &g, const double2 *tw,
               double *u_out, const double *fsrc) {
    // 4 rows per tile (2 for 32-point register FFTs): <= 384 threads, 3-4 tiles per SM
    constexpr bool big = N1 >= 32;
    if (g.dim == 2) return run_rows_t<N1, N2, 2, big ? 2 : 4>(ctx, fwd, rho, g, tw, u_out, fsrc);
    static int rows_env = -1;
    if (rows_env < 0) {
        const char *e = getenv("MM_PLANE_ROWS");
        rows_env = e ? atoi(e) : 4;
    }
    // plane layout: ROWS consecutive rows give ROWS x 16 B runs per (c, k2)
    if constexpr (!big)
        if (g.plane && rows_env == 8) return run_rows_t<N1, N2, 3, 8>(ctx, fwd, rho, g, tw, u_out, fsrc);
    return run_rows_t<N1, N2, 3, big ? 2 : 4>(ctx, fwd, rho, g, tw, u_out, fsrc);
}

int run_rows(mm_ctx *ctx, bool fwd, double rho, double *u_out = nullptr,
             const double *fsrc = nullptr, bool plane = false) {
    RowGeom g;
    g.plane = plane ? 1 : 0;
    g.n = ctx->n;
    g.dim = ctx->dim;
    g.M = ctx->M;
    g.nrows = ctx->nrows;
    g.P = ctx->P;
    g.packed = (ctx->n % 2 == 0) ? 1 : 0;
    g.N = g.packed ? ctx->n / 2 : ctx->n;
    g.nl = ctx->slab_mode ? ctx->slab_nl : ctx->n;
    g.hlo = ctx->slab_mode ? ctx->halo_in_lo : nullptr;
    g.hhi = ctx->slab_mode ? ctx->halo_in_hi : nullptr;
    g.uM = ctx->uM;
    const double2 *tw = g.packed ? ctx->tw_half : ctx->tw_full;
    int N1, N2;
    factor(g.N, N1, N2);
    switch (N1 * 100 + N2) {
#define CASE(a, b) \
    case a * 100 + b: return run_rows_n<a, b>(ctx, fwd, rho, g, tw, u_out, fsrc);
        CASE(1, 1) CASE(2, 1) CASE(4, 1) CASE(8, 1) CASE(4, 4) CASE(8, 4) CASE(8, 8)
        CASE(16, 8) CASE(16, 16) CASE(32, 16) CASE(32, 32)
#undef CASE
        default: return run_rows_n<0, 0>(ctx, fwd, rho, g, tw, u_out, fsrc);
    }
}

template <int N1, int N2, int MODE>
int run_col_t(mm_ctx *ctx, const ColGeom &g, int n_outer) {
    constexpr int TK = ColCfg<N1, N2>::TK;
    const int threads = ColCfg<N1, N2>::NT;
    if constexpr (N1 * N2 >= 16 && (MODE == COL_FWD || MODE == COL_INV)) {
        // persistent pipelined variant
        const size_t smem2 = sizeof(double2) * (size_t)g.N * (TK + 1) * 2;
        auto kern = k_colp<N1, N2, MODE>;
        int rc = launch_smem(ctx, kern, dim3(1), threads, smem2);
        if (rc) return rc;
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem2);
        if (per_sm < 1) per_sm = 1;
        TileMap tm{(g.ncol + TK - 1) / TK, n_outer};
        const int ntiles = tm.ntk * n_outer * ctx->dim;
        const int blocks = std::min(ntiles, per_sm * ctx->num_sms);
        kern<<<blocks, threads, smem2, ctx->stream>>>(ctx->spec, g, ctx->tw_full, tm, ntiles);
        MM_LAUNCH_CHECK(ctx);
        return MM_OK;
    }
    const size_t smem = sizeof(double2) * (size_t)g.N * (TK + 1) * (N1 ? 1 : 2);
    dim3 grid((unsigned)((g.ncol + TK - 1) / TK), (unsigned)n_outer, (unsigned)ctx->dim);
    auto kern = k_col<N1, N2, MODE>;
    int rc = launch_smem(ctx, kern, grid, threads, smem);
    if (rc) return rc;
    kern<<<grid, threads, smem, ctx->stream>>>(ctx->spec, g, ctx->tw_full);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

template <int MODE>
int run_col(mm_ctx *ctx, const ColGeom &g, int n_outer) {
    int N1, N2;
    factor(g.N, N1, N2);
    switch (N1 * 100 + N2) {
#define CASE(a, b) \
    case a * 100 + b: return run_col_t<a, b, MODE>(ctx, g, n_outer);
        CASE(1, 1) CASE(2, 1) CASE(4, 1) CASE(8, 1) CASE(4, 4) CASE(8, 4) CASE(8, 8)
        CASE(16, 8) CASE(16, 16) CASE(32, 16) CASE(32, 32)
#undef CASE
        default: return run_col_t<0, 0, MODE>(ctx, g, n_outer);
    }
}

#ifndef MM_PLANE_TMA  // 1: pass 2 of the plane FFT through TMA + mbarrier (plane_col_tma);
#define MM_PLANE_TMA 2  // 2: passes 1 and 3 too at n = 256 (plane_row_tma)
#endif

// Tensor map of the plane-layout spectrum for plane_col_tma: doubles, dims
// {2N (re/im along axis 1), N (axis 0), planes}, box {2 TK, N, 1}.  Encoded
// once per context through the driver entry point (no libcuda link).
int mm_plane_tensor_map(mm_ctx *ctx, int N, int TK, bool swz) {
    // the cache key includes the swizzle: tmap_n = N, negated for the swizzled map
    if (ctx->tmap_ok && ctx->tmap_src == ctx->spec && ctx->tmap_n == (swz ? -N : N)) return MM_OK;
    ctx->tmap_ok = false;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            cudaGetLastError();
            return MM_OK;  // no TMA: plane_pass's cp.async path
        }
        encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint64_t dims[3] = {(cuuint64_t)2 * N, (cuuint64_t)N,
                                (cuuint64_t)ctx->dim * (cuuint64_t)ctx->nh};
    const cuuint64_t strides[2] = {(cuuint64_t)N * 16, (cuuint64_t)N * N * 16};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * TK), (cuuint32_t)N, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    // swz (n = 256, TK = 8, 128 threads, MM_PLANE_TMA >= 2): the column tiles
    // use the 128-byte swizzle that col_fft_solve_256 indexes
    CUresult r = encode(&ctx->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ctx->spec, dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return mm_fail(ctx, MM_ERR_CUDA, "cuTensorMapEncodeTiled: %d", (int)r);
    // row tiles (passes 1 and 3, n = 256): doubles {256 (half a row), 2 halves,
    // N rows, planes}, box {256, 2, TK, 1}: TK whole rows, dense
    ctx->rmap_ok = false;
    if (N == 256) {
        const cuuint64_t rd[4] = {256, 2, (cuuint64_t)N, dims[2]};
        const cuuint64_t rs[3] = {256 * 8, (cuuint64_t)N * 16, (cuuint64_t)N * N * 16};
        const cuuint32_t rb[4] = {256, 2, (cuuint32_t)TK, 1};
        const cuuint32_t re[4] = {1, 1, 1, 1};
        r = encode(&ctx->rmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, ctx->spec, rd, rs, rb, re,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return mm_fail(ctx, MM_ERR_CUDA, "cuTensorMapEncodeTiled (rows): %d", (int)r);
        ctx->rmap_ok = true;
    }
    ctx->tmap_ok = true;
    ctx->tmap_src = ctx->spec;
    ctx->tmap_n = swz ? -N : N;
    return MM_OK;
}

template <int N1, int N2, int TK, int CS>
int run_plane_t(mm_ctx *ctx, const PlaneGeom &g) {
    using C = PlaneCfg<N1, N2, TK>;
    const size_t smem = sizeof(double2) * (size_t)C::N * (TK + 1) * 2;
    auto kern = k_plane<N1, N2, TK, CS>;
    int rc = launch_smem(ctx, kern, dim3(1), C::NT, smem);
    if (rc) return rc;
    if (CS > 8) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess)
            return mm_fail(ctx, MM_ERR_CUDA, "cluster size %d: %s", CS, cudaGetErrorString(e));
    }
    const int blocks = CS * ctx->dim * g.nh;
    int use_tma = 0;
    if (C::PPT == 16 && MM_PLANE_TMA) {
        // use_tma == 3 <=> the column map is swizzled (plane_col_swz)
        const bool swz =
            MM_PLANE_TMA >= 2 && MM_PLANE_COLSWZ && C::N == 256 && TK == 8 && C::NT == 128;
        if ((rc = mm_plane_tensor_map(ctx, C::N, TK, swz))) return rc;
        use_tma = ctx->tmap_ok ? 1 : 0;
        if (use_tma && MM_PLANE_TMA >= 2 && C::N == 256 && TK == 8 && C::NT == 128 &&
            ctx->rmap_ok)
            use_tma = swz ? 3 : 2;
    }
    kern<<<blocks, C::NT, smem, ctx->stream>>>(ctx->spec, g, ctx->tw_full, ctx->tmap, use_tma,
                                               ctx->rmap);
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

// cluster size per plane (MM_PLANE_CS overrides; tiles per pass must divide).
// 256^3: 8 CTAs per plane keeps ~52 planes (52 MB) in flight, which stay in
// L2 between the passes (DRAM 1.11x the algorithmic bytes); 4 per plane ran
// 104 planes and moved 2.2x at the same time (ncu, tools/gpu_ncu_plane.sh)
template <int N1, int N2, int TK>
int run_plane_tk(mm_ctx *ctx, const PlaneGeom &g) {
    constexpr int NTILE = N1 * N2 / TK;
    static int cs_env = -1;
    if (cs_env < 0) {
        const char *e = getenv("MM_PLANE_CS");
        cs_env = e ? atoi(e) : 0;
    }
    int cs = cs_env > 0 ? cs_env : (N1 * N2 >= 256 ? 8 : N1 * N2 >= 128 ? 4 : N1 * N2 >= 64 ? 2 : 1);
    while (cs > 1 && (cs > NTILE || NTILE % cs)) cs >>= 1;
    switch (cs) {
        case 16: if constexpr (NTILE % 16 == 0) return run_plane_t<N1, N2, TK, 16>(ctx, g); [[fallthrough]];
        case 8: if constexpr (NTILE % 8 == 0) return run_plane_t<N1, N2, TK, 8>(ctx, g); [[fallthrough]];
        case 4: if constexpr (NTILE % 4 == 0) return run_plane_t<N1, N2, TK, 4>(ctx, g); [[fallthrough]];
        case 2: if constexpr (NTILE % 2 == 0) return run_plane_t<N1, N2, TK, 2>(ctx, g); [[fallthrough]];
        default: return run_plane_t<N1, N2, TK, 1>(ctx, g);
    }
}

template <int N1, int N2>
int run_plane_n(mm_ctx *ctx, const PlaneGeom &g) {
    static int tk_env = -1;
    if (tk_env < 0) {
        const char *e = getenv("MM_PLANE_TK");
        tk_env = e ? atoi(e) : 8;
    }
    if (tk_env == 16 && N1 * N2 >= 64) return run_plane_tk<N1, N2, 16>(ctx, g);
    if (tk_env == 4) return run_plane_tk<N1, N2, 4>(ctx, g);
    return run_plane_tk<N1, N2, 8>(ctx, g);
}

bool plane_eligible(const mm_ctx *ctx) {
    return ctx->opt_plane && ctx->dim == 3 && !ctx->slab_mode && is_pow2(ctx->n) && ctx->n >= 16 &&
           ctx->n <= 256;
}

int run_plane(mm_ctx *ctx, double scale) {
    PlaneGeom g;
    g.n = ctx->n;
    g.nh = ctx->nh;
    g.sym = ctx->sym;
    g.thresh = ctx->sym_thresh;
    g.scale = scale;
    switch (ctx->n) {
        case 16: return run_plane_n<4, 4>(ctx, g);
        case 32: return run_plane_n<8, 4>(ctx, g);
        case 64: return run_plane_n<8, 8>(ctx, g);
        case 128: return run_plane_n<16, 8>(ctx, g);
        case 256:
            if (MM_PLANE_HW) {
                constexpr int NTH = MM_PLANE_HW_NT, CS = 8;
                const size_t smem = sizeof(double2) * 2 * 256 * (NTH / 16);
                auto kern = k_plane_hw<NTH, CS>;
                int rc = launch_smem(ctx, kern, dim3(1), NTH, smem);
                if (rc) return rc;
                kern<<<CS * ctx->dim * g.nh, NTH, smem, ctx->stream>>>(ctx->spec, g, ctx->tw_full);
                MM_LAUNCH_CHECK(ctx);
                return MM_OK;
            }
            return run_plane_n<16, 16>(ctx, g);
        default: return mm_fail(ctx, MM_ERR_CONFIG, "plane FFT needs n in 16..256 (pow2)");
    }
}

bool g_const_ready[64] = {false};

int ensure_constants(mm_ctx *ctx) {
    if (ctx->device >= 0 && ctx->device < 64 && g_const_ready[ctx->device]) return MM_OK;
    double2 w[32];
    for (int k = 0; k < 32; ++k) {
        long double a = -2.0L * 3.141592653589793238462643383279502884L * k / 32.0L;
        w[k].x = (double)cosl(a);
        w[k].y = (double)sinl(a);
    }
    MM_CUDA(ctx, cudaMemcpyToSymbol(c_w32, w, sizeof w));
    if (ctx->device >= 0 && ctx->device < 64) g_const_ready[ctx->device] = true;
    return MM_OK;
}

}  // namespace

// A (divergence + R2C rows), the column passes with the solve, E (C2R rows
// -> u_new): the part of the projection that does not need u_mean
int mm_run_project_front(mm_ctx *ctx, double rho, int update, double **u_new_out) {
    int rc = ensure_constants(ctx);
    if (rc) return rc;
    const int n = ctx->n, d = ctx->dim;
    const bool plane = plane_eligible(ctx);
    // A: divergence + R2C rows (of the T field the fused pass left, when
    // it is current for this rho)
    {
        StageScope ss(ctx, MM_STAGE_ROW_FWD);
        const bool useT = ctx->T_valid && ctx->Tbuf && ctx->T_rho == rho && !ctx->slab_mode;
        if ((rc = run_rows(ctx, true, rho, nullptr, useT ? ctx->Tbuf : nullptr, plane))) return rc;
    }
    ColGeom g;
    g.N = n;
    g.ncol = ctx->nh;
    g.n = n;
    g.dim = d;
    g.sym = ctx->sym;
    g.thresh = ctx->sym_thresh;
    double nd = 1.0;
    for (int i = 0; i < d; ++i) nd *= (double)n;
    g.scale = 1.0 / (2.0 * ctx->h) / nd;
    if (plane) {
        // B + C + D: one cluster per (component, k2) plane
        StageScope ss(ctx, MM_STAGE_PLANE);
        if ((rc = run_plane(ctx, g.scale))) return rc;
    } else if (d == 3) {
        // spectral index ((c*n + i0)*n + i1)*P + k2
        ColGeom gy = g;
        gy.es = ctx->P;
        gy.os = (int64_t)n * ctx->P;
        gy.cs = (int64_t)n * n * ctx->P;
        ColGeom gz = g;
        gz.es = (int64_t)n * ctx->P;
        gz.os = ctx->P;
        gz.cs = gy.cs;
        {
            StageScope ss(ctx, MM_STAGE_COL_FWD);
            if ((rc = run_col<COL_FWD>(ctx, gy, n))) return rc;
        }
        {
            StageScope ss(ctx, MM_STAGE_COL_SOLVE);
            if ((rc = run_col<COL_SOLVE>(ctx, gz, n))) return rc;
        }
        {
            StageScope ss(ctx, MM_STAGE_COL_INV);
            if ((rc = run_col<COL_INV>(ctx, gy, n))) return rc;
        }
    } else {
        ColGeom gz = g;
        gz.es = ctx->P;
        gz.os = 0;
        gz.cs = (int64_t)n * ctx->P;
        StageScope ss(ctx, MM_STAGE_COL_SOLVE);
        if ((rc = run_col<COL_SOLVE>(ctx, gz, 1))) return rc;
    }
    // E: C2R rows -> u (new buffer on the solver path)
    double *u_new = ctx->Ut;
    if (update == 2 || (update && ctx->opt_implicit_g)) {
        if (!ctx->Ut2 && (rc = mm_alloc(ctx, (void **)&ctx->Ut2, sizeof(double) * d * ctx->M)))
            return rc;
        u_new = ctx->Ut2;
    }
    {
        StageScope ss(ctx, MM_STAGE_ROW_INV);
        if ((rc = run_rows(ctx, false, rho, u_new, nullptr, plane))) return rc;
    }
    *u_new_out = u_new;
    return MM_OK;
}

int mm_run_project(mm_ctx *ctx, double rho, const double *u_mean, int update,
                   mm_update_stats *out) {
    int rc;
    const int n = ctx->n, d = ctx->dim;
    double *u_new = nullptr;
    if (update == 2 && ctx->front_valid && ctx->front_rho == rho && ctx->front_gen == ctx->gen &&
        ctx->Ut2) {
        u_new = ctx->Ut2;  // launched by mm_update_and_sweep behind the fused pass
    } else if ((rc = mm_run_project_front(ctx, rho, update, &u_new))) {
        ctx->front_valid = false;
        return rc;
    }
    ctx->front_valid = false;
    // F: gradient (+ ascent and residual sums)
    Mean9 um, umo;
    for (int i = 0; i < 9; ++i) {
        um.v[i] = i < ctx->D ? u_mean[i] : 0.0;
        umo.v[i] = ctx->ubar[i];
    }
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((ctx->M + threads - 1) / threads, 148 * 8);
    if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
    const double inv2h = 1.0 / (2.0 * ctx->h);
    const int lgn = ilog2_(n);
    const int mode = !update ? GRAD_WRITE
                     : update == 2 ? (ctx->g_implicit ? GRAD_RES_IMPL : GRAD_RES_EXPL)
                     : !ctx->opt_implicit_g ? GRAD_EXPLW
                     : (ctx->g_implicit ? GRAD_IMPL : GRAD_EXPL);
    double *rout = ctx->k1_dst ? ctx->k1_dst : ctx->red_out;  // pipelined step: second slot
    DecideArgs dec = ctx->k1_decide;
    if (update != 2) dec.on = 0;
#define LAUNCH(DIM, MODE)                                                                       \
    k_grad<DIM, MODE><<<blocks, threads, 0, ctx->stream>>>(u_new, ctx->Ut, ctx->G, ctx->F,       \
                                                           ctx->Lam, n, lgn, ctx->M, inv2h, rho, \
                                                           um, umo, ctx->partials, rout,         \
                                                           ctx->red_count, ctx->uM,              \
                                                           ctx->slab_mode ? 0 : 1, dec)
    const int nplanes = ctx->slab_mode ? ctx->slab_nl : n;
    const bool march = d == 3 && mode == GRAD_RES_IMPL && n % RT_X == 0 && n % RT_Y == 0 &&
                       nplanes % RT_ZC == 0 && ctx->opt_march;
    if (march) {
        StageScope ss(ctx, MM_STAGE_GRAD);
        dim3 grid(n / RT_X, n / RT_Y, nplanes / RT_ZC);
        if ((rc = mm_ensure_partials(ctx, (int64_t)grid.x * grid.y * grid.z))) return rc;
        k_res_march<<<grid, RT_X * RT_Y, 0, ctx->stream>>>(
            u_new, ctx->Ut, ctx->F, n, ctx->M, inv2h, um, umo, ctx->partials, rout,
            ctx->red_count, ctx->uM, ctx->slab_mode ? 0 : 1, dec);
    } else {
        StageScope ss(ctx, MM_STAGE_GRAD);
        if (d == 2) {
            if (mode == GRAD_WRITE) LAUNCH(2, GRAD_WRITE);
            else if (mode == GRAD_EXPL) LAUNCH(2, GRAD_EXPL);
            else if (mode == GRAD_EXPLW) LAUNCH(2, GRAD_EXPLW);
            else if (mode == GRAD_RES_EXPL) LAUNCH(2, GRAD_RES_EXPL);
            else if (mode == GRAD_RES_IMPL) LAUNCH(2, GRAD_RES_IMPL);
            else LAUNCH(2, GRAD_IMPL);
        } else {
            if (mode == GRAD_WRITE) LAUNCH(3, GRAD_WRITE);
            else if (mode == GRAD_EXPL) LAUNCH(3, GRAD_EXPL);
            else if (mode == GRAD_EXPLW) LAUNCH(3, GRAD_EXPLW);
            else if (mode == GRAD_RES_EXPL) LAUNCH(3, GRAD_RES_EXPL);
            else if (mode == GRAD_RES_IMPL) LAUNCH(3, GRAD_RES_IMPL);
            else LAUNCH(3, GRAD_IMPL);
        }
    }
#undef LAUNCH
    MM_LAUNCH_CHECK(ctx);
    for (int i = 0; i < 9; ++i) ctx->ubar[i] = um.v[i];
    if (!update) {
        // grad_u written explicitly
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
        return MM_OK;
    }
    if (update == 1) ctx->T_valid = false;  // lam changed
    if (update == 2 || ctx->opt_implicit_g) {
        // new u becomes current; grad_u is now ubar + D u (implicit)
        std::swap(ctx->Ut, ctx->Ut2);
        ctx->g_implicit = true;
        ctx->g_buf_valid = false;
    } else {
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    }
    if (update == 2) {
        ctx->lam_pending = true;  // lam += rho (grad_u - F) deferred (mm_run_update)
        ctx->pending_rho = rho;
    }
    if (!out) return MM_OK;  // pipelined step: the sums are read later (k1_dst)
    double r[MM_MAX_PARTIALS];
    const int K = 2 + ctx->D;
    if ((rc = mm_fetch_reduction(ctx, K, r))) return rc;
    out->sum_dG2 = r[0];
    out->sum_mis2 = r[1];
    for (int i = 0; i < 9; ++i) out->sum_lam[i] = (i < ctx->D && update != 2) ? r[2 + i] : 0.0;
    return MM_OK;
}

// ||div P||_{H^-1} / npts of a stress field P (SoA, d*d components):
// stencil divergence + R2C rows, FFT along axis 1 (3D), then the FFT along
// axis 0 with the weighted |.|^2 sum in the same pass (COL_NORM).  The
// spectral divergence of the reference (solver.py:364-371) is the DFT of the
// central-difference divergence, which the row pass computes unscaled
// (2h times larger): the 1/(4h^2) is applied to the sum.
int mm_run_eq_residual(mm_ctx *ctx, const double *P, double *out) {
    int rc = ensure_constants(ctx);
    if (rc) return rc;
    const int n = ctx->n, d = ctx->dim;
    {
        StageScope ss(ctx, MM_STAGE_OTHER);
        if ((rc = run_rows(ctx, true, 1.0, nullptr, P))) return rc;
    }
    ColGeom g;
    g.N = n;
    g.ncol = ctx->nh;
    g.n = n;
    g.dim = d;
    g.sym = ctx->sym;
    g.thresh = ctx->sym_thresh;
    g.scale = 1.0;
    ColGeom gz = g;
    if (d == 3) {
        ColGeom gy = g;
        gy.es = ctx->P;
        gy.os = (int64_t)n * ctx->P;
        gy.cs = (int64_t)n * n * ctx->P;
        gz.es = (int64_t)n * ctx->P;
        gz.os = ctx->P;
        gz.cs = gy.cs;
        StageScope ss(ctx, MM_STAGE_OTHER);
        if ((rc = run_col<COL_FWD>(ctx, gy, n))) return rc;
    } else {
        gz.es = ctx->P;
        gz.os = 0;
        gz.cs = (int64_t)n * ctx->P;
    }
    const int n_outer = d == 3 ? n : 1;
    const int64_t nb = (int64_t)((ctx->nh + 7) / 8) * n_outer * d;
    if ((rc = mm_ensure_partials(ctx, nb))) return rc;
    gz.partials = ctx->partials;
    gz.red_out = ctx->red_out;
    gz.count = ctx->red_count;
    {
        StageScope ss(ctx, MM_STAGE_OTHER);
        if ((rc = run_col<COL_NORM>(ctx, gz, n_outer))) return rc;
    }
    double total;
    if ((rc = mm_fetch_reduction(ctx, 1, &total))) return rc;
    const double h = ctx->h;
    *out = sqrt(total / (4.0 * h * h)) / (double)ctx->M;
    return MM_OK;
}

int mm_ilog2(int n) { return ilog2_(n); }

GSrc mm_gsrc(mm_ctx *ctx) {
    GSrc s;
    const bool impl = ctx->g_implicit && !ctx->g_buf_valid;
    s.G = impl ? nullptr : ctx->G;
    s.U = ctx->Ut;
    for (int i = 0; i < 9; ++i) s.ubar[i] = ctx->ubar[i];
    s.n = ctx->n;
    s.lgn = ctx->points_only ? -1 : ilog2_(ctx->n);
    s.inv2h = ctx->points_only ? 0.0 : 1.0 / (2.0 * ctx->h);
    s.M = ctx->M;
    s.uM = ctx->uM;
    s.wrap0 = ctx->slab_mode ? 0 : 1;
    return s;
}

// fill the G buffer from the implicit form (ubar + D u_tilde)
int mm_materialize_G(mm_ctx *ctx) {
    if (!ctx->g_implicit || ctx->g_buf_valid) return MM_OK;
    Mean9 um, umo;
    for (int i = 0; i < 9; ++i) um.v[i] = umo.v[i] = ctx->ubar[i];
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((ctx->M + threads - 1) / threads, 148 * 8);
    const double inv2h = 1.0 / (2.0 * ctx->h);
    const int lgn = ilog2_(ctx->n);
    {
        StageScope ss(ctx, MM_STAGE_OTHER);
        if (ctx->dim == 2)
            k_grad<2, GRAD_WRITE><<<blocks, threads, 0, ctx->stream>>>(
                ctx->Ut, ctx->Ut, ctx->G, ctx->F, ctx->Lam, ctx->n, lgn, ctx->M, inv2h, 0.0, um,
                umo, nullptr, nullptr, nullptr, ctx->uM, ctx->slab_mode ? 0 : 1, DecideArgs{});
        else
            k_grad<3, GRAD_WRITE><<<blocks, threads, 0, ctx->stream>>>(
                ctx->Ut, ctx->Ut, ctx->G, ctx->F, ctx->Lam, ctx->n, lgn, ctx->M, inv2h, 0.0, um,
                umo, nullptr, nullptr, nullptr, ctx->uM, ctx->slab_mode ? 0 : 1, DecideArgs{});
    }
    MM_LAUNCH_CHECK(ctx);
    ctx->g_buf_valid = true;
    return MM_OK;
}

int mm_run_stencil(mm_ctx *ctx, int op) {
    StageScope ss(ctx, MM_STAGE_OTHER);
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((ctx->M + threads - 1) / threads, 148 * 8);
    const double inv2h = 1.0 / (2.0 * ctx->h);
    if (op == 0) {
        Mean9 um;
        for (int i = 0; i < 9; ++i) um.v[i] = 0.0;
        if (ctx->dim == 2)
            k_grad<2, GRAD_WRITE><<<blocks, threads, 0, ctx->stream>>>(
                ctx->Ut, ctx->Ut, ctx->G, ctx->F, ctx->Lam, ctx->n, ilog2_(ctx->n), ctx->M, inv2h,
                0.0, um, um, nullptr, nullptr, nullptr, ctx->uM, 1, DecideArgs{});
        else
            k_grad<3, GRAD_WRITE><<<blocks, threads, 0, ctx->stream>>>(
                ctx->Ut, ctx->Ut, ctx->G, ctx->F, ctx->Lam, ctx->n, ilog2_(ctx->n), ctx->M, inv2h,
                0.0, um, um, nullptr, nullptr, nullptr, ctx->uM, 1, DecideArgs{});
        ctx->g_implicit = false;
        ctx->g_buf_valid = true;
    } else {
        if (ctx->dim == 2)
            k_div<2><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->Ut, ctx->n, ilog2_(ctx->n),
                                                          ctx->M, inv2h);
        else
            k_div<3><<<blocks, threads, 0, ctx->stream>>>(ctx->F, ctx->Ut, ctx->n, ilog2_(ctx->n),
                                                          ctx->M, inv2h);
    }
    MM_LAUNCH_CHECK(ctx);
    return MM_OK;
}

// ===========================================================================
// Slab decomposition (one rank's part of a 3D grid split along axis 0).
// The host moves halos and runs the two all-to-all transposes with NCCL
// (paper_2010_06697_b200/slab.py); these entry points are the per-rank compute.
// ===========================================================================
namespace {

// T_c0 (or u) of the first / last local plane -> halo send buffers [c][i1*n + x]
__global__ void k_slab_halo(const double *__restrict__ A, const double *__restrict__ B,
                            double irho, int stride_c, int nc, int n, int nl, int64_t M,
                            double *__restrict__ lo, double *__restrict__ hi) {
    const int64_t nn = (int64_t)n * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc * nn;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i / nn);
        const int64_t q = i - c * nn;
        const int64_t comp = (int64_t)c * stride_c * M;
        const int64_t o0 = comp + q, o1 = comp + (int64_t)(nl - 1) * nn + q;
        if (B) {  // T = F - lam * (1/rho), the expression the divergence uses
            lo[i] = A[o0] - B[o0] * irho;
            hi[i] = A[o1] - B[o1] * irho;
        } else {
            lo[i] = A[o0];
            hi[i] = A[o1];
        }
    }
}

// column transform with two-level line addressing, out of place:
// element j of a line sits at (j / blk) * sq + (j % blk) * es (+ outer, comp, column)
struct SlabCol {
    const double2 *src;
    double2 *dst;
    int blk_s, blk_d;
    int64_t s_sq, s_es, s_os, s_cs;
    int64_t d_sq, d_es, d_os, d_cs;
    int outer_off;  // global index of outer line 0 along axis 1 (solve symbols)
    // peer stores: block q of the destination lives in peers[q] + peer_off
    // (d_sq unused); nullptr = local destination
    double2 *const *peers;
    int64_t peer_off;
};

template <int N1, int N2, int MODE>
__global__ void __launch_bounds__(ColCfg<N1, N2>::NT)
k_col_slab(ColGeom g, SlabCol sc, const double2 *__restrict__ tw) {
    constexpr int TK = ColCfg<N1, N2>::TK, LD = TK + 1;
    extern __shared__ double2 smem_c[];
    double2 *buf = smem_c;
    double2 *scr = smem_c + (size_t)g.N * LD;
    const int k0 = blockIdx.x * TK;
    const int outer = blockIdx.y;
    const int comp = blockIdx.z;
    const int N = g.N;
    const double2 *sb = sc.src + comp * sc.s_cs + outer * sc.s_os + k0;
    double2 *db = sc.dst + comp * sc.d_cs + outer * sc.d_os + k0;
    for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
        const int n = w / TK, c = w - n * TK;
        double2 v = make_double2(0.0, 0.0);
        if (k0 + c < g.ncol) v = sb[(n / sc.blk_s) * sc.s_sq + (n % sc.blk_s) * sc.s_es + c];
        buf[n * LD + c] = v;
    }
    __syncthreads();
    if constexpr (MODE == COL_FWD || MODE == COL_SOLVE || MODE == COL_NORM)
        line_transform<N1, N2, TK, false>(buf, scr, N, tw);
    else
        line_transform<N1, N2, TK, true>(buf, scr, N, tw);
    if constexpr (MODE == COL_NORM) {
        __shared__ double red_sm[32];
        const double *s0 = g.sym;
        const double *slast = g.sym + (int64_t)(g.dim - 1) * g.n;
        const double s1 = (g.dim == 3) ? g.sym[g.n + outer] : 0.0;
        const int nyq = (g.n % 2 == 0) ? g.n / 2 : -1;
        double acc[1] = {0.0};
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int kl = w / TK, c = w - kl * TK;
            const int k2 = k0 + c;
            if (k2 >= g.ncol) continue;
            double gsq = s0[kl];
            if (g.dim == 3) gsq = gsq + s1;
            gsq = gsq + slast[k2];
            if (!(gsq > g.thresh)) continue;
            const double2 X = buf[kl * LD + c];
            const double m = (k2 == 0 || k2 == nyq) ? 1.0 : 2.0;
            acc[0] += m * (X.x * X.x + X.y * X.y) / gsq;
        }
        const int ops[1] = {RED_SUM};
        block_reduce<1>(acc, ops, red_sm);
        grid_finalize<1>(acc, ops, g.partials, g.red_out, g.count, red_sm);
        return;
    }
    if constexpr (MODE == COL_SOLVE) {
        const double *s0 = g.sym;
        const double *slast = g.sym + (int64_t)(g.dim - 1) * g.n;
        const double s1 = g.sym[g.n + sc.outer_off + outer];
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int kl = w / TK, c = w - kl * TK;
            double gsq = s0[kl];
            gsq = gsq + s1;
            gsq = gsq + slast[min(k0 + c, g.n - 1)];
            const double inv = (gsq > g.thresh) ? 1.0 / gsq : 0.0;
            buf[kl * LD + c] = cscale(buf[kl * LD + c], -inv * g.scale);
        }
        __syncthreads();
        line_transform<N1, N2, TK, true>(buf, scr, N, tw);
    }
    if (sc.peers) {
        // fused transpose: each element goes straight to the rank that owns
        // it (NVLink peer store); line element n belongs to block n / blk_d
        const int64_t loc = comp * sc.d_cs + outer * sc.d_os + k0 + sc.peer_off;
        for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
            const int n = w / TK, c = w - n * TK;
            if (k0 + c < g.ncol)
                sc.peers[n / sc.blk_d][loc + (n % sc.blk_d) * sc.d_es + c] = buf[n * LD + c];
        }
        // the peer stores are complete and visible system-wide before this
        // CTA retires, hence before the barrier that follows the kernel
        __threadfence_system();
        return;
    }
    for (int w = threadIdx.x; w < N * TK; w += blockDim.x) {
        const int n = w / TK, c = w - n * TK;
        if (k0 + c < g.ncol) db[(n / sc.blk_d) * sc.d_sq + (n % sc.blk_d) * sc.d_es + c] = buf[n * LD + c];
    }
}

template <int MODE>
int run_col_slab(mm_ctx *ctx, const ColGeom &g, const SlabCol &sc, int n_outer) {
    int N1, N2;
    factor(g.N, N1, N2);
    auto go = [&](auto kern, int threads, size_t smem) -> int {
        int rc = launch_smem(ctx, kern, dim3(1), threads, smem);
        if (rc) return rc;
        dim3 grid((unsigned)((g.ncol + 7) / 8), (unsigned)n_outer, 3u);
        kern<<<grid, threads, smem, ctx->stream>>>(g, sc, ctx->tw_full);
        MM_LAUNCH_CHECK(ctx);
        return MM_OK;
    };
    switch (N1 * 100 + N2) {
#define CASE(a, b)                                                                          \
    case a * 100 + b:                                                                       \
        return go(k_col_slab<a, b, MODE>, ColCfg<a, b>::NT,                                 \
                  sizeof(double2) * (size_t)g.N * 9);
        CASE(2, 1) CASE(4, 1) CASE(8, 1) CASE(4, 4) CASE(8, 4) CASE(8, 8) CASE(16, 8)
        CASE(16, 16) CASE(32, 16) CASE(32, 32)
#undef CASE
        default:
            return go(k_col_slab<0, 0, MODE>, 256, sizeof(double2) * (size_t)g.N * 9 * 2);
    }
}

}  // namespace

// K1 of the fused schedule on a slab (mm_run_project's residual pass): the
// u_new buffer (Ut2) was written by MM_SLAB_INV and its ghost planes filled
// by the halo exchange; u_old (Ut) keeps the ghosts of the previous
// exchange.  Then u_new becomes current, grad_u = ubar + D u (implicit) and
// the ascent is left pending for the fused update + local pass.
int mm_slab_res(mm_ctx *ctx, double rho, const double *u_mean, double *sums) {
    int rc;
    const int n = ctx->n;
    Mean9 um, umo;
    for (int i = 0; i < 9; ++i) {
        um.v[i] = u_mean[i];
        umo.v[i] = ctx->ubar[i];
    }
    const double inv2h = 1.0 / (2.0 * ctx->h);
    const int lgn = ilog2_(n);
    const int mode = ctx->g_implicit && !ctx->g_buf_valid ? GRAD_RES_IMPL : GRAD_RES_EXPL;
    double *u_new = ctx->Ut2;
    const int nl = ctx->slab_nl;
    const bool march = mode == GRAD_RES_IMPL && n % RT_X == 0 && n % RT_Y == 0 &&
                       nl % RT_ZC == 0 && ctx->opt_march;
    {
        StageScope ss(ctx, MM_STAGE_GRAD);
        if (march) {
            dim3 grid(n / RT_X, n / RT_Y, nl / RT_ZC);
            if ((rc = mm_ensure_partials(ctx, (int64_t)grid.x * grid.y * grid.z))) return rc;
            k_res_march<<<grid, RT_X * RT_Y, 0, ctx->stream>>>(
                u_new, ctx->Ut, ctx->F, n, ctx->M, inv2h, um, umo, ctx->partials, ctx->red_out,
                ctx->red_count, ctx->uM, 0, DecideArgs{});
        } else {
            const int threads = 256;
            const int blocks = (int)std::min<int64_t>((ctx->M + threads - 1) / threads, 148 * 8);
            if ((rc = mm_ensure_partials(ctx, blocks))) return rc;
            if (mode == GRAD_RES_IMPL)
                k_grad<3, GRAD_RES_IMPL><<<blocks, threads, 0, ctx->stream>>>(
                    u_new, ctx->Ut, ctx->G, ctx->F, ctx->Lam, n, lgn, ctx->M, inv2h, rho, um, umo,
                    ctx->partials, ctx->red_out, ctx->red_count, ctx->uM, 0, DecideArgs{});
            else
                k_grad<3, GRAD_RES_EXPL><<<blocks, threads, 0, ctx->stream>>>(
                    u_new, ctx->Ut, ctx->G, ctx->F, ctx->Lam, n, lgn, ctx->M, inv2h, rho, um, umo,
                    ctx->partials, ctx->red_out, ctx->red_count, ctx->uM, 0, DecideArgs{});
        }
    }
    MM_LAUNCH_CHECK(ctx);
    for (int i = 0; i < 9; ++i) ctx->ubar[i] = um.v[i];
    std::swap(ctx->Ut, ctx->Ut2);
    ctx->g_implicit = true;
    ctx->g_buf_valid = false;
    ctx->lam_pending = true;
    ctx->pending_rho = rho;
    double r[MM_MAX_PARTIALS];
    const int K = march ? 2 : 2 + ctx->D;
    if ((rc = mm_fetch_reduction(ctx, K, r))) return rc;
    sums[0] = r[0];
    sums[1] = r[1];
    return MM_OK;
}

int mm_run_slab_step(mm_ctx *ctx, int step, double rho, const double *u_mean, double *sums) {
    int rc = ensure_constants(ctx);
    if (rc) return rc;
    const int n = ctx->n, nl = ctx->slab_nl, P = ctx->slab_P;
    const int64_t M = ctx->M, nn = (int64_t)n * n;
    const int Pp = ctx->P;  // spectral pitch
    const int threads = 256;
    ColGeom g;
    g.N = n;
    g.ncol = ctx->nh;
    g.n = n;
    g.dim = 3;
    g.sym = ctx->sym;
    g.thresh = ctx->sym_thresh;
    g.scale = 1.0 / (2.0 * ctx->h) / ((double)n * n * n);
    g.es = g.os = g.cs = 0;
    // layouts: spec [c][i0l][i1][k2]; send/recv [q][c][i0l][i1l][k2]
    const int64_t spec_cs = (int64_t)nl * n * Pp, spec_os = (int64_t)n * Pp;
    const int64_t blk = 3LL * nl * nl * Pp;  // one destination block
    switch (step) {
        case MM_SLAB_HALO_T: {
            // T_c0 = (F - lam / rho)_{i0} of the first / last local plane: from
            // the T field the fused pass left when it is current for rho
            StageScope ss(ctx, MM_STAGE_OTHER);
            const bool tf = ctx->T_valid && ctx->T_rho == rho && ctx->Tbuf;
            const int blocks = (int)std::min<int64_t>((3 * nn + threads - 1) / threads, 148 * 8);
            k_slab_halo<<<blocks, threads, 0, ctx->stream>>>(
                tf ? ctx->Tbuf : ctx->F, tf ? nullptr : ctx->Lam, 1.0 / rho, 3, 3, n, nl, M,
                ctx->halo_out_lo, ctx->halo_out_hi);
            MM_LAUNCH_CHECK(ctx);
            return MM_OK;
        }
        case MM_SLAB_FWD:
        case MM_SLAB_FWD_PUSH: {
            const bool push = step == MM_SLAB_FWD_PUSH;
            if (push && !ctx->peer_recv)
                return mm_fail(ctx, MM_ERR_CONFIG, "FWD_PUSH: peer RECV buffers were never set");
            const bool tf = ctx->T_valid && ctx->T_rho == rho && ctx->Tbuf;
            {
                StageScope ss(ctx, MM_STAGE_ROW_FWD);
                if ((rc = run_rows(ctx, true, rho, nullptr, tf ? ctx->Tbuf : nullptr))) return rc;
            }
            SlabCol sc;
            sc.peers = push ? ctx->peer_recv : nullptr;
            sc.peer_off = (int64_t)ctx->slab_rank * blk;
            sc.src = ctx->spec;
            sc.dst = ctx->sendbuf;
            sc.blk_s = n;
            sc.s_sq = 0; sc.s_es = Pp; sc.s_os = spec_os; sc.s_cs = spec_cs;
            sc.blk_d = nl;  // i1 = q * nl + i1l
            sc.d_sq = blk; sc.d_es = Pp; sc.d_os = (int64_t)nl * Pp; sc.d_cs = (int64_t)nl * nl * Pp;
            sc.outer_off = 0;
            StageScope ss(ctx, MM_STAGE_COL_FWD);
            return run_col_slab<COL_FWD>(ctx, g, sc, nl);
        }
        case MM_SLAB_SOLVE:
        case MM_SLAB_SOLVE_PUSH: {
            // recv [s][c][i0l][i1l][k2]: line along i0 = s * nl + i0l, outer = i1l
            const bool push = step == MM_SLAB_SOLVE_PUSH;
            if (push && !ctx->peer_send)
                return mm_fail(ctx, MM_ERR_CONFIG, "SOLVE_PUSH: peer SEND buffers were never set");
            SlabCol sc;
            sc.peers = push ? ctx->peer_send : nullptr;
            sc.peer_off = (int64_t)ctx->slab_rank * blk;
            sc.src = ctx->recvbuf;
            sc.dst = ctx->recvbuf;
            sc.blk_s = sc.blk_d = nl;
            sc.s_sq = sc.d_sq = blk;
            sc.s_es = sc.d_es = (int64_t)nl * Pp;
            sc.s_os = sc.d_os = Pp;
            sc.s_cs = sc.d_cs = (int64_t)nl * nl * Pp;
            sc.outer_off = ctx->slab_rank * nl;
            StageScope ss(ctx, MM_STAGE_COL_SOLVE);
            return run_col_slab<COL_SOLVE>(ctx, g, sc, nl);
        }
        case MM_SLAB_INV: {
            // inverse axis-1 FFT from the returned send buffer, C2R rows into
            // the u_new buffer (data planes; its ghosts come from the exchange)
            SlabCol sc;
            sc.peers = nullptr;
            sc.peer_off = 0;
            sc.src = ctx->sendbuf;
            sc.dst = ctx->spec;
            sc.blk_s = nl;
            sc.s_sq = blk; sc.s_es = Pp; sc.s_os = (int64_t)nl * Pp; sc.s_cs = (int64_t)nl * nl * Pp;
            sc.blk_d = n;
            sc.d_sq = 0; sc.d_es = Pp; sc.d_os = spec_os; sc.d_cs = spec_cs;
            sc.outer_off = 0;
            {
                StageScope ss(ctx, MM_STAGE_COL_INV);
                if ((rc = run_col_slab<COL_INV>(ctx, g, sc, nl))) return rc;
            }
            StageScope ss(ctx, MM_STAGE_ROW_INV);
            return run_rows(ctx, false, rho, ctx->Ut2);
        }
        case MM_SLAB_RES: return mm_slab_res(ctx, rho, u_mean, sums);
        default: return mm_fail(ctx, MM_ERR_PARAM, "unknown slab step %d", step);
    }
    (void)P;
    (void)u_mean;
    (void)sums;
}
