/*
 * mm_admm.h — C-ABI of the B200-native ADMM outer iteration (arXiv 2010.06697).
 *
 * Drop-in boundary for the hot path of the reference package `micromech`
 * (paths relative to /root/reference/pkg/src/micromech).  Every entry point
 * names the reference interface it replaces.  Plain pointers, sizes and
 * doubles only; host arrays are C-order float64 in the reference's own
 * layout (grid axes first, tensor components innermost: "AoS"), borrowed for
 * the duration of the call.  Device fields are owned by the context and
 * kept component-major ("SoA") in HBM.
 *
 * Error convention (errors.py:21-69): every int-returning call returns one
 * of the MM_* status codes below; mm_last_error() gives the message.
 * Status -> Python exception mapping used by the host package:
 *   MM_ERR_PARAM        -> ParameterError
 *   MM_ERR_CONFIG       -> ConfigurationError
 *   MM_ERR_INADMISSIBLE -> InadmissibleStateError
 *   MM_ERR_DIVERGED     -> DivergenceError
 *   MM_ERR_CUDA         -> RuntimeError (device / driver failure)
 *
 * Threading: one context per GPU, not re-entrant; all work is issued on the
 * context's stream (solver.py runs a single orchestrating thread).
 */
#ifndef MM_ADMM_H
#define MM_ADMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MM_ABI_VERSION 2  /* 2: mm_local_stats gained sum_nsw; mm_struct_size */

enum mm_status {
    MM_OK = 0,
    MM_ERR_PARAM = 1,
    MM_ERR_CONFIG = 2,
    MM_ERR_INADMISSIBLE = 3,
    MM_ERR_DIVERGED = 4,
    MM_ERR_CUDA = 5
};

/* Field identifiers for mm_upload / mm_download / mm_field_sums.
 * "ncomp" is the number of doubles per grid point in the host AoS array. */
enum mm_field {
    MM_FIELD_F = 0,      /* ADMMState.F      grid+(d,d)  solver.py:112 */
    MM_FIELD_G = 1,      /* ADMMState.grad_u grid+(d,d)  solver.py:111 */
    MM_FIELD_LAM = 2,    /* ADMMState.lam    grid+(d,d)  solver.py:113 */
    MM_FIELD_UT = 3,     /* ADMMState.u_tilde grid+(d,)  solver.py:110 */
    MM_FIELD_PREV_F = 4, /* ADMMState.prev_F grid+(d,d)  solver.py:120 */
    MM_FIELD_MOD_A = 5,  /* per-point modulus: mu (MR) or c (quadratic), (npts,) */
    MM_FIELD_MOD_B = 6,  /* per-point modulus: kappa (MR), (npts,) */
    MM_FIELD_ANG = 7,    /* LCE internal["angles"]  (npts,) 2D / (npts,2) 3D  lce.py:116-124 */
    MM_FIELD_CHART = 8,  /* LCE internal["chart"]   (npts,3,3) 3D only */
    MM_FIELD_PINC = 9,   /* LCE internal["p_inc"]   (npts,) */
    MM_FIELD_N0 = 10,    /* LCE imprinted director n0 (npts,d)  lce.py:96 */
    MM_FIELD_FF = 11,    /* LCE frozen Frank force (npts,d)      lce.py:223-229 */
    MM_FIELD_PREV_ANG = 12,   /* prev_internal["angles"] */
    MM_FIELD_PREV_CHART = 13, /* prev_internal["chart"] */
    MM_FIELD_PREV_PINC = 14,  /* prev_internal["p_inc"] */
    MM_FIELD_COUNT = 15
};

/* Materials for mm_local_sweeps. */
enum mm_material {
    MM_MAT_MR = 0,        /* MooneyRivlin, mooney_rivlin.py:56 */
    MM_MAT_QUADRATIC = 1, /* QuadraticMaterial, quadratic.py:22 */
    MM_MAT_LCE = 2,       /* LiquidCrystalElastomer, lce.py:73 */
    MM_MAT_MR_DESCENT = 3 /* MooneyRivlin through the vectorised-descent algorithm in any
                             dim (MooneyRivlin._sweeps_numpy, mooney_rivlin.py:126-162) */
};

typedef struct mm_ctx mm_ctx;

/* Outcome of one metered batch (LocalStats, base.py:44-55) plus the sums the
 * solver needs afterwards.  sum_F holds sum over points of F_ij (d*d, the
 * numerator of mean_field(F), grid.py:266). */
typedef struct {
    int64_t sweeps;       /* LocalStats.sweeps (max over points) */
    int64_t n_conv;       /* points counted as converged (converged_frac * npts) */
    double sum_res2;      /* sum of res_pts^2 (solver.py:266 r_l numerator) */
    double sum_F[9];
    double sum_nsw;       /* sum over points of the sweeps each took (work measure) */
} mm_local_stats;

/* Solver tail: projection + r_d + multiplier ascent + r_p (solver.py:268-279). */
typedef struct {
    double sum_dG2;       /* sum |grad_u_new - grad_u_old|^2  (r_d, solver.py:271) */
    double sum_mis2;      /* sum |grad_u_new - F|^2           (r_p, solver.py:278) */
    double sum_lam[9];    /* sum of lam after the ascent (next mean_field(lam)) */
} mm_update_stats;

/* Pipeline stages for mm_profile_read (one outer iteration runs them in
 * this order). */
enum mm_stage {
    MM_STAGE_LOCAL = 0,     /* local constitutive step (all chunks) */
    MM_STAGE_ROW_FWD = 1,   /* divergence + R2C along the contiguous axis */
    MM_STAGE_COL_FWD = 2,   /* FFT along axis 1 (3D) */
    MM_STAGE_COL_SOLVE = 3, /* FFT + solve + inverse FFT along axis 0 */
    MM_STAGE_COL_INV = 4,   /* inverse FFT along axis 1 (3D) */
    MM_STAGE_ROW_INV = 5,   /* C2R along the contiguous axis -> u_tilde */
    MM_STAGE_GRAD = 6,      /* gradient + multiplier ascent + residual sums */
    MM_STAGE_FROZEN = 7,    /* LCE director + Frank stencil */
    MM_STAGE_OTHER = 8,     /* transfers, sums, checks */
    MM_STAGE_FUSED = 9,     /* multiplier ascent fused with the next first local chunk */
    MM_STAGE_PLANE = 10,    /* COL_FWD + COL_SOLVE + COL_INV in one cluster pass (3D) */
    MM_NSTAGE = 11
};

typedef struct {
    double ms[MM_NSTAGE];          /* device time per stage (CUDA events), since reset */
    int64_t launches[MM_NSTAGE];   /* kernels launched per stage, since reset */
} mm_profile;

/* LCE scalar parameters (lce.py:78-107, 233-275). */
typedef struct {
    double mu, r1d, rr, alpha, gamma_inc, vis_F, vis_n, det_tol;
    double phiF_scale, phin_scale, frank_kappa;
} mm_lce_params;

int mm_abi_version(void);
/* sizeof of the public structs, so a binding can check its declarations:
 * which = MM_STRUCT_* below; -1 for an unknown id. */
enum mm_struct_id {
    MM_STRUCT_LOCAL_STATS = 0, MM_STRUCT_UPDATE_STATS = 1, MM_STRUCT_STEP_PARAMS = 2,
    MM_STRUCT_STEP_RESULT = 3, MM_STRUCT_PROFILE = 4, MM_STRUCT_LCE_PARAMS = 5,
    MM_STRUCT_SOLVE_PARAMS = 6, MM_STRUCT_SOLVE_RESULT = 7
};
int64_t mm_struct_size(int which);

/* Context = one periodic grid on one device (Grid, grid.py:55-122).
 * dim in {2,3}, n >= 4, length > 0 (half edge L). */
int mm_create(int dim, int n, double length, int device, mm_ctx **out);
/* Point-set context for the pointwise operator alone (local_sweeps called on
 * (npts, d, d) arrays that are not a grid, as in materials tests): only the
 * per-point fields exist; projection calls fail with MM_ERR_CONFIG. */
int mm_create_points(int dim, int64_t npts, int device, mm_ctx **out);
void mm_destroy(mm_ctx *ctx);
const char *mm_last_error(const mm_ctx *ctx);
int mm_synchronize(mm_ctx *ctx);
/* Bytes of device memory currently held by the context. */
int64_t mm_device_bytes(const mm_ctx *ctx);

/* Host AoS <-> device SoA.  count = number of doubles in the host array
 * (npts * ncomp of the field); a mismatch is MM_ERR_CONFIG. */
int mm_upload(mm_ctx *ctx, int field, const double *host, int64_t count);
/* field += host array (AoS, same count as mm_upload), rounded once per
 * element like numpy's `state.F = state.F + dF`: the seeded perturbation
 * of the load-stepping drivers (scenarios.py:801-805) without a round trip
 * of the field.  field in {F, LAM, PREV_F}. */
int mm_add_field(mm_ctx *ctx, int field, const double *host, int64_t count);
int mm_download(mm_ctx *ctx, int field, double *host, int64_t count);
/* Device-to-device copy of a whole field (e.g. begin_time_step, solver.py:230-233). */
int mm_copy_field(mm_ctx *ctx, int dst_field, int src_field);
/* Per-component sums over all points (mean_field numerator, grid.py:266). */
int mm_field_sums(mm_ctx *ctx, int field, double *out);

/* Modified central-difference symbols (grid.py:161-184): per-axis tables of
 * |g_j(m)|^2 = (sin(h xi_m)/h)^2 in FFT order, axis_tab[j*n + m], the last
 * axis holding only m = 0..n/2; `threshold` = 1e-14 * max |g|^2 (the live
 * mask of projection.py:155-157).  Tables are built on the host exactly as
 * the reference builds them and uploaded once per grid. */
int mm_set_symbols(mm_ctx *ctx, const double *axis_tab, double threshold);

/* One metered batch of local sweeps, MaterialModel.local_sweeps
 * (base.py:104-112): MR -> mooney_rivlin.py:108-124 (2D kernel :169-255,
 * 3D descent :126-162 + base.py:124-230); quadratic -> quadratic.py:46-69;
 * LCE -> lce.py:233-275 (2D :371-584, 3D :676-995).
 * tol is absolute (point_tol * mu_rep).  phi_scale: MR/quadratic energy
 * scale (max mu + max kappa, resp. max c).  want_points != 0 keeps per-point
 * res / nsw / ok for mm_download_points.  F (and LCE internals) are updated
 * in place on the device.  Returns MM_ERR_INADMISSIBLE when the 3D MR
 * gradient meets det F <= 0 (base.py:116-121); F is then unchanged. */
int mm_local_sweeps(mm_ctx *ctx, int material, double rho, double tol, int64_t max_sweeps,
                    double phi_scale, int want_points, mm_local_stats *out);
int mm_set_lce(mm_ctx *ctx, const mm_lce_params *p);
int mm_download_points(mm_ctx *ctx, double *res, int64_t *nsw, uint8_t *ok, int64_t npts);

/* LCE frozen data (lce.py:223-229): director from angles/chart, then the
 * Frank force 2 kappa (D^T D) n as the exact radius-2 real-space stencil
 * (equal to the reference's spectral form, lce.py:213-221). */
int mm_prepare_frozen(mm_ctx *ctx);
/* The same stencil applied to a director field the caller uploaded into the
 * MM_FIELD_FF slot (LiquidCrystalElastomer.frank_force, lce.py:213-221);
 * the force replaces it in that slot. */
int mm_frank_stencil(mm_ctx *ctx);

/* Diagnostics: work counters of the 3D LCE Newton kernel, 8 doubles
 * (multiplier-only sweeps, Newton steps, eliminations, Armijo evaluations,
 * det-guard trials, fallback passes, fallback evaluations, warp Newton
 * iterations x 32).  Zeros unless the library was built with
 * -DMM_LCE_STATS=1 (MM_NVCC_FLAGS); reset != 0 clears them. */
int mm_debug_lce_counters(double *out, int reset);

/* Helmholtz projection of (F, lam) (projection.py:132-168): writes
 * u_tilde and grad_u = u_mean + D u_tilde on the device.  u_mean (d*d,
 * from macro_gradient, projection.py:125-129) is supplied by the host. */
int mm_project(mm_ctx *ctx, double rho, const double *u_mean);

/* Fused solver tail (solver.py:268-279): projection, then one pass that
 * forms grad_u_new, accumulates |dG|^2 for r_d, misfit^2 for r_p, applies
 * lam += rho (grad_u_new - F) and sums lam for the next macro control. */
int mm_project_update(mm_ctx *ctx, double rho, const double *u_mean, mm_update_stats *out);

/* Stage profiling: when on, each stage is bracketed by CUDA events on the
 * context stream; mm_profile_read returns accumulated device milliseconds and
 * kernel-launch counts (launch counts are kept even when off). */
int mm_profile_enable(mm_ctx *ctx, int on);
int mm_profile_read(mm_ctx *ctx, mm_profile *out, int reset);

/* Split form of the solver tail used by solve() to fuse the multiplier
 * ascent of iteration k with the first local chunk of iteration k+1:
 *  mm_project_residuals: projection + sums for r_d and r_p only
 *    (solver.py:268-278); the ascent lam += rho (grad_u - F) is left pending
 *    and grad_u becomes implicit (u_mean + D u_tilde);
 *  mm_update_multiplier: apply the pending ascent (sum_lam filled);
 *  mm_update_and_sweep: apply it and, in the same pass, run the first local
 *    chunk of the next iteration with rho_next / tol (at most 64 sweeps;
 *    MR and quadratic).  Any other call first applies a pending ascent. */
int mm_project_residuals(mm_ctx *ctx, double rho, const double *u_mean, mm_update_stats *out);
int mm_update_multiplier(mm_ctx *ctx, mm_update_stats *out);
/* One step of solve()'s fused loop without a host round trip in between
 * (solver.py:268-296 + the next call's first chunk): the residual sums
 * (mm_project_residuals), then r_d, r_p, the divergence guard, the penalty
 * update, the convergence test and the policy tolerance exactly as the
 * Python loop computes them, then either the ascent alone (the last
 * iteration, or divergence) or the ascent fused with the next first local
 * chunk (mm_update_and_sweep). */
typedef struct {
    double u_mean[9];        /* macro gradient for this projection */
    double rho;              /* penalty of this iteration */
    double npts, mu_rep;
    double r_l;              /* this iteration's local residual */
    double r_p_tol, r_d_tol, r_l_tol, divergence_limit;
    int adapt;               /* SolverParams.adapt */
    double tau_adapt, kappa_adapt, rho_floor;  /* rho_floor = rho_min_factor * rho_ref */
    int64_t outer_iter;      /* the iteration counter after this iteration */
    int last_allowed;        /* this is the last iteration max_outer allows */
    int ratio_policy;        /* 1: RatioToDual (tol = max(point_tol, ratio r_d)) */
    double point_tol, ratio;
    int material;
    double phi_scale;
    int64_t chunk;           /* first local chunk of the next iteration */
} mm_step_params;

typedef struct {
    double r_p, r_d, rho_next;
    int diverged, done, swept;  /* swept: the next first chunk ran (ls valid) */
    double sum_lam[9];          /* sum of lam after the ascent */
} mm_step_result;

int mm_residuals_and_step(mm_ctx *ctx, const mm_step_params *p, mm_step_result *out,
                          mm_local_stats *ls);
int mm_update_and_sweep(mm_ctx *ctx, int material, double rho_next, double tol,
                        int64_t max_sweeps, double phi_scale, int want_points,
                        mm_local_stats *ls, mm_update_stats *us);

/* solve()'s whole fused loop in the library (solver.py:305-339 with the
 * fused schedule, solver.py:252-302 per iteration): the policy's metered
 * local chunks, macro_gradient (projection.py:125-129), mm_residuals_and_step,
 * the convergence test -- the same decisions in the Python loop's float
 * order, without a Python round trip per iteration.  `step` carries the
 * per-solve constants of mm_step_params (its u_mean / rho / r_l /
 * outer_iter / last_allowed fields are ignored).  hist receives 4 doubles
 * per completed iteration (r_p, r_d, r_l, rho after the update).  Returns
 * MM_ERR_DIVERGED when the guard trips (the result is filled up to that
 * iteration, whose history entry is not written). */
enum mm_policy_kind { MM_POLICY_EXACT = 0, MM_POLICY_FRACTION = 1, MM_POLICY_RATIO = 2 };
typedef struct {
    mm_step_params step;
    double bc_mask[9], bc_value[9];  /* MacroBC (strain_mask as 0/1, value), d*d used */
    double rho, r_d_prev;            /* state.rho, state.r_d_prev on entry */
    double lam_sum[9];               /* sum of lam over points on entry */
    int64_t outer_iter, max_outer, max_local;
    int policy;                      /* mm_policy_kind */
    int64_t policy_chunk;
    double fraction;                 /* FractionConverged.fraction */
} mm_solve_params;
typedef struct {
    int64_t iterations, outer_iter, total_sweeps;
    int converged, diverged;
    double rho, r_d_prev, point_sweeps;
    double lam_sum[9], u_mean[9];
} mm_solve_result;
int mm_solve_fused(mm_ctx *ctx, const mm_solve_params *p, mm_solve_result *r, double *hist);

/* Slab decomposition: rank `rank` of `nranks` holds planes
 * [rank*n/nranks, (rank+1)*n/nranks) of a 3D n^3 grid (n divisible by
 * nranks, n even).  Fields (upload/download/local sweeps/the fused update
 * calls) are the local slab's; mm_local_sweeps, mm_update_and_sweep and
 * mm_update_multiplier run unchanged on a slab context (their u stencil
 * reads the ghost planes below).  The projection + residual pass of the
 * fused schedule (mm_project_residuals on one context) is the step sequence
 *   HALO_T, [T halo exchange: HALO_OUT_LO -> lower neighbour's HALO_IN_HI,
 *            HALO_OUT_HI -> upper neighbour's HALO_IN_LO],
 *   FWD, [all-to-all SEND -> RECV], SOLVE, [all-to-all RECV -> SEND], INV,
 *   [u ghost exchange of the MM_SLAB_FIELD_U_NEW buffer], RES
 * and the LCE frozen data (mm_prepare_frozen on one context) is
 *   DIRECTOR, [2-plane ghost exchange of MM_SLAB_FIELD_DIRECTOR], FRANK.
 * Ghost exchange of a field (mm_slab_field: ncomp components, component
 * stride cs doubles, g ghost planes of n*n doubles on each face, base = plane
 * 0): planes 0..g-1 go to the lower neighbour's planes nl..nl+g-1, planes
 * nl-g..nl-1 to the upper neighbour's planes -g..-1.
 * Every step only enqueues work on the context stream (mm_slab_stream), so
 * NCCL exchanges issued on that stream between the steps need no host
 * synchronisation; RES returns its two local sums (|dG|^2, |misfit|^2) and
 * is the one step that waits for the stream.
 * Buffers: MM_SLAB_BUF_SEND / RECV  nranks * 3 * (n/nranks)^2 * pitch complex,
 * [peer][c][i0l][i1l][k2]; HALO_*  3 * n^2 doubles [c][i1][i2]. */
/* Peer-memory variant of the two transposes (no separate all-to-all):
 * MM_SLAB_FWD_PUSH is MM_SLAB_FWD whose axis-1 FFT stores each output tile
 * straight into the RECV buffer of the rank that owns it (block `rank` of
 * that buffer), and MM_SLAB_SOLVE_PUSH is MM_SLAB_SOLVE storing each solved
 * tile into the SEND buffer of its source rank -- the transfer overlaps the
 * FFT tile by tile over NVLink/NVSwitch peer stores.  Sequence:
 *   HALO_T, [exchange], FWD_PUSH, [barrier], SOLVE_PUSH, [barrier], INV, ...
 * The barrier orders every rank's push kernel before the next step on any
 * rank (a stream-ordered collective, or a host barrier after a stream
 * synchronise); no kernel waits on another rank.  Peer buffers are
 * registered with mm_slab_set_peers (device pointers usable in this process,
 * e.g. ranks sharing one process) or mm_slab_open_peers (CUDA IPC handles of
 * the other processes' buffers, from mm_slab_ipc_handle). */
enum mm_slab_step {
    MM_SLAB_HALO_T = 0, MM_SLAB_FWD = 1, MM_SLAB_SOLVE = 2, MM_SLAB_INV = 3,
    /* 4..6 retired in ABI 2 (explicit-gradient slab steps) */
    MM_SLAB_FWD_PUSH = 7, MM_SLAB_SOLVE_PUSH = 8, MM_SLAB_RES = 9, MM_SLAB_DIRECTOR = 10,
    MM_SLAB_FRANK = 11
};
enum mm_slab_buffer {
    MM_SLAB_BUF_SEND = 0, MM_SLAB_BUF_RECV = 1, MM_SLAB_BUF_HALO_OUT_LO = 2,
    MM_SLAB_BUF_HALO_OUT_HI = 3, MM_SLAB_BUF_HALO_IN_LO = 4, MM_SLAB_BUF_HALO_IN_HI = 5
};
enum mm_slab_field_id {
    MM_SLAB_FIELD_U_NEW = 0,    /* u_tilde being produced by INV (consumed by RES) */
    MM_SLAB_FIELD_U = 1,        /* current u_tilde */
    MM_SLAB_FIELD_DIRECTOR = 2  /* LCE director written by DIRECTOR (consumed by FRANK) */
};
int mm_create_slab(int n, double length, int nranks, int rank, int device, mm_ctx **out);
int mm_slab_buffer(mm_ctx *ctx, int which, void **dev_ptr, int64_t *nbytes);
/* u_mean (9 doubles) is read by RES only; sums (>= 2 doubles) written by RES only. */
int mm_slab_step(mm_ctx *ctx, int step, double rho, const double *u_mean, double *sums);
int mm_slab_field(mm_ctx *ctx, int which, void **base, int64_t *cstride, int *ncomp,
                  int *ghost);
/* The context's CUDA stream (cudaStream_t), for collectives ordered with its work. */
int mm_slab_stream(mm_ctx *ctx, void **stream);
/* which = MM_SLAB_BUF_RECV (targets of FWD_PUSH) or MM_SLAB_BUF_SEND (targets
 * of SOLVE_PUSH).  ptrs[q] = rank q's buffer, P = nranks. */
int mm_slab_set_peers(mm_ctx *ctx, int which, void *const *ptrs, int P);
/* 64-byte CUDA IPC handle of this rank's SEND or RECV buffer. */
int mm_slab_ipc_handle(mm_ctx *ctx, int which, void *handle_out);
/* handles = P consecutive 64-byte handles (entry `rank` is ignored: the own
 * buffer is used); opened with cudaIpcOpenMemHandle, closed by mm_destroy. */
int mm_slab_open_peers(mm_ctx *ctx, int which, const void *handles, int P);

/* Options.  MM_OPT_IMPLICIT_GRAD (default 0): after a fused projection keep
 * grad_u implicitly as u_mean + D u_tilde instead of storing the 9-component
 * field (the local step and the next update rebuild it with the same
 * stencil expression; a download materialises it). */
/* MM_OPT_STENCIL_MARCH (default 1): the 3D residual pass of
 * mm_project_residuals uses the plane-marching kernel (register/shared-memory
 * stencil reuse) when n is a multiple of 32; 0 selects the per-voxel kernel
 * (the two differ only in the order of the residual sums). */
/* MM_OPT_T_FIELD (default 1): the fused update + local pass also stores
 * T = F - lam/rho_next, and the next projection differentiates it instead of
 * re-reading F and lam (even n, single-context grids). */
/* MM_OPT_PLANE_FFT (default 1): 3D single-GPU grids with power-of-two
 * n <= 256 keep the half spectrum as (component, k2) planes and run the
 * axis-1 / axis-0 transforms and the solve in one launch, one thread-block
 * cluster per plane with the plane resident in L2 (bitwise identical to the
 * three-launch column sequence). */
enum mm_option {
    MM_OPT_IMPLICIT_GRAD = 0,
    MM_OPT_STENCIL_MARCH = 1,
    MM_OPT_T_FIELD = 2,
    MM_OPT_PLANE_FFT = 3,
    MM_OPT_ROWINV_PIPE = 4, /* default 1: persistent double-buffered C2R rows (plane layout) */
    MM_OPT_SPECULATE = 5,   /* default 1: mm_update_and_sweep queues the next projection's
                             * A / column passes / E behind the fused pass; mm_project_residuals
                             * uses them if no other call intervened and rho matches */
    MM_OPT_ROWFWD_WARP = 6, /* default 1: single-GPU n = 256 R2C rows with one warp per
                             * 4-row task (k_row_fwd_w): the block-tiled kernel's four-step
                             * in the same order (equal to roundoff) */
    MM_OPT_PIPELINE = 7     /* default 1: mm_residuals_and_step queues K1, the decision (on
                             * the device) and the next fused pass back to back; the host
                             * takes the same decision and checks it (bitwise equal loop) */
};
int mm_set_option(mm_ctx *ctx, int option, int64_t value);

/* Central-difference stencils on the grid fields (grid.py:227-249):
 * op 0: grad_u = D u_tilde (discrete_grad);  op 1: u_tilde = div F
 * (discrete_div).  Both equal the reference's spectral forms to roundoff. */
int mm_stencil(mm_ctx *ctx, int op);

/* equilibrium_residual (solver.py:346-371): || div P ||_{H^-1} / npts of
 * the total stress P(F, internal; dt) of `material` on the device state
 * (MR / quadratic: mooney_rivlin.py:78-85, quadratic.py:34-36; LCE:
 * lce.py:186-196 incl. reaction and viscous terms; the viscous coefficient
 * is the vis_F = nu_F / dt of the last mm_set_lce, applied when dt > 0).
 * MR with det F <= 0 returns MM_ERR_INADMISSIBLE like the reference's
 * stress(). */
int mm_equilibrium_residual(mm_ctx *ctx, int material, double dt, double *out);

/* Bloch-wave stability (stability.py:171-289): smallest eigenvalue of the
 * shifted acoustic operator at one multiplicity, by the splitting iteration.
 * Setup (per solve): Minv = (L + rho I)^-1 and L per point (npts x D x D,
 * D = d^2, row-major blocks), shift = xi + omega per point (npts x d), |b|^2
 * and the live mask per point (full spectrum, the reference's
 * bloch_symbols), rho, target = npts^2.  start: p (npts x d complex,
 * re/im interleaved) -> p_hat = FFT(p) masked and normalised, g = 0.
 * iterate: up to max_iter iterations; out = {beta, primal, iterations,
 * converged, diverged}.  mode: p = IFFT(p_hat) as complex AoS. */
int mm_bloch_setup(mm_ctx *ctx, const double *Minv, const double *Lmat, const double *shift,
                   const double *bsq, const uint8_t *live, double rho, double target);
int mm_bloch_start(mm_ctx *ctx, const double *p);
int mm_bloch_iterate(mm_ctx *ctx, int max_iter, double tol_beta, double tol_primal,
                     double floor_, double mu_rep, double *out);
int mm_bloch_mode(mm_ctx *ctx, double *p_out);

/* Test hook: y[i] = the device natural logarithm the Mooney-Rivlin objective
 * uses (table-driven, csrc/mm_local.cu log_pos) for host arrays x, y. */
int mm_selftest_log(mm_ctx *ctx, const double *x, double *y, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* MM_ADMM_H */
