"""ADMM outer iteration on the device — drop-in for micromech/solver.py.

Same public surface as the reference module (solver.py:45-59): parameters,
residual record, state, local policies, ``init_state``, ``begin_time_step``,
``outer_iteration``, ``solve``, ``equilibrium_residual``, ``macro_stress``.

One outer iteration (solver.py:236-302) is, on the B200:
  1. [LCE] frozen Frank force: one stencil kernel;
  2. local step: one kernel launch per metered chunk (the policy decides on
     the host from a 13-double reduction read back per chunk);
  3. projection + multiplier ascent + residuals: six kernels (d-component
     FFT pipeline and one fused gradient/update/reduction pass), one
     11-double readback for r_p, r_d, the divergence guard and rho adaptation.
Fields stay resident in HBM between iterations and across solve() calls on
the same state; the host only ever sees reductions.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from ._engine import STATE_FIELDS, Engine, field_shape
from .errors import ConfigurationError, ConvergenceError, DivergenceError, ParameterError
from .grid import Grid, mean_field
from .materials.base import DeviceLocalStats
from .projection import MacroBC, macro_gradient

# state fields the reference mutates in place during solve()
INPLACE_FIELDS = ("F", "lam")

__all__ = [
    "SolverParams",
    "Residuals",
    "ADMMState",
    "LocalPolicy",
    "ExactAll",
    "FractionConverged",
    "RatioToDual",
    "init_state",
    "outer_iteration",
    "solve",
    "begin_time_step",
    "equilibrium_residual",
    "macro_stress",
]


@dataclass
class SolverParams:
    """Outer-loop tolerances and penalty schedule (solver.py:66-93)."""

    r_p_tol: float = 1e-6
    r_d_tol: float = 1e-6
    r_l_tol: float | None = None
    point_tol: float = 1e-11
    max_outer: int = 20000
    max_local: int = 2000
    rho_init: float | None = None
    rho_min_factor: float = 1e-3
    kappa_adapt: float = 1.3
    tau_adapt: float = 10.0
    adapt: bool = True
    divergence_limit: float = 1e8

    def __post_init__(self):
        if self.r_p_tol <= 0 or self.r_d_tol <= 0:
            raise ParameterError("residual tolerances must be positive")
        if self.kappa_adapt <= 1.0:
            raise ParameterError("kappa_adapt must exceed 1")
        if self.tau_adapt < 1.0:
            raise ParameterError("tau_adapt must be at least 1")


class Residuals(NamedTuple):
    outer_iter: int
    r_p: float
    r_d: float
    r_l: float
    rho: float
    wall_ms: float


# ---------------------------------------------------------------------------
# state: host views over device-resident fields
# ---------------------------------------------------------------------------

class ADMMState:
    """Complete solver state (solver.py:105-121).

    Field attributes (F, grad_u, lam, u_tilde, prev_F, internal, prev_internal)
    are device-resident while the state is attached to an engine.  Reading one
    returns a read-only numpy snapshot (downloaded on first access after the
    device changed it); assigning a new array (``state.F = state.F + dF``)
    uploads it before the next device operation.  In-place edits of a snapshot
    raise instead of being silently lost.  A snapshot read before a solve is
    not updated by it — read the attribute again afterwards.
    """

    _FIELD_NAMES = tuple(STATE_FIELDS)

    def __init__(self, u_mean, u_tilde, grad_u, F, lam, internal, rho, outer_iter=0,
                 r_d_prev=np.inf, total_sweeps=0, history=None, prev_F=None,
                 prev_internal=None):
        object.__setattr__(self, "_host", {})
        object.__setattr__(self, "_dev", set())     # names valid on the device
        object.__setattr__(self, "_stale", set())   # host copy out of date
        object.__setattr__(self, "_dirty", set())   # host copy must be uploaded
        object.__setattr__(self, "_engine", None)
        # communicator of a slab-decomposed state (slab.py); None: one GPU
        object.__setattr__(self, "_comm", None)
        # caller arrays updated in place at the end of solve() (F, lam)
        object.__setattr__(self, "_inplace", {})
        self.u_mean = np.asarray(u_mean, dtype=float)
        self.F = F
        self.grad_u = grad_u
        self.lam = lam
        self.u_tilde = u_tilde
        self.prev_F = prev_F
        self.internal = internal if internal is not None else {}
        self.prev_internal = prev_internal
        self.rho = float(rho)
        self.outer_iter = int(outer_iter)
        self.r_d_prev = r_d_prev
        self.total_sweeps = int(total_sweeps)
        self.history = list(history) if history is not None else []

    # -- field access ----------------------------------------------------------
    def _get(self, name):
        eng = self._engine
        if name in self._stale and eng is not None:
            grid = eng.grid
            if name in STATE_FIELDS:
                fid, rank = STATE_FIELDS[name]
                val = eng.ctx.download(fid, eng.field_shape(rank))
                val.flags.writeable = False
            else:
                val = eng.model._download_internal(eng.ctx, name)
                for a in val.values():
                    a.flags.writeable = False
            self._host[name] = val
            self._stale.discard(name)
        return self._host.get(name)

    def _set(self, name, value):
        given = value
        if value is not None and name in STATE_FIELDS:
            value = np.asarray(value, dtype=float)
        # The reference updates F (local_sweeps, base.py:109-111) and lam
        # (solver.py:279) in place: a writeable contiguous caller array for
        # either is written back at the end of solve() (_writeback_inplace)
        if name in INPLACE_FIELDS:
            if (value is given and isinstance(value, np.ndarray) and value.dtype == np.float64
                    and value.flags.c_contiguous and value.flags.writeable):
                self._inplace[name] = value
            else:
                self._inplace.pop(name, None)
        self._host[name] = value
        self._stale.discard(name)
        self._dev.discard(name)
        if value is not None:
            self._dirty.add(name)
        else:
            self._dirty.discard(name)

    def _prefault_downloads(self, grid):
        """Fields the caller holds on the host (other than the in-place F and
        lam) are re-read after the solve as fresh arrays: prepare those host
        arrays while the device iterates (_lib.prefault_async)."""
        if self._comm is not None:
            return  # slab fields: local shapes, not worth it
        shapes = []
        for nm in ("grad_u", "u_tilde"):
            if self._host.get(nm) is not None:
                shapes.append(field_shape(grid, STATE_FIELDS[nm][1]))
        if shapes:
            _lib.prefault_async(shapes)

    def _writeback_inplace(self):
        """Download F and lam into the caller's arrays they were given as
        (the reference mutates those arrays in place).  The arrays stay
        registered, so every later solve() on this state writes into them
        again and ``state.F is F0`` holds throughout, as in the reference;
        they become read-only, so an in-place edit between solves raises
        instead of being silently lost (assign ``state.F = ...`` instead:
        the device copy is authoritative while the state is attached)."""
        eng = self._engine
        if eng is None:
            return
        for nm in INPLACE_FIELDS:
            target = self._inplace.get(nm)
            if target is None or nm not in self._stale:
                continue
            fid, rank = STATE_FIELDS[nm]
            if target.shape != eng.field_shape(rank):
                continue
            eng.ctx.download_into(fid, target)
            target.flags.writeable = False
            self._host[nm] = target
            self._stale.discard(nm)

    def detach_caller_arrays(self):
        """Stop writing solve() results back into the F / lam arrays the
        caller handed in (see _writeback_inplace).  Those arrays keep the
        values of the last solve; the state's attributes keep returning the
        current (device) values.  For device-resident loops that never read
        the caller's arrays: saves one D2H of F and lam per solve() call."""
        self._inplace.clear()

    def _mark_device(self, *names):
        """Fields just rewritten on the device: host copies are stale."""
        for nm in names:
            self._dev.add(nm)
            self._stale.add(nm)
            self._dirty.discard(nm)
            self._host[nm] = None

    def __getstate__(self):
        for nm in list(self._stale):
            self._get(nm)
        d = {k: self._host.get(k) for k in self._FIELD_NAMES + ("internal", "prev_internal")}
        d.update(u_mean=self.u_mean, rho=self.rho, outer_iter=self.outer_iter,
                 r_d_prev=self.r_d_prev, total_sweeps=self.total_sweeps,
                 history=list(self.history))
        return d

    def __setstate__(self, d):
        self.__init__(d["u_mean"], d["u_tilde"], d["grad_u"], d["F"], d["lam"],
                      d["internal"], d["rho"], d["outer_iter"], d["r_d_prev"],
                      d["total_sweeps"], d["history"], d["prev_F"], d["prev_internal"])

    # -- device attachment -------------------------------------------------------
    def _attach(self, grid: Grid, model) -> Engine:
        eng = self._engine
        if eng is None or not eng.matches(grid, self._comm):
            if eng is not None:
                # leaving an old engine: bring everything home first
                for nm in list(self._stale):
                    self._get(nm)
            eng = Engine(grid, comm=self._comm)
            object.__setattr__(self, "_engine", eng)
            self._dev.clear()
            self._stale.clear()
            self._dirty.update(k for k, v in self._host.items() if v is not None)
        eng.bind_model(model)
        ctx = eng.ctx
        d = grid.dim
        for nm, (fid, rank) in STATE_FIELDS.items():
            val = self._host.get(nm)
            if nm in self._stale:
                continue
            if val is None:
                continue
            if nm in self._dirty or nm not in self._dev:
                eng.check_field(val, rank, nm)
                ctx.upload(fid, val)
                if nm == "lam":
                    eng.lam_sum = None
            # the caller keeps its array; ours is re-read from the device
            self._mark_device(nm)
        for nm in ("internal", "prev_internal"):
            if nm in self._stale:
                continue
            val = self._host.get(nm)
            if val and (nm in self._dirty or nm not in self._dev):
                model._upload_internal(ctx, nm, val)
                self._mark_device(nm)
        self._dirty.clear()
        return eng


def _field_property(name):
    def fget(self):
        return self._get(name)

    def fset(self, value):
        self._set(name, value)

    return property(fget, fset)


for _nm in ADMMState._FIELD_NAMES + ("internal", "prev_internal"):
    setattr(ADMMState, _nm, _field_property(_nm))


# ---------------------------------------------------------------------------
# local inexactness policies (solver.py:128-199)
# ---------------------------------------------------------------------------

class LocalPolicy:
    """Meters the local sweeps spent per outer iteration; ``target_tol`` is
    the pointwise tolerance (relative to mu_rep), ``is_done`` judges a batch."""

    name = "base"
    chunk = 50

    def target_tol(self, params: SolverParams, r_d_prev: float) -> float:
        return params.point_tol

    def is_done(self, stats, sweeps_total: int) -> bool:
        raise NotImplementedError


class ExactAll(LocalPolicy):
    """Every point to the pointwise tolerance."""

    name = "exact"
    chunk = 50

    def is_done(self, stats, sweeps_total):
        return stats.converged_frac >= 1.0


class FractionConverged(LocalPolicy):
    """Stop once ``fraction`` of the points meet the tolerance, checking
    every ``check_every`` sweeps."""

    name = "fraction"

    def __init__(self, fraction: float = 0.9, check_every: int = 2):
        if not 0.0 < fraction <= 1.0:
            raise ParameterError("fraction must lie in (0, 1]")
        self.fraction = float(fraction)
        self.chunk = int(check_every)

    def is_done(self, stats, sweeps_total):
        return stats.converged_frac >= self.fraction


class RatioToDual(LocalPolicy):
    """Pointwise tolerance tied to the previous dual residual: tol =
    max(point_tol, ratio * r_d_prev), unbounded (1.0) before any r_d exists."""

    name = "ratio"
    chunk = 25

    def __init__(self, ratio: float = 0.3):
        if ratio <= 0:
            raise ParameterError("ratio must be positive")
        self.ratio = float(ratio)

    def target_tol(self, params, r_d_prev):
        if not np.isfinite(r_d_prev):
            return 1.0
        return max(params.point_tol, self.ratio * r_d_prev)

    def is_done(self, stats, sweeps_total):
        return stats.converged_frac >= 1.0


_BUILTIN_POLICIES = (ExactAll, FractionConverged, RatioToDual)


def _needs_points(policy) -> bool:
    """Custom policies may inspect res_pts: keep per-point residuals then."""
    return type(policy) not in _BUILTIN_POLICIES


# ---------------------------------------------------------------------------
# state setup and the outer iteration
# ---------------------------------------------------------------------------

def init_state(grid: Grid, model, bc: MacroBC, params: SolverParams, rng=None,
               comm=None) -> ADMMState:
    """Uniform state at the pinned macroscopic strain (solver.py:206-227).
    With a communicator (slab decomposition, slab.py) the fields are this
    rank's slab (n/P, n, n, ...) and the model holds this rank's per-point
    parameters."""
    d = grid.dim
    if bc.strain_mask.shape != (d, d):
        raise ParameterError("boundary control dimension mismatch")
    comm = _as_comm(comm, grid)
    shape = grid.shape
    npts = grid.npoints
    if comm is not None:
        from .slab import SlabLayout
        lay = SlabLayout(grid.n, comm.P, comm.rank, grid.length, grid.dim)
        shape, npts = lay.local_shape, lay.npts_local
    Fbar0 = np.where(bc.strain_mask, bc.value, np.eye(d))
    F = np.empty(shape + (d, d))
    F[...] = Fbar0
    state = ADMMState(
        u_mean=Fbar0.copy(), u_tilde=np.zeros(shape + (d,)), grad_u=F.copy(), F=F,
        lam=np.zeros(shape + (d, d)), internal=model.init_internal(npts, rng),
        rho=float(params.rho_init if params.rho_init is not None else model.mu_rep))
    object.__setattr__(state, "_comm", comm)
    if state.rho <= 0:
        raise ParameterError("initial penalty must be positive")
    return state


def _as_comm(comm, grid):
    if comm is None:
        return None
    from .slab import as_comm
    comm = as_comm(comm)
    if grid.dim != 3:
        raise ConfigurationError("the slab decomposition is implemented for 3D grids")
    return comm


def begin_time_step(state: ADMMState):
    """Freeze the current fields as the previous-step reference
    (solver.py:230-233); device-to-device copies when the state is resident."""
    eng = state._engine
    resident = eng is not None and "F" in state._dev and "F" not in state._dirty
    if resident:
        eng.ctx.copy_field(_lib.FIELD_PREV_F, _lib.FIELD_F)
        state._mark_device("prev_F")
    else:
        state.prev_F = state.F.copy()
    model = eng.model if eng is not None else None
    if (resident and model is not None and hasattr(model, "_copy_internal_to_prev")
            and "internal" in state._dev and "internal" not in state._dirty):
        model._copy_internal_to_prev(eng.ctx)
        state._mark_device("prev_internal")
    else:
        state.prev_internal = {k: v.copy() for k, v in state.internal.items()}


def outer_iteration(grid: Grid, model, state: ADMMState, params: SolverParams, bc: MacroBC,
                    policy: LocalPolicy, dt: float = 0.0, freqs=None) -> Residuals:
    """One splitting round on the device; updates state in place
    (solver.py:236-302)."""
    t_start = time.perf_counter()
    if bc.dim != grid.dim:
        from .errors import ConfigurationError
        raise ConfigurationError(f"MacroBC dim {bc.dim} does not match grid dim {grid.dim}")
    eng = state._attach(grid, model)
    if eng.distributed and _needs_points(policy):
        raise ConfigurationError("slab decomposition: custom policies see only this rank's "
                                 "points; use a built-in policy")
    ctx = eng.ctx
    d = grid.dim
    npts = grid.npoints
    mu_rep = model.mu_rep

    if hasattr(model, "_device_prepare_frozen"):
        model._device_prepare_frozen(ctx)

    # ---- step 1: metered local solves (solver.py:252-266)
    tol_pt = policy.target_tol(params, state.r_d_prev)
    want_points = _needs_points(policy)
    if getattr(model, "_material_id", None) == _lib.MAT_LCE and dt > 0.0 and \
            (model.nu_F > 0.0 or model.nu_n > 0.0) and \
            (state._host.get("prev_F") is None and "prev_F" not in state._dev
             or not state._host.get("prev_internal") and "prev_internal" not in state._dev):
        raise ParameterError("viscous update needs the previous step (begin_time_step)")
    sweeps_total = 0
    while True:
        chunk = min(policy.chunk, params.max_local - sweeps_total)
        stats = model._device_local(ctx, npts, state.rho, dt, chunk, tol_pt, want_points)
        sweeps_total += stats.sweeps
        eng.point_sweeps += stats.sum_nsw
        if (policy.is_done(stats, sweeps_total) or stats.sweeps < chunk
                or sweeps_total >= params.max_local):
            break
    state.total_sweeps += sweeps_total
    state._mark_device("F")
    if getattr(model, "_material_id", None) == _lib.MAT_LCE:
        state._mark_device("internal")
    r_l = float(np.sqrt(stats.sum_res2 / npts)) / mu_rep

    # ---- step 2 + 3: projection, dual residual, multiplier ascent (:268-279)
    F_mean = (stats.sum_F[: d * d] / npts).reshape(d, d)
    u_mean = macro_gradient(bc, F_mean, eng.lam_mean(), state.rho)
    up = ctx.project_update(state.rho, u_mean)
    state._mark_device("grad_u", "lam", "u_tilde")
    eng.lam_sum = np.array(up.sum_lam[: d * d])
    r_d = state.rho * float(np.sqrt(up.sum_dG2 / npts)) / mu_rep
    r_p = float(np.sqrt(up.sum_mis2 / npts))
    state.u_mean = u_mean

    state.outer_iter += 1
    state.r_d_prev = r_d

    if not np.isfinite(r_p) or r_p > params.divergence_limit:
        raise DivergenceError(f"primal residual {r_p:.3e} at outer iteration {state.outer_iter}")

    # ---- penalty rebalancing (:288-296)
    if params.adapt and state.outer_iter > 1:
        rho_ref = params.rho_init if params.rho_init is not None else model.mu_rep
        if r_p > params.tau_adapt * r_d:
            state.rho *= params.kappa_adapt
        elif r_d > params.tau_adapt * r_p:
            state.rho = max(state.rho / params.kappa_adapt, params.rho_min_factor * rho_ref)

    wall_ms = (time.perf_counter() - t_start) * 1e3
    resid = Residuals(state.outer_iter, float(r_p), float(r_d), float(r_l), float(state.rho),
                      wall_ms)
    state.history.append(resid)
    return resid


def solve(grid: Grid, model, bc: MacroBC, params: SolverParams,
          policy: LocalPolicy | None = None, state: ADMMState | None = None, dt: float = 0.0,
          rng=None, callback=None, raise_on_max: bool = True, comm=None):
    """Iterate to joint primal/dual/local tolerance; returns (state, converged)
    (solver.py:305-339).

    ``comm`` (extension): a communicator (slab.TorchComm /
    ThreadComm, or torch.distributed) -- the grid is split along axis 0 over
    its ranks, one GPU each; `state` and the model's per-point parameters
    are this rank's slab (init_state(..., comm=comm)), and every rank takes
    identical decisions from rank-ordered global sums."""
    if policy is None:
        policy = ExactAll()
    comm = _as_comm(comm, grid)
    if state is None:
        state = init_state(grid, model, bc, params, rng, comm=comm)
    elif comm is not None and state._comm is not comm:
        if state._engine is not None:
            raise ConfigurationError("state is attached to another communicator")
        object.__setattr__(state, "_comm", comm)
    r_l_tol = params.r_l_tol if params.r_l_tol is not None else max(params.r_p_tol,
                                                                   params.r_d_tol)
    converged = False
    resid = None
    state._prefault_downloads(grid)
    if callback is None and _fusable(model, policy, bc, grid) and os.environ.get(
            "MM_FUSE", "1") != "0":
        converged, resid = _solve_fused(grid, model, bc, params, policy, state, r_l_tol)
    else:
        for _ in range(params.max_outer):
            resid = outer_iteration(grid, model, state, params, bc, policy, dt=dt)
            if callback is not None:
                callback(state, resid)
            if (resid.r_p <= params.r_p_tol and resid.r_d <= params.r_d_tol
                    and resid.r_l <= r_l_tol):
                converged = True
                break
    state._writeback_inplace()
    if not converged and raise_on_max:
        raise ConvergenceError(
            f"no convergence in {params.max_outer} outer iterations "
            f"(r_p={resid.r_p:.3e}, r_d={resid.r_d:.3e})" if resid is not None else
            "no outer iterations allowed", history=state.history)
    return state, converged


# ---------------------------------------------------------------------------
# fused schedule: ascent of iteration k + first local chunk of iteration k+1
# ---------------------------------------------------------------------------

def _fusable(model, policy, bc, grid) -> bool:
    """The fused pass covers the Mooney-Rivlin and quadratic local steps with
    a built-in policy whose chunk fits one launch; no callback may observe
    the state between iterations (solve() checks that)."""
    if getattr(model, "_fused_material", None) is None or model._fused_material() is None:
        return False
    if type(policy) not in _BUILTIN_POLICIES or policy.chunk > 64:
        return False
    return bc.dim == grid.dim


def _solve_fused(grid, model, bc, params, policy, state, r_l_tol):
    """solve()'s loop with the multiplier ascent of iteration k and the first
    local chunk of iteration k+1 in one device pass (mm_update_and_sweep).

    Every decision the reference takes between those two steps (divergence
    guard, history, convergence test, penalty update, the policy tolerance
    from the new r_d) only needs r_p and r_d, which mm_project_residuals
    returns before the ascent is applied; the per-point arithmetic is the
    reference's, in the same order.  The last iteration (converged or at
    max_outer) applies the ascent alone, so the state on return is exactly
    the unfused one."""
    eng = state._attach(grid, model)
    ctx = eng.ctx
    d = grid.dim
    npts = grid.npoints
    mu_rep = model.mu_rep
    mat, phi_scale = model._fused_material()
    pending = None  # stats of a first local chunk already run by the fused pass
    converged = False
    resid = None
    # the decisions between the residuals and the next fused pass taken in
    # the library (MM_HOST_DECIDE=1: here, through two calls)
    device_step = os.environ.get("MM_HOST_DECIDE", "0") != "1" and not eng.distributed
    if device_step:
        prm = _lib.StepParamsC()
        prm.npts = float(npts)
        prm.mu_rep = mu_rep
        prm.r_p_tol, prm.r_d_tol = params.r_p_tol, params.r_d_tol
        prm.r_l_tol = r_l_tol
        prm.divergence_limit = params.divergence_limit
        prm.adapt = 1 if params.adapt else 0
        prm.tau_adapt, prm.kappa_adapt = params.tau_adapt, params.kappa_adapt
        rho_ref = params.rho_init if params.rho_init is not None else model.mu_rep
        prm.rho_floor = params.rho_min_factor * rho_ref
        prm.ratio_policy = 1 if isinstance(policy, RatioToDual) else 0
        prm.point_tol = params.point_tol
        prm.ratio = getattr(policy, "ratio", 0.0)
        prm.material = mat
        prm.phi_scale = phi_scale
        prm.chunk = min(policy.chunk, params.max_local)
    if device_step and os.environ.get("MM_C_LOOP", "1") != "0":
        return _solve_fused_c(eng, grid, model, bc, params, policy, state, prm, mat, phi_scale)
    for it in range(params.max_outer):
        t_start = time.perf_counter()
        tol_pt = policy.target_tol(params, state.r_d_prev)
        sweeps_total = 0
        stats = None
        while True:
            chunk = min(policy.chunk, params.max_local - sweeps_total)
            if pending is not None:
                stats, pending = pending, None
            else:
                stats = model._device_local(ctx, npts, state.rho, 0.0, chunk, tol_pt, False)
            sweeps_total += stats.sweeps
            eng.point_sweeps += stats.sum_nsw
            if (policy.is_done(stats, sweeps_total) or stats.sweeps < chunk
                    or sweeps_total >= params.max_local):
                break
        state.total_sweeps += sweeps_total
        state._mark_device("F")
        r_l = float(np.sqrt(stats.sum_res2 / npts)) / mu_rep
        F_mean = (stats.sum_F[: d * d] / npts).reshape(d, d)
        u_mean = macro_gradient(bc, F_mean, eng.lam_mean(), state.rho)
        if device_step:
            # residuals, the decisions below and the next ascent + first chunk
            # in one library call (mm_residuals_and_step): same arithmetic
            prm.u_mean[:] = np.zeros(9)
            prm.u_mean[: d * d] = np.asarray(u_mean, dtype=float).reshape(-1)
            prm.rho = state.rho
            prm.r_l = r_l
            prm.outer_iter = state.outer_iter + 1
            prm.last_allowed = 1 if it == params.max_outer - 1 else 0
            res, ls = ctx.residuals_and_step(prm)
            state._mark_device("grad_u", "u_tilde", "lam")
            r_d, r_p = res.r_d, res.r_p
            state.u_mean = u_mean
            state.outer_iter += 1
            state.r_d_prev = r_d
            eng.lam_sum = np.array(res.sum_lam[: d * d])
            if res.diverged:
                raise DivergenceError(
                    f"primal residual {r_p:.3e} at outer iteration {state.outer_iter}")
            state.rho = res.rho_next
            done = bool(res.done)
            if res.swept:
                pending = DeviceLocalStats(None, ls.sweeps,
                                           float(ls.n_conv) / npts if npts else 1.0,
                                           ls.sum_res2, list(ls.sum_F), ls.sum_nsw)
            wall_ms = (time.perf_counter() - t_start) * 1e3
            resid = Residuals(state.outer_iter, float(r_p), float(r_d), float(r_l),
                              float(state.rho), wall_ms)
            state.history.append(resid)
            if done:
                converged = True
                break
            continue
        up = ctx.project_residuals(state.rho, u_mean)
        state._mark_device("grad_u", "u_tilde", "lam")
        r_d = state.rho * float(np.sqrt(up.sum_dG2 / npts)) / mu_rep
        r_p = float(np.sqrt(up.sum_mis2 / npts))
        state.u_mean = u_mean
        state.outer_iter += 1
        state.r_d_prev = r_d
        if not np.isfinite(r_p) or r_p > params.divergence_limit:
            eng.lam_sum = np.array(ctx.update_multiplier().sum_lam[: d * d])
            raise DivergenceError(
                f"primal residual {r_p:.3e} at outer iteration {state.outer_iter}")
        if params.adapt and state.outer_iter > 1:
            rho_ref = params.rho_init if params.rho_init is not None else model.mu_rep
            if r_p > params.tau_adapt * r_d:
                state.rho *= params.kappa_adapt
            elif r_d > params.tau_adapt * r_p:
                state.rho = max(state.rho / params.kappa_adapt, params.rho_min_factor * rho_ref)
        done = r_p <= params.r_p_tol and r_d <= params.r_d_tol and r_l <= r_l_tol
        last = done or it == params.max_outer - 1
        if last:
            eng.lam_sum = np.array(ctx.update_multiplier().sum_lam[: d * d])
        else:
            # ascent of this iteration + first local chunk of the next one
            tol_next = policy.target_tol(params, r_d)
            chunk = min(policy.chunk, params.max_local)
            ls, us = ctx.update_and_sweep(mat, state.rho, tol_next * mu_rep, chunk, phi_scale)
            eng.lam_sum = np.array(us.sum_lam[: d * d])
            pending = DeviceLocalStats(None, ls.sweeps, float(ls.n_conv) / npts if npts else 1.0,
                                       ls.sum_res2, list(ls.sum_F), ls.sum_nsw)
        wall_ms = (time.perf_counter() - t_start) * 1e3
        resid = Residuals(state.outer_iter, float(r_p), float(r_d), float(r_l), float(state.rho),
                          wall_ms)
        state.history.append(resid)
        if done:
            converged = True
            break
    return converged, resid


def _solve_fused_c(eng, grid, model, bc, params, policy, state, prm, mat, phi_scale):
    """The fused loop of _solve_fused run inside the library (mm_solve_fused):
    the same policy metering, macro control, residuals, decisions and float
    order as the Python loop above, no Python round trip per iteration
    (bitwise identical; MM_C_LOOP=0 runs the Python loop).  Residuals.wall_ms
    is the loop's average per iteration."""
    d = grid.dim
    sp = _lib.SolveParamsC()
    sp.step = prm
    mask = np.zeros(9)
    val = np.zeros(9)
    mask[: d * d] = np.asarray(bc.strain_mask, dtype=bool).reshape(-1)
    val[: d * d] = np.asarray(bc.value, dtype=float).reshape(-1)
    sp.bc_mask[:] = mask
    sp.bc_value[:] = val
    sp.rho = state.rho
    sp.r_d_prev = float(state.r_d_prev)
    lam = np.zeros(9)
    if eng.lam_sum is None:
        eng.lam_mean()
    lam[: d * d] = np.asarray(eng.lam_sum, dtype=float).reshape(-1)
    sp.lam_sum[:] = lam
    sp.outer_iter = state.outer_iter
    sp.max_outer = params.max_outer
    sp.max_local = params.max_local
    sp.policy = (_lib.POLICY_RATIO if isinstance(policy, RatioToDual) else
                 _lib.POLICY_FRACTION if isinstance(policy, FractionConverged) else
                 _lib.POLICY_EXACT)
    sp.policy_chunk = policy.chunk
    sp.fraction = getattr(policy, "fraction", 1.0)
    t0 = time.perf_counter()
    res, hist, rc, msg = eng.ctx.solve_fused(sp, params.max_outer)
    wall = (time.perf_counter() - t0) * 1e3 / max(int(res.iterations), 1)
    state._mark_device("F", "grad_u", "u_tilde", "lam")
    base = state.outer_iter
    for i, (r_p, r_d, r_l, rho) in enumerate(hist):
        state.history.append(Residuals(base + i + 1, float(r_p), float(r_d), float(r_l),
                                       float(rho), wall))
    state.outer_iter = int(res.outer_iter)
    state.total_sweeps += int(res.total_sweeps)
    state.r_d_prev = float(res.r_d_prev)
    state.rho = float(res.rho)
    if res.iterations:
        state.u_mean = np.array(res.u_mean[: d * d]).reshape(d, d)
    eng.lam_sum = np.array(res.lam_sum[: d * d])
    eng.point_sweeps += float(res.point_sweeps)
    if rc == _lib.MM_ERR_DIVERGED:
        raise DivergenceError(msg)
    resid = state.history[-1] if len(hist) else None
    return bool(res.converged), resid


# ---------------------------------------------------------------------------
# diagnostics
# ---------------------------------------------------------------------------

def equilibrium_residual(grid: Grid, model, state: ADMMState, dt: float = 0.0) -> float:
    """Negative norm of div P of the total stress (solver.py:346-371), on the
    device (mm_equilibrium_residual): the material's total stress into a
    scratch field, its central-difference divergence fused with the R2C row
    transform (the reference's spectral divergence with g_j = i sin(h xi)/h
    is exactly the DFT of that stencil), the column FFTs, and the sum of
    |div P_hat|^2 / |g|^2 over live modes in the last column pass (half
    spectrum, conjugate columns counted twice)."""
    mat = getattr(model, "_material_id", None)
    if mat is None:
        raise ConfigurationError(f"{getattr(model, 'name', model)} has no device stress")
    if getattr(model, "dim", grid.dim) != grid.dim:
        raise ConfigurationError("model and grid dimensions differ")
    if mat == _lib.MAT_LCE and dt > 0.0 and model.nu_F > 0.0 and state.prev_F is None:
        raise ParameterError("viscous stress needs prev_F (call begin_time_step)")
    eng = state._attach(grid, model)
    model._prepare_stress(eng.ctx, dt)
    return eng.ctx.equilibrium_residual(mat, dt)


def macro_stress(grid: Grid, state: ADMMState) -> np.ndarray:
    """Volume average of the multiplier (solver.py:374-377); from the device
    reduction when the state is resident."""
    eng = state._engine
    if eng is not None and eng.matches(grid, state._comm) and "lam" in state._dev \
            and "lam" not in state._dirty:
        return eng.lam_mean().copy()
    if state._comm is not None:
        # this rank holds a slab: rank-ordered global sum of the local sums
        d = grid.dim
        loc = np.asarray(state.lam, dtype=float).reshape(-1, d * d).sum(axis=0)
        return (state._comm.ordered_sum(loc) / grid.npoints).reshape(d, d)
    return mean_field(grid, state.lam)
