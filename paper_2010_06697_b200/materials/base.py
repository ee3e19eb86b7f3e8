"""Material contract (micromech/materials/base.py:44-121) for the B200 path.

A material keeps its pointwise physics on the host for diagnostics
(``energy``, ``stress``, ``tangent``) exactly as the reference does, and
runs its local solver — the hot per-voxel step — on the device through
libmm_admm.  ``local_sweeps`` keeps the reference signature and in-place
semantics for callers holding numpy arrays; the solver instead calls the
device-resident ``_device_local`` on its engine context.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .. import _lib
from ..errors import InadmissibleStateError

__all__ = ["MaterialModel", "LocalStats", "BACKTRACK_SHRINK", "BACKTRACK_DECREASE",
           "MAX_BACKTRACKS", "MEAS_EPS", "descent_sweeps_numpy"]

# Armijo constants of the reference (base.py:36-41); the CUDA kernels use the
# same values (csrc/mm_local.cu, csrc/mm_lce.cu).
BACKTRACK_DECREASE = 1e-4
BACKTRACK_SHRINK = 0.5
MAX_BACKTRACKS = 60
MEAS_EPS = 64.0 * np.finfo(float).eps


@dataclass
class LocalStats:
    """Outcome of one metered batch of local sweeps (base.py:44-55)."""

    res_pts: np.ndarray
    sweeps: int
    converged_frac: float


class DeviceLocalStats(LocalStats):
    """LocalStats from a device batch.  ``res_pts`` is materialised only when
    the batch kept per-point residuals (custom policies); the solver needs
    only the reductions (sum res^2 for r_l, the converged count, max sweeps)."""

    def __init__(self, res_pts, sweeps, converged_frac, sum_res2, sum_F, sum_nsw=0.0):
        self._res = res_pts
        self.sweeps = int(sweeps)
        self.converged_frac = float(converged_frac)
        self.sum_res2 = float(sum_res2)
        self.sum_F = np.asarray(sum_F, dtype=float)
        self.sum_nsw = float(sum_nsw)  # sweeps summed over points (work done)

    @property
    def res_pts(self):
        if self._res is None:
            raise AttributeError("per-point residuals were not kept for this batch")
        return self._res

    @res_pts.setter
    def res_pts(self, v):
        self._res = v


class MaterialModel:
    """Base class; concrete models override the pointwise physics."""

    dim: int = 2
    name: str = "base"
    mu_rep: float = 1.0
    internal_spec: dict = {}
    has_tangent: bool = False
    has_dissipation: bool = False
    #: libmm_admm material id
    _material_id = None

    def init_internal(self, npts: int, rng=None) -> dict:
        return {}

    def energy(self, F, internal):
        raise NotImplementedError

    def stress(self, F, internal):
        raise NotImplementedError

    def stress_total(self, F, internal, prev_F, prev_internal, dt):
        return self.stress(F, internal)

    def tangent(self, F, internal):
        raise NotImplementedError(f"{self.name} has no analytic tangent")

    def dissipation_density(self, dF, dinternal, dt):
        return np.zeros(dF.shape[0])

    def prepare_frozen(self, grid, F, internal) -> dict:
        return {}

    def local_sweeps(self, F, internal, grad_u, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol) -> LocalStats:
        raise NotImplementedError

    def _check_det(self, J):
        if np.any(J <= 0.0):
            bad = int(np.argmax(J <= 0.0))
            raise InadmissibleStateError(f"det F = {J.reshape(-1)[bad]:.3e} <= 0 at point {bad}")

    # -- device plumbing -----------------------------------------------------
    def _device_bind(self, ctx, npts):
        """Upload the per-point parameters of this model to a context."""
        raise NotImplementedError(f"{self.name} has no device local step")

    def _prepare_stress(self, ctx, dt):
        """Scalars the device stress needs for time step dt (none by default)."""

    def _points_context(self, npts):
        """Cached point-set context for direct local_sweeps calls."""
        ctx = getattr(self, "_pts_ctx", None)
        if ctx is None or ctx.npts != npts or ctx.dim != self.dim:
            ctx = _lib.Context(self.dim, npts=npts)
            self._device_bind(ctx, npts)
            self._pts_ctx = ctx
        return ctx


def descent_sweeps_numpy(*args, **kwargs):
    """The reference's generic vectorised descent takes arbitrary Python
    objective/gradient callables (base.py:124-230); on the B200 path that
    algorithm is compiled per material (csrc/mm_local.cu, k_descent) and
    reached through the materials' local_sweeps."""
    raise NotImplementedError(
        "descent_sweeps_numpy with Python callables has no device form; use a material's "
        "local_sweeps (MooneyRivlin, QuadraticMaterial), which runs the same algorithm on the GPU")
