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

__all__ = ["MaterialModel", "LocalStats", "DeviceParam", "BACKTRACK_SHRINK", "BACKTRACK_DECREASE",
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


class DeviceParam:
    """A model parameter array that is mirrored on the device.

    The reference re-reads its moduli on every ``local_sweeps`` call
    (mooney_rivlin.py:111-116); the device keeps an uploaded copy and a cached
    energy scale instead.  To keep the two consistent the value is stored as
    a private read-only copy: assigning a new value bumps the model's
    ``_device_version`` (the engine and the point-set context re-upload, the
    cached maxima are recomputed), and an in-place edit raises instead of
    silently leaving stale moduli on the device."""

    def __init__(self, convert=None):
        self.convert = convert

    def __set_name__(self, owner, name):
        self.name = name
        self.slot = "_param_" + name

    def __get__(self, obj, objtype=None):
        if obj is None:
            return self
        return obj.__dict__[self.slot]

    def __set__(self, obj, value):
        a = self.convert(value) if self.convert is not None else np.array(value, dtype=float)
        if a is value or (isinstance(value, np.ndarray) and np.shares_memory(a, value)):
            a = a.copy()
        a.flags.writeable = False
        obj.__dict__[self.slot] = a
        obj.__dict__["_device_version"] = obj.__dict__.get("_device_version", 0) + 1


class MaterialModel:
    """Base class; concrete models override the pointwise physics."""

    #: bumped whenever a DeviceParam is assigned (see DeviceParam)
    _device_version = 0

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
            self._pts_ctx = ctx
            self._pts_ver = None
        if self._pts_ver != self._device_version:
            self._device_bind(ctx, npts)
            self._pts_ver = self._device_version
        return ctx

    def _cached_max(self, key, fn):
        """Host maxima of the moduli (the energy scale), recomputed only when
        a DeviceParam was reassigned."""
        cache = self.__dict__.setdefault("_max_cache", {})
        hit = cache.get(key)
        if hit is None or hit[0] != self._device_version:
            hit = (self._device_version, float(fn()))
            cache[key] = hit
        return hit[1]

    def _globalize(self, comm):
        """Slab ranks hold part of the per-point parameters: pin the cached
        energy scales to their global values and check that every rank
        uses the same mu_rep (the default max(mu) of a rank's own part would
        differ between ranks)."""
        reps = comm.gather_objects(float(self.mu_rep))
        if any(r != reps[0] for r in reps):
            from ..errors import ConfigurationError
            raise ConfigurationError(f"mu_rep differs between ranks {reps}: pass the global value")
        for key, fn in self._scale_terms().items():
            loc = [float(np.max(a)) if np.size(a) else -np.inf for a in fn()]
            glob = comm.ordered_sum(loc, ops=[1] * len(loc))
            self._override_max(key, float(np.sum(glob)))

    def _scale_terms(self):
        """Cached maxima: key -> arrays whose maxima sum to the scale."""
        return {}

    def _override_max(self, key, value):
        """Pin a cached maximum (slab ranks hold part of the moduli: the
        energy scale is the global one, reduced across ranks)."""
        self.__dict__.setdefault("_max_cache", {})[key] = (self._device_version, float(value))


def descent_sweeps_numpy(*args, **kwargs):
    """The reference's generic vectorised descent takes arbitrary Python
    objective/gradient callables (base.py:124-230); on the B200 path that
    algorithm is compiled per material (csrc/mm_local.cu, k_descent) and
    reached through the materials' local_sweeps."""
    raise NotImplementedError(
        "descent_sweeps_numpy with Python callables has no device form; use a material's "
        "local_sweeps (MooneyRivlin, QuadraticMaterial), which runs the same algorithm on the GPU")
