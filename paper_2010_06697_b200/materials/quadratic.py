"""Quadratic reference material W = c/2 |F|^2 (micromech/materials/quadratic.py).

Every piece of the splitting has a closed form against it (local step
F = (lam + rho G)/(c + rho)), which makes it the dense-KKT parity fixture.
Its local step runs the reference's vectorised descent (quadratic.py:46-69)
on the device (csrc/mm_local.cu, k_descent<QUAD, D>).
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from ..errors import ParameterError
from .base import DeviceLocalStats, DeviceParam, LocalStats, MaterialModel

__all__ = ["QuadraticMaterial"]


class QuadraticMaterial(MaterialModel):
    name = "quadratic"
    has_tangent = True
    _material_id = _lib.MAT_QUADRATIC
    c = DeviceParam()

    def __init__(self, c, dim: int = 2, mu_rep: float | None = None):
        self.dim = int(dim)
        self.c = c
        if np.any(self.c <= 0):
            raise ParameterError("QuadraticMaterial needs c > 0")
        self.mu_rep = float(mu_rep) if mu_rep is not None else float(np.max(self.c))

    def energy(self, F, internal=None):
        return 0.5 * self.c * np.einsum("...ij,...ij->...", F, F)

    def stress(self, F, internal=None):
        c = self.c[..., None, None] if self.c.ndim else self.c
        return c * F

    def tangent(self, F, internal=None):
        d = self.dim
        lead = F.shape[:-2]
        eye = np.eye(d)
        c = np.broadcast_to(self.c, lead)
        return c[..., None, None, None, None] * np.einsum("ik,jl->ijkl", eye, eye)

    def _cmax(self):
        return self._cached_max("cmax", lambda: np.max(self.c))

    def _scale_terms(self):
        return {"cmax": lambda: (self.c,)}

    def _fused_material(self):
        return _lib.MAT_QUADRATIC, self._cmax()

    def _device_bind(self, ctx, npts):
        ctx.upload(_lib.FIELD_MOD_A, np.ascontiguousarray(np.broadcast_to(self.c, (npts,)),
                                                          dtype=float))

    def _device_local(self, ctx, npts, rho, dt, max_sweeps, point_tol, want_points=False):
        tol = point_tol * self.mu_rep
        st = ctx.local_sweeps(self._material_id, rho, tol, max_sweeps, self._cmax(), want_points)
        res = None
        if want_points:
            res, _, _ = ctx.download_points()
        frac = float(st.n_conv) / npts if npts else 1.0
        return DeviceLocalStats(res, st.sweeps, frac, st.sum_res2, list(st.sum_F), st.sum_nsw)

    def local_sweeps(self, F, internal, grad_u, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol) -> LocalStats:
        npts = F.shape[0]
        d = self.dim
        if npts == 0:
            return LocalStats(res_pts=np.empty(0), sweeps=0, converged_frac=1.0)
        ctx = self._points_context(npts)
        ctx.upload(_lib.FIELD_F, F.reshape(npts, d * d))
        ctx.upload(_lib.FIELD_G, np.asarray(grad_u).reshape(npts, d * d))
        ctx.upload(_lib.FIELD_LAM, np.asarray(lam).reshape(npts, d * d))
        st = self._device_local(ctx, npts, rho, dt, max_sweeps, point_tol, True)
        F[...] = ctx.download(_lib.FIELD_F, (npts, d, d)).reshape(F.shape)
        return LocalStats(res_pts=st.res_pts, sweeps=st.sweeps,
                          converged_frac=st.converged_frac)
