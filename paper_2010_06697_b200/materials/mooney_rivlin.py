"""Compressible Mooney-Rivlin (neo-Hookean) solid, reference
micromech/materials/mooney_rivlin.py.

    W(F) = mu/2 (|F|^2 - 2 ln J - d) + kappa/2 (J - 1)^2,   J = det F

Closed forms (energy / stress / tangent) stay on the host for diagnostics.
The local step runs on the device (csrc/mm_local.cu):
  * 2D: ``k_mr2d``, the reference's compiled kernel (mooney_rivlin.py:169-255);
  * 3D: ``k_descent<MR, 9>``, the reference's vectorised numpy descent
    (mooney_rivlin.py:126-162 + base.py:124-230), including its per-call
    step-length reset and the 32-sweep stall guard.
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from ..errors import ParameterError
from .base import DeviceLocalStats, DeviceParam, LocalStats, MaterialModel

__all__ = ["MooneyRivlin"]


class MooneyRivlin(MaterialModel):
    name = "mooney_rivlin"
    has_tangent = True
    _material_id = _lib.MAT_MR
    mu = DeviceParam()
    kappa = DeviceParam()

    def __init__(self, mu, kappa, dim: int = 2, mu_rep: float | None = None):
        self.dim = int(dim)
        self.mu = mu
        self.kappa = kappa
        if np.any(self.mu <= 0) or np.any(self.kappa < 0):
            raise ParameterError("MooneyRivlin needs mu > 0 and kappa >= 0")
        self.mu_rep = float(mu_rep) if mu_rep is not None else float(np.max(self.mu))

    # -- closed forms (host diagnostics) -------------------------------------
    def energy(self, F, internal=None):
        J = np.linalg.det(F)
        self._check_det(J)
        I1 = np.einsum("...ij,...ij->...", F, F)
        return 0.5 * self.mu * (I1 - 2.0 * np.log(J) - self.dim) \
            + 0.5 * self.kappa * (J - 1.0) ** 2

    def stress(self, F, internal=None):
        """S = mu (F - F^{-T}) + kappa (J^2 - J) F^{-T}."""
        J = np.linalg.det(F)
        self._check_det(J)
        FinvT = np.swapaxes(np.linalg.inv(F), -2, -1)
        mu = self.mu[..., None, None] if self.mu.ndim else self.mu
        kap = self.kappa[..., None, None] if self.kappa.ndim else self.kappa
        Jc = J[..., None, None]
        return mu * (F - FinvT) + kap * (Jc * Jc - Jc) * FinvT

    def tangent(self, F, internal=None):
        """dS/dF (mooney_rivlin.py:313-329)."""
        J = np.linalg.det(F)
        self._check_det(J)
        Finv = np.linalg.inv(F)
        FinvT = np.swapaxes(Finv, -2, -1)
        d = self.dim
        lead = F.shape[:-2]
        eye = np.eye(d)
        mu = np.broadcast_to(self.mu, lead)
        kap = np.broadcast_to(self.kappa, lead)
        out = mu[..., None, None, None, None] * np.einsum("ik,jl->ijkl", eye, eye)
        out = out + (kap * (2.0 * J - 1.0) * J)[..., None, None, None, None] * \
            np.einsum("...ij,...kl->...ijkl", FinvT, FinvT)
        out = out + (mu - kap * (J * J - J))[..., None, None, None, None] * \
            np.einsum("...jk,...li->...ijkl", Finv, Finv)
        return out

    # -- device local step -----------------------------------------------------
    def _flat_moduli(self, npts):
        mu = np.ascontiguousarray(np.broadcast_to(self.mu, (npts,)), dtype=float)
        kap = np.ascontiguousarray(np.broadcast_to(self.kappa, (npts,)), dtype=float)
        return mu, kap

    def _phi_scale(self):
        """max mu + max kappa (mooney_rivlin.py:116), cached until the moduli
        are reassigned (a host max over the full grid would otherwise cost
        more than the device local step)."""
        return self._cached_max("phi", lambda: np.max(self.mu) + np.max(self.kappa))

    def _scale_terms(self):
        return {"phi": lambda: (self.mu, self.kappa)}

    def _fused_material(self):
        """Material id and energy scale for the fused ascent + first chunk."""
        return _lib.MAT_MR, self._phi_scale()

    def _device_bind(self, ctx, npts):
        mu, kap = self._flat_moduli(npts)
        ctx.upload(_lib.FIELD_MOD_A, mu)
        ctx.upload(_lib.FIELD_MOD_B, kap)

    def _device_local(self, ctx, npts, rho, dt, max_sweeps, point_tol, want_points=False,
                      material=None, abs_tol=None):
        tol = point_tol * self.mu_rep if abs_tol is None else abs_tol  # mooney_rivlin.py:112
        mat = self._material_id if material is None else material
        st = ctx.local_sweeps(mat, rho, tol, max_sweeps, self._phi_scale(), want_points)
        res = None
        if want_points:
            res, _, _ = ctx.download_points()
        frac = float(st.n_conv) / npts if npts else 1.0
        return DeviceLocalStats(res, st.sweeps, frac, st.sum_res2, list(st.sum_F), st.sum_nsw)

    def _run_points(self, F, grad_u, lam, rho, max_sweeps, point_tol, material, abs_tol=None):
        npts = F.shape[0]
        d = self.dim
        if npts == 0:
            return LocalStats(res_pts=np.empty(0), sweeps=0, converged_frac=1.0)
        ctx = self._points_context(npts)
        ctx.upload(_lib.FIELD_F, F.reshape(npts, d * d))
        ctx.upload(_lib.FIELD_G, np.asarray(grad_u).reshape(npts, d * d))
        ctx.upload(_lib.FIELD_LAM, np.asarray(lam).reshape(npts, d * d))
        st = self._device_local(ctx, npts, rho, 0.0, max_sweeps, point_tol, True, material,
                                abs_tol)
        Fn = ctx.download(_lib.FIELD_F, (npts, d, d))
        F[...] = Fn.reshape(F.shape)
        return LocalStats(res_pts=st.res_pts, sweeps=st.sweeps,
                          converged_frac=st.converged_frac)

    def local_sweeps(self, F, internal, grad_u, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol) -> LocalStats:
        """MaterialModel.local_sweeps (mooney_rivlin.py:108-124), on the device;
        F (npts, d, d) is updated in place."""
        return self._run_points(F, grad_u, lam, rho, max_sweeps, point_tol, None)

    def _sweeps_numpy(self, F, grad_u, lam, mu, kap, rho, tol, max_sweeps):
        """The vectorised-descent path in any dimension (mooney_rivlin.py:126-162),
        on the device.  ``tol`` is absolute, as in the reference."""
        st = self._run_points(F, grad_u, lam, rho, max_sweeps, None, _lib.MAT_MR_DESCENT,
                              abs_tol=tol)
        return st.res_pts, st.sweeps
