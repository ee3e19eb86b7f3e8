"""Incompressible nematic liquid-crystal elastomer (micromech/materials/lce.py).

    W_el = mu/2 r^{1/d} (|F|^2 - (r-1)/r |F^T n|^2),
    W_ni = mu a/2 (|F^T n|^2 - ((F^T n).n0)^2),
    Frank: kappa |grad n|^2 (central differences), det F = 1 by a nested
    per-point multiplier, director as one angle (2D) or spherical angles on
    a per-point chart (3D).

Host side: parameters, director storage, closed forms for diagnostics.
Device side (csrc/mm_lce.cu): the joint damped-Newton local kernels
(lce.py:371-584 in 2D, 5x5; lce.py:676-995 in 3D, 11x11) in the reference's
operation order, and the frozen Frank force as the exact radius-2 real-space
stencil of 2 kappa (D^T D) n (lce.py:213-229).  The Newton iterations of
non-converging (polydomain) points are chaotic: an ulp-level difference in
sin/cos grows to O(1) within ~50 sweeps, so parity is pinned per call, on
local-convergent configurations, and statistically.
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from ..errors import ParameterError
from .base import DeviceLocalStats, DeviceParam, LocalStats, MaterialModel

__all__ = ["LiquidCrystalElastomer", "step_length_tensor", "step_length_sqrt"]


def step_length_tensor(n, r):
    """l(n) = r^{-1/d} (I + (r-1) n n) (lce.py:47-53)."""
    n = np.asarray(n, dtype=float)
    d = n.shape[-1]
    nn = np.einsum("...i,...j->...ij", n, n)
    return r ** (-1.0 / d) * (np.eye(d) + (r - 1.0) * nn)


def step_length_sqrt(n, r):
    """Principal square root of l(n) (lce.py:56-62)."""
    n = np.asarray(n, dtype=float)
    d = n.shape[-1]
    nn = np.einsum("...i,...j->...ij", n, n)
    return r ** (-0.5 / d) * (np.eye(d) + (np.sqrt(r) - 1.0) * nn)


def _unit_rows(v, what):
    v = np.asarray(v, dtype=float)
    norms = np.linalg.norm(v, axis=-1)
    if np.any(norms < 1e-12):
        raise ParameterError(f"{what} contains (near-)zero directors")
    return v / norms[..., None]


def _set_chart(angles, chart, n, idx):
    """Equatorial chart per director: e1 = n, phi = pi/2, theta = 0
    (lce.py:278-290)."""
    e1 = n[idx]
    helper = np.zeros_like(e1)
    helper[np.arange(len(idx)), np.argmin(np.abs(e1), axis=1)] = 1.0
    e3 = helper - np.sum(helper * e1, axis=1, keepdims=True) * e1
    e3 /= np.linalg.norm(e3, axis=1, keepdims=True)
    e2 = np.cross(e3, e1)
    chart[idx, :, 0] = e1
    chart[idx, :, 1] = e2
    chart[idx, :, 2] = e3
    angles[idx, 0] = 0.5 * np.pi
    angles[idx, 1] = 0.0


class LiquidCrystalElastomer(MaterialModel):
    name = "lce"
    has_tangent = False
    has_dissipation = True
    _material_id = _lib.MAT_LCE
    n0 = DeviceParam(lambda v: _unit_rows(np.atleast_2d(np.asarray(v, dtype=float)), "n0"))

    def __init__(self, mu, r, alpha, frank_kappa, n0, dim: int = 2, nu_F: float = 0.0,
                 nu_n: float = 0.0, gamma_inc: float | None = None, det_tol: float = 1e-8,
                 mu_rep: float | None = None):
        self.dim = int(dim)
        if self.dim not in (2, 3):
            raise ParameterError("dim must be 2 or 3")
        self.mu, self.r, self.alpha = float(mu), float(r), float(alpha)
        self.frank_kappa = float(frank_kappa)
        self.nu_F, self.nu_n = float(nu_F), float(nu_n)
        if self.mu <= 0 or self.r < 1.0 or self.alpha < 0 or self.frank_kappa < 0 \
                or self.nu_F < 0 or self.nu_n < 0:
            raise ParameterError("LCE needs mu > 0, r >= 1, alpha >= 0, frank_kappa >= 0 "
                                 "and nonnegative viscosities")
        self.n0 = n0
        if self.n0.shape[-1] != self.dim:
            raise ParameterError(f"n0 has {self.n0.shape[-1]} components, model is {self.dim}D")
        self.gamma_inc = float(gamma_inc) if gamma_inc is not None else 50.0 * self.mu
        if self.gamma_inc <= 0:
            raise ParameterError("gamma_inc must be positive")
        self.det_tol = float(det_tol)
        self.mu_rep = float(mu_rep) if mu_rep is not None else self.mu
        self.internal_spec = {"angles": 1, "p_inc": 1} if self.dim == 2 \
            else {"angles": 2, "chart": 9, "p_inc": 1}

    # -- director storage ------------------------------------------------------
    def init_internal(self, npts: int, rng=None) -> dict:
        if self.n0.shape[0] != npts:
            raise ParameterError(f"n0 holds {self.n0.shape[0]} points, grid has {npts}")
        internal = {"p_inc": np.zeros(npts)}
        if self.dim == 2:
            internal["angles"] = np.arctan2(self.n0[:, 1], self.n0[:, 0])
        else:
            internal["angles"] = np.empty((npts, 2))
            internal["chart"] = np.empty((npts, 3, 3))
            _set_chart(internal["angles"], internal["chart"], self.n0, np.arange(npts))
        return internal

    def director(self, internal) -> np.ndarray:
        if self.dim == 2:
            th = internal["angles"]
            return np.stack([np.cos(th), np.sin(th)], axis=-1)
        ph, th = internal["angles"][:, 0], internal["angles"][:, 1]
        local = np.stack([np.sin(ph) * np.cos(th), np.sin(ph) * np.sin(th), np.cos(ph)], axis=-1)
        return np.einsum("pij,pj->pi", internal["chart"], local)

    def set_director(self, internal, n):
        n = _unit_rows(n, "director")
        if self.dim == 2:
            internal["angles"][...] = np.arctan2(n[:, 1], n[:, 0])
        else:
            _set_chart(internal["angles"], internal["chart"], n, np.arange(n.shape[0]))

    # -- closed forms (host diagnostics) -----------------------------------------
    def _terms(self, F, n):
        r1d = self.r ** (1.0 / self.dim)
        rr = (self.r - 1.0) / self.r
        Ftn = np.einsum("...ji,...j->...i", F, n)
        c = np.sum(Ftn * self.n0, axis=-1)
        return r1d, rr, Ftn, c

    def energy(self, F, internal=None, n=None):
        if n is None:
            n = self.director(internal)
        r1d, rr, Ftn, c = self._terms(F, n)
        fsq = np.einsum("...ij,...ij->...", F, F)
        tsq = np.sum(Ftn * Ftn, axis=-1)
        return 0.5 * self.mu * r1d * (fsq - rr * tsq) + 0.5 * self.mu * self.alpha * (tsq - c * c)

    def stress(self, F, internal=None, n=None):
        if n is None:
            n = self.director(internal)
        r1d, rr, Ftn, c = self._terms(F, n)
        nF = n[..., :, None] * Ftn[..., None, :]
        nn0 = n[..., :, None] * self.n0[..., None, :]
        return self.mu * r1d * (F - rr * nF) + self.mu * self.alpha * (nF - c[..., None, None] * nn0)

    def dW_dn(self, F, internal=None, n=None):
        if n is None:
            n = self.director(internal)
        r1d, rr, Ftn, c = self._terms(F, n)
        h = np.einsum("...ij,...j->...i", F, Ftn)
        Fn0 = np.einsum("...ij,...j->...i", F, self.n0)
        return -self.mu * r1d * rr * h + self.mu * self.alpha * (h - c[..., None] * Fn0)

    def stress_total(self, F, internal, prev_F, prev_internal, dt):
        n = self.director(internal)
        J = np.linalg.det(F)
        cof = J[..., None, None] * np.swapaxes(np.linalg.inv(F), -2, -1)
        react = (internal["p_inc"] + self.gamma_inc * (J - 1.0))[..., None, None]
        S = self.stress(F, n=n) + react * cof
        if dt > 0.0 and self.nu_F > 0.0:
            S = S + (self.nu_F / dt) * (F - prev_F)
        return S

    def dissipation_density(self, dF, dinternal, dt):
        D = 0.5 * self.nu_F * np.einsum("...ij,...ij->...", dF, dF)
        if dinternal and "n" in dinternal:
            D = D + 0.5 * self.nu_n * np.sum(dinternal["n"] ** 2, axis=-1)
        return D

    def frank_energy(self, grid, internal=None, n_field=None) -> float:
        from ..grid import discrete_grad
        if n_field is None:
            n_field = self.director(internal).reshape(grid.shape + (self.dim,))
        gn = discrete_grad(grid, n_field)
        return self.frank_kappa * float(np.mean(np.sum(gn * gn, axis=(-2, -1))))

    # -- device ------------------------------------------------------------------
    def _prepare_stress(self, ctx, dt):
        ctx.set_lce(**self._scalars(dt))  # viscous coefficient nu_F / dt

    def _scalars(self, dt):
        d = self.dim
        r1d = self.r ** (1.0 / d)
        if dt > 0.0 and (self.nu_F > 0.0 or self.nu_n > 0.0):
            vis_F, vis_n = self.nu_F / dt, self.nu_n / dt
        else:
            vis_F = vis_n = 0.0
        return dict(mu=self.mu, r1d=r1d, rr=(self.r - 1.0) / self.r, alpha=self.alpha,
                    gamma_inc=self.gamma_inc, vis_F=vis_F, vis_n=vis_n, det_tol=self.det_tol,
                    phiF_scale=self.mu * (r1d * (d + 1.0) + self.alpha * d) + self.gamma_inc,
                    phin_scale=self.mu * (r1d + self.alpha) * d * self.r ** (2.0 / d),
                    frank_kappa=self.frank_kappa)

    def _device_bind(self, ctx, npts):
        if self.n0.shape[0] != npts:
            raise ParameterError(f"n0 holds {self.n0.shape[0]} points, grid has {npts}")
        ctx.upload(_lib.FIELD_N0, self.n0)
        ctx.set_lce(**self._scalars(0.0))

    # -- state <-> device (used by ADMMState) ----------------------------------
    _INTERNAL_FIELDS = {"angles": _lib.FIELD_ANG, "chart": _lib.FIELD_CHART,
                        "p_inc": _lib.FIELD_PINC}
    _PREV_FIELDS = {"angles": _lib.FIELD_PREV_ANG, "chart": _lib.FIELD_PREV_CHART,
                    "p_inc": _lib.FIELD_PREV_PINC}

    def _internal_shapes(self, npts):
        shp = {"p_inc": (npts,)}
        if self.dim == 2:
            shp["angles"] = (npts,)
        else:
            shp["angles"] = (npts, 2)
            shp["chart"] = (npts, 3, 3)
        return shp

    def _upload_internal(self, ctx, which, val):
        fields = self._INTERNAL_FIELDS if which == "internal" else self._PREV_FIELDS
        for k, fid in fields.items():
            if k in val and val[k] is not None:
                ctx.upload(fid, val[k])

    def _download_internal(self, ctx, which):
        fields = self._INTERNAL_FIELDS if which == "internal" else self._PREV_FIELDS
        shp = self._internal_shapes(ctx.npts)
        return {k: ctx.download(fields[k], shp[k]) for k in shp}

    def _copy_internal_to_prev(self, ctx):
        for k in self._internal_shapes(ctx.npts):
            ctx.copy_field(self._PREV_FIELDS[k], self._INTERNAL_FIELDS[k])

    def _device_prepare_frozen(self, ctx):
        ctx.set_lce(**self._scalars(0.0))
        ctx.prepare_frozen()

    def _device_local(self, ctx, npts, rho, dt, max_sweeps, point_tol, want_points=False):
        ctx.set_lce(**self._scalars(dt))
        tol = point_tol * self.mu_rep
        st = ctx.local_sweeps(self._material_id, rho, tol, max_sweeps, 0.0, want_points)
        res = None
        if want_points:
            res, _, _ = ctx.download_points()
        frac = float(st.n_conv) / npts if npts else 1.0
        return DeviceLocalStats(res, st.sweeps, frac, st.sum_res2, list(st.sum_F), st.sum_nsw)

    def frank_force(self, grid, n_field) -> np.ndarray:
        """2 kappa (D^T D) n (lce.py:213-221) as the radius-2 stencil, on the device."""
        from .._engine import field_shape, scratch_engine
        eng = scratch_engine(grid)
        ctx = eng.ctx
        d = self.dim
        nf = np.asarray(n_field, dtype=float).reshape(grid.npoints, d)
        ctx.set_lce(**self._scalars(0.0))
        ctx.upload(_lib.FIELD_FF, nf)       # director goes in through the FF slot
        ctx.check(ctx.lib.mm_frank_stencil(ctx.h))
        return ctx.download(_lib.FIELD_FF, field_shape(grid, 1))

    def prepare_frozen(self, grid, F, internal) -> dict:
        """Frozen Frank force for one outer iteration (lce.py:223-229)."""
        n_field = self.director(internal).reshape(grid.shape + (self.dim,))
        if self.frank_kappa > 0.0:
            ff = self.frank_force(grid, n_field).reshape(-1, self.dim)
        else:
            ff = np.zeros((grid.npoints, self.dim))
        return {"frank_force": np.ascontiguousarray(ff)}

    def local_sweeps(self, F, internal, grad_u, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol) -> LocalStats:
        """lce.py:233-275 on the device; F and internal updated in place."""
        npts = F.shape[0]
        d = self.dim
        if npts == 0:
            return LocalStats(res_pts=np.empty(0), sweeps=0, converged_frac=1.0)
        viscous = dt > 0.0 and (self.nu_F > 0.0 or self.nu_n > 0.0)
        if viscous and (prev_F is None or prev_internal is None):
            raise ParameterError("viscous update needs the previous step (begin_time_step)")
        ctx = self._points_context(npts)
        ctx.upload(_lib.FIELD_F, F.reshape(npts, d * d))
        ctx.upload(_lib.FIELD_G, np.asarray(grad_u).reshape(npts, d * d))
        ctx.upload(_lib.FIELD_LAM, np.asarray(lam).reshape(npts, d * d))
        ctx.upload(_lib.FIELD_ANG, internal["angles"])
        ctx.upload(_lib.FIELD_PINC, internal["p_inc"])
        if d == 3:
            ctx.upload(_lib.FIELD_CHART, internal["chart"])
        ff = frozen.get("frank_force") if frozen else None
        ctx.upload(_lib.FIELD_FF, np.zeros((npts, d)) if ff is None else ff)
        if viscous:
            ctx.upload(_lib.FIELD_PREV_F, np.asarray(prev_F).reshape(npts, d * d))
            self._upload_internal(ctx, "prev_internal", prev_internal)
        st = self._device_local(ctx, npts, rho, dt, max_sweeps, point_tol, True)
        F[...] = ctx.download(_lib.FIELD_F, (npts, d, d)).reshape(F.shape)
        internal["angles"][...] = ctx.download(_lib.FIELD_ANG, internal["angles"].shape)
        internal["p_inc"][...] = ctx.download(_lib.FIELD_PINC, internal["p_inc"].shape)
        if d == 3:
            internal["chart"][...] = ctx.download(_lib.FIELD_CHART, internal["chart"].shape)
        return LocalStats(res_pts=st.res_pts, sweeps=st.sweeps, converged_frac=st.converged_frac)
