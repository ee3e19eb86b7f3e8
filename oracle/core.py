"""ORACLE (test infrastructure only) — numpy restatement of the reference's
ADMM iteration.  See oracle/__init__.py for the usage rule.

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/micromech).  Transforms use numpy.fft (pocketfft, C)
where the reference uses scipy.fft (pocketfft, C++): same algorithm family,
results agree to roundoff.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "lib", "symbols", "project", "rms", "mean_field",
    "MR", "Quadratic", "LCE", "set_chart",
    "Params", "State", "ExactAll", "FractionConverged", "RatioToDual",
    "init_state", "begin_time_step", "outer_iteration", "solve", "macro_stress",
    "OracleInadmissible", "OracleDivergence", "OracleConvergence",
    "composite_moduli", "polydomain_n0", "set_threads", "set_fft",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OracleInadmissible(Exception):
    pass


class OracleDivergence(Exception):
    pass


class OracleConvergence(Exception):
    pass


def lib():
    """Load (building on first use) the C restatement of the local kernels."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.path.join(_HERE, "_build", "liboracle.so")
    src = os.path.join(_HERE, "oracle_kernels.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    D = ctypes.c_double
    I = ctypes.c_int64
    L.orc_mr2d_sweeps.argtypes = [I, P, P, P, P, P, D, D, I, D, P, P]
    L.orc_mr2d_sweeps.restype = None
    L.orc_descent_sweeps.argtypes = [ctypes.c_int, ctypes.c_int, I, P, P, P, P, P, D, D, I, D, P]
    L.orc_descent_sweeps.restype = I
    L.orc_lce2d_sweeps.argtypes = [I, P, P, P, P, P, P, P, P, P] + [D] * 10 + [I, D, D, P, P, P]
    L.orc_lce2d_sweeps.restype = None
    L.orc_lce3d_sweeps.argtypes = [I, P, P, P, P, P, P, P, P, P, P] + [D] * 10 + [I, D, D, P, P, P]
    L.orc_lce3d_sweeps.restype = None
    L.orc_set_threads.argtypes = [ctypes.c_int]
    L.orc_get_threads.restype = ctypes.c_int
    _LIB = L
    return L


_FFT = np.fft  # transforms of project / frank_force (set_fft)


def set_fft(name: str, workers: int | None = None):
    """Transforms of the projection and the Frank force: "numpy" (pocketfft,
    numpy's build; the default the goldens pin) or "scipy" (scipy.fft, the
    module the reference itself calls, grid.py:32,195-220).  The two are the
    same algorithm family and differ by roundoff, which measures how far two
    faithful CPU runs of the reference algorithm drift apart."""
    global _FFT
    if name == "numpy":
        _FFT = np.fft
    elif name == "scipy":
        import scipy.fft
        _FFT = scipy.fft if workers is None else _ScipyWorkers(scipy.fft, int(workers))
    else:
        raise ValueError(name)
    return _FFT


class _ScipyWorkers:
    """scipy.fft with a fixed worker count, as the reference calls it
    (grid.py:213-220: ``workers=get_workers()``)."""

    def __init__(self, mod, workers):
        self.mod, self.workers = mod, workers

    def rfftn(self, a, **kw):
        return self.mod.rfftn(a, workers=self.workers, **kw)

    def irfftn(self, a, **kw):
        return self.mod.irfftn(a, workers=self.workers, **kw)


def set_threads(n: int) -> int:
    lib().orc_set_threads(int(n))
    return lib().orc_get_threads()


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# grid primitives (grid.py:161-268)
# ---------------------------------------------------------------------------

def symbols(dim, n, L, real=True):
    """Modified central-difference symbols g_j = i sin(h xi_j)/h
    (grid.py:161-184); returns (grad_sym (*spec, dim) complex, grad_sq)."""
    h = 2.0 * L / n
    per_axis = []
    for ax in range(dim):
        last = ax == dim - 1
        if real and last:
            m = np.arange(n // 2 + 1, dtype=float)
        else:
            m = np.fft.fftfreq(n, d=1.0 / n)
        per_axis.append(np.pi * m / L)
    mesh = np.meshgrid(*per_axis, indexing="ij")
    xi = np.stack(mesh, axis=-1)
    g = 1j * np.sin(h * xi) / h
    gsq = np.sum(np.abs(g) ** 2, axis=-1)
    return g, gsq


def rms(f, npts):
    """grid.py:256-263"""
    a = np.ascontiguousarray(f).reshape(-1)
    return float(np.sqrt(np.sum(a * a) / npts))


def mean_field(f, dim):
    """grid.py:266-268"""
    return np.mean(f, axis=tuple(range(dim)))


def project(dim, n, L, F, lam, rho, strain_mask, value, sym=None):
    """Helmholtz projection, projection.py:132-168 (+ macro_gradient :125).

    Returns (u_mean (d,d), u_tilde (*grid, d), grad_u (*grid, d, d))."""
    axes = tuple(range(dim))
    g, gsq = sym if sym is not None else symbols(dim, n, L)
    T = F - lam / rho
    That = _FFT.rfftn(T, axes=axes)
    live = gsq > 1e-14 * gsq.max()
    inv = np.where(live, 1.0 / np.where(live, gsq, 1.0), 0.0)
    uhat = -np.einsum("...ij,...j,...->...i", That, g, inv)
    ghat = uhat[..., :, None] * g[..., None, :]
    shape = (n,) * dim
    u_tilde = _FFT.irfftn(uhat, s=shape, axes=axes)
    grad_fluct = _FFT.irfftn(ghat, s=shape, axes=axes)
    Fm = mean_field(F, dim)
    Lm = mean_field(lam, dim)
    stress_update = Fm - (Lm - value) / rho
    u_mean = np.where(strain_mask, value, stress_update)
    return u_mean, u_tilde, grad_fluct + u_mean


def stencil_grad(dim, n, L, u):
    """Central-difference gradient (u(x+h e_j) - u(x-h e_j))/(2h), the
    real-space form of grid.py:227-239."""
    h = 2.0 * L / n
    out = np.empty(u.shape + (dim,))
    for j in range(dim):
        out[..., j] = (np.roll(u, -1, axis=j) - np.roll(u, 1, axis=j)) / (2.0 * h)
    return out


# ---------------------------------------------------------------------------
# materials
# ---------------------------------------------------------------------------

class MR:
    """Compressible Mooney-Rivlin, materials/mooney_rivlin.py:56-162."""

    def __init__(self, mu, kappa, dim=2, mu_rep=None):
        self.dim = int(dim)
        self.mu = np.asarray(mu, dtype=float)
        self.kappa = np.asarray(kappa, dtype=float)
        self.mu_rep = float(mu_rep) if mu_rep is not None else float(np.max(self.mu))

    def init_internal(self, npts, rng=None):
        return {}

    def prepare_frozen(self, dim, n, L, F, internal):
        return {}

    def energy(self, F):
        J = np.linalg.det(F)
        I1 = np.sum(F * F, axis=(-2, -1))
        return 0.5 * self.mu * (I1 - 2.0 * np.log(J) - self.dim) + 0.5 * self.kappa * (J - 1.0) ** 2

    def stress(self, F):
        J = np.linalg.det(F)
        FinvT = np.swapaxes(np.linalg.inv(F), -2, -1)
        mu = self.mu[..., None, None] if self.mu.ndim else self.mu
        kap = self.kappa[..., None, None] if self.kappa.ndim else self.kappa
        Jc = J[..., None, None]
        return mu * (F - FinvT) + kap * (Jc * Jc - Jc) * FinvT

    def flat_moduli(self, npts):
        mu = _c(np.broadcast_to(self.mu, (npts,)))
        kap = _c(np.broadcast_to(self.kappa, (npts,)))
        return mu, kap

    def local_sweeps(self, F, internal, G, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol):
        """mooney_rivlin.py:108-124; F (npts,d,d) updated in place."""
        npts = F.shape[0]
        mu, kap = self.flat_moduli(npts)
        tol = point_tol * self.mu_rep
        phi_scale = float(np.max(mu) + np.max(kap))
        Fc = _c(F)
        Gc, Lc = _c(G), _c(lam)
        res = np.empty(npts)
        if self.dim == 2:
            nsw = np.zeros(npts, dtype=np.int64)
            lib().orc_mr2d_sweeps(npts, _p(Fc), _p(Gc), _p(Lc), _p(mu), _p(kap), float(rho),
                                  float(tol), int(max_sweeps), phi_scale, _p(res), _p(nsw))
            sweeps = int(nsw.max()) if npts else 0
        else:
            sweeps = self.descent(Fc, Gc, Lc, mu, kap, rho, tol, max_sweeps, res)
            nsw = None
        F[...] = Fc
        frac = float(np.mean(res < tol)) if npts else 1.0
        return res, sweeps, frac, nsw

    def descent(self, Fc, Gc, Lc, mu, kap, rho, tol, max_sweeps, res):
        """Vectorised-numpy path (mooney_rivlin.py:126-162 / base.py:124-230)."""
        npts = Fc.shape[0]
        sweeps = lib().orc_descent_sweeps(0, self.dim, npts, _p(Fc), _p(Gc), _p(Lc), _p(mu),
                                          _p(kap), float(rho), float(tol), int(max_sweeps),
                                          float(np.max(mu) + np.max(kap)), _p(res))
        if sweeps < 0:
            raise OracleInadmissible("det F <= 0")
        return int(sweeps)


class Quadratic:
    """W = c/2 |F|^2, materials/quadratic.py:22-69."""

    def __init__(self, c, dim=2, mu_rep=None):
        self.dim = int(dim)
        self.c = np.asarray(c, dtype=float)
        self.mu_rep = float(mu_rep) if mu_rep is not None else float(np.max(self.c))

    def init_internal(self, npts, rng=None):
        return {}

    def prepare_frozen(self, dim, n, L, F, internal):
        return {}

    def local_sweeps(self, F, internal, G, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol):
        npts = F.shape[0]
        c = _c(np.broadcast_to(self.c, (npts,)))
        tol = point_tol * self.mu_rep
        Fc, Gc, Lc = _c(F), _c(G), _c(lam)
        res = np.empty(npts)
        sweeps = lib().orc_descent_sweeps(1, self.dim, npts, _p(Fc), _p(Gc), _p(Lc), _p(c),
                                          _p(c), float(rho), float(tol), int(max_sweeps),
                                          float(np.max(c)), _p(res))
        F[...] = Fc
        frac = float(np.mean(res < tol)) if npts else 1.0
        return res, int(sweeps), frac, None


def set_chart(angles, chart, n, idx):
    """Chart directors at the equator, lce.py:278-290."""
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


class LCE:
    """Liquid-crystal elastomer, materials/lce.py:73-275."""

    def __init__(self, mu, r, alpha, frank_kappa, n0, dim=2, nu_F=0.0, nu_n=0.0,
                 gamma_inc=None, det_tol=1e-8, mu_rep=None):
        self.dim = int(dim)
        self.mu, self.r, self.alpha = float(mu), float(r), float(alpha)
        self.frank_kappa = float(frank_kappa)
        self.nu_F, self.nu_n = float(nu_F), float(nu_n)
        n0 = np.atleast_2d(np.asarray(n0, dtype=float))
        self.n0 = n0 / np.linalg.norm(n0, axis=-1)[..., None]
        self.gamma_inc = float(gamma_inc) if gamma_inc is not None else 50.0 * self.mu
        self.det_tol = float(det_tol)
        self.mu_rep = float(mu_rep) if mu_rep is not None else self.mu

    def init_internal(self, npts, rng=None):
        internal = {"p_inc": np.zeros(npts)}
        if self.dim == 2:
            internal["angles"] = np.arctan2(self.n0[:, 1], self.n0[:, 0])
        else:
            internal["angles"] = np.empty((npts, 2))
            internal["chart"] = np.empty((npts, 3, 3))
            set_chart(internal["angles"], internal["chart"], self.n0, np.arange(npts))
        return internal

    def director(self, internal):
        """lce.py:126-134"""
        if self.dim == 2:
            th = internal["angles"]
            return np.stack([np.cos(th), np.sin(th)], axis=-1)
        ph, th = internal["angles"][:, 0], internal["angles"][:, 1]
        nloc = np.stack([np.sin(ph) * np.cos(th), np.sin(ph) * np.sin(th), np.cos(ph)], axis=-1)
        return np.einsum("pij,pj->pi", internal["chart"], nloc)

    def frank_force(self, dim, n, L, n_field):
        """2 kappa (D^T D) n through the spectrum, lce.py:213-221."""
        _, gsq = symbols(dim, n, L)
        axes = tuple(range(dim))
        nhat = _FFT.rfftn(n_field, axes=axes)
        f = _FFT.irfftn(gsq[..., None] * nhat, s=(n,) * dim, axes=axes)
        return 2.0 * self.frank_kappa * f

    def prepare_frozen(self, dim, n, L, F, internal):
        """lce.py:223-229"""
        npts = n ** dim
        n_field = self.director(internal).reshape((n,) * dim + (dim,))
        if self.frank_kappa > 0.0:
            ff = self.frank_force(dim, n, L, n_field).reshape(-1, dim)
        else:
            ff = np.zeros((npts, dim))
        return {"frank_force": np.ascontiguousarray(ff)}

    def local_sweeps(self, F, internal, G, lam, rho, dt, prev_F, prev_internal, frozen,
                     max_sweeps, point_tol):
        """lce.py:233-275"""
        npts = F.shape[0]
        d = self.dim
        tol = point_tol * self.mu_rep
        ff = frozen.get("frank_force") if frozen else None
        if ff is None:
            ff = np.zeros((npts, d))
        if dt > 0.0 and (self.nu_F > 0.0 or self.nu_n > 0.0):
            if prev_F is None or prev_internal is None:
                raise ValueError("viscous update needs the previous step")
            vis_F, vis_n = self.nu_F / dt, self.nu_n / dt
            Fk = prev_F
            nk = self.director(prev_internal)
        else:
            vis_F = vis_n = 0.0
            Fk = np.zeros_like(F)
            nk = np.zeros((npts, d))
        r1d = self.r ** (1.0 / d)
        phiF_scale = self.mu * (r1d * (d + 1.0) + self.alpha * d) + self.gamma_inc
        phin_scale = self.mu * (r1d + self.alpha) * d * self.r ** (2.0 / d)
        res = np.empty(npts)
        nsw = np.zeros(npts, dtype=np.int64)
        ok = np.zeros(npts, dtype=np.uint8)
        Fc, Gc, Lc = _c(F), _c(G), _c(lam)
        n0, ffc, Fkc, nkc = _c(self.n0), _c(ff), _c(Fk), _c(nk)
        ang = _c(internal["angles"])
        pinc = _c(internal["p_inc"])
        scal = [self.mu, r1d, (self.r - 1.0) / self.r, self.alpha, self.gamma_inc, float(rho),
                vis_F, vis_n, tol, self.det_tol]
        if d == 2:
            lib().orc_lce2d_sweeps(npts, _p(Fc), _p(ang), _p(pinc), _p(Gc), _p(Lc), _p(n0),
                                   _p(ffc), _p(Fkc), _p(nkc), *scal, int(max_sweeps),
                                   phiF_scale, phin_scale, _p(res), _p(nsw), _p(ok))
        else:
            chart = _c(internal["chart"])
            lib().orc_lce3d_sweeps(npts, _p(Fc), _p(ang), _p(chart), _p(pinc), _p(Gc), _p(Lc),
                                   _p(n0), _p(ffc), _p(Fkc), _p(nkc), *scal, int(max_sweeps),
                                   phiF_scale, phin_scale, _p(res), _p(nsw), _p(ok))
            internal["chart"][...] = chart
        F[...] = Fc
        internal["angles"][...] = ang
        internal["p_inc"][...] = pinc
        sweeps = int(nsw.max()) if npts else 0
        frac = float(np.mean(ok)) if npts else 1.0
        return res, sweeps, frac, (nsw, ok)


# ---------------------------------------------------------------------------
# solver (solver.py:66-339)
# ---------------------------------------------------------------------------

@dataclass
class Params:
    """solver.py:66-93"""
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


class ExactAll:
    """solver.py:147-154"""
    chunk = 50

    def target_tol(self, params, r_d_prev):
        return params.point_tol

    def is_done(self, frac):
        return frac >= 1.0


class FractionConverged(ExactAll):
    """solver.py:157-173"""

    def __init__(self, fraction=0.9, check_every=2):
        self.fraction = float(fraction)
        self.chunk = int(check_every)

    def is_done(self, frac):
        return frac >= self.fraction


class RatioToDual(ExactAll):
    """solver.py:176-199"""
    chunk = 25

    def __init__(self, ratio=0.3):
        self.ratio = float(ratio)

    def target_tol(self, params, r_d_prev):
        if not np.isfinite(r_d_prev):
            return 1.0
        return max(params.point_tol, self.ratio * r_d_prev)


@dataclass
class State:
    """solver.py:105-121"""
    u_mean: np.ndarray
    u_tilde: np.ndarray
    grad_u: np.ndarray
    F: np.ndarray
    lam: np.ndarray
    internal: dict
    rho: float
    outer_iter: int = 0
    r_d_prev: float = np.inf
    total_sweeps: int = 0
    history: list = field(default_factory=list)
    prev_F: np.ndarray | None = None
    prev_internal: dict | None = None


def init_state(dim, n, model, strain_mask, value, params, rng=None):
    """solver.py:206-227"""
    Fbar0 = np.where(strain_mask, value, np.eye(dim))
    shape = (n,) * dim
    F = np.empty(shape + (dim, dim))
    F[...] = Fbar0
    return State(u_mean=Fbar0.copy(), u_tilde=np.zeros(shape + (dim,)), grad_u=F.copy(), F=F,
                 lam=np.zeros(shape + (dim, dim)), internal=model.init_internal(n ** dim, rng),
                 rho=float(params.rho_init if params.rho_init is not None else model.mu_rep))


def begin_time_step(state):
    """solver.py:230-233"""
    state.prev_F = state.F.copy()
    state.prev_internal = {k: v.copy() for k, v in state.internal.items()}


def outer_iteration(dim, n, L, model, state, params, strain_mask, value, policy, dt=0.0,
                    sym=None, timings=None):
    """solver.py:236-302; returns (outer_iter, r_p, r_d, r_l, rho)."""
    t0 = time.perf_counter()
    npts = n ** dim
    mu_rep = model.mu_rep
    Ff = state.F.reshape(npts, dim, dim)
    Gf = state.grad_u.reshape(npts, dim, dim)
    Lf = state.lam.reshape(npts, dim, dim)
    prev_Ff = state.prev_F.reshape(npts, dim, dim) if state.prev_F is not None else None
    frozen = model.prepare_frozen(dim, n, L, state.F, state.internal)
    tol_pt = policy.target_tol(params, state.r_d_prev)
    sweeps_total = 0
    while True:
        chunk = min(policy.chunk, params.max_local - sweeps_total)
        res, sweeps, frac, _ = model.local_sweeps(Ff, state.internal, Gf, Lf, state.rho, dt,
                                                  prev_Ff, state.prev_internal, frozen, chunk,
                                                  tol_pt)
        sweeps_total += sweeps
        if policy.is_done(frac) or sweeps < chunk or sweeps_total >= params.max_local:
            break
    state.total_sweeps += sweeps_total
    r_l = float(np.sqrt(np.sum(res ** 2) / npts)) / mu_rep
    t1 = time.perf_counter()
    u_mean, u_tilde, grad_u = project(dim, n, L, state.F, state.lam, state.rho, strain_mask,
                                      value, sym=sym)
    r_d = state.rho * rms(grad_u - state.grad_u, npts) / mu_rep
    state.u_mean, state.u_tilde, state.grad_u = u_mean, u_tilde, grad_u
    misfit = state.grad_u - state.F
    r_p = rms(misfit, npts)
    state.lam += state.rho * misfit
    state.outer_iter += 1
    state.r_d_prev = r_d
    if timings is not None:
        timings["local"] = timings.get("local", 0.0) + (t1 - t0)
        timings["global"] = timings.get("global", 0.0) + (time.perf_counter() - t1)
    if not np.isfinite(r_p) or r_p > params.divergence_limit:
        raise OracleDivergence(f"primal residual {r_p:.3e} at outer iteration {state.outer_iter}")
    if params.adapt and state.outer_iter > 1:
        rho_ref = params.rho_init if params.rho_init is not None else model.mu_rep
        if r_p > params.tau_adapt * r_d:
            state.rho *= params.kappa_adapt
        elif r_d > params.tau_adapt * r_p:
            state.rho = max(state.rho / params.kappa_adapt, params.rho_min_factor * rho_ref)
    rec = (state.outer_iter, float(r_p), float(r_d), float(r_l), float(state.rho))
    state.history.append(rec)
    return rec


def solve(dim, n, L, model, strain_mask, value, params, policy=None, state=None, dt=0.0,
          max_outer=None, raise_on_max=True):
    """solver.py:305-339"""
    policy = policy or ExactAll()
    if state is None:
        state = init_state(dim, n, model, strain_mask, value, params)
    sym = symbols(dim, n, L)
    r_l_tol = params.r_l_tol if params.r_l_tol is not None else max(params.r_p_tol, params.r_d_tol)
    converged = False
    rec = None
    for _ in range(params.max_outer if max_outer is None else max_outer):
        rec = outer_iteration(dim, n, L, model, state, params, strain_mask, value, policy, dt,
                              sym=sym)
        if rec[1] <= params.r_p_tol and rec[2] <= params.r_d_tol and rec[3] <= r_l_tol:
            converged = True
            break
    if not converged and raise_on_max:
        raise OracleConvergence("no convergence")
    return state, converged


def macro_stress(state, dim):
    """solver.py:374-377"""
    return mean_field(state.lam, dim)


# ---------------------------------------------------------------------------
# synthetic-input generators (scenarios.py)
# ---------------------------------------------------------------------------

def composite_moduli(phase, mu_matrix=1.0, contrast=20.0, kappa_ratio=9.8):
    """scenarios.py:311-324"""
    chi = np.clip(np.asarray(phase).ravel().astype(float), 0.0, 1.0)
    mu = mu_matrix + (mu_matrix / contrast - mu_matrix) * chi
    return mu, kappa_ratio * mu


def polydomain_n0(dim, n, L, correlation_length, seed, angle_std=0.5 * np.pi):
    """scenarios.py:380-422"""
    h = 2.0 * L / n
    shape = (n,) * dim
    rng = np.random.default_rng(seed)
    cut = 2.0 * np.pi / correlation_length
    xi2 = np.zeros(shape)
    for ax in range(dim):
        sh = [1] * dim
        sh[ax] = n
        xi = np.fft.fftfreq(n, d=h) * 2.0 * np.pi
        xi2 = xi2 + (xi.reshape(sh)) ** 2
    kernel = np.exp(-0.5 * xi2 / cut ** 2)

    def filtered():
        w = rng.standard_normal(shape)
        return np.fft.ifftn(np.fft.fftn(w) * kernel).real

    if dim == 2:
        theta = filtered()
        spread = theta.std()
        if spread > 0:
            theta = theta * (angle_std / spread)
        return np.stack([np.cos(theta), np.sin(theta)], axis=-1).reshape(-1, 2)
    v = np.stack([filtered() for _ in range(3)], axis=-1).reshape(-1, 3)
    nrm = np.linalg.norm(v, axis=1)
    bad = nrm < 1e-12
    if np.any(bad):
        v[bad] = (1.0, 0.0, 0.0)
        nrm[bad] = 1.0
    return v / nrm[:, None]
