"""Load-stepping drivers on the device-resident solver.

Mirrors the LCE/protocol half of ``micromech.scenarios``
(scenarios.py:79-187 ProtocolSpec, :311-324 composite_moduli, :380-456
director generators, :511-536 diagnostics, :680-836 records, relaxation and
the protocol driver).  The solver state stays on the GPU across load steps:
each step changes the macroscopic control on the host (a few scalars), adds
the seeded perturbation of F on the device (``mm_add_field``: the host draws
the same numpy random numbers and uploads them; the field itself never makes
a round trip), and warm-starts ``solve``.  Only the per-step records (mean
stress from the device reduction of lam, mean deformation, the orientation
tensor) come back to the host.

The composite bifurcation study (scenarios.py:537-666) runs its three
branches (unit cell, 2x2 supercell, eigenmode-seeded supercell) as
device-resident solves, with the Bloch eigenvalue sweep of stability.py on
the device between them; the microstructure (build_composite, the
MicrostructureSpec kinds), supercell tiling (tile_field / tile_state),
perturb_state and the stripe compatibility check are host utilities, as in
the reference (once per study, or per step on a few thousand points).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigurationError, ConvergenceError, ParameterError
from .grid import Grid, discrete_grad, mean_field
from .projection import MacroBC
from .solver import (ADMMState, RatioToDual, SolverParams, begin_time_step, init_state,
                     macro_stress, solve)

__all__ = ["ProtocolSpec", "StepRecord", "ProtocolStudy", "composite_moduli",
           "generate_polydomain_n0", "make_stripe_n0", "orientation_tensor", "true_stress",
           "perturb_F", "relax_zero_stress", "run_lce_protocol", "MICROSTRUCTURE_KINDS",
           "MicrostructureSpec", "build_composite", "tile_field", "tile_state", "perturb_state",
           "CompatibilityResult", "check_stripe_compatibility", "BifurcationStudy",
           "run_bifurcation"]

PROTOCOL_KINDS = ("eb_compression", "uni", "pe", "eb", "monodomain", "custom")

# pinned mean components per named protocol (scenarios.py:79-84); all other
# components are stress-controlled at zero
_PINNED = {
    "uni": [(0, 0)],
    "pe": [(0, 0), (0, 1), (1, 1)],
    "eb": [(0, 0), (0, 1), (1, 1)],
    "monodomain": [(0, 0), (0, 1), (1, 0)],
}


def _same(a, b):
    if isinstance(a, np.ndarray) or isinstance(b, np.ndarray):
        return a is not None and b is not None and np.array_equal(a, b)
    return a == b


@dataclass(frozen=True, eq=False)
class ProtocolSpec:
    """Stretch schedule lam_start -> lam_end (step lam_step) applied to the
    pinned mean components of ``kind``; ``rate`` > 0 with ``dt`` == 0 sets
    dt = |lam_step| / rate (scenarios.py:87-135)."""

    kind: str
    lam_start: float = 1.0
    lam_end: float = 1.0
    lam_step: float = 0.0
    rate: float = 0.0
    dt: float = 0.0
    strain_mask: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in PROTOCOL_KINDS:
            raise ConfigurationError(f"unknown protocol kind {self.kind!r}; expected one of "
                                     f"{PROTOCOL_KINDS}")
        span = self.lam_end - self.lam_start
        if span != 0.0 and self.lam_step == 0.0:
            raise ConfigurationError("lam_step must be nonzero for a nontrivial stretch schedule")
        if span * self.lam_step < 0.0:
            raise ConfigurationError("lam_step direction must match the schedule (monotone)")
        if self.rate < 0.0 or self.dt < 0.0:
            raise ConfigurationError("rate and dt must be nonnegative")
        if self.kind == "custom":
            if self.strain_mask is None:
                raise ConfigurationError("custom protocol needs a strain_mask")
            m = np.asarray(self.strain_mask, dtype=bool)
            if m.ndim != 2 or m.shape[0] != m.shape[1]:
                raise ConfigurationError("strain_mask must be square")
            object.__setattr__(self, "strain_mask", m)
        if self.rate > 0.0 and self.dt == 0.0:
            object.__setattr__(self, "dt", abs(self.lam_step) / self.rate)

    def __eq__(self, other):
        if not isinstance(other, ProtocolSpec):
            return NotImplemented
        return all(_same(getattr(self, f), getattr(other, f)) for f in self.__dataclass_fields__)

    def schedule(self) -> np.ndarray:
        """Stretch values, both ends included."""
        span = self.lam_end - self.lam_start
        if span == 0.0:
            return np.array([self.lam_start])
        count = int(round(span / self.lam_step))
        return self.lam_start + self.lam_step * np.arange(count + 1)

    def deformation(self, lam: float, dim: int) -> np.ndarray:
        if self.kind == "eb_compression":
            return lam * np.eye(dim)
        P = np.eye(dim)
        P[0, 0] = lam
        if self.kind == "eb":
            P[1, 1] = lam
        return P

    def mask(self, dim: int) -> np.ndarray:
        if self.kind == "eb_compression":
            return np.ones((dim, dim), dtype=bool)
        if self.kind == "custom":
            if self.strain_mask.shape != (dim, dim):
                raise ConfigurationError(f"strain_mask is {self.strain_mask.shape}, grid is "
                                         f"{dim}D")
            return self.strain_mask.copy()
        m = np.zeros((dim, dim), dtype=bool)
        for ij in _PINNED[self.kind]:
            m[ij] = True
        return m

    def macro_bc(self, lam: float, dim: int, reference: np.ndarray | None = None) -> MacroBC:
        """Pinned components = (P(lam) @ reference), the rest zero stress."""
        ref = np.eye(dim) if reference is None else np.asarray(reference)
        target = self.deformation(lam, dim) @ ref
        m = self.mask(dim)
        return MacroBC(strain_mask=m, value=np.where(m, target, 0.0))


# ---------------------------------------------------------------------------
# microstructure helpers (host, once per study)
# ---------------------------------------------------------------------------

def composite_moduli(phase: np.ndarray, mu_matrix: float = 1.0, contrast: float = 20.0,
                     kappa_ratio: float = 9.8):
    """Per-point (mu, kappa): mu linear in the clipped phase field between the
    matrix value and matrix/contrast, kappa = kappa_ratio mu
    (scenarios.py:311-324)."""
    if contrast <= 0 or mu_matrix <= 0 or kappa_ratio < 0:
        raise ConfigurationError("moduli and contrast must be positive")
    chi = np.clip(np.asarray(phase).ravel().astype(float), 0.0, 1.0)
    mu = mu_matrix + (mu_matrix / contrast - mu_matrix) * chi
    return mu, kappa_ratio * mu


def generate_polydomain_n0(grid: Grid, correlation_length: float, seed: int,
                           angle_std: float = 0.5 * np.pi) -> np.ndarray:
    """Seeded random director field (npoints, dim): Gaussian-filtered white
    noise, cut-off 2 pi / correlation_length; 2D as an angle field scaled to
    ``angle_std``, 3D as three filtered components normalised pointwise
    (scenarios.py:380-422).  Same random stream and transform sequence as the
    reference, so the fields agree to roundoff."""
    if not 0.0 < correlation_length <= 2.0 * grid.length:
        raise ConfigurationError("correlation_length must lie in (0, cell edge]")
    rng = np.random.default_rng(seed)
    cut = 2.0 * np.pi / correlation_length
    k2 = np.zeros(grid.shape)
    for ax in range(grid.dim):
        kax = 2.0 * np.pi * np.fft.fftfreq(grid.n, d=grid.h)
        shape = [1] * grid.dim
        shape[ax] = grid.n
        k2 = k2 + kax.reshape(shape) ** 2
    lowpass = np.exp(-0.5 * k2 / cut ** 2)

    def smooth_noise():
        white = rng.standard_normal(grid.shape)
        return np.fft.ifftn(np.fft.fftn(white) * lowpass).real

    if grid.dim == 2:
        theta = smooth_noise()
        spread = theta.std()
        if spread > 0:
            theta = theta * (angle_std / spread)
        return np.stack([np.cos(theta), np.sin(theta)], axis=-1).reshape(-1, 2)
    v = np.stack([smooth_noise() for _ in range(3)], axis=-1).reshape(-1, 3)
    norm = np.linalg.norm(v, axis=1)
    degenerate = norm < 1e-12
    if np.any(degenerate):
        v[degenerate] = (1.0, 0.0, 0.0)
        norm[degenerate] = 1.0
    return v / norm[:, None]


def _unit_vector(v, what):
    v = np.asarray(v, dtype=float)
    nv = np.linalg.norm(v)
    if not np.isfinite(nv) or nv < 1e-12:
        raise ConfigurationError(f"{what} must be a nonzero vector")
    return v / nv


def make_stripe_n0(grid: Grid, n0_plus, n0_minus, stripes: int) -> np.ndarray:
    """Alternating director bands normal to axis 1 (scenarios.py:425-456)."""
    if stripes < 2:
        raise ConfigurationError("need at least two stripes")
    a = _unit_vector(n0_plus, "n0_plus")
    b = _unit_vector(n0_minus, "n0_minus")
    if len(a) != grid.dim or len(b) != grid.dim:
        raise ConfigurationError("stripe directors must match the grid dimension")
    y = grid.coords()[..., 1]
    band = np.floor((y + grid.length) / (2.0 * grid.length) * stripes)
    band = np.clip(band, 0, stripes - 1).astype(int)
    n = np.where((band % 2 == 0)[..., None], a, b)
    return np.ascontiguousarray(n.reshape(-1, grid.dim))


# ---------------------------------------------------------------------------
# diagnostics
# ---------------------------------------------------------------------------

def orientation_tensor(n: np.ndarray) -> np.ndarray:
    """Nematic order tensor 3/2 (<n n> - I/3), 3x3; planar fields embedded
    (scenarios.py:511-524)."""
    n = np.asarray(n, dtype=float)
    if n.ndim != 2 or n.shape[1] not in (2, 3):
        raise ConfigurationError("director sample must be (npoints, 2|3)")
    if n.shape[1] == 2:
        n = np.concatenate([n, np.zeros((len(n), 1))], axis=1)
    second_moment = (n[:, :, None] * n[:, None, :]).mean(axis=0)
    return 1.5 * (second_moment - np.eye(3) / 3.0)


def true_stress(nominal: np.ndarray, Fbar: np.ndarray) -> np.ndarray:
    """Cauchy stress from mean nominal stress and mean deformation."""
    return nominal @ Fbar.T / np.linalg.det(Fbar)


# ---------------------------------------------------------------------------
# records
# ---------------------------------------------------------------------------

@dataclass
class StepRecord:
    """Macroscopic observables after one protocol step (scenarios.py:680-690)."""

    lam: float
    Fbar: np.ndarray
    nominal: np.ndarray
    true: np.ndarray
    S: np.ndarray
    outer_iters: int
    n_field: np.ndarray | None = None


@dataclass
class ProtocolStudy:
    records: list = field(default_factory=list)
    reference: np.ndarray | None = None
    state: ADMMState | None = None
    completed: bool = False

    @property
    def lams(self):
        return np.array([r.lam for r in self.records])

    @property
    def nominal(self):
        return np.array([r.nominal for r in self.records])

    @property
    def true(self):
        return np.array([r.true for r in self.records])

    @property
    def S(self):
        return np.array([r.S for r in self.records])


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------

def perturb_F(state: ADMMState, dF: np.ndarray) -> None:
    """``state.F = state.F + dF`` with F left on the device when it is there
    (one addition per element on the GPU, the same rounding as numpy)."""
    eng = state._engine
    if eng is not None and "F" in state._dev and "F" not in state._dirty:
        dF = np.asarray(dF, dtype=float)
        eng.grid.check_field(dF, 2, "F perturbation")
        eng.ctx.add_field(_lib.FIELD_F, dF)
        state._mark_device("F")
    else:
        state.F = state.F + dF


def _viscous(model, dt):
    return dt > 0.0 and (getattr(model, "nu_F", 0.0) > 0.0 or getattr(model, "nu_n", 0.0) > 0.0)


def relax_zero_stress(grid: Grid, model, params: SolverParams | None = None, policy=None,
                      dt: float = 0.0, max_steps: int = 200, stress_tol: float = 1e-4,
                      state: ADMMState | None = None, callback=None) -> ADMMState:
    """All components stress-controlled at zero; viscous models take implicit
    time steps until |<P>| < stress_tol mu_rep, others one equilibrium solve
    (scenarios.py:712-756)."""
    params = SolverParams() if params is None else params
    policy = RatioToDual() if policy is None else policy
    if max_steps < 1:
        raise ParameterError("max_steps must be at least 1")
    d = grid.dim
    bc = MacroBC.stress(np.zeros((d, d)))
    if state is None:
        state = init_state(grid, model, bc, params)
    viscous = _viscous(model, dt)
    level = np.inf
    for step in range(max_steps):
        if viscous:
            begin_time_step(state)
        state, ok = solve(grid, model, bc, params, policy=policy, state=state,
                          dt=dt if viscous else 0.0, raise_on_max=False)
        if not ok:
            raise ConvergenceError(f"zero-stress relaxation stalled at step {step}",
                                   history=state.history)
        level = np.linalg.norm(macro_stress(grid, state)) / model.mu_rep
        if callback is not None:
            callback(step, level, state)
        if level < stress_tol:
            return state
        if not viscous:
            break
    if level >= stress_tol:
        raise ConvergenceError(f"mean stress {level:.3e} did not relax below {stress_tol}")
    return state


def run_lce_protocol(grid: Grid, model, protocol: ProtocolSpec,
                     params: SolverParams | None = None, policy=None, relax: bool = True,
                     seed: int = 0, perturb: float = 1e-4, store_fields_at=(),
                     callback=None) -> ProtocolStudy:
    """Quasistatic / viscous loading through ``protocol.schedule()``
    (scenarios.py:759-836): per step, the mixed control relative to the
    relaxed reference, ``begin_time_step`` when viscous, the seeded
    perturbation F += perturb N(0, 1) (SeedSequence((seed, step))), a
    warm-started solve, and a record.  A failed step raises ConvergenceError
    with the partial study attached as ``partial``."""
    params = SolverParams() if params is None else params
    policy = RatioToDual() if policy is None else policy
    if protocol.kind == "eb_compression":
        raise ConfigurationError("the compression protocol belongs to the composite study")
    study = ProtocolStudy()
    state = (relax_zero_stress(grid, model, params, policy=policy, dt=protocol.dt)
             if relax else None)
    if state is None:
        state = init_state(grid, model, protocol.macro_bc(protocol.lam_start, grid.dim), params)
    ref = state.u_mean.copy()
    study.reference = ref
    viscous = _viscous(model, protocol.dt)
    keep_at = np.asarray(store_fields_at, dtype=float)
    try:
        for step, lam in enumerate(protocol.schedule()):
            bc = protocol.macro_bc(lam, grid.dim, reference=ref)
            if viscous:
                begin_time_step(state)
            if perturb > 0.0:
                rng = np.random.default_rng(np.random.SeedSequence((seed, step)))
                noise = rng.standard_normal(grid.shape + (grid.dim, grid.dim))
                perturb_F(state, perturb * noise)
            state, ok = solve(grid, model, bc, params, policy=policy, state=state,
                              dt=protocol.dt if viscous else 0.0, raise_on_max=False)
            if not ok:
                raise ConvergenceError(f"protocol step at stretch {lam:.6g} did not converge",
                                       history=state.history)
            nominal = macro_stress(grid, state)
            n = model.director(state.internal) if hasattr(model, "director") else None
            keep = keep_at.size and np.any(
                np.isclose(keep_at, lam, atol=1e-9 + 0.5 * abs(protocol.lam_step)))
            rec = StepRecord(lam=float(lam), Fbar=state.u_mean.copy(), nominal=nominal,
                             true=true_stress(nominal, state.u_mean),
                             S=orientation_tensor(n) if n is not None else np.zeros((3, 3)),
                             outer_iters=state.outer_iter,
                             n_field=n.copy() if keep and n is not None else None)
            study.records.append(rec)
            if callback is not None:
                callback(step, lam, state, rec)
    except ConvergenceError as err:
        err.partial = study
        study.state = state
        raise
    study.state = state
    study.completed = True
    return study


# ---------------------------------------------------------------------------
# microstructure specification and the composite geometry (scenarios.py:186-310)
# ---------------------------------------------------------------------------

MICROSTRUCTURE_KINDS = ("circular_inclusion", "stripe_director", "random_director",
                        "uniform_director")


def _unit(v, what):
    v = np.asarray(v, dtype=float)
    nrm = np.linalg.norm(v)
    if not np.isfinite(nrm) or nrm < 1e-12:
        raise ConfigurationError(f"{what} must be a nonzero vector")
    return v / nrm


@dataclass(frozen=True, eq=False)
class MicrostructureSpec:
    """Initial microstructure: composite phase layout or imprinted director
    field; director values renormalised to unit norm (scenarios.py:199-265)."""

    kind: str
    volume_fraction: float = 0.0
    interface_width: float = 0.02
    n0_plus: np.ndarray | None = None
    n0_minus: np.ndarray | None = None
    stripes: int = 0
    correlation_length: float = 0.0
    seed: int = 0
    n0: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in MICROSTRUCTURE_KINDS:
            raise ConfigurationError(f"unknown microstructure kind {self.kind!r}; expected one "
                                     f"of {MICROSTRUCTURE_KINDS}")
        if self.kind == "circular_inclusion":
            if not 0.0 < self.volume_fraction < 1.0:
                raise ConfigurationError("volume_fraction must lie in (0, 1)")
            if self.interface_width < 0.0:
                raise ConfigurationError("interface_width must be nonnegative")
        elif self.kind == "stripe_director":
            if self.stripes < 2:
                raise ConfigurationError("need at least two stripes")
            object.__setattr__(self, "n0_plus", _unit(self.n0_plus, "n0_plus"))
            object.__setattr__(self, "n0_minus", _unit(self.n0_minus, "n0_minus"))
        elif self.kind == "random_director":
            if self.correlation_length <= 0.0:
                raise ConfigurationError("correlation_length must be positive")
        elif self.kind == "uniform_director":
            object.__setattr__(self, "n0", _unit(self.n0, "n0"))

    def __eq__(self, other):
        if not isinstance(other, MicrostructureSpec):
            return NotImplemented
        return all(_same(getattr(self, f), getattr(other, f)) for f in self.__dataclass_fields__)

    def build(self, grid: Grid) -> np.ndarray:
        """Phase field (grid shape) or n0 field (npoints, dim)."""
        if self.kind == "circular_inclusion":
            return build_composite(grid, self.volume_fraction, self.interface_width)
        if self.kind == "stripe_director":
            return make_stripe_n0(grid, self.n0_plus, self.n0_minus, self.stripes)
        if self.kind == "random_director":
            return generate_polydomain_n0(grid, self.correlation_length, self.seed)
        if len(self.n0) != grid.dim:
            raise ConfigurationError("uniform director dimension must match the grid")
        return np.tile(self.n0, (grid.npoints, 1))


def build_composite(grid: Grid, volume_fraction: float,
                    interface_width: float = 0.02) -> np.ndarray:
    """Centred circular inclusion with an erf-graded boundary whose cell mean
    is exactly ``volume_fraction`` (scenarios.py:271-308): the erf disc
    carries area pi (radius^2 + width^2), so the radius is shrunk by the
    width; width 0 is the sharp pixel disc."""
    from scipy import special
    if grid.dim != 2:
        raise ConfigurationError("the composite layout is two-dimensional")
    if not 0.0 < volume_fraction < 1.0:
        raise ConfigurationError("volume_fraction must lie in (0, 1)")
    if not 0.0 <= interface_width < grid.length:
        raise ConfigurationError(
            f"interface_width {interface_width} must lie in [0, {grid.length})")
    L = grid.length
    r0sq = (2.0 * L) ** 2 * volume_fraction / np.pi
    if r0sq <= interface_width ** 2:
        raise ConfigurationError(f"volume fraction {volume_fraction} gives an inclusion smaller "
                                 f"than interface_width {interface_width}")
    radius = np.sqrt(r0sq - interface_width ** 2)
    if radius > L:
        raise ConfigurationError(f"volume fraction {volume_fraction} needs inclusion radius "
                                 f"{radius:.3f} > half cell {L}")
    x = grid.coords()
    r = np.sqrt(np.sum(x * x, axis=-1))
    if interface_width == 0.0:
        return (r <= radius).astype(float)
    return 0.5 * special.erfc((r - radius) / (np.sqrt(2.0) * interface_width))


# ---------------------------------------------------------------------------
# supercell tiling (scenarios.py:331-378)
# ---------------------------------------------------------------------------

def tile_field(grid: Grid, f: np.ndarray, k: int) -> np.ndarray:
    """Replicate a cell field onto the k x ... x k supercell."""
    extra = f.ndim - grid.dim
    if f.shape[: grid.dim] != grid.shape:
        raise ConfigurationError("field does not live on this grid")
    return np.tile(f, (k,) * grid.dim + (1,) * extra)


def _tile_points(grid: Grid, a: np.ndarray, k: int) -> np.ndarray:
    shaped = a.reshape(grid.shape + a.shape[1:])
    tiled = tile_field(grid, shaped, k)
    return np.ascontiguousarray(tiled.reshape((-1,) + a.shape[1:]))


def tile_state(grid: Grid, state: ADMMState, k: int) -> ADMMState:
    """Solver state replicated onto the supercell, counters reset; the
    fields are read from the device once and the new state uploads on its
    first solve.  Point-indexed internals are re-flattened in the
    supercell's row-major point order."""
    return ADMMState(
        u_mean=np.array(state.u_mean, dtype=float),
        u_tilde=tile_field(grid, np.asarray(state.u_tilde), k),
        grad_u=tile_field(grid, np.asarray(state.grad_u), k),
        F=tile_field(grid, np.asarray(state.F), k),
        lam=tile_field(grid, np.asarray(state.lam), k),
        internal={key: _tile_points(grid, np.asarray(a), k)
                  for key, a in (state.internal or {}).items()},
        rho=state.rho,
    )


def perturb_state(grid: Grid, state: ADMMState, v: np.ndarray) -> None:
    """Add a displacement field to the compatible iterate (scenarios.py:
    361-374): u_tilde += v - <v>, grad_u += D(v - <v>); F keeps its warm
    values, so the local admissibility guards see the perturbation through
    the projected gradient.  Assigning the fields uploads them before the
    next device operation."""
    grid.check_field(v, 1, "perturbation")
    v = v - mean_field(grid, v)
    state.u_tilde = np.asarray(state.u_tilde) + v
    state.grad_u = np.asarray(state.grad_u) + discrete_grad(grid, v)


# ---------------------------------------------------------------------------
# stripe compatibility (scenarios.py:451-508)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CompatibilityResult:
    compatible: bool
    Q: np.ndarray | None
    a: np.ndarray | None
    residual: float


def check_stripe_compatibility(n0_plus, n0_minus, r: float, normal=None, tol: float = 1e-8,
                               seed: int = 0) -> CompatibilityResult:
    """Rank-one compatibility Q U+ = U- + a (x) normal of the two spontaneous
    stretches: multi-start least squares on the rotation-free normal
    equation (U- + a (x) nu)^T (U- + a (x) nu) = U+^2, Q recovered after."""
    from scipy.optimize import least_squares

    from .materials.lce import step_length_sqrt
    np0 = _unit(n0_plus, "n0_plus")
    nm0 = _unit(n0_minus, "n0_minus")
    d = len(np0)
    if len(nm0) != d:
        raise ConfigurationError("directors must have equal dimension")
    if normal is None:
        normal = np.zeros(d)
        normal[1] = 1.0
    nu = _unit(normal, "normal")
    Up = step_length_sqrt(np0[None], r)[0]
    Um = step_length_sqrt(nm0[None], r)[0]
    target = Up @ Up
    scale = np.linalg.norm(target)

    def resid(a):
        M = Um + np.outer(a, nu)
        return ((M.T @ M) - target)[np.triu_indices(d)]

    rng = np.random.default_rng(seed)
    starts = [np.zeros(d)] + [0.5 * rng.standard_normal(d) for _ in range(7)]
    best = None
    for a0 in starts:
        sol = least_squares(resid, a0, xtol=1e-15, ftol=1e-15, gtol=1e-15)
        M = Um + np.outer(sol.x, nu)
        if np.linalg.det(M) <= 0:
            continue
        res = np.linalg.norm(resid(sol.x)) / scale
        if best is None or res < best[0]:
            best = (res, sol.x, M)
    if best is None or best[0] > tol:
        return CompatibilityResult(False, None, None, np.inf if best is None else best[0])
    res, a, M = best
    return CompatibilityResult(True, M @ np.linalg.inv(Up), a, res)


# ---------------------------------------------------------------------------
# composite bifurcation study (scenarios.py:537-666)
# ---------------------------------------------------------------------------

@dataclass
class BifurcationStudy:
    """Three stress-stretch curves plus the cell stability trace."""

    lams: np.ndarray
    stress_unit: np.ndarray      # (nstep, d, d) nominal, unit cell
    stress_super: np.ndarray     # supercell from the tiled state
    stress_pert: np.ndarray      # supercell with eigenmode-seeded guesses
    betas: dict                  # multiplicity -> (nstep,) eigenvalue trace
    completed: bool = True

    def beta_zero_lam(self, k=(2, 2)) -> float | None:
        """First schedule point where the k eigenvalue is <= 0."""
        tr = self.betas[tuple(k)]
        hit = np.nonzero(tr <= 0.0)[0]
        return None if hit.size == 0 else float(self.lams[hit[0]])

    def departure_lam(self, rel: float = 1e-3) -> float | None:
        """First point where the perturbed curve leaves the unperturbed one
        by more than ``rel`` of the curve's stress scale."""
        a = self.stress_super[:, 0, 0]
        b = self.stress_pert[:, 0, 0]
        scale = np.nanmax(np.abs(a))
        if not np.isfinite(scale) or scale == 0.0:
            scale = 1.0
        hit = np.nonzero(np.abs(a - b) > rel * scale)[0]
        return None if hit.size == 0 else float(self.lams[hit[0]])


def _solve_step(grid, model, bc, params, policy, state, label, lam):
    state, ok = solve(grid, model, bc, params, policy=policy, state=state, raise_on_max=False)
    if not ok:
        raise ConvergenceError(f"{label} branch did not converge at stretch {lam:.6g}",
                               history=state.history)
    return state


def run_bifurcation(grid: Grid, protocol: ProtocolSpec, volume_fraction: float = 0.3,
                    interface_width: float = 0.02, mu_matrix: float = 1.0,
                    contrast: float = 20.0, kappa_ratio: float = 9.8,
                    params: SolverParams | None = None, policy=None, seed: int = 0,
                    k_max: int = 2, perturb_amplitude: float = 1e-3,
                    stability_tol: float = 1e-8, callback=None) -> BifurcationStudy:
    """Equi-biaxial compression of the circular-inclusion composite
    (scenarios.py:575-666): per stretch value the unit cell, the 2x2
    supercell continued from the tiled unit state, and the supercell with
    the dominant Bloch eigenmode added to its initial guess, plus the Bloch
    eigenvalue trace for every multiplicity up to ``k_max``.  The three
    states stay resident on the device across the schedule (one engine
    each); the Bloch sweep runs on the device between the solves.  On solver
    failure the partial study is attached to the raised error."""
    from .materials import MooneyRivlin
    from .stability import mode_to_perturbation, stability_sweep
    if params is None:
        params = SolverParams()
    if policy is None:
        policy = RatioToDual()
    phase = build_composite(grid, volume_fraction, interface_width)
    mu, kappa = composite_moduli(phase, mu_matrix, contrast, kappa_ratio)
    model = MooneyRivlin(mu, kappa, dim=grid.dim, mu_rep=mu_matrix)
    grid2 = grid.supercell(2)
    mu2 = _tile_points(grid, mu[:, None], 2)[:, 0]
    model2 = MooneyRivlin(mu2, kappa_ratio * mu2, dim=grid.dim, mu_rep=mu_matrix)

    lams = protocol.schedule()
    ks = [tuple(x + 1 for x in flat) for flat in np.ndindex(*(k_max,) * grid.dim)]
    study = BifurcationStudy(
        lams=lams,
        stress_unit=np.full((len(lams), grid.dim, grid.dim), np.nan),
        stress_super=np.full((len(lams), grid.dim, grid.dim), np.nan),
        stress_pert=np.full((len(lams), grid.dim, grid.dim), np.nan),
        betas={k: np.full(len(lams), np.nan) for k in ks},
        completed=False,
    )
    s_unit = s_super = s_pert = None
    warm_modes = None
    try:
        for i, lam in enumerate(lams):
            bc = protocol.macro_bc(lam, grid.dim)
            s_unit = _solve_step(grid, model, bc, params, policy, s_unit, "unit-cell", lam)
            study.stress_unit[i] = macro_stress(grid, s_unit)

            sweep = stability_sweep(grid, model, s_unit, k_max=k_max, seed=seed,
                                    p0_map=warm_modes, tol_beta=stability_tol)
            warm_modes = {res.k: res.p for res in sweep}
            for res in sweep:
                study.betas[res.k][i] = res.beta

            if s_super is None:
                s_super = tile_state(grid, s_unit, 2)
            s_super = _solve_step(grid2, model2, bc, params, policy, s_super, "supercell", lam)
            study.stress_super[i] = macro_stress(grid2, s_super)

            if s_pert is None:
                s_pert = tile_state(grid, s_unit, 2)
            if perturb_amplitude > 0.0:
                # seed with the period-doubling eigenmode; fall back to the
                # softest multi-cell mode
                k22 = (2,) * grid.dim
                multi = [rr for rr in sweep if max(rr.k) > 1]
                lead = next((rr for rr in multi if rr.k == k22),
                            min(multi, key=lambda rr: rr.beta))
                v = mode_to_perturbation(grid, lead, perturb_amplitude)
                if lead.k != k22:
                    v = np.tile(v, tuple(2 // kk for kk in lead.k) + (1,))
                perturb_state(grid2, s_pert, v)
            s_pert = _solve_step(grid2, model2, bc, params, policy, s_pert,
                                 "perturbed supercell", lam)
            study.stress_pert[i] = macro_stress(grid2, s_pert)

            if callback is not None:
                callback(i, lam, study)
    except ConvergenceError as err:
        err.partial = study
        raise
    study.completed = True
    return study
