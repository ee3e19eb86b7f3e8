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

Not here: the composite bifurcation study (``run_bifurcation``, needs the
Bloch stability analysis of ``stability.py``), supercell tiling and
``check_stripe_compatibility`` (host-side utilities off the hot path).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigurationError, ConvergenceError, ParameterError
from .grid import Grid
from .projection import MacroBC
from .solver import (ADMMState, RatioToDual, SolverParams, begin_time_step, init_state,
                     macro_stress, solve)

__all__ = ["ProtocolSpec", "StepRecord", "ProtocolStudy", "composite_moduli",
           "generate_polydomain_n0", "make_stripe_n0", "orientation_tensor", "true_stress",
           "perturb_F", "relax_zero_stress", "run_lce_protocol"]

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
