"""Bloch-wave stability of converged periodic states (
micromech/stability.py).

A converged unit-cell state is stable against perturbations periodic on a
(k_1 x ... x k_d) supercell iff the smallest eigenvalue beta of the
Hermitian acoustic operator (A p)_i = B*_j L_ijkl B_l p_k, B_j = d_j + i
omega_j, omega_j = pi / (L k_j), is nonnegative.  beta comes from the
reference's splitting iteration (stability.py:171-289), which runs on the
device (csrc/mm_bloch.cu): the pointwise (L + rho I)^-1 apply, the
full-spectrum complex transforms of the d^2 gradient components, the
sphere-constrained projection (its secular equation solved by bisection in
one CTA with deterministic reductions) and the Rayleigh quotient /
multiplier ascent.  Per solve, the host prepares what the reference
prepares with numpy -- the tangent field, its pointwise spectrum (for the
default penalty), (L + rho I)^-1 and the shifted symbols with their live
mask -- and keeps the reference's restart policy (penalty x4 on divergence).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._engine import scratch_engine
from .errors import ParameterError
from .grid import Grid, modified_symbols

__all__ = ["BlochResult", "tangent_field", "bloch_symbols", "bloch_min_eigen",
           "stability_sweep", "first_unstable", "mode_to_perturbation", "BAND_FRACTION"]

BAND_FRACTION = 0.75


@dataclass
class BlochResult:
    """Smallest Bloch eigenvalue for one supercell multiplicity."""

    k: tuple
    omega: np.ndarray
    beta: float
    p: np.ndarray          # complex mode, grid.shape + (d,), unit mean-square norm
    iterations: int
    converged: bool


def tangent_field(grid: Grid, model, state) -> np.ndarray:
    """Incremental moduli at the state, (npts, d, d, d, d), checked for the
    major symmetry the Hermitian eigenproblem needs (stability.py:61-78)."""
    if not getattr(model, "has_tangent", False):
        raise ParameterError(f"model '{model.name}' provides no incremental tangent")
    d = grid.dim
    npts = grid.npoints
    L = model.tangent(np.asarray(state.F).reshape(npts, d, d), state.internal)
    asym = np.abs(L - np.transpose(L, (0, 3, 4, 1, 2))).max()
    scale = np.abs(L).max()
    if asym > 1e-8 * max(scale, 1e-300):
        raise ParameterError(f"tangent field lacks major symmetry (error {asym:.3e})")
    return L


def bloch_symbols(grid: Grid, k) -> tuple:
    """(omega, b, |b|^2, live) on the full spectrum for multiplicity k
    (stability.py:83-117): b = i (xi + omega); live drops the rigid
    translation and every frequency with a component beyond BAND_FRACTION of
    the band edge (collocation aliasing)."""
    k = tuple(int(x) for x in np.atleast_1d(k))
    if len(k) != grid.dim or any(x < 1 for x in k):
        raise ParameterError(f"multiplicity {k} invalid for dim {grid.dim}")
    omega = np.pi / (grid.length * np.asarray(k, dtype=float))
    xi = modified_symbols(grid).xi
    shifted = xi + omega
    b = 1j * shifted
    bsq = np.sum(shifted * shifted, axis=-1)
    edge = np.pi / grid.h
    band = np.all(np.abs(xi) <= (BAND_FRACTION + 1e-12) * edge, axis=-1)
    live = (bsq > 1e-14 * bsq.max()) & band
    return omega, b, bsq, live


def bloch_min_eigen(grid: Grid, Lfield: np.ndarray, k, mu_rep: float,
                    rho: float | None = None, seed: int = 0, tol_beta: float = 1e-10,
                    tol_primal: float = 1e-8, max_iter: int = 20000,
                    p0: np.ndarray | None = None) -> BlochResult:
    """Smallest eigenvalue of the Bloch acoustic operator at multiplicity k
    (stability.py:171-289).  The default penalty is the spread of the
    pointwise tangent spectrum, lambda_max + |lambda_min|_-; without an
    explicit rho a diverging solve restarts with the penalty x4 (up to four
    attempts)."""
    d = grid.dim
    npts = grid.npoints
    D = d * d
    Lmat = np.ascontiguousarray(np.asarray(Lfield, dtype=float).reshape(npts, D, D))
    spec = np.linalg.eigvalsh(Lmat)
    lam_min, lam_max = float(spec.min()), float(spec.max())
    user_rho = rho is not None
    if rho is None:
        rho = lam_max + max(0.0, -lam_min)
        if rho <= 0.0:
            rho = mu_rep
    elif rho <= -lam_min:
        raise ParameterError(f"penalty {rho} does not dominate the tangent spectrum "
                             f"(lambda_min = {lam_min:.3e})")
    omega, _, bsq, live = bloch_symbols(grid, k)
    shifted = modified_symbols(grid).xi + omega
    target = float(npts) ** 2  # Parseval image of a unit mean-square norm
    floor = min(0.0, lam_min) * float(bsq[live].max())
    if p0 is not None:
        grid.check_field(p0, 1, "p0")
    ctx = scratch_engine(grid).ctx
    beta, iters, converged = np.inf, 0, False
    for _attempt in range(4):
        Minv = np.linalg.inv(Lmat + rho * np.eye(D))
        ctx.bloch_setup(Minv, Lmat, shifted.reshape(npts, d), bsq.reshape(npts),
                        live.reshape(npts), rho, target)
        if p0 is not None:
            p = np.asarray(p0, dtype=complex)
        else:
            rng = np.random.default_rng(seed)
            p = np.full(grid.shape + (d,), 1.0 / np.sqrt(d), dtype=complex)
            p += 1e-3 * (rng.standard_normal(p.shape) + 1j * rng.standard_normal(p.shape))
        ctx.bloch_start(p.reshape(npts, d))
        beta, _primal, iters, converged, diverged = ctx.bloch_iterate(
            max_iter, tol_beta, tol_primal, floor, mu_rep)
        if not diverged or user_rho:
            break
        rho *= 4.0
    mode = ctx.bloch_mode((npts, d)).reshape(grid.shape + (d,))
    return BlochResult(k=tuple(int(x) for x in np.atleast_1d(k)), omega=omega, beta=beta,
                       p=mode, iterations=iters, converged=converged)


def stability_sweep(grid: Grid, model, state, k_max: int = 4, seed: int = 0,
                    p0_map: dict | None = None, **kwargs) -> list[BlochResult]:
    """One result per multiplicity 1 <= k_j <= k_max, lexicographic
    (stability.py:292-310)."""
    if k_max < 1:
        raise ParameterError("k_max must be at least 1")
    Lfield = tangent_field(grid, model, state)
    out = []
    for flat in np.ndindex(*(k_max,) * grid.dim):
        k = tuple(x + 1 for x in flat)
        p0 = p0_map.get(k) if p0_map else None
        out.append(bloch_min_eigen(grid, Lfield, k, model.mu_rep, seed=seed, p0=p0, **kwargs))
    return out


def first_unstable(results: list[BlochResult], mu_rep: float, tol: float = 1e-8):
    """Lowest-|k| multiplicity with a negative eigenvalue, or None."""
    bad = [r for r in results if r.beta < -tol * mu_rep]
    if not bad:
        return None
    return min(bad, key=lambda r: (float(np.sum(np.square(r.k))), r.k))


def mode_to_perturbation(grid: Grid, result: BlochResult, amplitude: float) -> np.ndarray:
    """Real displacement of the Bloch mode tiled over its supercell, scaled so
    the largest pointwise magnitude is amplitude x cell edge
    (stability.py:322-341)."""
    k = result.k
    tiled = np.tile(result.p, tuple(k) + (1,))
    axes = [-grid.length * kj + grid.h * np.arange(grid.n * kj) for kj in k]
    x = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)
    carrier = np.exp(1j * np.einsum("...j,j->...", x, result.omega))
    v = np.real(tiled * carrier[..., None])
    peak = np.abs(v).max()
    if peak > 0:
        v *= amplitude * (2.0 * grid.length) / peak
    return v
