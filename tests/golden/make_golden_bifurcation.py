"""Golden fixture of the composite bifurcation study, by running the REAL
reference (`micromech.scenarios.run_bifurcation`, scenarios.py:575-666) in
the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_bifurcation.py

Writes tests/golden/bifurcation_16.npz (stress curves of the three branches,
Bloch eigenvalue traces, the tiling / perturbation helpers on the final
unit-cell state, the composite phase field, one compatibility check).
"""

import os

import numpy as np

import micromech as mm
from micromech import scenarios

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    grid = mm.Grid(2, 16, 0.5)
    proto = scenarios.ProtocolSpec("eb_compression", 1.0, 0.94, -0.02)
    params = mm.SolverParams(r_p_tol=1e-8, r_d_tol=1e-8)
    study = scenarios.run_bifurcation(grid, proto, volume_fraction=0.3, interface_width=0.06,
                                      params=params, seed=0, k_max=2)
    out = dict(n=16, L=0.5, lams=study.lams, stress_unit=study.stress_unit,
               stress_super=study.stress_super, stress_pert=study.stress_pert,
               completed=study.completed)
    for k, v in study.betas.items():
        out["beta_%d%d" % k] = v
    phase = scenarios.build_composite(grid, 0.3, 0.06)
    out["phase"] = phase
    # helpers on a small deterministic state
    rng = np.random.default_rng(5)
    st = mm.solver.init_state(grid, mm.MooneyRivlin(1.0, 9.8, dim=2), mm.MacroBC.strain(np.eye(2)),
                              mm.SolverParams())
    st.u_tilde = 0.01 * rng.standard_normal(st.u_tilde.shape)
    st.grad_u = st.grad_u + 0.01 * rng.standard_normal(st.grad_u.shape)
    st.F = st.F + 0.01 * rng.standard_normal(st.F.shape)
    st.lam = 0.01 * rng.standard_normal(st.lam.shape)
    for k in ("u_tilde", "grad_u", "F", "lam"):
        out["h_" + k] = getattr(st, k)
    t = scenarios.tile_state(grid, st, 2)
    for k in ("u_tilde", "grad_u", "F", "lam"):
        out["t_" + k] = getattr(t, k)
    v = 1e-3 * rng.standard_normal(grid.shape + (2,))
    out["v"] = v
    scenarios.perturb_state(grid, st, v)
    out["p_u_tilde"] = st.u_tilde
    out["p_grad_u"] = st.grad_u
    c = scenarios.check_stripe_compatibility([1.0, 0.3], [0.3, 1.0], 1.5)
    out["compat"] = np.array([c.compatible, c.residual], dtype=float)
    out["compat_Q"] = c.Q if c.Q is not None else np.full((2, 2), np.nan)
    np.savez_compressed(os.path.join(HERE, "bifurcation_16.npz"), **out)
    print({k: np.asarray(v).ravel()[:4] for k, v in out.items() if k.startswith("beta")},
          study.completed, study.beta_zero_lam(), study.departure_lam())


if __name__ == "__main__":
    main()
