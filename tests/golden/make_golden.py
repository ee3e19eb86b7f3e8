"""Generate golden fixtures by running the REAL reference (`micromech`).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each fixture stores the seeded inputs and the
reference's outputs, so tests can replay the same call through the oracle
(CPU) and through the CUDA product path (GPU) and compare both against the
reference's own numbers.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import micromech as mm  # noqa: E402
from micromech.materials import lce as lce_mod  # noqa: E402
from micromech import scenarios  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def random_states(rng, npts, dim, spread=0.3, min_det=0.2):
    """test_materials.py:37-47"""
    out = np.empty((npts, dim, dim))
    n = 0
    while n < npts:
        F = np.eye(dim) + spread * rng.standard_normal((dim, dim))
        if np.linalg.det(F) > min_det:
            out[n] = F
            n += 1
    return out


def local_mr(dim, seed, npts, max_sweeps, point_tol, rho, two_phase=True):
    rng = np.random.default_rng(seed)
    if two_phase:
        mu = np.where(rng.random(npts) < 0.3, 1.0, 20.0)
    else:
        mu = np.full(npts, 1.0)
    kap = 9.8 * mu
    m = mm.MooneyRivlin(mu=mu, kappa=kap, dim=dim, mu_rep=float(mu.max()))
    G = random_states(rng, npts, dim, spread=0.15)
    lam = 0.3 * rng.standard_normal((npts, dim, dim))
    F0 = G + 0.02 * rng.standard_normal((npts, dim, dim))
    F = F0.copy()
    st = m.local_sweeps(F, {}, G, lam, rho, 0.0, None, None, {}, max_sweeps, point_tol)
    return dict(mu=mu, kappa=kap, mu_rep=m.mu_rep, G=G, lam=lam, F0=F0, rho=rho,
                max_sweeps=max_sweeps, point_tol=point_tol, F=F, res=st.res_pts,
                sweeps=st.sweeps, frac=st.converged_frac)


def local_quad(seed, npts, dim, max_sweeps, point_tol, rho):
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.5, 3.0, npts)
    q = mm.QuadraticMaterial(c=c, dim=dim)
    G = 0.2 * rng.standard_normal((npts, dim, dim))
    lam = 0.3 * rng.standard_normal((npts, dim, dim))
    F0 = G.copy()
    F = F0.copy()
    st = q.local_sweeps(F, {}, G, lam, rho, 0.0, None, None, {}, max_sweeps, point_tol)
    return dict(c=c, mu_rep=q.mu_rep, G=G, lam=lam, F0=F0, rho=rho, max_sweeps=max_sweeps,
                point_tol=point_tol, F=F, res=st.res_pts, sweeps=st.sweeps,
                frac=st.converged_frac)


def unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def local_lce(dim, seed, npts, max_sweeps, point_tol, rho, dt=0.0, nu_F=0.0, nu_n=0.0,
              frank=True):
    rng = np.random.default_rng(seed)
    n0 = unit(rng.standard_normal((npts, dim)))
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim,
                                  nu_F=nu_F, nu_n=nu_n)
    internal = m.init_internal(npts)
    # perturb the stored director angles a little so the director is loaded
    internal["angles"] = internal["angles"] + 0.2 * rng.standard_normal(internal["angles"].shape)
    G = random_states(rng, npts, dim, spread=0.1, min_det=0.5)
    lam = 0.2 * rng.standard_normal((npts, dim, dim))
    F0 = G + 0.01 * rng.standard_normal((npts, dim, dim))
    ff = 1e-3 * rng.standard_normal((npts, dim)) if frank else np.zeros((npts, dim))
    prev_F = prev_internal = None
    if dt > 0:
        prev_F = F0 + 0.01 * rng.standard_normal(F0.shape)
        prev_internal = {k: v.copy() for k, v in internal.items()}
        prev_internal["angles"] = prev_internal["angles"] + 0.05
    inputs = {k + "0": v.copy() for k, v in internal.items()}
    F = F0.copy()
    st = m.local_sweeps(F, internal, G, lam, rho, dt, prev_F, prev_internal,
                        {"frank_force": ff}, max_sweeps, point_tol)
    # per-point nsw / ok straight from the kernels (lce.py:256-272)
    out = dict(n0=n0, G=G, lam=lam, F0=F0, ff=ff, rho=rho, dt=dt, nu_F=nu_F, nu_n=nu_n,
               max_sweeps=max_sweeps, point_tol=point_tol, F=F, res=st.res_pts,
               sweeps=st.sweeps, frac=st.converged_frac, **inputs,
               **{k: v for k, v in internal.items()})
    if prev_F is not None:
        out["prev_F"] = prev_F
        for k, v in prev_internal.items():
            out["prev_" + k] = v
    # rerun on copies through the raw kernel to get per-point nsw and ok
    Fr = F0.copy()
    intr = {k: inputs[k + "0"].copy() for k in internal}
    d = dim
    r1d = m.r ** (1.0 / d)
    phiF_scale = m.mu * (r1d * (d + 1.0) + m.alpha * d) + m.gamma_inc
    phin_scale = m.mu * (r1d + m.alpha) * d * m.r ** (2.0 / d)
    if dt > 0:
        vis_F, vis_n = nu_F / dt, nu_n / dt
        Fk, nk = prev_F, m.director(prev_internal)
    else:
        vis_F = vis_n = 0.0
        Fk, nk = np.zeros_like(Fr), np.zeros((npts, d))
    res = np.empty(npts)
    nsw = np.zeros(npts, dtype=np.int64)
    ok = np.zeros(npts, dtype=np.bool_)
    args = (m.mu, r1d, (m.r - 1.0) / m.r, m.alpha, m.gamma_inc, float(rho), vis_F, vis_n,
            point_tol * m.mu_rep, m.det_tol, int(max_sweeps), phiF_scale, phin_scale, res, nsw, ok)
    if d == 2:
        lce_mod._lce_sweeps_2d(Fr, intr["angles"], intr["p_inc"], G, lam, m.n0, ff, Fk, nk, *args)
    else:
        lce_mod._lce_sweeps_3d(Fr, intr["angles"], intr["chart"], intr["p_inc"], G, lam, m.n0, ff,
                               Fk, nk, *args)
    assert np.array_equal(Fr, F)
    out["nsw"] = nsw
    out["ok"] = ok
    return out


def projection(dim, n, seed, L=0.5):
    rng = np.random.default_rng(seed)
    g = mm.Grid(dim, n, L)
    F = np.eye(dim) + 0.1 * rng.standard_normal(g.shape + (dim, dim))
    lam = 0.3 * rng.standard_normal(g.shape + (dim, dim))
    rho = 3.7
    mask = rng.random((dim, dim)) < 0.5
    value = np.where(mask, np.eye(dim) + 0.05 * rng.standard_normal((dim, dim)),
                     0.1 * rng.standard_normal((dim, dim)))
    bc = mm.MacroBC(mask, value)
    pr = mm.helmholtz_project(g, F, lam, rho, bc)
    return dict(dim=dim, n=n, L=L, F=F, lam=lam, rho=rho, mask=mask, value=value,
                u_mean=pr.u_mean, u_tilde=pr.u_tilde, grad_u=pr.grad_u)


def hist_arr(history):
    return np.array([[r.outer_iter, r.r_p, r.r_d, r.r_l, r.rho] for r in history])


def trajectory_mr2d(K=12):
    rng = np.random.default_rng(9)
    g = mm.Grid(2, 8)
    mu = np.where(rng.random(g.npoints) < 0.3, 1.0, 20.0)
    m = mm.MooneyRivlin(mu=mu, kappa=9.8 * mu, dim=2, mu_rep=20.0)
    bc = mm.MacroBC.strain(np.array([[0.92, 0.05], [0.0, 1.03]]))
    params = mm.SolverParams(max_outer=K)
    st, conv = mm.solve(g, m, bc, params, policy=mm.RatioToDual(0.3), raise_on_max=False)
    return dict(n=8, L=0.5, mu=mu, kappa=9.8 * mu, mu_rep=20.0, mask=bc.strain_mask,
                value=bc.value, K=K, F=st.F, lam=st.lam, grad_u=st.grad_u, u_tilde=st.u_tilde,
                u_mean=st.u_mean, hist=hist_arr(st.history), total_sweeps=st.total_sweeps)


def trajectory_mr3d(K=6, n=8):
    g = mm.Grid(3, n, 0.5)
    x = g.coords()[..., 0]
    phase = ((x + g.length) / (2 * g.length) < 0.5)
    mu, kap = scenarios.composite_moduli(phase, 1.0, 20.0, 9.8)
    m = mm.MooneyRivlin(mu=mu, kappa=kap, dim=3, mu_rep=1.0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    params = mm.SolverParams(max_outer=K)
    st = mm.solver.init_state(g, m, bc, params)
    st.F = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
    F0 = st.F.copy()
    st, conv = mm.solve(g, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                        raise_on_max=False)
    return dict(n=n, L=0.5, mu=mu, kappa=kap, mu_rep=1.0, mask=bc.strain_mask, value=bc.value,
                K=K, F0=F0, F=st.F, lam=st.lam, grad_u=st.grad_u, u_tilde=st.u_tilde,
                u_mean=st.u_mean, hist=hist_arr(st.history), total_sweeps=st.total_sweeps)


def config1_protocol():
    """2D 64^2 laminate, monodomain lam 1.0 -> 0.8."""
    g = mm.Grid(2, 64, 0.5)
    y = g.coords()[..., 1]
    phase = ((y + g.length) / (2 * g.length) < 0.5)
    mu, kap = scenarios.composite_moduli(phase, 1.0, 20.0, 9.8)
    m = mm.MooneyRivlin(mu=mu, kappa=kap, dim=2, mu_rep=1.0)
    proto = mm.ProtocolSpec("monodomain", 1.0, 0.8, -0.02)
    study = mm.run_lce_protocol(g, m, proto, relax=True, seed=0, perturb=1e-4)
    recs = study.records
    return dict(n=64, L=0.5, mu=mu, kappa=kap,
                lams=np.array([r.lam for r in recs]),
                outer_iters=np.array([r.outer_iters for r in recs]),
                nominal=np.array([r.nominal for r in recs]),
                Fbar=np.array([r.Fbar for r in recs]),
                F=study.state.F, lam=study.state.lam, grad_u=study.state.grad_u,
                hist=hist_arr(study.state.history))


def lce_uniform_solve():
    """test_lce.py:531-544 fixture (uniform n0, strain control, ExactAll):
    local-convergent, so full-trajectory parity is well posed."""
    g = mm.Grid(2, 12, 0.5)
    n0 = np.tile([np.cos(0.35), np.sin(0.35)], (g.npoints, 1))
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=n0, dim=2)
    bc = mm.MacroBC.strain(np.diag([1.03, 1.0 / 1.03]))
    params = mm.SolverParams(r_p_tol=1e-8, r_d_tol=1e-8, point_tol=1e-12, max_outer=4000)
    st, conv = mm.solve(g, m, bc, params)
    assert conv
    return dict(n=12, L=0.5, n0=n0, mask=bc.strain_mask, value=bc.value, F=st.F, lam=st.lam,
                grad_u=st.grad_u, angles=st.internal["angles"], p_inc=st.internal["p_inc"],
                hist=hist_arr(st.history), total_sweeps=st.total_sweeps)


def lce_stripe_iters(K=6):
    """Two-director stripes under strain control, ExactAll, K iterations."""
    g = mm.Grid(2, 16, 0.5)
    n0 = scenarios.make_stripe_n0(g, [1.0, 0.2], [0.2, 1.0], 4)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=n0, dim=2)
    bc = mm.MacroBC.strain(np.diag([1.02, 1.0 / 1.02]))
    params = mm.SolverParams(point_tol=1e-12, max_outer=K)
    st, _ = mm.solve(g, m, bc, params, raise_on_max=False)
    return dict(n=16, L=0.5, n0=n0, mask=bc.strain_mask, value=bc.value, K=K, F=st.F,
                lam=st.lam, grad_u=st.grad_u, angles=st.internal["angles"],
                p_inc=st.internal["p_inc"], hist=hist_arr(st.history),
                total_sweeps=st.total_sweeps)


def lce_poly_one_iter(dim, n, seed=1, max_local=10):
    """One outer iteration of polydomain LCE (chaotic beyond)."""
    g = mm.Grid(dim, n, 0.5)
    n0 = scenarios.generate_polydomain_n0(g, 0.25, seed=seed)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim)
    bc = mm.MacroBC.stress(np.zeros((dim, dim)))
    params = mm.SolverParams(max_outer=1, max_local=max_local)
    st = mm.solver.init_state(g, m, bc, params)
    st.F = st.F + 1e-3 * np.random.default_rng(seed).standard_normal(st.F.shape)
    F0 = st.F.copy()
    st, _ = mm.solve(g, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    out = dict(dim=dim, n=n, L=0.5, n0=n0, F0=F0, max_local=max_local, F=st.F, lam=st.lam,
               grad_u=st.grad_u, u_tilde=st.u_tilde, hist=hist_arr(st.history),
               total_sweeps=st.total_sweeps)
    for k, v in st.internal.items():
        out["int_" + k] = v
    return out


def frank(dim, n, seed=4):
    rng = np.random.default_rng(seed)
    g = mm.Grid(dim, n, 0.5)
    nf = unit(rng.standard_normal((g.npoints, dim)))
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=0.3, n0=nf, dim=dim)
    ff = m.frank_force(g, nf.reshape(g.shape + (dim,)))
    return dict(dim=dim, n=n, L=0.5, n_field=nf, kappa=0.3, ff=ff)


def eq_residual_cases():
    """equilibrium_residual (solver.py:346-371) on seeded non-equilibrium
    states: MR 2D/3D, quadratic on an odd grid, LCE 2D viscous, LCE 3D."""
    rng = np.random.default_rng(601)
    out = {}

    def state_for(g, model, F, internal=None, prev_F=None, prev_internal=None):
        d = g.dim
        z = np.zeros(g.shape + (d, d))
        return mm.ADMMState(u_mean=np.eye(d), u_tilde=np.zeros(g.shape + (d,)), grad_u=z.copy(),
                            F=F, lam=z.copy(), internal=internal or {}, rho=1.0,
                            prev_F=prev_F, prev_internal=prev_internal)

    # MR 2D, two-phase
    g = mm.Grid(2, 16, 0.5)
    y = g.coords()[..., 1]
    mu, kap = scenarios.composite_moduli((y + 0.5) < 0.5, 1.0, 20.0, 9.8)
    F = np.eye(2) + 0.05 * rng.standard_normal(g.shape + (2, 2))
    m = mm.MooneyRivlin(mu, kap, dim=2, mu_rep=1.0)
    out["mr2d_F"], out["mr2d_mu"], out["mr2d_kappa"] = F, mu, kap
    out["mr2d_val"] = mm.equilibrium_residual(g, m, state_for(g, m, F))
    # MR 3D
    g = mm.Grid(3, 8, 0.5)
    x = g.coords()[..., 0]
    mu, kap = scenarios.composite_moduli((x + 0.5) < 0.5, 1.0, 20.0, 9.8)
    F = np.eye(3) + 0.05 * rng.standard_normal(g.shape + (3, 3))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    out["mr3d_F"], out["mr3d_mu"], out["mr3d_kappa"] = F, mu, kap
    out["mr3d_val"] = mm.equilibrium_residual(g, m, state_for(g, m, F))
    # quadratic, odd n
    g = mm.Grid(2, 9, 0.5)
    c = 1.0 + rng.random(g.npoints)
    F = np.eye(2) + 0.1 * rng.standard_normal(g.shape + (2, 2))
    m = mm.QuadraticMaterial(c, dim=2)
    out["quad_F"], out["quad_c"] = F, c
    out["quad_val"] = mm.equilibrium_residual(g, m, state_for(g, m, F))
    # LCE 2D, viscous time step
    g = mm.Grid(2, 16, 0.5)
    n0 = scenarios.make_stripe_n0(g, [1.0, 0.2], [0.2, 1.0], 4)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=n0, dim=2,
                                  nu_F=0.5, nu_n=0.2)
    internal = m.init_internal(g.npoints)
    internal["angles"] = internal["angles"] + 0.1 * rng.standard_normal(g.npoints)
    internal["p_inc"] = 0.05 * rng.standard_normal(g.npoints)
    F = np.eye(2) + 0.05 * rng.standard_normal(g.shape + (2, 2))
    Fk = np.eye(2) + 0.05 * rng.standard_normal(g.shape + (2, 2))
    st = state_for(g, m, F, internal, prev_F=Fk, prev_internal=m.init_internal(g.npoints))
    out["lce2d_n0"], out["lce2d_F"], out["lce2d_Fk"] = n0, F, Fk
    out["lce2d_angles"], out["lce2d_p_inc"] = internal["angles"], internal["p_inc"]
    out["lce2d_val"] = mm.equilibrium_residual(g, m, st, dt=0.1)
    # LCE 3D
    g = mm.Grid(3, 8, 0.5)
    n0 = scenarios.generate_polydomain_n0(g, 0.25, seed=7)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=3)
    internal = m.init_internal(g.npoints)
    internal["angles"] = internal["angles"] + 0.1 * rng.standard_normal((g.npoints, 2))
    internal["p_inc"] = 0.05 * rng.standard_normal(g.npoints)
    F = np.eye(3) + 0.05 * rng.standard_normal(g.shape + (3, 3))
    out["lce3d_n0"], out["lce3d_F"] = n0, F
    out["lce3d_angles"], out["lce3d_chart"] = internal["angles"], internal["chart"]
    out["lce3d_p_inc"] = internal["p_inc"]
    out["lce3d_val"] = mm.equilibrium_residual(g, m, state_for(g, m, F, internal))
    return out


def scenario_fields():
    """Host microstructure generators and protocol bookkeeping."""
    g2, g3 = mm.Grid(2, 16, 0.5), mm.Grid(3, 8, 0.5)
    p = mm.ProtocolSpec("custom", 1.0, 0.9, -0.025,
                        strain_mask=[[1, 1, 1], [1, 0, 1], [1, 1, 0]])
    bc = p.macro_bc(0.95, 3, reference=np.diag([1.0, 1.1, 0.9]))
    pv = mm.ProtocolSpec("monodomain", 1.0, 1.1, 0.05, rate=0.25)
    n3 = scenarios.generate_polydomain_n0(g3, 0.3, seed=2)
    return dict(poly2d=scenarios.generate_polydomain_n0(g2, 0.25, seed=3), poly3d=n3,
                stripe2d=scenarios.make_stripe_n0(g2, [1.0, 0.3], [-0.2, 1.0], 4),
                stripe3d=scenarios.make_stripe_n0(g3, [1.0, 0.0, 0.3], [0.0, 1.0, 0.0], 2),
                moduli=np.stack(scenarios.composite_moduli(np.linspace(-0.2, 1.2, 11), 2.0,
                                                           10.0, 5.0)),
                S3=scenarios.orientation_tensor(n3),
                S2=scenarios.orientation_tensor(scenarios.make_stripe_n0(g2, [1, 0], [0, 1], 2)),
                sched=p.schedule(), bc_mask=bc.strain_mask, bc_value=bc.value,
                visc_dt=pv.dt, visc_sched=pv.schedule())


def lce_protocol_visc():
    """Viscous load stepping of a 2D stripe LCE (run_lce_protocol with
    relaxation and rate-derived time step; local-convergent inputs)."""
    g = mm.Grid(2, 16, 0.5)
    n0 = scenarios.make_stripe_n0(g, [1.0, 0.2], [0.2, 1.0], 4)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=n0, dim=2,
                                  nu_F=0.5, nu_n=0.2)
    proto = mm.ProtocolSpec("monodomain", 1.0, 1.04, 0.02, rate=0.2)
    study = mm.run_lce_protocol(g, m, proto, relax=True, seed=3, perturb=1e-4)
    recs = study.records
    st = study.state
    return dict(n=16, L=0.5, n0=n0, lams=study.lams,
                outer_iters=np.array([r.outer_iters for r in recs]),
                nominal=study.nominal, S=study.S, Fbar=np.array([r.Fbar for r in recs]),
                reference=study.reference, F=st.F, lam=st.lam, angles=st.internal["angles"],
                p_inc=st.internal["p_inc"], total_sweeps=st.total_sweeps)


def bloch_cases():
    """Bloch stability (stability.py:171-289) on the reference's own test
    inputs: identity moduli (2D, 3D), random major-symmetric PD fields,
    fields that lose ellipticity, and a converged compressed MR state."""
    from micromech import stability as stab
    out = {}

    def rand_tangent(npts, dim, lo, hi, rng):
        m = dim * dim
        Q = np.linalg.qr(rng.standard_normal((npts, m, m)))[0]
        eigs = rng.uniform(lo, hi, size=(npts, m))
        return np.einsum("pab,pb,pcb->pac", Q, eigs, Q).reshape(npts, dim, dim, dim, dim)

    def ident(npts, dim):
        eye = np.eye(dim * dim).reshape(dim, dim, dim, dim)
        return np.broadcast_to(eye, (npts,) + eye.shape).copy()

    cases = []
    g8 = mm.Grid(2, 8, 0.5)
    for k in [(2, 2), (3, 2), (4, 3), (1, 1)]:
        cases.append((f"id8_{k[0]}{k[1]}", g8, ident(g8.npoints, 2), k, 3))
    cases.append(("id8b", g8, ident(g8.npoints, 2), (2, 3), 1))
    g4 = mm.Grid(3, 4, 0.5)
    cases.append(("id3d", g4, ident(g4.npoints, 3), (2, 1, 1), 0))
    g6 = mm.Grid(2, 6, 0.5)
    for seed in range(5):
        rng = np.random.default_rng(100 + seed)
        Lf = rand_tangent(g6.npoints, 2, 0.5, 3.0, rng)
        k = [(2, 1), (1, 2), (2, 2), (3, 1), (2, 3)][seed]
        cases.append((f"pd{seed}", g6, Lf, k, seed))
    for seed in range(3):
        rng = np.random.default_rng(200 + seed)
        a = rng.standard_normal(2)
        a /= np.linalg.norm(a)
        v = rng.standard_normal(2)
        v /= np.linalg.norm(v)
        x = g6.coords().reshape(-1, 2)
        env = 1.0 + 0.5 * np.cos(np.pi * x[:, 0] / g6.length)
        eye = np.eye(4).reshape(2, 2, 2, 2)
        neg = np.einsum("i,j,k,l->ijkl", a, v, a, v)
        Lf = eye[None] - 2.5 * env[:, None, None, None, None] * neg[None]
        k = [(2, 1), (2, 2), (1, 1)][seed]
        cases.append((f"unst{seed}", g6, Lf, k, seed))
    names = []
    for name, g, Lf, k, seed in cases:
        r = stab.bloch_min_eigen(g, Lf, k, mu_rep=1.0, seed=seed)
        out[name + "_L"] = Lf
        out[name + "_meta"] = np.array([g.dim, g.n, seed] + list(k) + [0] * (3 - len(k)), float)
        out[name + "_beta"] = np.array(r.beta)
        out[name + "_iters"] = np.array(r.iterations)
        out[name + "_conv"] = np.array(r.converged)
        names.append(name)
    # converged compressed MR state (test_stability.py:217-269)
    model = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    st, conv = mm.solve(g6, model, mm.MacroBC.strain(0.97 * np.eye(2)),
                        mm.SolverParams(r_p_tol=1e-9, r_d_tol=1e-9, max_outer=4000))
    assert conv
    res = stab.stability_sweep(g6, model, st, k_max=2, seed=0)
    out["mr_F"] = st.F
    out["mr_betas"] = np.array([r.beta for r in res])
    out["mr_ks"] = np.array([r.k for r in res])
    out["names"] = np.array(names)
    return out


def main():
    only = sys.argv[1:]
    if only:  # regenerate the named fixtures only
        for name in only:
            save(name, **globals()[name]())
        return 0
    save("local_mr2d", **local_mr(2, 101, 256, 25, 1e-11, 5.0))
    save("local_mr2d_long", **local_mr(2, 102, 64, 8000, 1e-11, 6.0))
    save("local_mr3d", **local_mr(3, 103, 200, 25, 1e-11, 5.0))
    save("local_mr3d_long", **local_mr(3, 104, 48, 8000, 1e-11, 6.0))
    save("local_mr3d_loose", **local_mr(3, 105, 300, 50, 1e-4, 2.0))
    save("local_quad", **local_quad(106, 40, 2, 8000, 1e-11, 4.0))
    save("local_quad3d", **local_quad(107, 40, 3, 30, 1e-8, 2.5))
    save("local_lce2d", **local_lce(2, 201, 128, 50, 1e-11, 3.0))
    save("local_lce2d_visc", **local_lce(2, 202, 64, 50, 1e-11, 3.0, dt=0.1, nu_F=0.5, nu_n=0.2))
    save("local_lce3d", **local_lce(3, 203, 96, 50, 1e-11, 3.0))
    save("local_lce3d_visc", **local_lce(3, 204, 48, 50, 1e-11, 3.0, dt=0.1, nu_F=0.5, nu_n=0.2))
    save("project_2d", **projection(2, 8, 301))
    save("project_2d_odd", **projection(2, 6, 302))
    save("project_3d", **projection(3, 8, 303))
    save("project_3d_n12", **projection(3, 12, 304))
    save("frank_2d", **frank(2, 16))
    save("frank_3d", **frank(3, 8))
    save("traj_mr2d", **trajectory_mr2d())
    save("traj_mr3d", **trajectory_mr3d())
    save("config1_protocol", **config1_protocol())
    save("lce_uniform_solve", **lce_uniform_solve())
    save("lce_stripe_iters", **lce_stripe_iters())
    save("lce_poly_2d", **lce_poly_one_iter(2, 16))
    # 3D Newton sweeps amplify roundoff faster: shorter budget
    save("lce_poly_3d", **lce_poly_one_iter(3, 8, max_local=5))
    save("eq_residual_cases", **eq_residual_cases())
    save("scenario_fields", **scenario_fields())
    save("lce_protocol_visc", **lce_protocol_visc())
    save("bloch_cases", **bloch_cases())


if __name__ == "__main__":
    sys.exit(main())
