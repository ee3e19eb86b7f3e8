"""The composite bifurcation study (scenarios.py:537-666) and its helpers
against a fixture made by running the reference itself
(tests/golden/make_golden_bifurcation.py)."""

import numpy as np
import pytest

from conftest import golden, rel_l2

mm = pytest.importorskip("paper_2010_06697_b200")


def test_build_composite_and_compatibility_match_reference():
    g = golden("bifurcation_16")
    grid = mm.Grid(2, int(g["n"]), float(g["L"]))
    assert np.array_equal(mm.build_composite(grid, 0.3, 0.06), g["phase"])
    c = mm.check_stripe_compatibility([1.0, 0.3], [0.3, 1.0], 1.5)
    assert c.compatible == bool(g["compat"][0])
    if c.compatible:
        np.testing.assert_allclose(c.Q, g["compat_Q"], atol=1e-8)
    with pytest.raises(mm.ConfigurationError):
        mm.build_composite(mm.Grid(3, 8), 0.3)
    with pytest.raises(mm.ConfigurationError):
        mm.MicrostructureSpec("circular_inclusion", volume_fraction=1.5)
    spec = mm.MicrostructureSpec("circular_inclusion", volume_fraction=0.3, interface_width=0.06)
    assert np.array_equal(spec.build(grid), g["phase"])
    assert spec == mm.MicrostructureSpec("circular_inclusion", 0.3, 0.06)


def test_tile_state_matches_reference():
    g = golden("bifurcation_16")
    grid = mm.Grid(2, int(g["n"]), float(g["L"]))
    st = mm.ADMMState(u_mean=np.eye(2), u_tilde=g["h_u_tilde"], grad_u=g["h_grad_u"],
                      F=g["h_F"], lam=g["h_lam"], internal={}, rho=1.0)
    t = mm.tile_state(grid, st, 2)
    for k in ("u_tilde", "grad_u", "F", "lam"):
        assert np.array_equal(getattr(t, k), g["t_" + k]), k
    assert t.outer_iter == 0 and t.history == []


@pytest.mark.gpu
def test_perturb_state_matches_reference():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = golden("bifurcation_16")
    grid = mm.Grid(2, int(g["n"]), float(g["L"]))
    st = mm.ADMMState(u_mean=np.eye(2), u_tilde=g["h_u_tilde"], grad_u=g["h_grad_u"],
                      F=g["h_F"], lam=g["h_lam"], internal={}, rho=1.0)
    mm.perturb_state(grid, st, g["v"])
    np.testing.assert_allclose(st.u_tilde, g["p_u_tilde"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(st.grad_u, g["p_grad_u"], rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_run_bifurcation_matches_reference():
    """Three device-resident branches + the device Bloch sweep per step:
    the stress curves to 1e-9 relative, the eigenvalue traces to 1e-6
    (the Bloch iteration stops at tol_beta = 1e-8)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = golden("bifurcation_16")
    grid = mm.Grid(2, int(g["n"]), float(g["L"]))
    proto = mm.ProtocolSpec("eb_compression", 1.0, 0.94, -0.02)
    params = mm.SolverParams(r_p_tol=1e-8, r_d_tol=1e-8)
    study = mm.run_bifurcation(grid, proto, volume_fraction=0.3, interface_width=0.06,
                               params=params, seed=0, k_max=2)
    assert study.completed
    np.testing.assert_allclose(study.lams, g["lams"])
    for k in ("stress_unit", "stress_super", "stress_pert"):
        e = rel_l2(getattr(study, k), g[k])
        print(f"{k}: {e:.3e}")
        assert e < 1e-9, k
    for k in ((1, 1), (1, 2), (2, 1), (2, 2)):
        np.testing.assert_allclose(study.betas[k], g["beta_%d%d" % k], rtol=1e-6)
