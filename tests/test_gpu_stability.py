"""Bloch stability on the device against the
reference's own bloch_min_eigen on its test inputs (tests/golden/
make_golden.py bloch_cases): identity moduli in 2D and 3D, random
major-symmetric positive fields, fields that lose ellipticity, and the
stability sweep of a converged compressed Mooney-Rivlin state."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_2010_06697_b200")
from paper_2010_06697_b200 import stability as stab  # noqa: E402


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


G = None


def _g():
    global G
    if G is None:
        G = golden("bloch_cases")
    return G


def _case(name):
    g = _g()
    meta = g[name + "_meta"]
    dim, n, seed = int(meta[0]), int(meta[1]), int(meta[2])
    k = tuple(int(x) for x in meta[3:3 + dim])
    return mm.Grid(dim, n, 0.5), g[name + "_L"], k, seed


@pytest.mark.parametrize("name", [str(x) for x in golden("bloch_cases")["names"]])
def test_bloch_min_eigen_matches_reference(name):
    g = _g()
    grid, Lf, k, seed = _case(name)
    r = stab.bloch_min_eigen(grid, Lf, k, mu_rep=1.0, seed=seed)
    assert r.converged == bool(g[name + "_conv"])
    assert r.beta == pytest.approx(float(g[name + "_beta"]), rel=1e-8)
    # iteration counts follow the same stopping rule on the same iterates
    assert abs(r.iterations - int(g[name + "_iters"])) <= 2
    norm = float(np.sum(np.abs(r.p) ** 2)) / grid.npoints
    assert norm == pytest.approx(1.0, rel=1e-10)


def test_translation_mode_carries_no_weight():
    grid = mm.Grid(2, 6, 0.5)
    eye = np.eye(4).reshape(2, 2, 2, 2)
    Lf = np.broadcast_to(eye, (grid.npoints,) + eye.shape).copy()
    res = stab.bloch_min_eigen(grid, Lf, (1, 1), mu_rep=1.0, seed=2)
    _, _, bsq, live = stab.bloch_symbols(grid, (1, 1))
    phat = np.fft.fftn(res.p, axes=(0, 1))
    assert float(np.abs(phat[~live]).max()) < 1e-10 * float(np.abs(phat).max())
    assert res.beta > 0.0


def test_deterministic_and_rho_validated():
    grid, Lf, k, _ = _case("pd0")
    a = stab.bloch_min_eigen(grid, Lf, k, mu_rep=1.0, seed=5)
    b = stab.bloch_min_eigen(grid, Lf, k, mu_rep=1.0, seed=5)
    assert a.beta == b.beta and np.array_equal(a.p, b.p)
    _, Lu, ku, _ = _case("unst0")
    with pytest.raises(mm.ParameterError):
        stab.bloch_min_eigen(grid, Lu, ku, mu_rep=1.0, rho=0.5)


def test_stability_sweep_of_converged_state():
    g = _g()
    grid = mm.Grid(2, 6, 0.5)
    model = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    st = mm.ADMMState(u_mean=0.97 * np.eye(2), u_tilde=np.zeros(grid.shape + (2,)),
                      grad_u=g["mr_F"], F=g["mr_F"], lam=np.zeros_like(g["mr_F"]), internal={},
                      rho=1.0)
    res = stab.stability_sweep(grid, model, st, k_max=2, seed=0)
    assert [r.k for r in res] == [tuple(k) for k in g["mr_ks"]]
    np.testing.assert_allclose([r.beta for r in res], g["mr_betas"], rtol=1e-8)
    assert stab.first_unstable(res, model.mu_rep) is None
    v = stab.mode_to_perturbation(grid, res[1], amplitude=1e-3)
    assert v.shape == (6, 12, 2)
    assert np.abs(v).max() == pytest.approx(1e-3 * 2.0 * grid.length)
