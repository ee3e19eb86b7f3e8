"""CPU-only checks of the boundary: the C-ABI library loads and exports
every symbol include/mm_admm.h declares, the host mirror of the reference
API validates like the reference, and the product path refuses to run
without a device (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2010_06697_b200 as mm
from paper_2010_06697_b200 import _lib
from conftest import ROOT


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "mm_admm.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("extension not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared) == set(_lib.EXPORTS)
    L = _lib.load_library()
    assert L.mm_abi_version() == 2


def test_status_mapping():
    for code, exc in ((1, mm.ParameterError), (2, mm.ConfigurationError),
                      (3, mm.InadmissibleStateError), (4, mm.DivergenceError)):
        with pytest.raises(exc):
            _lib.Context._raise(code, "x")
    with pytest.raises(RuntimeError):
        _lib.Context._raise(5, "x")


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    g = mm.Grid(2, 8)
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    with pytest.raises(RuntimeError):
        mm.solve(g, m, mm.MacroBC.strain(np.eye(2)), mm.SolverParams(max_outer=1))
    with pytest.raises(RuntimeError):
        m.local_sweeps(np.tile(np.eye(2), (4, 1, 1)), {}, np.tile(np.eye(2), (4, 1, 1)),
                       np.zeros((4, 2, 2)), 1.0, 0.0, None, None, {}, 5, 1e-11)


def test_exceptions_hierarchy():
    assert issubclass(mm.ParameterError, mm.ConfigurationError)
    assert issubclass(mm.DivergenceError, mm.ConvergenceError)
    e = mm.ConvergenceError("m", history=[1, 2])
    assert e.history == [1, 2]
    assert mm.ConfigurationError("a").errors == ["a"]


def test_params_and_policy_validation():
    with pytest.raises(mm.ParameterError):
        mm.SolverParams(r_p_tol=0.0)
    with pytest.raises(mm.ParameterError):
        mm.SolverParams(kappa_adapt=1.0)
    with pytest.raises(mm.ParameterError):
        mm.SolverParams(tau_adapt=0.5)
    with pytest.raises(mm.ParameterError):
        mm.FractionConverged(0.0)
    with pytest.raises(mm.ParameterError):
        mm.RatioToDual(-1.0)
    p = mm.SolverParams()
    assert mm.RatioToDual(0.3).target_tol(p, np.inf) == 1.0
    assert mm.RatioToDual(0.3).target_tol(p, 1e-3) == pytest.approx(3e-4)
    assert mm.RatioToDual(0.3).target_tol(p, 1e-20) == p.point_tol
    assert mm.ExactAll.chunk == 50 and mm.RatioToDual.chunk == 25
    assert mm.FractionConverged(0.9, 3).chunk == 3


def test_grid_and_macro_bc_validation():
    with pytest.raises(mm.ConfigurationError):
        mm.Grid(4, 8)
    with pytest.raises(mm.ConfigurationError):
        mm.Grid(2, 2)
    with pytest.raises(mm.ConfigurationError):
        mm.Grid(2, 8, -1.0)
    with pytest.raises(mm.ConfigurationError):
        mm.MacroBC(np.ones((2, 2), bool), np.ones((3, 3)))
    with pytest.raises(mm.ConfigurationError):
        mm.MacroBC.mixed({(0, 0): 1.0}, {(0, 0): 0.0}, 2)
    with pytest.raises(mm.ConfigurationError):
        mm.MacroBC.mixed({(0, 0): 1.0}, {}, 2)
    bc = mm.MacroBC.mixed({(0, 0): 0.9, (1, 1): 1.0}, {(0, 1): 0.0, (1, 0): 0.0}, 2)
    assert bc.strain_mask.tolist() == [[True, False], [False, True]]


@pytest.mark.parametrize("dim,n,L", [(2, 8, 0.5), (2, 6, 1.0), (3, 8, 0.5), (3, 9, 0.7),
                                     (3, 256, 0.5)])
def test_axis_symbol_tables_reproduce_grad_sq(dim, n, L):
    """The per-axis tables the device sums give the reference's |g|^2 and
    live-mode threshold bit for bit (grid.py:167-184, projection.py:155)."""
    import oracle
    grid = mm.Grid(dim, n, L)
    tab, thr = mm.grid.axis_symbol_tables(grid)
    if n ** dim <= 4096:
        _, gsq = oracle.symbols(dim, n, L)
        m = np.meshgrid(*[np.arange(n)] * (dim - 1) + [np.arange(n // 2 + 1)], indexing="ij")
        acc = tab[0][m[0]]
        for ax in range(1, dim):
            acc = acc + tab[ax][m[ax]]
        assert np.array_equal(acc, gsq)
        assert thr == 1e-14 * gsq.max()
    assert thr > 0


def test_state_host_views_round_trip():
    g = mm.Grid(2, 4)
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    st = mm.solver.init_state(g, m, mm.MacroBC.strain(np.diag([0.9, 1.0])), mm.SolverParams())
    assert st.F.shape == (4, 4, 2, 2)
    np.testing.assert_array_equal(st.F[0, 0], np.diag([0.9, 1.0]))
    st.lam += 1.0
    assert np.all(st.lam == 1.0)
    st.F = st.F * 2
    assert st.F[1, 1, 0, 0] == 1.8
    assert st.internal == {}
    assert st.r_d_prev == np.inf


def test_inplace_targets_are_only_writeable_contiguous_float64():
    """F and lam handed in as writeable C-contiguous float64 arrays are the
    arrays solve() writes back into (the reference mutates them in place);
    anything else is copied and left alone."""
    z = np.zeros((4, 4, 2, 2))
    ok = np.ones((4, 4, 2, 2))
    ro = np.ones((4, 4, 2, 2))
    ro.flags.writeable = False
    st = mm.ADMMState(u_mean=np.eye(2), u_tilde=np.zeros((4, 4, 2)), grad_u=z.copy(), F=ok,
                      lam=ro, internal={}, rho=1.0)
    assert st._inplace.get("F") is ok and "lam" not in st._inplace
    st.F = np.asfortranarray(np.ones((4, 4, 2, 2)))   # not C-contiguous: a copy is kept
    assert "F" not in st._inplace
    st.lam = np.ones((4, 4, 2, 2), dtype=np.float32)  # converted: not the caller's array
    assert "lam" not in st._inplace
    assert "grad_u" not in st._inplace and "u_tilde" not in st._inplace


def test_bench_fp64_peak_is_the_measured_one():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    pk, src = bench.fp64_peak_tflops()
    assert 30.0 < pk < 45.0
    assert "measured" in src


def test_moduli_are_read_only_and_reassignment_bumps_the_device_version():
    """Device-mirrored moduli cannot drift from their device copy: in-place
    edits raise, reassignment re-versions the model (engine re-upload) and
    recomputes the energy scale."""
    mu = np.ones(8)
    m = mm.MooneyRivlin(mu, 9.8 * mu, dim=3)
    mu[0] = 5.0                      # the caller's array is not aliased
    assert m.mu[0] == 1.0
    with pytest.raises(ValueError):
        m.mu[0] = 2.0
    v, phi = m._device_version, m._phi_scale()
    m.kappa = 20.0 * np.ones(8)
    assert m._device_version > v and m._phi_scale() == 21.0 != phi
    q = mm.QuadraticMaterial(np.full(4, 2.0), dim=2)
    assert q._cmax() == 2.0
    q.c = np.full(4, 3.0)
    assert q._cmax() == 3.0
