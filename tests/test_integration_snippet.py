"""INTEGRATION.md's Option-2 binding (the ctypes module a reference
maintainer would add as micromech/_b200.py), executed verbatim.

CPU: the module loads the built library, its ABI-version check passes and
its ctypes struct declarations have the sizes the library reports
(mm_struct_size).  GPU: its outer iteration reproduces the oracle's
trajectory on a small 3D laminate (fields 1e-10 relative L2, sweep counts
exact)."""

import os
import re
import types

import numpy as np
import pytest

from conftest import ROOT, rel_l2

from paper_2010_06697_b200 import _lib


def _snippet_source():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        md = f.read()
    blocks = re.findall(r"```python\n(.*?)```", md, flags=re.S)
    src = [b for b in blocks if b.startswith("# micromech/_b200.py")]
    assert len(src) == 1, "Option-2 module block not found in INTEGRATION.md"
    return src[0]


def _load_snippet(monkeypatch):
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("extension not built (run __graft_entry__.build())")
    monkeypatch.setenv("MM_ADMM_LIB", _lib.LIB_PATH)
    mod = types.ModuleType("micromech_b200_snippet")
    exec(compile(_snippet_source(), "INTEGRATION.md:micromech/_b200.py", "exec"), mod.__dict__)
    return mod


def test_snippet_struct_sizes_match_library(monkeypatch):
    import ctypes
    mod = _load_snippet(monkeypatch)
    L = mod.lib
    assert L.mm_abi_version() == 2
    assert ctypes.sizeof(mod.LocalStats) == L.mm_struct_size(0) == 104
    assert ctypes.sizeof(mod.UpdateStats) == L.mm_struct_size(1)
    # the host package's own declarations agree too
    assert ctypes.sizeof(_lib.LocalStatsC) == L.mm_struct_size(0)
    assert ctypes.sizeof(_lib.UpdateStatsC) == L.mm_struct_size(1)
    assert ctypes.sizeof(_lib.StepParamsC) == L.mm_struct_size(2)
    assert ctypes.sizeof(_lib.StepResultC) == L.mm_struct_size(3)
    assert ctypes.sizeof(_lib.ProfileC) == L.mm_struct_size(4)
    assert ctypes.sizeof(_lib.LCEParamsC) == L.mm_struct_size(5)
    assert L.mm_struct_size(99) == -1


def test_snippet_axis_tables_match_package():
    import paper_2010_06697_b200 as mm
    from paper_2010_06697_b200.grid import axis_symbol_tables
    mod = types.ModuleType("s")
    src = _snippet_source()
    # only the pure-numpy helper (no library needed)
    fn = src[src.index("def axis_tables"):src.index("class DeviceGrid")]
    exec("import numpy as np\n" + fn, mod.__dict__)
    for dim, n, L in ((2, 16, 0.5), (3, 12, 0.4), (3, 9, 1.0)):
        tab, thr = mod.axis_tables(dim, n, L)
        ref_tab, ref_thr = axis_symbol_tables(mm.Grid(dim, n, L))
        assert np.array_equal(tab, ref_tab) and thr == ref_thr


@pytest.mark.gpu
def test_snippet_outer_iterations_match_oracle(monkeypatch):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    import paper_2010_06697_b200 as mm
    from paper_2010_06697_b200.projection import macro_gradient

    mod = _load_snippet(monkeypatch)
    n, K = 12, 5
    grid = mm.Grid(3, n, 0.5)
    x = grid.coords()[..., 0]
    chi = ((x + 0.5) < 0.5).ravel().astype(float)
    mu = 1.0 + (0.05 - 1.0) * chi
    kap = 9.8 * mu
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    params = mm.SolverParams()
    model = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    policy = mm.RatioToDual(0.3)
    st = mm.solver.init_state(grid, model, bc, params)
    F0 = st.F + 1e-3 * np.random.default_rng(0).standard_normal(st.F.shape)
    hst = types.SimpleNamespace(F=F0.copy(), grad_u=np.array(st.grad_u), lam=np.array(st.lam),
                                u_tilde=np.array(st.u_tilde), u_mean=np.array(st.u_mean),
                                rho=st.rho, r_d_prev=np.inf, total_sweeps=0, outer_iter=0)
    dev = mod.DeviceGrid(grid, model, hst)
    hist = []
    try:
        for _ in range(K):
            r_p, r_d, r_l = dev.outer_iteration(hst, params, bc, policy, macro_gradient)
            # solver.py:281-296, kept by the maintainer
            hst.outer_iter += 1
            hst.r_d_prev = r_d
            if params.adapt and hst.outer_iter > 1:
                if r_p > params.tau_adapt * r_d:
                    hst.rho *= params.kappa_adapt
                elif r_d > params.tau_adapt * r_p:
                    hst.rho = max(hst.rho / params.kappa_adapt, params.rho_min_factor * 1.0)
            hist.append((r_p, r_d, r_l))
        dev.fetch(hst)
    finally:
        dev.close()

    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    op = oracle.Params(max_outer=K)
    ost = oracle.init_state(3, n, om, bc.strain_mask, bc.value, op)
    ost.F = F0.copy()
    ost, _ = oracle.solve(3, n, 0.5, om, bc.strain_mask, bc.value, op,
                          policy=oracle.RatioToDual(0.3), state=ost, raise_on_max=False)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(hst, k), getattr(ost, k)) < 1e-10, k
    assert hst.total_sweeps == ost.total_sweeps
    np.testing.assert_allclose(np.array(hist), np.array([h[1:4] for h in ost.history]),
                               rtol=1e-9)
