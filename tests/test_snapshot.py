"""Snapshot IO (SPEC.md cli-io write_snapshot / read_snapshot): bit-exact
round trips, versioned format, truncation detected with its byte offset,
and (GPU) a run resumed from a mid-run snapshot equal to the continuous run."""

import os

import numpy as np
import pytest

mm = pytest.importorskip("paper_2010_06697_b200")
from paper_2010_06697_b200.snapshot import FORMAT_VERSION, read_snapshot, write_snapshot  # noqa


def _host_state(rng, n=6, dim=2, lce=False):
    shape = (n,) * dim
    npts = n ** dim
    internal = {}
    prev_internal = None
    if lce:
        internal = {"angles": rng.standard_normal(npts), "p_inc": rng.standard_normal(npts)}
        prev_internal = {"angles": rng.standard_normal(npts), "p_inc": np.zeros(npts)}
    hist = [mm.solver.Residuals(i + 1, *rng.random(4), 0.125 * i) for i in range(5)]
    return mm.ADMMState(u_mean=np.eye(dim) + 0.01 * rng.standard_normal((dim, dim)),
                        u_tilde=rng.standard_normal(shape + (dim,)),
                        grad_u=rng.standard_normal(shape + (dim, dim)),
                        F=rng.standard_normal(shape + (dim, dim)),
                        lam=rng.standard_normal(shape + (dim, dim)), internal=internal,
                        rho=np.pi, outer_iter=17, r_d_prev=1.0 / 3.0, total_sweeps=12345,
                        history=hist, prev_F=rng.standard_normal(shape + (dim, dim)) if lce
                        else None, prev_internal=prev_internal)


@pytest.mark.parametrize("lce", [False, True])
def test_roundtrip_bit_exact(tmp_path, lce):
    rng = np.random.default_rng(3)
    st = _host_state(rng, lce=lce)
    stem = write_snapshot(st, str(tmp_path / "s"), grid=mm.Grid(2, 6, 0.5))
    back = read_snapshot(stem)
    for k in ("F", "grad_u", "lam", "u_tilde", "u_mean"):
        assert np.array_equal(getattr(back, k), getattr(st, k)), k
    if lce:
        assert np.array_equal(back.prev_F, st.prev_F)
        for k in st.internal:
            assert np.array_equal(back.internal[k], st.internal[k])
            assert np.array_equal(back.prev_internal[k], st.prev_internal[k])
    assert (back.rho, back.outer_iter, back.r_d_prev, back.total_sweeps) == \
        (st.rho, st.outer_iter, st.r_d_prev, st.total_sweeps)
    assert back.history == st.history
    assert not os.path.exists(stem + ".bin.tmp")


def test_fresh_state_roundtrip(tmp_path):
    st = mm.ADMMState(u_mean=np.eye(2), u_tilde=np.zeros((4, 4, 2)),
                      grad_u=np.broadcast_to(np.eye(2), (4, 4, 2, 2)).copy(),
                      F=np.broadcast_to(np.eye(2), (4, 4, 2, 2)).copy(),
                      lam=np.zeros((4, 4, 2, 2)), internal={}, rho=1.0)
    back = read_snapshot(write_snapshot(st, str(tmp_path / "f")))
    assert back.history == [] and back.r_d_prev == np.inf
    assert np.array_equal(back.F, st.F)


def test_truncated_and_version_mismatch(tmp_path):
    st = _host_state(np.random.default_rng(4))
    stem = write_snapshot(st, str(tmp_path / "t"))
    with open(stem + ".bin", "r+b") as f:
        f.truncate(1000)
    with pytest.raises(mm.SnapshotError) as e:
        read_snapshot(stem)
    assert e.value.offset is not None and e.value.offset <= 1000
    stem = write_snapshot(st, str(tmp_path / "v"))
    meta = open(stem + ".meta").read().replace(FORMAT_VERSION, "mm-snapshot/0")
    open(stem + ".meta", "w").write(meta)
    with pytest.raises(mm.SnapshotError, match="version"):
        read_snapshot(stem)


@pytest.mark.gpu
def test_resume_from_snapshot_equals_continuous_run(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(41)
    grid = mm.Grid(2, 8)
    mu = np.where(rng.random(grid.npoints) < 0.3, 1.0, 20.0)
    m = mm.MooneyRivlin(mu=mu, kappa=9.8 * mu, dim=2, mu_rep=20.0)
    bc = mm.MacroBC.strain(np.array([[0.95, 0.02], [0.0, 1.01]]))
    st_a, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=7), raise_on_max=False)
    stem = write_snapshot(st_a, str(tmp_path / "mid"), grid=grid)
    st_r = read_snapshot(stem)
    st_r, conv_r = mm.solve(grid, m, bc, mm.SolverParams(max_outer=600), state=st_r)
    st_b, conv_b = mm.solve(grid, m, bc, mm.SolverParams(max_outer=600))
    assert conv_r and conv_b
    assert st_r.outer_iter == st_b.outer_iter
    assert np.array_equal(st_r.grad_u, st_b.grad_u)
    assert np.array_equal(st_r.lam, st_b.lam)
    assert st_r.history[-1][:5] == st_b.history[-1][:5]
