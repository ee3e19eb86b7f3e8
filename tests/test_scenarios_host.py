"""Host-side scenario helpers (CPU): the microstructure generators and the
protocol bookkeeping of paper_2010_06697_b200.scenarios against fixtures
produced by the reference's micromech.scenarios (tests/golden/make_golden.py
scenario_fields)."""

import numpy as np
import pytest

from conftest import golden

mm = pytest.importorskip("paper_2010_06697_b200")


def test_generators_and_protocol_match_reference():
    g = golden("scenario_fields")
    g2, g3 = mm.Grid(2, 16, 0.5), mm.Grid(3, 8, 0.5)
    np.testing.assert_allclose(mm.generate_polydomain_n0(g2, 0.25, seed=3), g["poly2d"],
                               rtol=0, atol=1e-14)
    np.testing.assert_allclose(mm.generate_polydomain_n0(g3, 0.3, seed=2), g["poly3d"],
                               rtol=0, atol=1e-14)
    assert np.array_equal(mm.make_stripe_n0(g2, [1.0, 0.3], [-0.2, 1.0], 4), g["stripe2d"])
    assert np.array_equal(mm.make_stripe_n0(g3, [1.0, 0.0, 0.3], [0.0, 1.0, 0.0], 2),
                          g["stripe3d"])
    mods = np.stack(mm.composite_moduli(np.linspace(-0.2, 1.2, 11), 2.0, 10.0, 5.0))
    assert np.array_equal(mods, g["moduli"])
    np.testing.assert_allclose(mm.orientation_tensor(g["poly3d"]), g["S3"], atol=1e-15)
    np.testing.assert_allclose(
        mm.orientation_tensor(mm.make_stripe_n0(g2, [1, 0], [0, 1], 2)), g["S2"], atol=1e-15)
    p = mm.ProtocolSpec("custom", 1.0, 0.9, -0.025,
                        strain_mask=[[1, 1, 1], [1, 0, 1], [1, 1, 0]])
    assert np.array_equal(p.schedule(), g["sched"])
    bc = p.macro_bc(0.95, 3, reference=np.diag([1.0, 1.1, 0.9]))
    assert np.array_equal(bc.strain_mask, g["bc_mask"])
    assert np.array_equal(bc.value, g["bc_value"])
    pv = mm.ProtocolSpec("monodomain", 1.0, 1.1, 0.05, rate=0.25)
    assert pv.dt == g["visc_dt"]
    assert np.array_equal(pv.schedule(), g["visc_sched"])


@pytest.mark.parametrize("kw", [dict(kind="bogus"), dict(kind="uni", lam_end=0.9),
                                dict(kind="uni", lam_end=0.9, lam_step=0.1),
                                dict(kind="custom"), dict(kind="uni", rate=-1.0)])
def test_protocol_validation(kw):
    with pytest.raises(mm.ConfigurationError):
        mm.ProtocolSpec(**kw)


def test_protocol_masks():
    assert mm.ProtocolSpec("uni").mask(2).tolist() == [[True, False], [False, False]]
    assert mm.ProtocolSpec("monodomain").mask(2).tolist() == [[True, True], [True, False]]
    assert mm.ProtocolSpec("eb_compression").mask(3).all()
    P = mm.ProtocolSpec("eb").deformation(0.9, 2)
    assert np.array_equal(P, np.diag([0.9, 0.9]))
    with pytest.raises(mm.ConfigurationError):
        mm.run_lce_protocol(mm.Grid(2, 4, 0.5), None, mm.ProtocolSpec("eb_compression"))
