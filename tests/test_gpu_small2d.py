"""The persistent one-cluster PCG of small 2-D scalar problems (small2d.cu,
the c1 path): the whole solve_pcg loop of proj/src/solver.cpp:50-97 in one
16-CTA cluster. Checked against the CPU oracle at fixed k (1e-10, the parity
protocol of test_gpu_baseline_parity.py) and against the library's
multi-kernel iteration of the same problem (HOMFE_SMALL2D=0), plus the
reference's early exits."""
import os

import numpy as np
import pytest

import parity_util
from oracle.cfgutil import newton_rhs, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2203_02962_b200 as mod
    return mod


def _three_phase():
    from paper_2203_02962_b200 import inputs
    dims = (256, 256)
    ph, _ = inputs.rsa_balls(dims, radius=9.0, seed=21, fraction=0.25)
    ph2, _ = inputs.rsa_balls(dims, radius=5.0, seed=22, fraction=0.10)
    ph = np.where(ph2 == 1, 2, ph).astype(np.uint8)
    rot = np.array([[np.cos(0.4), -np.sin(0.4)], [np.sin(0.4), np.cos(0.4)]])
    aniso = rot @ np.diag([30.0, 3.0]) @ rot.T
    cm = np.stack([np.eye(2), aniso, 0.05 * np.eye(2)])
    return dims, ph, cm


def _multi_kernel_grid(hb, dims):
    os.environ["HOMFE_SMALL2D"] = "0"
    try:
        g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
        g.context(1)
    finally:
        del os.environ["HOMFE_SMALL2D"]
    return g


def test_small2d_fixed_k_matches_oracle_three_phases(hb, oracle_mod):
    """Three phases (one anisotropic), explicit anisotropic reference: fixed k
    against the oracle with the exact symbol."""
    dims, ph, cm = _three_phase()
    cref = cm[1]
    b = newton_rhs(dims, [1.0, 1.0], 1, cm, ph, (0.3, 1.0))
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    og = oracle_mod.Grid(dims, [1.0, 1.0], "two-triangles")
    mats = [hb.Material(t, True, 2) for t in cm]
    pre = hb.assemble_preconditioner(g, cref, 1)
    for k in (parity_util.STRICT_K, 25):
        got = hb.pcg_solve(g, mats, ph, pre, b, 0.0, k)
        assert "small2d" in g.context(1).path()
        ref = parity_util.oracle_fixed_k(oracle_mod, og, 1, cm, ph, cref, b, k)
        assert got["iterations"] == ref["iterations"] == k
        parity_util.check_fixed_k(f"small2d three-phase fixed k={k}", k, got["x"], ref, dict(path=["small2d"]))
        np.testing.assert_allclose(got["history"], ref["history"], rtol=1e-9, atol=1e-9 * ref["history"][0])


def test_small2d_matches_multi_kernel_path(hb):
    """Tolerance mode: the one-cluster loop and the multi-kernel iteration
    (cuFFT + element kernel + scalar kernels) stop at the same iteration with
    the same iterate to rounding."""
    dims, ph, cm = _three_phase()
    b = newton_rhs(dims, [1.0, 1.0], 1, cm, ph, (1.0, 0.0))
    mats = [hb.Material(t, True, 2) for t in cm]
    g1 = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    g2 = _multi_kernel_grid(hb, dims)
    pre1 = hb.assemble_preconditioner(g1, np.eye(2), 1)
    pre2 = hb.assemble_preconditioner(g2, np.eye(2), 1)
    a = hb.pcg_solve(g1, mats, ph, pre1, b, 1e-8, 1000)
    m = hb.pcg_solve(g2, mats, ph, pre2, b, 1e-8, 1000)
    assert "small2d" in g1.context(1).path() and "small2d" not in g2.context(1).path()
    assert a["converged"] and m["converged"]
    assert abs(a["iterations"] - m["iterations"]) <= 1, (a["iterations"], m["iterations"])
    assert rel(a["x"], m["x"]) <= 1e-9
    np.testing.assert_allclose(a["history"][:5], m["history"][:5], rtol=1e-11)


def test_small2d_c1_newton_and_determinism(hb):
    """The c1 configuration through newton_solve: converged, bitwise
    reproducible run to run, mean-free fluctuation field."""
    from paper_2203_02962_b200 import inputs
    cfg = inputs.config("c1")
    ph = cfg.phases()
    mats = [hb.Material(t, True, 2) for t in cfg.tangents()]
    g = hb.Grid(cfg.dims, [1.0, 1.0], cfg.stencil)
    kw = dict(eta_cg=cfg.eta_cg, reference=cfg.reference, reference_matrix=cfg.reference_matrix())
    s = hb.Solver(g, mats, ph, **kw)
    o1 = s.solve(np.asarray(cfg.load))
    o2 = s.solve(np.asarray(cfg.load))
    assert "small2d" in g.context(1).path()
    assert o1["converged"]
    assert np.array_equal(o1["u"], o2["u"]) and np.array_equal(o1["average_stress"], o2["average_stress"])
    assert abs(o1["u"].mean()) <= 1e-14 * np.abs(o1["u"]).max()


def test_small2d_zero_rhs_and_cap(hb):
    """b = 0: converged before the first iteration with x = 0
    (solver.cpp:66-70); it_max = 3: exactly three iterations, not converged."""
    dims, ph, cm = _three_phase()
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    mats = [hb.Material(t, True, 2) for t in cm]
    pre = hb.assemble_preconditioner(g, np.eye(2), 1)
    z = hb.pcg_solve(g, mats, ph, pre, np.zeros((1, g.num_nodes)), 1e-8, 100)
    assert z["iterations"] == 0 and z["converged"] and not np.any(z["x"])
    b = newton_rhs(dims, [1.0, 1.0], 1, cm, ph, (1.0, 0.0))
    c = hb.pcg_solve(g, mats, ph, pre, b, 1e-8, 3)
    assert c["iterations"] == 3 and not c["converged"]
