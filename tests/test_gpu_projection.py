"""Strain-based scheme and spectral bounds on the GPU
against the oracle (projection.cpp, spectral.cpp restated) and the
reference's own test_projection / test_spectral properties."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2203_02962_b200 as mod
    return mod


@pytest.mark.parametrize("dims,stencil,c", [((8, 6), "two-triangles", 2), ((6, 8), "bilinear-quad", 1),
                                            ((4, 6, 8), "trilinear-hex", 3), ((32, 32, 32), "trilinear-hex", 3)])
def test_gamma_matches_oracle(hb, oracle_mod, dims, stencil, c):
    g = hb.Grid(dims, [1.0] * len(dims), stencil)
    og = oracle_mod.Grid(dims, [1.0] * len(dims), stencil)
    m = g.dim if c == 1 else (3 if g.dim == 2 else 6)
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (m, m))
    cref = a @ a.T + m * np.eye(m)
    s = rng.uniform(-1, 1, (g.num_quads, m))
    pre = hb.assemble_preconditioner(g, cref, c, weighted=False)
    got = hb.gamma_apply(g, pre, s)
    want = oracle_mod.gamma_apply(og, cref, c, s)
    assert np.abs(got - want).max() <= 1e-11 * np.abs(want).max()
    # Gamma C_ref Gamma = Gamma (a projection in the C_ref pairing), kills
    # constants (test_projection.cpp:26-87)
    again = hb.gamma_apply(g, pre, got @ cref.T)
    assert np.abs(again - got).max() <= 1e-10 * np.abs(got).max()
    const = np.tile(rng.uniform(-1, 1, m), (g.num_quads, 1))
    assert np.abs(hb.gamma_apply(g, pre, const)).max() < 1e-12
    with pytest.raises(hb.ValidationError):
        hb.gamma_apply(g, hb.assemble_preconditioner(g, cref, c), s)


@pytest.mark.parametrize("plastic", [False, True])
def test_sb_matches_oracle_and_db(hb, oracle_mod, plastic):
    """sb_newton_solve vs the oracle, and the DB/SB equivalence of
    test_projection.cpp:125-170 through compare_db_sb."""
    dims = (8, 8)
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    og = oracle_mod.Grid(dims, [1.0, 1.0], "two-triangles")
    ph = (oracle_mod.uniform(1001 if not plastic else 77, 64) > 0.0).astype(np.uint8)
    if plastic:
        mats = [hb.Material.j2_plastic(0.833, 0.385, 3e-3, 0.08, 2), hb.Material.j2_plastic(0.833, 0.385, 6e-3, 0.16, 2)]
        omats = [oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=3e-3, hardening=0.08),
                 oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=6e-3, hardening=0.16)]
        loads = [np.array([4e-3, -4e-3, 0.0]), np.array([6e-3, -6e-3, 0.0])]
    else:
        c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(35.0, 17.0, 2)
        mats = [hb.Material.linear_elastic(c0), hb.Material.linear_elastic(c1)]
        omats = [oracle_mod.material("linear", c0), oracle_mod.material("linear", c1)]
        loads = [np.array([1.0, -0.2, 0.35])]
    # tight tolerances: GPU vs oracle
    kw = dict(eta_newton=1e-10, eta_cg=1e-12)
    g_sb = None
    w_sb = None
    g_or = None
    w_or = None
    for e in loads:
        got = hb.sb_newton_solve(g, mats, ph, e, np.eye(3), internal=g_sb, warm_strain=w_sb, **kw)
        ref = oracle_mod.sb_newton_solve_models(og, False, omats, ph, e, np.eye(3), g0=g_or, warm_strain=w_or, **kw)
        assert got["converged"] and ref["converged"]
        assert len(got["report"]["steps"]) == len(ref["steps"])
        assert all(abs(a["cg_iterations"] - b["cg_iterations"]) <= 1
                   for a, b in zip(got["report"]["steps"], ref["steps"]))
        assert np.abs(got["strain"] - ref["strain"]).max() <= 1e-8 * np.abs(ref["strain"]).max()
        assert np.abs(got["average_stress"] - ref["average_stress"]).max() <= 1e-9 * np.abs(ref["average_stress"]).max()
        g_sb, w_sb = got.get("internal"), got["strain"]
        g_or, w_or = ref["internal"], ref["strain"]
    # reference harness at the reference's tolerances
    cmp = hb.compare_db_sb(g, mats, ph, loads, np.eye(3), eta_newton=1e-5, eta_cg=1e-5)
    assert cmp["converged"]
    for a, b in zip(cmp["db_reports"], cmp["sb_reports"]):
        assert a["newton_steps"] == b["newton_steps"]
        assert all(abs(x["cg_iterations"] - y["cg_iterations"]) <= 1 for x, y in zip(a["steps"], b["steps"]))
    assert max(cmp["strain_discrepancy"]) < (1e-6 if plastic else 1e-8)


def test_bounds_match_oracle(hb, oracle_mod):
    """eigenvalue_bounds: GPU vs oracle on a two-phase elastic hex tangent,
    plus test_spectral.cpp:52-61 (perfect reference collapses to one)."""
    dims = (6, 4, 8)
    g = hb.Grid(dims, [1.0] * 3, "trilinear-hex")
    og = oracle_mod.Grid(dims, [1.0] * 3, "trilinear-hex")
    c0, c1 = hb.isotropic_stiffness(1.0, 0.4, 3), hb.isotropic_stiffness(20.0, 9.0, 3)
    ph = (oracle_mod.uniform(17, g.num_pixels, 0.0, 1.0) < 0.3)
    t = np.where(np.repeat(ph, g.quads_per_pixel)[:, None, None], c1[None], c0[None])
    cref = 0.5 * (c0 + c1)
    lo, hi, cond = hb.eigenvalue_bounds(g, t, cref, 3, pixel_constant=True)
    olo, ohi, ocond = oracle_mod.eigenvalue_bounds(og, t, cref, 3, pixel_constant=True)
    assert np.abs(lo - olo).max() <= 1e-12 * np.abs(olo).max()
    assert np.abs(hi - ohi).max() <= 1e-12 * np.abs(ohi).max()
    assert abs(cond - ocond) <= 1e-12 * ocond
    t1 = np.repeat(c0[None], g.num_quads, axis=0)
    lo1, hi1, cond1 = hb.eigenvalue_bounds(g, t1, c0, 3)
    assert np.abs(lo1 - 1.0).max() < 1e-12 and np.abs(hi1 - 1.0).max() < 1e-12 and abs(cond1 - 1.0) < 1e-12
