"""FourTrianglesTwoNode (two node types per pixel, complex Hermitian Fourier
blocks) on the GPU against the oracle."""
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


DIMS = (6, 8)
LEN = (1.1, 0.9)


def _grid(hb, oracle_mod):
    return hb.Grid(DIMS, LEN, "four-triangles-two-node"), oracle_mod.Grid(DIMS, LEN, "four-triangles-two-node")


@pytest.mark.parametrize("c", [1, 2])
def test_operators_match_oracle(hb, oracle_mod, c):
    g, og = _grid(hb, oracle_mod)
    m = 2 if c == 1 else 3
    rng = np.random.default_rng(3 + c)
    u = rng.uniform(-1, 1, (c, g.num_nodes))
    gr = hb.gradient_apply(g, u)
    ogr = oracle_mod.gradient(og, c, u)
    assert np.abs(gr - ogr).max() <= 1e-13 * np.abs(ogr).max()
    sq = rng.uniform(-1, 1, (g.num_quads, m))
    dv = hb.divergence_apply(g, sq)
    odv = oracle_mod.divergence(og, c, sq).reshape(c, -1)
    assert np.abs(dv - odv).max() <= 1e-13 * np.abs(odv).max()
    a = rng.uniform(-1, 1, (m, m))
    cm = np.stack([a @ a.T + m * np.eye(m), 3.0 * np.eye(m)])
    ph = (rng.random(g.num_pixels) < 0.4).astype(np.uint8)
    ku = hb.apply_operator(g, cm[np.repeat(ph, g.quads_per_pixel)], u)
    oku = oracle_mod.apply_phase(og, c, cm, ph, u).reshape(c, -1)
    assert np.abs(ku - oku).max() <= 1e-12 * np.abs(oku).max()


@pytest.mark.parametrize("c", [1, 2])
def test_probed_blocks_and_minv_match_oracle(hb, oracle_mod, c):
    g, og = _grid(hb, oracle_mod)
    m = 2 if c == 1 else 3
    rng = np.random.default_rng(11 + c)
    a = rng.uniform(-1, 1, (m, m))
    cref = a @ a.T + m * np.eye(m)
    pre = hb.assemble_preconditioner(g, cref, c)
    blocks = pre.symbol()
    op = oracle_mod.Preconditioner(og, cref, c, invert=False)
    ob = op.blocks()
    assert np.abs(blocks - ob).max() <= 1e-11 * np.abs(ob).max()
    r = rng.uniform(-1, 1, (c, g.num_nodes))
    z = hb.apply_preconditioner(g, pre, r)
    oz = oracle_mod.Preconditioner(og, cref, c).apply(r).reshape(c, -1)
    assert np.abs(z - oz).max() <= 1e-10 * np.abs(oz).max()


def test_newton_matches_oracle(hb, oracle_mod):
    g, og = _grid(hb, oracle_mod)
    c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(12.0, 7.0, 2)
    ph = (oracle_mod.uniform(21, g.num_pixels, 0.0, 1.0) < 0.35).astype(np.uint8)
    e = np.array([0.01, -0.003, 0.004])
    for kw in (dict(eta_cg=1e-10, eta_newton=1e-8),
               dict(eta_cg=1e-10, eta_newton=1e-8, reference="explicit", reference_matrix=np.eye(3))):
        got = hb.newton_solve(g, [hb.Material.linear_elastic(c0), hb.Material.linear_elastic(c1)], ph, e, **kw)
        ref = oracle_mod.newton_solve(og, False, [c0, c1], ph, e, **kw)
        assert got["converged"] and ref["converged"]
        kg = got["report"]["steps"][0]["cg_iterations"]
        ko = ref["steps"][0]["cg_iterations"]
        assert abs(kg - ko) <= 1
        rel = np.linalg.norm(got["u"].ravel() - ref["u"]) / np.linalg.norm(ref["u"])
        assert rel < 1e-8
        assert np.abs(got["average_stress"] - ref["average_stress"]).max() <= 1e-9 * np.abs(ref["average_stress"]).max()


def test_j2_sb_and_bounds_on_two_node_grid(hb, oracle_mod):
    """The f1 / f4 paths on the two-node stencil: J2 Newton, strain-based
    Newton and eigenvalue bounds against the oracle."""
    g, og = _grid(hb, oracle_mod)
    ph = (oracle_mod.uniform(77, g.num_pixels) > 0.0).astype(np.uint8)
    mats = [hb.Material.j2_plastic(0.833, 0.385, 3e-3, 0.08, 2), hb.Material.j2_plastic(0.833, 0.385, 6e-3, 0.16, 2)]
    omats = [oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=3e-3, hardening=0.08),
             oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=6e-3, hardening=0.16)]
    e = np.array([5e-3, -5e-3, 1e-3])
    kw = dict(eta_newton=1e-10, eta_cg=1e-12)
    got = hb.Solver(g, mats, ph, reference="explicit", reference_matrix=np.eye(3), **kw).solve(e)
    ref = oracle_mod.newton_solve_models(og, False, omats, ph, e, reference="explicit", reference_matrix=np.eye(3),
                                         **kw)
    assert got["converged"] and ref["converged"]
    assert len(got["report"]["steps"]) == len(ref["steps"])
    assert np.linalg.norm(got["u"].ravel() - ref["u"]) <= 1e-8 * np.linalg.norm(ref["u"])
    assert np.abs(got["internal"] - ref["internal"].reshape(-1, 7)).max() <= 1e-9 * np.abs(ref["internal"]).max()
    sb = hb.sb_newton_solve(g, mats, ph, e, np.eye(3), **kw)
    osb = oracle_mod.sb_newton_solve_models(og, False, omats, ph, e, np.eye(3), **kw)
    assert sb["converged"] and osb["converged"]
    assert np.abs(sb["strain"] - osb["strain"]).max() <= 1e-8 * np.abs(osb["strain"]).max()
    c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(12.0, 7.0, 2)
    t = np.where(np.repeat(ph.astype(bool), g.quads_per_pixel)[:, None, None], c1[None], c0[None])
    lo, hi, cond = hb.eigenvalue_bounds(g, t, c0, 2, pixel_constant=True)
    olo, ohi, ocond = oracle_mod.eigenvalue_bounds(og, t, c0, 2, pixel_constant=True)
    assert np.abs(lo - olo).max() <= 1e-12 * np.abs(olo).max() and np.abs(hi - ohi).max() <= 1e-12 * np.abs(ohi).max()
