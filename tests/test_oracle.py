"""Pins the CPU oracle (test infrastructure) against the golden fixtures made
from dense oracles (tests/golden/make_golden.py) and against the reference's
known-answer tests. Tolerances are the reference's own:
  K vs dense D^T W C D < 1e-12     proj/tests/test_operators.cpp:168-193
  D vs dense < 1e-13               proj/tests/test_operators.cpp:79-91
  blocks vs F K F^H < 1e-11 scale  proj/tests/test_precond.cpp:47-82
  M^-1 vs dense pinv < 1e-10       proj/tests/test_precond.cpp:201-252
  PCG vs dense solve < 1e-8 max|x| proj/tests/test_solver.cpp:82-103
"""
import numpy as np
import pytest


def _grid(oracle_mod, meta):
    return oracle_mod.Grid(meta["dims"], meta["lengths"], meta["stencil"])


def test_mt19937_64_known_answer(oracle_mod, golden):
    gen = golden.MT19937_64(77)
    ref = np.array([gen.uniform() for _ in range(1000)])
    np.testing.assert_array_equal(oracle_mod.uniform(77, 1000), ref)
    g2 = golden.MT19937_64(5489)
    for _ in range(9999):
        g2()
    assert g2() == 9981545732273789042


@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (4, 6), (6, 5), (5, 3, 2), (2, 2, 2), (8, 4, 6), (16, 12),
                                   (7, 9), (32, 32, 8)])
def test_fft_matches_numpy(oracle_mod, shape):
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal(shape)
    X = oracle_mod.fft_forward(x)
    ref = np.fft.rfftn(x)
    assert np.abs(X - ref).max() <= 1e-12 * np.abs(ref).max()
    y = oracle_mod.fft_inverse(X, shape)
    assert np.abs(y / x.size - x).max() <= 1e-13 * np.abs(x).max()


def test_operators_match_dense_oracles(oracle_mod, golden):
    for case in golden.load("operators.npz"):
        g = _grid(oracle_mod, case["meta"])
        c = case["meta"]["c"]
        ku = oracle_mod.apply_phase(g, c, case["cmats"], case["phase"], case["u"])
        assert np.abs(ku - case["Ku"]).max() < 1e-12, case["meta"]
        grad = oracle_mod.gradient(g, c, case["u"])
        assert np.abs(grad - case["grad"]).max() < 1e-13, case["meta"]
        div = oracle_mod.divergence(g, c, case["s"])
        assert np.abs(div - case["div"]).max() < 1e-13, case["meta"]
        # per-quad tangent path is bitwise the phase-indexed one
        nq = g.quads_per_pixel
        tangent = case["cmats"][np.repeat(case["phase"], nq)]
        np.testing.assert_array_equal(oracle_mod.apply_tangent(g, c, tangent, case["u"]), ku)


def test_precond_blocks_and_pinv(oracle_mod, golden):
    for case in golden.load("precond.npz"):
        g = _grid(oracle_mod, case["meta"])
        c = case["meta"]["c"]
        raw = oracle_mod.Preconditioner(g, case["c_ref"], c, invert=False).blocks()
        scale = np.abs(case["blocks"]).max()
        assert np.abs(raw - case["blocks"]).max() < 1e-11 * scale, case["meta"]
        inv = oracle_mod.Preconditioner(g, case["c_ref"], c)
        z = inv.apply(case["r"])
        assert np.abs(z - case["z"]).max() < 1e-10, case["meta"]


def test_pcg_matches_dense_solve(oracle_mod, golden):
    for case in golden.load("pcg.npz"):
        g = _grid(oracle_mod, case["meta"])
        c = case["meta"]["c"]
        pre = oracle_mod.Preconditioner(g, case["c_ref"], c)
        out = oracle_mod.pcg(g, c, case["cmats"], case["phase"], pre, case["b"], 1e-10, 500)
        assert out["converged"]
        x = case["x"]
        assert np.abs(out["x"] - x).max() < 1e-8 * np.abs(x).max(), case["meta"]


def test_isotropic_stiffness_kat(oracle_mod):
    """proj/tests/test_mandel.cpp special values."""
    c_id = oracle_mod.isotropic_stiffness(1.0 / 3.0, 0.5, 3)
    assert np.abs(c_id - np.eye(6)).max() < 1e-15
    c = oracle_mod.isotropic_stiffness(1.0, 0.6, 3)
    assert abs(c[0, 0] - 1.8) < 1e-15 * 1.8
    lam = np.linalg.eigvalsh(c)
    assert abs(lam[5] - 3.0) < 1e-13 * 3
    assert np.abs(lam[:5] - 1.2).max() < 1e-13 * 1.2
    c2 = oracle_mod.isotropic_stiffness(1.0, 0.6, 2)
    np.testing.assert_array_equal(c2, c[np.ix_([0, 1, 5], [0, 1, 5])])


def test_one_iteration_when_reference_equals_material(oracle_mod):
    """acceptance.cpp:45-80 / test_solver.cpp:47-65."""
    for dims, kind in [((6, 5), "two-triangles"), ((4, 4, 4), "trilinear-hex"), ((5, 6), "bilinear-quad")]:
        g = oracle_mod.Grid(dims, [1.0] * len(dims), kind)
        for c in (1, g.dim):
            m = g.m(c)
            rng = np.random.default_rng(9001 + c)
            a = rng.uniform(-1, 1, (m, m))
            cm = a @ a.T + 0.5 * np.eye(m)
            s = rng.uniform(-1, 1, (g.num_quads, m))
            b = -oracle_mod.divergence(g, c, s)
            pre = oracle_mod.Preconditioner(g, cm, c)
            out = oracle_mod.pcg(g, c, cm[None], np.zeros(g.num_pixels, np.uint8), pre, b, 1e-12, 10)
            assert out["iterations"] == 1
            assert out["history"][-1] < 1e-12 * out["history"][0]


def test_uniform_material_no_fluctuation(oracle_mod):
    """test_solver.cpp:177-198."""
    g = oracle_mod.Grid((6, 6), (1.0, 1.0), "bilinear-quad")
    c = oracle_mod.isotropic_stiffness(1.3, 0.5, 2)
    e = np.array([0.2, 0.0, 0.7])
    out = oracle_mod.newton_solve(g, False, c[None], np.zeros(36, np.uint8), e)
    assert out["converged"] and len(out["steps"]) == 1
    assert out["steps"][0]["cg_iterations"] == 0
    assert np.abs(out["u"]).max() < 1e-12
    assert np.abs(out["average_stress"] - c @ e).max() < 1e-12


def test_linear_newton_one_step_and_errors(oracle_mod):
    g = oracle_mod.Grid((8, 8), (1.0, 1.0), "two-triangles")
    cm = np.stack([oracle_mod.isotropic_stiffness(1.0, 0.5, 2), oracle_mod.isotropic_stiffness(25.0, 14.0, 2)])
    ph = np.zeros((8, 8), np.uint8)
    ph[3:5, 3:5] = 1
    out = oracle_mod.newton_solve(g, False, cm, ph, [1.0, -0.3, 0.4], eta_cg=1e-6)
    assert out["converged"] and len(out["steps"]) == 1 and out["assemblies"] == 1
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.newton_solve(g, False, cm, ph, [1.0, -0.3, 0.4], eta_newton=0.0)
    assert ei.value.code == 2
    with pytest.raises(oracle_mod.OracleError) as ei:
        oracle_mod.Preconditioner(g, -np.eye(3), 2)
    assert ei.value.code == 2


# ------------------------------------------------------------ J2
def _von_mises_mandel6(s):
    tr = s[:3].sum()
    dev = s.copy()
    dev[:3] -= tr / 3.0
    return np.sqrt(1.5) * np.linalg.norm(dev)


def test_j2_elastic_below_yield(oracle_mod):
    """test_material.cpp:68-81: J2 below the yield surface equals the
    isotropic elastic model, state untouched."""
    eps = np.zeros(6)
    eps[5] = 0.2
    sig, tan, gn = oracle_mod.j2_evaluate(3, 1.0, 0.7, 1.0, 0.5, eps, np.zeros(7))
    c = oracle_mod.isotropic_stiffness(1.0, 0.7, 3)
    assert np.abs(sig - c @ eps).max() < 1e-14
    assert np.abs(tan - c).max() < 1e-14
    assert np.abs(gn).max() == 0.0


def test_j2_consistency_condition(oracle_mod):
    """test_material.cpp:83-101: accumulated plastic strain never decreases and
    a plastic state sits on the yield surface."""
    k, g_mod, tau0, hard = 1.2, 0.8, 0.01, 0.25
    g = np.zeros(7)
    draws = oracle_mod.uniform(17, 24)
    for step in range(4):
        eps = 0.05 * draws[6 * step:6 * step + 6]
        sig, _, gn = oracle_mod.j2_evaluate(3, k, g_mod, tau0, hard, eps, g)
        assert gn[6] >= g[6]
        if gn[6] > g[6]:
            assert abs(_von_mises_mandel6(sig) - (tau0 + hard * gn[6])) < 1e-10 * tau0
        g = gn


@pytest.mark.parametrize("d", [3, 2])
def test_j2_tangent_matches_finite_differences(oracle_mod, d):
    """test_material.cpp:103-139."""
    k, g_mod, tau0, hard = 1.2, 0.8, 0.01, 0.25
    n = 6 if d == 3 else 3
    eps0 = np.zeros(n)
    eps0[0] = 0.04
    eps0[n - 1] = 0.02
    _, _, g1 = oracle_mod.j2_evaluate(d, k, g_mod, tau0, hard, eps0, np.zeros(7))
    assert g1[6] > 0.0
    eps = eps0.copy()
    eps[1] += 0.015
    _, tan, g2 = oracle_mod.j2_evaluate(d, k, g_mod, tau0, hard, eps, g1)
    assert g2[6] > g1[6]
    h = 1e-6
    fd = np.zeros((n, n))
    for j in range(n):
        ep, em = eps.copy(), eps.copy()
        ep[j] += h
        em[j] -= h
        fd[:, j] = (oracle_mod.j2_evaluate(d, k, g_mod, tau0, hard, ep, g1)[0] -
                    oracle_mod.j2_evaluate(d, k, g_mod, tau0, hard, em, g1)[0]) / (2 * h)
    assert np.abs(fd - tan).max() / np.abs(tan).max() < 1e-5
    assert np.abs(tan - tan.T).max() < 1e-12 * np.abs(tan).max()


def test_models_newton_linear_catalog_equals_linear_newton(oracle_mod):
    """The general-catalog Newton reduces to the linear one for linear models."""
    og = oracle_mod.Grid((12, 10), (1.0, 1.0), "two-triangles")
    c0 = oracle_mod.isotropic_stiffness(1.0, 0.5, 2)
    c1 = oracle_mod.isotropic_stiffness(12.0, 7.0, 2)
    ph = (oracle_mod.uniform(5, 120, 0.0, 1.0) < 0.4).astype(np.uint8)
    e = np.array([0.01, -0.002, 0.003])
    ref = oracle_mod.newton_solve(og, False, [c0, c1], ph, e, eta_cg=1e-10, eta_newton=1e-8)
    got = oracle_mod.newton_solve_models(og, False, [oracle_mod.material("linear", c0),
                                                     oracle_mod.material("linear", c1)], ph, e,
                                         eta_cg=1e-10, eta_newton=1e-8)
    assert got["converged"] and ref["converged"]
    assert [s["cg_iterations"] for s in got["steps"]] == [s["cg_iterations"] for s in ref["steps"]]
    np.testing.assert_allclose(got["u"], ref["u"], rtol=0, atol=1e-14 * np.abs(ref["u"]).max())
    np.testing.assert_allclose(got["average_stress"], ref["average_stress"], rtol=1e-13)


def test_models_newton_j2_plastic_flow(oracle_mod):
    """acceptance.cpp:333-345 plastic instances: two J2 phases on an 8x8
    plane-strain grid converge, plastify and keep the reference's state
    contract (trial state returned on convergence)."""
    og = oracle_mod.Grid((8, 8), (1.0, 1.0), "two-triangles")
    mats = [oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=3e-3, hardening=0.08),
            oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=6e-3, hardening=0.16)]
    ph = (oracle_mod.uniform(7007, 64, 0.0, 1.0) < 0.5).astype(np.uint8)
    e = np.array([5e-3, -5e-3, 1e-3])
    out = oracle_mod.newton_solve_models(og, False, mats, ph, e, eta_newton=1e-5, eta_cg=1e-5,
                                         reference="explicit", reference_matrix=np.eye(3))
    assert out["converged"]
    g = out["internal"].reshape(-1, 7)
    assert g[:, 6].max() > 0.0 and g[:, 6].min() >= 0.0
    assert len(out["steps"]) >= 2  # nonlinear: more than one Newton step


# ---------------------------------------- strain-based scheme, bounds (8 f4)
def test_gamma_fixes_compatible_fields_and_kills_constants(oracle_mod):
    """test_projection.cpp:26-47."""
    og = oracle_mod.Grid((4, 4), (1.0, 1.0), "two-triangles")
    u = oracle_mod.uniform(401, 2 * 16)
    du = oracle_mod.gradient(og, 2, u)
    proj = oracle_mod.gamma_apply(og, np.eye(3), 2, du)
    assert np.abs(proj - du).max() < 1e-10 * np.abs(du).max()
    const = np.tile([1.0, -2.0, 0.5], (og.num_quads, 1))
    assert np.abs(oracle_mod.gamma_apply(og, np.eye(3), 2, const)).max() < 1e-12


def test_gamma_matches_dense_pinv_composition(oracle_mod, golden):
    """test_projection.cpp:49-64: Gamma = D (D^T D)^+ D^T."""
    dims = (3, 3)
    og = oracle_mod.Grid(dims, (1.0, 1.0), "two-triangles")
    D, _ = golden.dense_gradient(dims, (1.0, 1.0), "two-triangles", 2)
    gd = D @ golden.dense_pinv(D.T @ D) @ D.T
    s = oracle_mod.uniform(409, og.num_quads * 3).reshape(og.num_quads, 3)
    flat = s.T.ravel()  # dense rows are component-major
    want = (gd @ flat).reshape(3, og.num_quads).T
    assert np.abs(oracle_mod.gamma_apply(og, np.eye(3), 2, s) - want).max() < 1e-10


def test_sb_uniform_material_converges_immediately(oracle_mod):
    """test_projection.cpp:108-123."""
    og = oracle_mod.Grid((6, 6), (1.0, 1.0), "two-triangles")
    mat = oracle_mod.material("linear", oracle_mod.isotropic_stiffness(1.0, 0.6, 2))
    out = oracle_mod.sb_newton_solve_models(og, False, [mat], np.zeros(36, np.uint8), [0.5, -0.1, 0.2], np.eye(3))
    assert out["converged"] and len(out["steps"]) == 1
    assert np.abs(out["strain"]).max() < 1e-12


@pytest.mark.parametrize("plastic", [False, True])
def test_db_sb_equivalence(oracle_mod, plastic):
    """test_projection.cpp:125-170: Newton counts equal, CG counts within 1,
    strain discrepancy small (linear 1e-8, J2 two steps 1e-6)."""
    og = oracle_mod.Grid((8, 8), (1.0, 1.0), "two-triangles")
    ph = (oracle_mod.uniform(1001 if not plastic else 77, 64) > 0.0).astype(np.uint8)
    if plastic:
        mats = [oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=3e-3, hardening=0.08),
                oracle_mod.material("j2", bulk=0.833, shear=0.385, yield_stress=6e-3, hardening=0.16)]
        loads = [np.array([4e-3, -4e-3, 0.0]), np.array([6e-3, -6e-3, 0.0])]
    else:
        mats = [oracle_mod.material("linear", oracle_mod.isotropic_stiffness(1.0, 0.5, 2)),
                oracle_mod.material("linear", oracle_mod.isotropic_stiffness(35.0, 17.0, 2))]
        loads = [np.array([1.0, -0.2, 0.35])]
    kw = dict(eta_newton=1e-5, eta_cg=1e-5)
    g_db = g_sb = None
    w_db = w_sb = None
    for e in loads:
        db = oracle_mod.newton_solve_models(og, False, mats, ph, e, g0=g_db, warm_u=w_db, reference="explicit",
                                            reference_matrix=np.eye(3), **kw)
        sb = oracle_mod.sb_newton_solve_models(og, False, mats, ph, e, np.eye(3), g0=g_sb, warm_strain=w_sb, **kw)
        assert db["converged"] and sb["converged"]
        assert len(db["steps"]) == len(sb["steps"])
        assert all(abs(a["cg_iterations"] - b["cg_iterations"]) <= 1 for a, b in zip(db["steps"], sb["steps"]))
        db_strain = oracle_mod.gradient(og, 2, db["u"])
        disc = np.abs(sb["strain"] - db_strain).max() / np.abs(db_strain).max()
        assert disc < (1e-6 if plastic else 1e-8)
        g_db, g_sb, w_db, w_sb = db["internal"], sb["internal"], db["u"], sb["strain"]
    if plastic:
        assert len(db["steps"]) > 1


def test_bounds_collapse_for_perfect_reference(oracle_mod):
    """test_spectral.cpp:52-61."""
    og = oracle_mod.Grid((4, 4), (1.0, 1.0), "two-triangles")
    c = oracle_mod.isotropic_stiffness(1.1, 0.7, 2)
    t = np.repeat(c[None], og.num_quads, axis=0)
    lo, hi, cond = oracle_mod.eigenvalue_bounds(og, t, c, 2)
    assert np.abs(lo - 1.0).max() < 1e-12 and np.abs(hi - 1.0).max() < 1e-12
    assert abs(cond - 1.0) < 1e-12


def test_thermal_bounds_match_support_sweep(oracle_mod, golden):
    """test_spectral.cpp:63-108."""
    dims = (4, 4)
    og = oracle_mod.Grid(dims, (1.0, 1.0), "two-triangles")
    ph = oracle_mod.uniform(307, 16) > 0.0
    kap = np.where(np.repeat(ph, og.quads_per_pixel), 20.0, 0.05)
    t = kap[:, None, None] * np.eye(2)[None]
    lo, hi, _ = oracle_mod.eigenvalue_bounds(og, t, np.eye(2), 1, pixel_constant=True)
    D, _ = golden.dense_gradient(dims, (1.0, 1.0), "two-triangles", 1)
    nq = og.num_quads
    blo, bhi = [], []
    for n in range(og.num_nodes):
        sup = [q for q in range(nq) if any(D[k * nq + q, n] != 0.0 for k in range(2))]
        blo.append(min(kap[q] for q in sup))
        bhi.append(max(kap[q] for q in sup))
    assert np.abs(lo - np.sort(blo)).max() < 1e-12
    assert np.abs(hi - np.sort(bhi)).max() < 1e-12


def test_threaded_timing_variant_matches_serial(oracle_mod):
    """The oracle's threaded variant (bench.py --impl reference on all host
    cores) runs the same algorithm: equal to the serial loop order up to
    summation order; the serial path is unchanged (bitwise repeatable)."""
    dims = (16, 12, 10)
    og = oracle_mod.Grid(dims, [1.0, 1.0, 1.0], "trilinear-hex")
    cm = np.stack([oracle_mod.isotropic_stiffness(0.83, 0.38, 3), oracle_mod.isotropic_stiffness(55.5, 41.7, 3)])
    ph = (oracle_mod.uniform(3, og.num_pixels, 0.0, 1.0) < 0.3).astype(np.uint8)
    pre = oracle_mod.Preconditioner(og, cm[0], 3)
    s = oracle_mod.uniform(4, og.num_quads * 6).reshape(og.num_quads, 6)
    b = -oracle_mod.divergence(og, 3, s)
    serial = oracle_mod.pcg(og, 3, cm, ph, pre, b, 0.0, 5)["x"]
    prev = oracle_mod.set_threads(4)
    try:
        threaded = oracle_mod.pcg(og, 3, cm, ph, pre, b, 0.0, 5)["x"]
    finally:
        oracle_mod.set_threads(prev)
    again = oracle_mod.pcg(og, 3, cm, ph, pre, b, 0.0, 5)["x"]
    assert np.array_equal(serial, again)
    assert np.linalg.norm(threaded - serial) <= 1e-12 * np.linalg.norm(serial)
