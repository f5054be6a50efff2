"""J2 plasticity Newton path on the GPU against the
oracle's restatement of material.cpp:122-226 and solver.cpp:120-319."""
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


def _rel(a, b):
    return np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def _pair(hb, oracle_mod, dims, stencil, mats_gpu, mats_or, ph, e, **kw):
    g = hb.Grid(dims, [1.0] * len(dims), stencil)
    og = oracle_mod.Grid(dims, [1.0] * len(dims), stencil)
    got = hb.Solver(g, mats_gpu, ph, **kw).solve(e, stress=True)
    okw = dict(kw)
    ref = oracle_mod.newton_solve_models(og, False, mats_or, ph, e, **okw)
    return got, ref


def _j2_pair(hb, oracle_mod, d, params):
    gpu = [hb.Material.j2_plastic(*p, d) for p in params]
    orc = [oracle_mod.material("j2", bulk=p[0], shear=p[1], yield_stress=p[2], hardening=p[3]) for p in params]
    return gpu, orc


@pytest.mark.parametrize("reference", ["explicit", "volume-mean"])
def test_j2_plane_strain_matches_oracle(hb, oracle_mod, reference):
    """acceptance.cpp:333-345 plastic instance (8x8 two triangles)."""
    gpu, orc = _j2_pair(hb, oracle_mod, 2, [(0.833, 0.385, 3e-3, 0.08), (0.833, 0.385, 6e-3, 0.16)])
    ph = (oracle_mod.uniform(7007, 64, 0.0, 1.0) < 0.5).astype(np.uint8)
    e = np.array([5e-3, -5e-3, 1e-3])
    kw = dict(eta_newton=1e-10, eta_cg=1e-12, reference=reference)
    if reference == "explicit":
        kw["reference_matrix"] = np.eye(3)
    got, ref = _pair(hb, oracle_mod, (8, 8), "two-triangles", gpu, orc, ph, e, **kw)
    assert got["converged"] and ref["converged"]
    steps_g = [s["cg_iterations"] for s in got["report"]["steps"]]
    steps_o = [s["cg_iterations"] for s in ref["steps"]]
    assert len(steps_g) == len(steps_o), (steps_g, steps_o)
    assert all(abs(a - b) <= 1 for a, b in zip(steps_g, steps_o)), (steps_g, steps_o)
    assert got["report"]["assemblies"] == ref["assemblies"]
    assert _rel(got["u"], ref["u"]) < 1e-8
    assert _rel(got["average_stress"], ref["average_stress"]) < 1e-9
    gi, oi = got["internal"], ref["internal"].reshape(-1, 7)
    assert np.abs(gi - oi).max() <= 1e-9 * np.abs(oi).max()
    assert oi[:, 6].max() > 0.0  # plastic flow happened


def test_j2_hex_mixed_catalog_matches_oracle(hb, oracle_mod):
    """3-D trilinear hex, linear elastic matrix + J2 inclusions."""
    d = 3
    c0 = hb.isotropic_stiffness(1.0, 0.6, 3)
    gpu = [hb.Material.linear_elastic(c0), hb.Material.j2_plastic(2.0, 1.2, 4e-3, 0.1, 3)]
    orc = [oracle_mod.material("linear", c0), oracle_mod.material("j2", bulk=2.0, shear=1.2, yield_stress=4e-3,
                                                                  hardening=0.1)]
    ph = (oracle_mod.uniform(99, 8 * 6 * 8, 0.0, 1.0) < 0.4).astype(np.uint8)
    e = np.array([4e-3, -1e-3, 0.0, 0.0, 2e-3, 3e-3])
    got, ref = _pair(hb, oracle_mod, (8, 6, 8), "trilinear-hex", gpu, orc, ph, e, eta_newton=1e-10, eta_cg=1e-12)
    assert got["converged"] and ref["converged"]
    assert len(got["report"]["steps"]) == len(ref["steps"])
    assert _rel(got["u"], ref["u"]) < 1e-8
    assert _rel(got["average_stress"], ref["average_stress"]) < 1e-9
    oi = ref["internal"].reshape(-1, 7)
    assert np.abs(got["internal"] - oi).max() <= 1e-9 * max(np.abs(oi).max(), 1e-30)


@pytest.mark.parametrize("fast", ["1", "0"])
def test_j2_hex_modal_operator_matches_oracle(hb, oracle_mod, fast, monkeypatch):
    """Hex grid eligible for the modal kernel: the J2 tangent operator runs on
    the z-march kernel with per-Gauss-point compact tangents (fast = 1) or on
    the generic two-pass path (0); both against the oracle."""
    monkeypatch.setenv("HOMFE_J2_FAST", fast)
    c0 = hb.isotropic_stiffness(1.0, 0.6, 3)
    gpu = [hb.Material.linear_elastic(c0), hb.Material.j2_plastic(2.0, 1.2, 4e-3, 0.1, 3)]
    orc = [oracle_mod.material("linear", c0), oracle_mod.material("j2", bulk=2.0, shear=1.2, yield_stress=4e-3,
                                                                  hardening=0.1)]
    dims = (16, 8, 32)
    ph = (oracle_mod.uniform(98, 16 * 8 * 32, 0.0, 1.0) < 0.4).astype(np.uint8)
    e = np.array([4e-3, -1e-3, 0.0, 0.0, 2e-3, 3e-3])
    got, ref = _pair(hb, oracle_mod, dims, "trilinear-hex", gpu, orc, ph, e, eta_newton=1e-10, eta_cg=1e-12)
    assert got["converged"] and ref["converged"]
    assert len(got["report"]["steps"]) == len(ref["steps"])
    assert all(abs(a["cg_iterations"] - b["cg_iterations"]) <= 1 for a, b in zip(got["report"]["steps"], ref["steps"]))
    assert _rel(got["u"], ref["u"]) < 1e-8
    assert _rel(got["average_stress"], ref["average_stress"]) < 1e-9
    oi = ref["internal"].reshape(-1, 7)
    assert oi[:, 6].max() > 0.0
    assert np.abs(got["internal"] - oi).max() <= 1e-9 * np.abs(oi).max()


def test_j2_load_program_commits_state(hb, oracle_mod):
    """run_load_program (solver.cpp:298-319): warm start + committed state."""
    gpu, orc = _j2_pair(hb, oracle_mod, 2, [(1.0, 0.5, 1e-3, 0.05), (10.0, 5.0, 2e-3, 0.5)])
    ph = np.zeros(100, np.uint8)
    ph.reshape(10, 10)[3:7, 3:7] = 1  # square inclusion (test_solver.cpp:353-354)
    loads = [np.array([2e-3, 0.0, 1e-3]), np.array([4e-3, 0.0, 2e-3])]
    kw = dict(eta_newton=1e-10, eta_cg=1e-12, reference="explicit", reference_matrix=np.eye(3))
    res = hb.run_load_program(hb.Grid((10, 10), (1.0, 1.0), "two-triangles"), gpu, ph, loads, **kw)
    og = oracle_mod.Grid((10, 10), (1.0, 1.0), "two-triangles")
    g = None
    warm = None
    for step, e in enumerate(loads):
        ref = oracle_mod.newton_solve_models(og, False, orc, ph, e, g0=g, warm_u=warm, **kw)
        assert res[step]["converged"] and ref["converged"]
        assert _rel(res[step]["average_stress"], ref["average_stress"]) < 1e-9
        assert _rel(res[step]["u"], ref["u"]) < 1e-8
        g = ref["internal"]
        warm = ref["u"]
    assert res[1]["internal"][:, 6].max() > res[0]["internal"][:, 6].max()


def test_j2_newton_cap_keeps_committed_state(hb):
    """test_solver.cpp:351-371: the iteration cap is reported, not thrown,
    and the committed state is returned unchanged."""
    g = hb.Grid((8, 8), (1.0, 1.0), "two-triangles")
    mats = [hb.Material.j2_plastic(1.0, 0.5, 1e-4, 0.05, 2), hb.Material.j2_plastic(10.0, 5.0, 2e-4, 0.5, 2)]
    ph = np.zeros(64, np.uint8)
    ph.reshape(8, 8)[2:6, 2:6] = 1
    s = hb.Solver(g, mats, ph, eta_newton=1e-12, max_newton=1)
    out = s.solve([0.05, 0.0, 0.02])
    assert not out["converged"] and out["report"]["cause"] == "newton-cap"
    assert out["report"]["newton_steps"] <= 1
    assert np.abs(out["internal"]).max() == 0.0


def test_linear_stress_field_matches_oracle(hb, oracle_mod):
    """NewtonOutcome::stress of a linear solve: sigma = C (e + D u)."""
    dims = (12, 10)
    c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(9.0, 4.0, 2)
    ph = (oracle_mod.uniform(3, 120, 0.0, 1.0) < 0.3).astype(np.uint8)
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    out = hb.newton_solve(g, [hb.Material.linear_elastic(c0), hb.Material.linear_elastic(c1)], ph,
                          [0.01, 0.0, 0.002], eta_cg=1e-10)
    og = oracle_mod.Grid(dims, [1.0, 1.0], "two-triangles")
    eps = oracle_mod.gradient(og, 2, out["u"]).reshape(-1, 3) + np.array([0.01, 0.0, 0.002])
    cm = np.stack([c0, c1])[np.repeat(ph, og.quads_per_pixel)]
    sig = np.einsum("qij,qj->qi", cm, eps)
    assert np.abs(out["stress"] - sig).max() <= 1e-12 * np.abs(sig).max()


def test_j2_load_program_shares_precond_manager(hb, oracle_mod):
    """run_load_program shares ONE PrecondManager over its steps
    (solver.cpp:306-318): with the volume-mean policy the reference is
    reassembled only when the averaged tangent drifts beyond the threshold
    (solver.cpp:120-142), so later steps may reuse an older C_ref. Per-step
    CG counts, reassembly flags and assembly counts match the oracle run with
    one shared manager."""
    gpu, orc = _j2_pair(hb, oracle_mod, 2, [(0.833, 0.385, 3e-3, 0.08), (0.833, 0.385, 6e-3, 0.16)])
    ph = (oracle_mod.uniform(7007, 256, 0.0, 1.0) < 0.5).astype(np.uint8)
    loads = [np.array([5e-3, -5e-3, 1e-3]) * s for s in (0.4, 0.7, 1.0, 1.3)]
    kw = dict(eta_newton=1e-9, eta_cg=1e-10, reference="volume-mean", reassembly_threshold=0.05)
    grid = hb.Grid((16, 16), (1.0, 1.0), "two-triangles")
    res = hb.run_load_program(grid, gpu, ph, loads, **kw)
    og = oracle_mod.Grid((16, 16), (1.0, 1.0), "two-triangles")
    mgr = oracle_mod.PrecondManager()
    g = warm = None
    flags_g, flags_o = [], []
    for step, e in enumerate(loads):
        ref = oracle_mod.newton_solve_models(og, False, orc, ph, e, g0=g, warm_u=warm, manager=mgr, **kw)
        got = res[step]
        assert got["converged"] and ref["converged"]
        assert got["report"]["newton_steps"] == len(ref["steps"]), step
        for sg, so in zip(got["report"]["steps"], ref["steps"]):
            assert abs(sg["cg_iterations"] - so["cg_iterations"]) <= 1, step
            flags_g.append(sg["precond_reassembled"])
            flags_o.append(so["precond_reassembled"])
        assert got["report"]["assemblies"] == ref["assemblies"], step
        assert _rel(got["average_stress"], ref["average_stress"]) < 1e-8
        g, warm = ref["internal"], ref["u"]
    assert flags_g == flags_o
    # the drift rule did skip reassemblies on later Newton steps
    assert sum(flags_o) < len(flags_o) and mgr.assemblies == sum(flags_o)
