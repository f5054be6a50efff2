"""Slab-mode context (homfe_gpu_create_dist) on one GPU (world = 1: the halo
ring and the transposes exchange with the rank itself through NCCL) against
the single-device context. Multi-rank host logic: tests/test_dist_host.py."""
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
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("dims,c", [((64, 128, 128), 3), ((128, 128, 128), 1)])
def test_slab_world1_matches_single_device(hb, dims, c):
    from paper_2203_02962_b200 import _native, dist, inputs
    ph, _ = inputs.rsa_balls(dims, radius=6.0, seed=3, fraction=0.25)
    if c == 1:
        cm = np.stack([np.eye(3), 100.0 * np.eye(3)])
        e = [1.0, 0.0, 0.0]
    else:
        cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)])
        e = [0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01]
    g = hb.Grid(dims, [1.0, 1.0, 1.0], "trilinear-hex")
    mats = [hb.Material(t, c == 1, 3) for t in cm]
    single = hb.Solver(g, mats, ph, eta_cg=1e-6, reference="explicit", reference_matrix=cm[0])
    ref = single.solve(e)
    sc = dist.SlabContext(g, c, 0, 1, dist.nccl_unique_id())
    sc.set_material(cm, ph)
    rng = np.random.default_rng(1)
    u = rng.uniform(-1, 1, (c, g.num_nodes))
    np.testing.assert_array_equal(sc.apply_K(u), hb.apply_operator(g, cm[np.repeat(ph, 8)], u))
    sc.set_reference(cm[0])
    r = u - u.mean(axis=1, keepdims=True)
    z1 = sc.apply_minv(r)
    z0 = hb.apply_preconditioner(g, hb.assemble_preconditioner(g, cm[0], c), r)
    assert _rel(z1, z0) < 1e-14
    out = sc.solve(e, single.cfg)
    assert out["converged"]
    assert out["report"]["steps"][0]["cg_iterations"] == ref["report"]["steps"][0]["cg_iterations"]
    assert _rel(out["u"], ref["u"]) < 1e-12
    assert _rel(out["average_stress"], ref["average_stress"]) < 1e-12
