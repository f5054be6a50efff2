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


@pytest.mark.parametrize("dims,c", [((64, 128, 128), 3), ((128, 128, 128), 1), ((32, 64, 64), 3)])
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


@pytest.mark.parametrize("world,dims,c,transport", [
    (2, (64, 128, 128), 3, "peer_pull"), (2, (128, 128, 128), 3, "peer_pull"), (4, (128, 128, 128), 1, "peer_pull"),
    (8, (128, 256, 256), 3, "peer_pull"), (2, (128, 128, 128), 3, "all_to_all"), (4, (128, 128, 128), 1, "all_to_all"),
    (8, (128, 256, 256), 3, "all_to_all"),
    # plane sizes outside the fused passes: slab spectra (cuFFT per rank + transposes, slabfft.cu)
    (2, (32, 64, 64), 3, "peer_pull"), (2, (32, 64, 64), 3, "all_to_all"), (4, (64, 96, 96), 1, "peer_pull"),
    (2, (16, 512, 512), 3, "peer_pull")])
def test_slab_multi_rank_in_process_matches_single_device(hb, world, dims, c, transport, monkeypatch):
    """World > 1 on one GPU through the in-process transport (host barriers
    instead of NCCL; no device-side waiting between ranks): the halo ring (sent
    planes, or the neighbours' p read in place by the K kernels), both
    peer-chunk transposes of the fused passes (all-to-all copies, or passes 2
    and 3 pulling the source ranks' chunks straight from their buffers), the
    pencil frequency offsets and the rank-ordered reductions against the
    single-device context."""
    import threading
    from paper_2203_02962_b200 import dist, inputs
    monkeypatch.setenv("HOMFE_P2P", "1" if transport == "peer_pull" else "0")
    ph, _ = inputs.rsa_balls(dims, radius=6.0, seed=5, fraction=0.25)
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
    rng = np.random.default_rng(2)
    u = rng.uniform(-1, 1, (c, g.num_nodes))
    ku_ref = hb.apply_operator(g, cm[np.repeat(ph, 8)], u)
    r = u - u.mean(axis=1, keepdims=True)
    z_ref = hb.apply_preconditioner(g, hb.assemble_preconditioner(g, cm[0], c), r)
    plane = dims[1] * dims[2]
    gid = 1000 + world * 10 + c + (0 if transport == "peer_pull" else 500) + dims[0]
    res = [None] * world
    errors = []

    def rank_main(rank):
        try:
            sc = dist.SlabContext(g, c, rank, world, dist.sim_group_id(gid))
            assert sc.transport == transport
            z0, nz = sc.z0, sc.nz
            sl = slice(z0 * plane, (z0 + nz) * plane)
            sc.set_material(cm, ph[sl])
            ku = sc.apply_K(u[:, sl])
            sc.set_reference(cm[0])
            z = sc.apply_minv(r[:, sl])
            out = sc.solve(e, single.cfg)
            res[rank] = (sl, ku, z, out)
        except Exception as ex:  # noqa: BLE001
            errors.append(repr(ex))

    threads = [threading.Thread(target=rank_main, args=(k,)) for k in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors
    ku = np.zeros_like(u)
    z = np.zeros_like(u)
    uu = np.zeros_like(u)
    for sl, kl, zl, out in res:
        ku[:, sl], z[:, sl], uu[:, sl] = kl, zl, out["u"]
    assert _rel(ku, ku_ref) < 1e-15, _rel(ku, ku_ref)
    np.testing.assert_array_equal(ku, ku_ref)
    assert _rel(z, z_ref) < 1e-13, _rel(z, z_ref)
    for sl, kl, zl, out in res:
        assert out["converged"]
        assert out["report"]["steps"][0]["cg_iterations"] == ref["report"]["steps"][0]["cg_iterations"]
        assert _rel(out["average_stress"], ref["average_stress"]) < 1e-12
    # 1e-10 (north_star): the slab spectra use 2-D + 1-D cuFFT plans instead of one 3-D plan
    assert _rel(uu, ref["u"]) < 1e-10


@pytest.mark.parametrize("world,n,c,transport", [
    (1, 256, 1, "single"), (2, 256, 1, "peer_pull"), (4, 512, 1, "all_to_all"), (8, 1024, 1, "peer_pull"),
    (8, 1024, 1, "all_to_all"), (2, 128, 2, "peer_pull"), (4, 256, 2, "all_to_all")])
def test_slab_2d_rows_match_single_device(hb, world, n, c, transport, monkeypatch):
    """2-D row slabs (c5 on 1 and 8 GPUs, BASELINE configs[4]): halo rows for
    K, 1-D r2c along axis 1 of the owned rows, all-to-all of half-spectrum
    column chunks (padded to G ceil(nh / G)), 1-D c2c along axis 0 and the
    spectral solve on the owned columns. W ranks in-process on one GPU
    against the single-device context (2-D cuFFT, warp-strip K)."""
    import threading
    from paper_2203_02962_b200 import dist, inputs
    monkeypatch.setenv("HOMFE_P2P", "1" if transport == "peer_pull" else "0")
    dims = (n, n)
    ph, _ = inputs.rsa_balls(dims, radius=12.0 * n / 256, seed=BASE_2D_SEED, fraction=0.30)
    if c == 1:
        cm = np.stack([np.eye(2), 1e3 * np.eye(2)])
        e = [1.0, 0.0]
        kw = dict(eta_cg=1e-8, reference="volume-mean")
    else:
        cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 2), hb.isotropic_stiffness(555.5, 416.7, 2)])
        e = [0.0, 0.0, np.sqrt(2.0) * 0.01]
        kw = dict(eta_cg=1e-8, reference="explicit", reference_matrix=cm[0])
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    mats = [hb.Material(t, c == 1, 2) for t in cm]
    single = hb.Solver(g, mats, ph, **kw)
    ref = single.solve(e)
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, (c, g.num_nodes))
    ku_ref = hb.apply_operator(g, cm[np.repeat(ph, 2)], u)
    r = u - u.mean(axis=1, keepdims=True)
    cref = cm[0] if c > 1 else (np.bincount(ph, minlength=2)[:, None, None] * cm).sum(0) / ph.size
    z_ref = hb.apply_preconditioner(g, hb.assemble_preconditioner(g, cref, c), r)
    row = n
    gid = 5000 + world * 10 + c + (0 if transport != "all_to_all" else 500) + n
    res = [None] * world
    errors = []

    def rank_main(rank):
        try:
            ident = dist.sim_group_id(gid) if world > 1 else dist.nccl_unique_id()
            sc = dist.SlabContext(g, c, rank, world, ident)
            assert sc.transport == transport, sc.transport
            sl = slice(sc.z0 * row, (sc.z0 + sc.nz) * row)
            sc.set_material(cm, ph[sl])
            ku = sc.apply_K(u[:, sl])
            sc.set_reference(cref)
            z = sc.apply_minv(r[:, sl])
            out = sc.solve(e, single.cfg)
            res[rank] = (sl, ku, z, out)
        except Exception as ex:  # noqa: BLE001
            errors.append(repr(ex))

    threads = [threading.Thread(target=rank_main, args=(k,)) for k in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors
    ku = np.zeros_like(u)
    z = np.zeros_like(u)
    uu = np.zeros_like(u)
    for sl, kl, zl, out in res:
        ku[:, sl], z[:, sl], uu[:, sl] = kl, zl, out["u"]
    # the slab K is the generic node-centric kernel, the single device's the warp-strip one
    assert _rel(ku, ku_ref) < 1e-13, _rel(ku, ku_ref)
    assert _rel(z, z_ref) < 1e-13, _rel(z, z_ref)
    for sl, kl, zl, out in res:
        assert out["converged"]
        assert abs(out["report"]["steps"][0]["cg_iterations"] - ref["report"]["steps"][0]["cg_iterations"]) <= 1
        assert _rel(out["average_stress"], ref["average_stress"]) < 1e-10
    assert _rel(uu, ref["u"]) < 1e-8


BASE_2D_SEED = 2203025


@pytest.mark.parametrize("n_gpus,dims,stencil,c", [(2, (64, 128, 128), "trilinear-hex", 3),
                                                   (4, (128, 128, 128), "trilinear-hex", 1),
                                                   (8, (1024, 1024), "two-triangles", 1),
                                                   (2, (32, 64, 64), "trilinear-hex", 3)])
def test_single_process_multi_gpu_context(hb, n_gpus, dims, stencil, c, monkeypatch):
    """homfe_gpu_create_multi (one host process driving n_gpus
    slab ranks, one host thread per rank inside each call) through the
    ordinary Python API with GLOBAL fields: Grid(..., n_gpus). On the one
    test GPU every rank runs on device 0 with the in-process transport
    (HOMFE_MULTI_SIM=1). Against the single-device context."""
    from paper_2203_02962_b200 import inputs
    monkeypatch.setenv("HOMFE_MULTI_SIM", "1")
    d = len(dims)
    ph, _ = inputs.rsa_balls(dims, radius=dims[0] / 16.0, seed=9, fraction=0.25)
    if c == 1:
        cm = np.stack([np.eye(d), 100.0 * np.eye(d)])
        e = np.zeros(d)
        e[0] = 1.0
    else:
        cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)])
        e = np.array([0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01])
    lengths = [x / dims[-1] for x in dims]
    mats = [hb.Material(t, c == 1, d) for t in cm]
    g1 = hb.Grid(dims, lengths, stencil)
    gm = hb.Grid(dims, lengths, stencil, n_gpus=n_gpus)
    kw = dict(eta_cg=1e-8, reference="explicit", reference_matrix=cm[0])
    ref = hb.Solver(g1, mats, ph, **kw).solve(e)
    sm = hb.Solver(gm, mats, ph, **kw)
    assert "multi" in gm.context(c).path() and "slab" in gm.context(c).path()
    out = sm.solve(e)
    assert out["converged"]
    assert abs(out["report"]["steps"][0]["cg_iterations"] - ref["report"]["steps"][0]["cg_iterations"]) <= 1
    assert _rel(out["average_stress"], ref["average_stress"]) < 1e-10
    assert _rel(out["u"], ref["u"]) < 1e-8
    # operators with global fields
    rng = np.random.default_rng(4)
    u = rng.uniform(-1, 1, (c, g1.num_nodes))
    nq = g1.quads_per_pixel
    assert _rel(hb.apply_operator(gm, cm[np.repeat(ph, nq)], u), hb.apply_operator(g1, cm[np.repeat(ph, nq)], u)) < 1e-13
    r = u - u.mean(axis=1, keepdims=True)
    zm = hb.apply_preconditioner(gm, hb.assemble_preconditioner(gm, cm[0], c), r)
    z1 = hb.apply_preconditioner(g1, hb.assemble_preconditioner(g1, cm[0], c), r)
    assert _rel(zm, z1) < 1e-13
