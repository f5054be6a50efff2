"""GPU parity of the fused three-pass preconditioner (fftfused.cu) against
the cuFFT path of the same library and against the CPU oracle."""
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


def _grid(hb, dims, monkeypatch, fused):
    monkeypatch.setenv("HOMFE_FUSED_FFT", "1" if fused else "0")
    return hb.Grid(dims, [1.0, 1.0, 1.0], "trilinear-hex")


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("dims,c", [((64, 128, 128), 1), ((64, 128, 128), 3), ((128, 128, 128), 1),
                                    ((64, 256, 256), 3), ((256, 128, 128), 3), ((256, 128, 128), 1)])
def test_minv_fused_matches_cufft(hb, monkeypatch, dims, c):
    rng = np.random.default_rng(5)
    m = 3 if c == 1 else 6
    a = rng.uniform(-1, 1, (m, m))
    c_ref = a @ a.T + 0.5 * np.eye(m)
    r = rng.uniform(-1, 1, (c, int(np.prod(dims))))
    r -= r.mean(axis=1, keepdims=True)
    gf = _grid(hb, dims, monkeypatch, True)
    zf = hb.apply_preconditioner(gf, hb.assemble_preconditioner(gf, c_ref, c), r)
    gc = _grid(hb, dims, monkeypatch, False)
    zc = hb.apply_preconditioner(gc, hb.assemble_preconditioner(gc, c_ref, c), r)
    assert _rel(zf, zc) < 1e-13


def test_minv_fused_matches_oracle(hb, oracle_mod, monkeypatch):
    dims = (64, 128, 128)
    og = oracle_mod.Grid(dims, [1.0] * 3, "trilinear-hex")
    c_ref = np.diag([1.0, 2.0, 3.0]) + 0.1
    r = oracle_mod.uniform(3, og.num_nodes)
    r -= r.mean()
    zo = oracle_mod.Preconditioner(og, c_ref, 1).apply(r)
    g = _grid(hb, dims, monkeypatch, True)
    z = hb.apply_preconditioner(g, hb.assemble_preconditioner(g, c_ref, 1), r.reshape(1, -1)).ravel()
    assert np.abs(z - zo).max() < 1e-10 * np.abs(zo).max()


@pytest.mark.parametrize("dims,c", [((64, 128, 128), 3), ((128, 128, 128), 1), ((64, 256, 256), 3)])
def test_pcg_fused_matches_cufft_path(hb, monkeypatch, dims, c):
    from paper_2203_02962_b200 import inputs
    ph, _ = inputs.rsa_balls(dims, radius=6.0, seed=3, fraction=0.25)
    d = 3
    if c == 1:
        cm = np.stack([np.eye(d), 100.0 * np.eye(d)])
        e = [1.0, 0.0, 0.0]
    else:
        cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)])
        e = [0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01]
    outs = []
    for fused in (True, False):
        g = _grid(hb, dims, monkeypatch, fused)
        mats = [hb.Material(t, c == 1, 3) for t in cm]
        outs.append(hb.newton_solve(g, mats, ph, e, eta_cg=1e-6, reference="explicit", reference_matrix=cm[0]))
    f, cu = outs
    assert f["converged"] and cu["converged"]
    kf, kc = f["report"]["steps"][0]["cg_iterations"], cu["report"]["steps"][0]["cg_iterations"]
    assert abs(kf - kc) <= 1
    tol = 1e-8 if kf == kc else 1e-5
    assert _rel(f["u"], cu["u"]) < tol
    assert _rel(f["average_stress"], cu["average_stress"]) < tol
