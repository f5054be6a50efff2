"""The BASELINE.json configurations c1-c5 at their full sizes on the GPU.

Oracle parity at these configurations (tolerance mode, fixed k at 1e-10, the
noise floor) is in test_gpu_baseline_parity.py. This file checks
size-independent properties of the problem at the full sizes, including the
ones the oracle cannot reach in test time (c4 at 512^3, c5 at 8192^2):

* linearity, bit-exact: u(2e) == 2 u(e) and <sigma>(2e) == 2 <sigma>(e) with
  the same iteration count (every PCG scalar is a ratio, so scaling by a power
  of two is exact in fp64);
* determinism: two solves are bitwise identical (fixed-order reductions);
* periodicity: rolling the microstructure rolls the solution;
* Voigt / Reuss bounds on the homogenized energy e.<sigma> (the energy of the
  total strain field, Hill-Mandel; PAPER section 4.3 bounds);
* mean-free fluctuation (solver.cpp:95) and the a-priori CG bound
  k <= sqrt(kappa)/2 ln(2/eta) of SURVEY 8(d);
* mesh independence of the iteration count over the c5 resolution sweep
  (the property the Fourier preconditioner is there for).
"""
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


_CACHE = {}


def _setup(hb, name, n=None, contrast=None):
    from paper_2203_02962_b200 import inputs
    key = (name, n, contrast)
    if key not in _CACHE:
        _CACHE.clear()  # one full-size config resident at a time
        cfg = inputs.config(name, n=n, contrast=contrast)
        _CACHE[key] = (cfg, cfg.phases(), cfg.tangents())
    return _CACHE[key]


def _solver(hb, cfg, ph, tans):
    g = hb.Grid(cfg.dims, [1.0] * cfg.dim, cfg.stencil)
    mats = [hb.Material(t, cfg.thermal, cfg.dim) for t in tans]
    return g, hb.Solver(g, mats, ph, eta_cg=cfg.eta_cg, eta_newton=cfg.eta_newton, reference=cfg.reference,
                        reference_matrix=cfg.reference_matrix())


def _bounds(cfg, ph, tans, e):
    """Reuss <= e.C_eff.e <= Voigt with phase volume fractions."""
    f = np.bincount(ph, minlength=len(tans)).astype(float) / ph.size
    voigt = np.einsum("p,pij->ij", f, tans)
    reuss = np.linalg.inv(np.einsum("p,pij->ij", f, np.linalg.inv(tans)))
    return float(e @ reuss @ e), float(e @ voigt @ e)


def _kbound(cfg, tans):
    """a-priori CG bound of SURVEY 8(d): kappa from the extreme generalised
    eigenvalues of C_ref^-1 C over the phases."""
    if cfg.reference == "explicit":
        cref = tans[cfg.reference_phase]
    else:
        return None  # volume-mean reference: no closed form here
    lam = np.concatenate([np.linalg.eigvals(np.linalg.solve(cref, t)).real for t in tans])
    kappa = lam.max() / lam.min()
    return 0.5 * np.sqrt(kappa) * np.log(2.0 / cfg.eta_cg)


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.mark.parametrize("name,n,contrast", [("c1", None, None), ("c2", None, None), ("c3", None, None),
                                             ("c4", None, None), ("c5", 1024, 1e1), ("c5", 1024, 1e5),
                                             ("c5", 8192, 1e3)])
def test_config_full_size_properties(hb, name, n, contrast):
    cfg, ph, tans = _setup(hb, name, n, contrast)
    g, s = _solver(hb, cfg, ph, tans)
    e = np.asarray(cfg.load, dtype=float)
    out = s.solve(e)
    assert out["converged"], (name, out["report"])
    rep = out["report"]
    k = rep["cg_total"]
    kb = _kbound(cfg, tans)
    if kb is not None:
        assert k <= kb, (name, k, kb)
    u = out["u"]
    means = np.abs(u.mean(axis=1))
    assert means.max() <= 1e-12 * max(np.abs(u).max(), 1e-300), (name, means)
    energy = float(e @ out["average_stress"])
    lo, hi = _bounds(cfg, ph, tans, e)
    assert lo * (1 - 1e-12) <= energy <= hi * (1 + 1e-12), (name, lo, energy, hi)
    # linearity, bit-exact
    out2 = s.solve(2.0 * e)
    assert out2["report"]["cg_total"] == k
    assert np.array_equal(out2["u"], 2.0 * u), name
    assert np.array_equal(out2["average_stress"], 2.0 * out["average_stress"]), name


def test_c3_deterministic_and_periodic(hb):
    """Bitwise run-to-run reproducibility, and a periodic roll of the
    microstructure rolls the solution (c3 at 256^3)."""
    cfg, ph, tans = _setup(hb, "c3")
    e = np.asarray(cfg.load, dtype=float)
    g, s = _solver(hb, cfg, ph, tans)
    a = s.solve(e)
    b = s.solve(e)
    assert np.array_equal(a["u"], b["u"]) and np.array_equal(a["average_stress"], b["average_stress"])
    shift = (37, 5, 100)
    ph3 = ph.reshape(cfg.dims)
    phr = np.ascontiguousarray(np.roll(ph3, shift, axis=(0, 1, 2))).ravel()
    del s
    g, sr = _solver(hb, cfg, phr, tans)
    r = sr.solve(e)
    ka, kr = a["report"]["cg_total"], r["report"]["cg_total"]
    assert abs(ka - kr) <= 1
    ua = np.roll(a["u"].reshape((3,) + cfg.dims), shift, axis=(1, 2, 3)).reshape(3, -1)
    tol = 1e-9 if ka == kr else 10 * cfg.eta_cg
    assert _rel(r["u"], ua) <= tol
    assert _rel(r["average_stress"], a["average_stress"]) <= max(tol, 1e-12)


def test_c5_sweep_mesh_independence(hb):
    """c5: N in {1024, 2048, 4096, 8192} at contrast 1e3, same physical
    geometry: the Fourier-preconditioned iteration count does not grow with
    N, and the effective conductivity converges."""
    its, kx = [], []
    for n in (1024, 2048, 4096, 8192):
        cfg, ph, tans = _setup(hb, "c5", n, 1e3)
        g, s = _solver(hb, cfg, ph, tans)
        out = s.solve(np.asarray(cfg.load, dtype=float))
        assert out["converged"]
        its.append(out["report"]["cg_total"])
        kx.append(out["average_stress"][0])
        del s
    assert max(its) <= 1.25 * min(its) + 2, its
    # discretisation error of k_eff shrinks under refinement
    assert abs(kx[3] - kx[2]) <= abs(kx[1] - kx[0]) + 1e-12, kx
