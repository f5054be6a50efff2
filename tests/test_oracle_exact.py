"""CPU checks of the parity-test infrastructure added for the BASELINE
configurations: the oracle's exact (long double) reference symbol against the
reference's impulse probing, and the numpy Newton RHS / homogenized-stress
helpers (oracle/cfgutil.py) against the oracle's divergence / volume average."""
import numpy as np
import pytest

from oracle.cfgutil import average_stress, newton_rhs, rel


def _spd(m, seed):
    a = np.random.default_rng(seed).uniform(-1, 1, (m, m))
    return a @ a.T + 0.5 * np.eye(m)


@pytest.mark.parametrize("dims,lengths,stencil,c", [
    ((6, 5), (1.0, 0.7), "two-triangles", 1), ((6, 5), (1.0, 0.7), "two-triangles", 2),
    ((5, 6), (1.0, 1.0), "bilinear-quad", 2), ((4, 3, 5), (1.0, 0.7, 1.3), "trilinear-hex", 3),
    ((8, 6, 10), (1.0, 1.0, 1.0), "trilinear-hex", 1), ((16, 16, 16), (1.0, 1.0, 1.0), "trilinear-hex", 3)])
def test_exact_symbol_matches_probed_blocks(oracle_mod, dims, lengths, stencil, c):
    """test_precond.cpp:47-82 tolerance (1e-11 scale): the exact symbol is the
    same block as the probed one, without the probing's rounding."""
    g = oracle_mod.Grid(dims, lengths, stencil)
    cr = _spd(g.m(c), 3 + c)
    pb = oracle_mod.Preconditioner(g, cr, c, invert=False).blocks()
    pe = oracle_mod.Preconditioner(g, cr, c, invert=False, exact=True).blocks()
    scale = np.abs(pe).max()
    assert np.abs(pb - pe).max() <= 1e-13 * scale
    # the zero-frequency block of the exact symbol vanishes (constants are in
    # the kernel of K_ref)
    assert np.abs(pe[0]).max() <= 1e-15 * scale


def test_exact_symbol_low_frequency_relative_accuracy(oracle_mod):
    """At the lowest frequency the block is O(theta^2); the probed block
    carries ~eps/theta^2 relative rounding there, the exact one does not:
    check the exact one against the closed form of the scalar TwoTriangles
    symbol, 2 k (1 - cos theta0)/h0^2 ... (weights V_p/2, k I)."""
    n = 512
    g = oracle_mod.Grid((n, n), (1.0, 1.0), "two-triangles")
    pe = oracle_mod.Preconditioner(g, np.eye(2), 1, invert=False, exact=True).blocks()
    h = 1.0 / n
    vp = h * h
    for f0, f1 in [(1, 0), (0, 1), (1, 1), (3, 2)]:
        t0, t1 = 2 * np.pi * f0 / n, 2 * np.pi * f1 / n
        # sum over both triangles of |grad phase|^2 w: lower 4 sin^2(t0/2)/h^2 + 4 sin^2(t1/2)/h^2, upper the same
        want = vp * (4 * np.sin(t0 / 2) ** 2 + 4 * np.sin(t1 / 2) ** 2) / h ** 2
        got = pe[f0 * (n // 2 + 1) + f1, 0, 0]
        assert abs(got.real - want) <= 4e-16 * want and abs(got.imag) <= 1e-16 * want, (f0, f1)


@pytest.mark.parametrize("dims,stencil,c", [((12, 10), "two-triangles", 1), ((10, 12), "two-triangles", 2),
                                            ((6, 5, 7), "trilinear-hex", 3), ((6, 8, 4), "trilinear-hex", 1)])
def test_newton_rhs_and_average_stress_helpers(oracle_mod, dims, stencil, c):
    lengths = tuple(1.0 + 0.1 * a for a in range(len(dims)))
    g = oracle_mod.Grid(dims, lengths, stencil)
    m = g.m(c)
    cm = np.stack([_spd(m, 1), _spd(m, 2), _spd(m, 3)])
    ph = np.random.default_rng(4).integers(0, 3, g.num_pixels).astype(np.uint8)
    e = np.random.default_rng(5).uniform(-1, 1, m)
    nq = g.quads_per_pixel
    sig = np.einsum("qij,j->qi", cm[np.repeat(ph, nq)], e)
    b_or = -oracle_mod.divergence(g, c, sig)
    b_np = newton_rhs(dims, lengths, c, cm, ph, e)
    assert rel(b_np, b_or) <= 1e-14
    u = oracle_mod.uniform(7, c * g.num_nodes)
    grad = oracle_mod.gradient(g, c, u)
    sq = np.einsum("qij,qj->qi", cm[np.repeat(ph, nq)], grad + e)
    s_or = oracle_mod.volume_average(g, sq)
    s_np = average_stress(dims, lengths, c, cm, ph, e, u)
    assert rel(s_np, s_or) <= 1e-13
