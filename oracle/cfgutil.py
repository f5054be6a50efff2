"""TEST INFRASTRUCTURE (with the oracle): the Newton right-hand side and the homogenized stress of a
pixel-constant linear material, in numpy, for grids too large for the
oracle's quadrature fields (c3: 6.4 GB per QuadField).

Both use one identity of the one-node stencils of the configurations
(TwoTriangles, TrilinearHex; grid.cpp:114-145,190-229): the quadrature-weighted
sum of a shape-function gradient over one pixel is V_p * dbar[o], with
dbar[o][a] = (2 o_a - 1) / (h_a 2^(d-1)) for the pixel corner o in {0,1}^d
(2-point Gauss integrates the bilinear gradients of the hex exactly; the two
triangles each carry half the pixel). With a pixel-constant stress sigma_p
(linear material, Newton step 0) this gives, exactly,
  b = -D^T W sigma      :  b[:, p + o] -= V_p * Bbar_o^T sigma_p
  <C (e + D u)>         :  sum_p C_p (e + Bbar u|_p) / N_p,
  Bbar u|_p = sum_o Bbar_o u[:, p + o]  (the pixel-average strain),
with the Mandel rows of operators.cpp:16-53. TEST INFRASTRUCTURE ONLY; checked
against the oracle's divergence / volume_average in tests/test_oracle.py.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

S2 = math.sqrt(2.0) / 2.0
_PAIRS = {2: [(0, 1)], 3: [(1, 2), (0, 2), (0, 1)]}  # Mandel shear slots after the diagonal


def _corners(d):
    return list(itertools.product((0, 1), repeat=d))


def _dbar(dims, lengths, o):
    d = len(dims)
    return np.array([(2 * o[a] - 1) / ((lengths[a] / dims[a]) * 2 ** (d - 1)) for a in range(d)])


def _strain_rows(d, c, db, u):
    """Mandel strain of one corner contribution: rows of operators.cpp:16-32
    applied to u (c, ...) with gradient weights db."""
    if c == 1:
        return np.stack([db[a] * u[0] for a in range(d)])
    rows = [db[a] * u[a] for a in range(d)]
    for i, j in _PAIRS[d]:
        rows.append(S2 * (db[j] * u[i] + db[i] * u[j]))
    return np.stack(rows)


def _adjoint_rows(d, c, db, s):
    """Transpose of _strain_rows (operators.cpp:36-53) on a stress s (m, ...)."""
    if c == 1:
        return (sum(db[a] * s[a] for a in range(d)))[None]
    out = [db[a] * s[a] for a in range(d)]
    for k, (i, j) in enumerate(_PAIRS[d]):
        sk = s[d + k]
        out[i] = out[i] + S2 * db[j] * sk
        out[j] = out[j] + S2 * db[i] * sk
    return np.stack(out)


def pixel_stress(cm, ph, e):
    """sigma_p = C_phase(p) e as (m, N_p)."""
    cm = np.asarray(cm, dtype=float)
    per_phase = cm @ np.asarray(e, dtype=float)  # (n_phases, m)
    return per_phase[ph].T.copy()


def newton_rhs(dims, lengths, c, cm, ph, e):
    """b = -D^T W C e (solver.cpp:189-196 at u = 0), shape (c, N_p)."""
    d = len(dims)
    vp = float(np.prod([lengths[a] / dims[a] for a in range(d)]))
    sig = pixel_stress(cm, ph, e).reshape((-1,) + tuple(dims))
    b = np.zeros((c,) + tuple(dims))
    for o in _corners(d):
        contrib = _adjoint_rows(d, c, _dbar(dims, lengths, o), sig)
        b -= vp * np.roll(contrib, shift=o, axis=tuple(range(1, d + 1)))
    return b.reshape(c, -1)


def average_stress(dims, lengths, c, cm, ph, e, u):
    """<sigma> = (1/|Y|) sum_q w_q C (e + (D u)_q) for a pixel-constant C."""
    d = len(dims)
    u = np.asarray(u, dtype=float).reshape((c,) + tuple(dims))
    m = np.asarray(cm).shape[1]
    strain = np.zeros((m,) + tuple(dims))
    for o in _corners(d):
        shifted = np.roll(u, shift=tuple(-x for x in o), axis=tuple(range(1, d + 1)))  # u[p + o]
        strain += _strain_rows(d, c, _dbar(dims, lengths, o), shifted)
    strain = strain.reshape(m, -1)
    n_p = strain.shape[1]
    cm = np.asarray(cm, dtype=float)
    out = np.zeros(m)
    for k in range(cm.shape[0]):
        sel = ph == k
        cnt = int(np.count_nonzero(sel))
        if cnt == 0:
            continue
        out += cm[k] @ (cnt * np.asarray(e, dtype=float) + strain[:, sel].sum(axis=1))
    return out / n_p


def rel(a, b):
    a = np.ravel(a)
    b = np.ravel(b)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
