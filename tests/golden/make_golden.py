#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from DENSE oracles.

The reference stores no golden vectors; its numerics are
pinned by dense oracles recomputed in its tests. This script restates those
dense oracles in numpy, independently of any matrix-free code in this repo:

  dense gradient D        proj/tests/support/oracles.hpp:20-69
  weights W               proj/tests/support/oracles.hpp:72-83
  material C              proj/tests/support/oracles.hpp:87-101
  K = D^T W C D           proj/tests/support/oracles.hpp:104-114
  pinv (SVD, rcond 1e-10) proj/tests/support/oracles.hpp:117-128
  unitary DFT             proj/tests/test_precond.cpp:14-32
  RNG mt19937_64 + (gen()>>11)*2^-53   proj/tests/support/oracles.hpp:154-160

with stencil tables restated from proj/src/grid.cpp:81-229 and the periodic
wrap of proj/src/grid.cpp:9-12,278-288. The inputs follow the structure of
the reference tests (test_operators.cpp:168-193, test_precond.cpp:47-82 and
201-252, test_solver.cpp:82-103, acceptance.cpp:83-144).

Run:  python tests/golden/make_golden.py      (writes tests/golden/*.npz)
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the C++ standard 64-bit Mersenne Twister)."""

    n, m = 312, 156
    a = 0xB5026F5AA96619E9
    upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed=5489):
        mt = [0] * self.n
        mt[0] = seed & MASK64
        for i in range(1, self.n):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
        self.mt, self.idx = mt, self.n

    def _twist(self):
        mt, n, m = self.mt, self.n, self.m
        for i in range(n):
            x = (mt[i] & self.upper) | (mt[(i + 1) % n] & self.lower)
            xa = x >> 1
            if x & 1:
                xa ^= self.a
            mt[i] = mt[(i + m) % n] ^ xa
        self.idx = 0

    def __call__(self):
        if self.idx >= self.n:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & MASK64

    def uniform(self, lo=-1.0, hi=1.0):
        return lo + (hi - lo) * ((self() >> 11) * 2.0 ** -53)


# ------------------------------------------------------------ stencil tables
QUAD_OFF = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0)]
HEX_OFF = [(0, 0, 0), (0, 0, 1), (0, 1, 0), (0, 1, 1), (1, 0, 0), (1, 0, 1), (1, 1, 0), (1, 1, 1)]


def stencil(dims, lengths, kind):
    """Returns (offsets, nodes_per_pixel, quads) with quads = [(w, [(off, node, dphi3)])]."""
    h = [lengths[a] / dims[a] for a in range(len(dims))]
    vp = float(np.prod(h))
    quads = []
    if kind == "two-triangles":
        quads.append((vp / 2, [(0, 0, (-1 / h[0], -1 / h[1], 0.0)), (1, 0, (1 / h[0], 0.0, 0.0)),
                               (2, 0, (0.0, 1 / h[1], 0.0))]))
        quads.append((vp / 2, [(3, 0, (1 / h[0], 1 / h[1], 0.0)), (2, 0, (-1 / h[0], 0.0, 0.0)),
                               (1, 0, (0.0, -1 / h[1], 0.0))]))
        return QUAD_OFF, 1, quads
    g = 0.5 / math.sqrt(3.0)
    gp = (0.5 - g, 0.5 + g)
    if kind == "bilinear-quad":
        for x in gp:
            for y in gp:
                ents = []
                for a in range(2):
                    for b in range(2):
                        xi, dxi = (1 - x, x)[a], (-1 / h[0], 1 / h[0])[a]
                        et, det = (1 - y, y)[b], (-1 / h[1], 1 / h[1])[b]
                        ents.append((a + 2 * b, 0, (dxi * et, xi * det, 0.0)))
                quads.append((vp / 4, ents))
        return QUAD_OFF, 1, quads
    if kind == "four-triangles-two-node":
        i0, i1 = 1 / h[0], 1 / h[1]
        quads = [
            (vp / 4, [(0, 0, (-i0, -i1, 0.0)), (1, 0, (i0, -i1, 0.0)), (0, 1, (0.0, 2 * i1, 0.0))]),
            (vp / 4, [(1, 0, (i0, -i1, 0.0)), (3, 0, (i0, i1, 0.0)), (0, 1, (-2 * i0, 0.0, 0.0))]),
            (vp / 4, [(3, 0, (i0, i1, 0.0)), (2, 0, (-i0, i1, 0.0)), (0, 1, (0.0, -2 * i1, 0.0))]),
            (vp / 4, [(2, 0, (-i0, i1, 0.0)), (0, 0, (-i0, -i1, 0.0)), (0, 1, (2 * i0, 0.0, 0.0))]),
        ]
        return QUAD_OFF, 2, quads
    assert kind == "trilinear-hex"
    for x in gp:
        for y in gp:
            for z in gp:
                ents = []
                for a in range(2):
                    for b in range(2):
                        for c in range(2):
                            xi, dxi = (1 - x, x)[a], (-1 / h[0], 1 / h[0])[a]
                            et, det = (1 - y, y)[b], (-1 / h[1], 1 / h[1])[b]
                            ze, dze = (1 - z, z)[c], (-1 / h[2], 1 / h[2])[c]
                            ents.append(((a * 2 + b) * 2 + c, 0, (dxi * et * ze, xi * det * ze, xi * et * dze)))
                quads.append((vp / 8, ents))
    return HEX_OFF, 1, quads


def mandel(d):
    return d * (d + 1) // 2


def pixel_coords(p, dims):
    out = []
    for a in range(len(dims)):
        stride = int(np.prod(dims[a + 1:]))
        out.append(p // stride)
        p -= out[-1] * stride
    return out


def wrap_index(coords, off, dims):
    flat = 0
    for a in range(len(dims)):
        stride = int(np.prod(dims[a + 1:]))
        flat += ((coords[a] + off[a]) % dims[a]) * stride
    return flat


def dense_gradient(dims, lengths, kind, c):
    d = len(dims)
    m = d if c == 1 else mandel(d)
    offs, nn_pp, quads = stencil(dims, lengths, kind)
    np_ = int(np.prod(dims))
    nq = len(quads)
    NQ, NI = np_ * nq, np_ * nn_pp
    D = np.zeros((m * NQ, c * NI))
    s2 = math.sqrt(2.0) / 2.0
    for p in range(np_):
        co = pixel_coords(p, dims)
        for lq, (_, ents) in enumerate(quads):
            q = p * nq + lq
            for off, node, dp in ents:
                nbr = wrap_index(co, offs[off], dims)
                nd = node * np_ + nbr
                dof = lambda comp: comp * NI + nd  # noqa: E731
                row = lambda k: k * NQ + q  # noqa: E731
                if c == 1:
                    for a in range(d):
                        D[row(a), dof(0)] += dp[a]
                elif d == 2:
                    D[row(0), dof(0)] += dp[0]
                    D[row(1), dof(1)] += dp[1]
                    D[row(2), dof(0)] += s2 * dp[1]
                    D[row(2), dof(1)] += s2 * dp[0]
                else:
                    D[row(0), dof(0)] += dp[0]
                    D[row(1), dof(1)] += dp[1]
                    D[row(2), dof(2)] += dp[2]
                    D[row(3), dof(1)] += s2 * dp[2]
                    D[row(3), dof(2)] += s2 * dp[1]
                    D[row(4), dof(0)] += s2 * dp[2]
                    D[row(4), dof(2)] += s2 * dp[0]
                    D[row(5), dof(0)] += s2 * dp[1]
                    D[row(5), dof(1)] += s2 * dp[0]
    return D, quads


def dense_weights(quads, np_, m):
    nq = len(quads)
    w = np.array([quads[q % nq][0] for q in range(np_ * nq)])
    return np.diag(np.tile(w, m))


def dense_material(tangent):  # tangent (NQ, m, m)
    NQ, m, _ = tangent.shape
    Cm = np.zeros((m * NQ, m * NQ))
    for q in range(NQ):
        for i in range(m):
            for j in range(m):
                Cm[i * NQ + q, j * NQ + q] = tangent[q, i, j]
    return Cm


def dense_operator(dims, lengths, kind, c, tangent, weighted=True):
    D, quads = dense_gradient(dims, lengths, kind, c)
    Cm = dense_material(tangent)
    if not weighted:
        return D.T @ Cm @ D
    W = dense_weights(quads, int(np.prod(dims)), tangent.shape[1])
    return D.T @ W @ Cm @ D


def dense_pinv(a, rcond=1e-10):
    u, s, vt = np.linalg.svd(a)
    inv = np.where(s > rcond * s.max(), 1.0 / np.where(s > 0, s, 1.0), 0.0)
    return (vt.T * inv) @ u.T


def unitary_dft(dims):
    np_ = int(np.prod(dims))
    F = np.zeros((np_, np_), dtype=complex)
    for k in range(np_):
        kc = pixel_coords(k, dims)
        for n in range(np_):
            nc = pixel_coords(n, dims)
            ph = sum(2 * math.pi * kc[a] * nc[a] / dims[a] for a in range(len(dims)))
            F[k, n] = complex(math.cos(ph), -math.sin(ph))
    return F / math.sqrt(np_)


def random_spd(n, gen, shift=0.5):
    a = np.array([[gen.uniform() for _ in range(n)] for _ in range(n)])
    return a @ a.T + shift * np.eye(n)


def two_phase(np_, m, gen, fraction=0.5):
    c0 = random_spd(m, gen)
    c1 = random_spd(m, gen)
    phase = np.array([1 if gen.uniform(0.0, 1.0) < fraction else 0 for _ in range(np_)], dtype=np.uint8)
    return np.stack([c0, c1]), phase


def rand_vec(n, gen):
    return np.array([gen.uniform() for _ in range(n)])


def spec_index_to_full(k, dims):
    spec = list(dims)
    spec[-1] = dims[-1] // 2 + 1
    f = []
    for a in range(len(dims) - 1, -1, -1):
        f.append(k % spec[a])
        k //= spec[a]
    f = f[::-1]
    flat = 0
    for a in range(len(dims)):
        flat = flat * dims[a] + f[a]
    return flat


# ------------------------------------------------------------------ cases
def operator_cases():
    gen = MT19937_64(41)
    layouts = [((3, 4), (1.0, 1.3), "bilinear-quad"), ((4, 3), (1.2, 1.0), "two-triangles"),
               ((3, 3), (1.0, 0.8), "four-triangles-two-node"), ((3, 2, 4), (1.0, 1.1, 0.9), "trilinear-hex"),
               ((5, 4), (1.0, 1.0), "two-triangles"), ((4, 3, 3), (1.0, 1.0, 1.0), "trilinear-hex")]
    cases = []
    for dims, lengths, kind in layouts:
        d = len(dims)
        for c in (1, d):
            m = d if c == 1 else mandel(d)
            np_ = int(np.prod(dims))
            _, nn_pp, quads = stencil(dims, lengths, kind)
            nq = len(quads)
            cm, phase = two_phase(np_, m, gen)
            u = rand_vec(c * np_ * nn_pp, gen)
            s = rand_vec(np_ * nq * m, gen)
            tangent = cm[np.repeat(phase, nq)]
            K = dense_operator(dims, lengths, kind, c, tangent)
            D, quads = dense_gradient(dims, lengths, kind, c)
            W = dense_weights(quads, np_, m)
            s_planar = s.reshape(np_ * nq, m).T.ravel()
            cases.append(dict(meta=dict(dims=dims, lengths=lengths, stencil=kind, c=c),
                              cmats=cm, phase=phase, u=u, s=s, Ku=K @ u,
                              grad=(D @ u).reshape(m, np_ * nq).T.copy(),
                              div=D.T @ W @ s_planar))
    return cases


def precond_cases():
    gen = MT19937_64(131)
    layouts = [((2, 2), (1.0, 1.0), "two-triangles"), ((3, 2), (1.2, 0.9), "bilinear-quad"),
               ((2, 2), (1.0, 0.8), "four-triangles-two-node"), ((2, 2, 2), (1.0, 1.1, 0.9), "trilinear-hex"),
               ((4, 5), (1.0, 1.2), "two-triangles"), ((3, 4, 2), (1.0, 1.0, 1.0), "trilinear-hex")]
    cases = []
    for dims, lengths, kind in layouts:
        d = len(dims)
        for c in (1, d):
            m = d if c == 1 else mandel(d)
            np_ = int(np.prod(dims))
            _, nn_pp, quads = stencil(dims, lengths, kind)
            c_ref = random_spd(m, gen)
            tangent = np.repeat(c_ref[None], np_ * len(quads), axis=0)
            K = dense_operator(dims, lengths, kind, c, tangent)
            F = unitary_dft(dims)
            bdim = c * nn_pp
            nf = int(np.prod(dims[:-1])) * (dims[-1] // 2 + 1)
            blocks = np.zeros((nf, bdim, bdim), dtype=complex)
            for a in range(bdim):
                for b in range(bdim):
                    hat = F @ K[a * np_:(a + 1) * np_, b * np_:(b + 1) * np_] @ F.conj().T
                    for k in range(nf):
                        full = spec_index_to_full(k, dims)
                        blocks[k, a, b] = hat[full, full]
            r = rand_vec(c * np_ * nn_pp, gen).reshape(c, -1)
            r -= r.mean(axis=1, keepdims=True)
            r = r.ravel()
            z = dense_pinv(K) @ r
            cases.append(dict(meta=dict(dims=dims, lengths=lengths, stencil=kind, c=c),
                              c_ref=c_ref, blocks=blocks, r=r, z=z))
    return cases


def pcg_cases():
    """Dense fluctuation-space solve (test_solver.cpp:82-103) on small grids."""
    gen = MT19937_64(223)
    layouts = [((3, 3), (1.0, 1.0), "two-triangles", 2), ((6, 5), (1.0, 1.0), "two-triangles", 1),
               ((4, 4, 3), (1.0, 1.0, 1.0), "trilinear-hex", 1), ((3, 3, 4), (1.0, 1.0, 1.0), "trilinear-hex", 3)]
    cases = []
    for dims, lengths, kind, c in layouts:
        d = len(dims)
        m = d if c == 1 else mandel(d)
        np_ = int(np.prod(dims))
        _, _, quads = stencil(dims, lengths, kind)
        nq = len(quads)
        cm, phase = two_phase(np_, m, gen)
        tangent = cm[np.repeat(phase, nq)]
        w = quads[0][0]
        c_ref = (tangent * w).sum(axis=0) / float(np.prod(lengths))
        s = rand_vec(np_ * nq * m, gen)
        D, quads = dense_gradient(dims, lengths, kind, c)
        W = dense_weights(quads, np_, m)
        b = -(D.T @ W @ s.reshape(np_ * nq, m).T.ravel())
        K = dense_operator(dims, lengths, kind, c, tangent)
        x = dense_pinv(K) @ b
        cases.append(dict(meta=dict(dims=dims, lengths=lengths, stencil=kind, c=c),
                          cmats=cm, phase=phase, c_ref=c_ref, b=b, x=x))
    return cases


def save(name, cases):
    arrays, metas = {}, []
    for i, case in enumerate(cases):
        metas.append(case.pop("meta"))
        for k, v in case.items():
            arrays[f"case{i}_{k}"] = np.asarray(v)
    arrays["manifest"] = np.array(json.dumps(metas))
    np.savez_compressed(os.path.join(HERE, name), **arrays)


def load(name):
    z = np.load(os.path.join(HERE, name))
    metas = json.loads(str(z["manifest"]))
    out = []
    for i, meta in enumerate(metas):
        case = dict(meta=meta)
        prefix = f"case{i}_"
        for k in z.files:
            if k.startswith(prefix):
                case[k[len(prefix):]] = z[k]
        out.append(case)
    return out


if __name__ == "__main__":
    gen = MT19937_64(5489)
    for _ in range(9999):
        gen()
    assert gen() == 9981545732273789042, "mt19937_64 known-answer failed"
    save("operators.npz", operator_cases())
    save("precond.npz", precond_cases())
    save("pcg.npz", pcg_cases())
    print("wrote", [f for f in os.listdir(HERE) if f.endswith(".npz")])
