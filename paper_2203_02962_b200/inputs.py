"""Seeded synthetic inputs for the five BASELINE.json configurations.

No dataset ships with the reference (the paper's SEM steel image is not in
this container and BASELINE.json names no suite), so the microstructures are
generated here, following SURVEY.md section 8(d):

  * RNG: std::mt19937_64(seed), u = (gen() >> 11) 2^-53 (the convention of
    proj/tests/support/oracles.hpp:154-160 and proj/src/microstructure.cpp:75-90);
  * inclusion membership tested at pixel centres (i + 1/2) h
    (proj/src/microstructure.cpp:10-14) with the periodic minimum image;
  * non-overlap by random sequential addition with rejection;
  * the Gaussian random field of c4 is white noise (Box-Muller on the same
    stream) filtered by exp(-(2 pi |f|)^2 l^2 / 4) and thresholded at the
    exact median.

Phase maps are flat uint8 arrays in row-major pixel order, the raw format of
proj/src/io.cpp:65-86, so the oracle and the GPU consume identical bytes.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 2203020

# The uniform stream (std::mt19937_64 + (gen() >> 11) 2^-53) comes from a C
# function `fn(seed, n, lo, hi, double* out)`: the product library's
# homfe_random_uniform by default. The CPU baseline arm of bench.py loads this
# module by path (no package import) and points it at the oracle's identical
# or_uniform, so that process never maps libhomfe_gpu.so.
_uniform_fn = None


def set_uniform_source(fn):
    global _uniform_fn
    _uniform_fn = fn


def uniform(seed, n, lo=0.0, hi=1.0):
    global _uniform_fn
    if _uniform_fn is None:
        from ._native import lib
        _uniform_fn = lib.homfe_random_uniform
    out = np.zeros(int(n))
    _uniform_fn(C.c_uint64(seed), C.c_int64(int(n)), C.c_double(lo), C.c_double(hi),
                out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def normal(seed, n):
    """Standard normals by Box-Muller on consecutive uniform pairs of the same
    stream (out[2i] = r cos, out[2i+1] = r sin)."""
    n = int(n)
    u = uniform(seed, 2 * ((n + 1) // 2))
    r = np.sqrt(-2.0 * np.log1p(-u[0::2]))
    t = 2.0 * math.pi * u[1::2]
    out = np.empty(2 * r.size)
    out[0::2] = r * np.cos(t)
    out[1::2] = r * np.sin(t)
    return out[:n]


def isotropic_stiffness(bulk, shear, dim):
    """3K P_vol + 2G P_dev in Mandel notation (mandel.cpp:114-134; plane
    strain in 2-D: the in-plane block of the 3-D tensor)."""
    vol = np.zeros((6, 6))
    vol[:3, :3] = 1.0
    pv = vol / 3.0
    pd = np.eye(6) - pv
    m3 = (3.0 * bulk) * pv + (2.0 * shear) * pd
    if dim == 3:
        return m3
    return m3[np.ix_([0, 1, 5], [0, 1, 5])].copy()


def youngs_to_bulk_shear(E, nu):
    return E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def _paint_ball(phase, dims, centre, radius):
    """Set phase 1 on pixels whose centre lies within `radius` (pixel units) of
    `centre` under the periodic minimum image; returns the newly set count."""
    d = len(dims)
    r = radius
    axes = []
    for a in range(d):
        lo = int(math.floor(centre[a] - 0.5 - r)) - 1
        hi = int(math.ceil(centre[a] - 0.5 + r)) + 1
        idx = np.arange(lo, hi + 1)
        dist = (idx + 0.5) - centre[a]
        axes.append((idx % dims[a], dist))
    grids = np.meshgrid(*[a[1] for a in axes], indexing="ij", sparse=True)
    inside = sum(g * g for g in grids) <= r * r
    idx = np.ix_(*[a[0] for a in axes])
    view = phase[idx]
    new = int(np.count_nonzero(inside & (view == 0)))
    view[inside] = 1
    phase[idx] = view
    return new


def rsa_balls(dims, radius, seed, count=None, fraction=None, max_tries=2_000_000):
    """Non-overlapping periodic balls (centre distance >= 2 r) by random
    sequential addition, until `count` balls are placed or the painted pixel
    fraction reaches `fraction`. Centres are drawn in unit-cell coordinates, so
    a grid refinement with radius scaled by N reproduces the same geometry."""
    d = len(dims)
    dims_f = np.asarray(dims, dtype=float)
    phase = np.zeros(dims, dtype=np.uint8)
    centres = np.zeros((0, d))
    chunk = 3 * 65536
    stream = uniform(seed, chunk)
    block = 0
    k = 0
    tries = 0
    painted = 0
    total = float(np.prod(dims))
    while True:
        if count is not None and centres.shape[0] >= count:
            break
        if fraction is not None and painted / total >= fraction:
            break
        if tries >= max_tries:
            raise RuntimeError("rsa: could not place inclusions")
        if k + d > stream.size:
            block += 1
            stream = uniform(seed + 7919 * block, chunk)
            k = 0
        cu = stream[k:k + d]
        k += d
        tries += 1
        if centres.shape[0]:
            dd = np.abs(centres - cu)
            dd = np.minimum(dd, 1.0 - dd) * dims_f
            if np.min(np.sum(dd * dd, axis=1)) < (2 * radius) ** 2:
                continue
        centres = np.vstack([centres, cu])
        painted += _paint_ball(phase, dims, cu * dims_f, radius)
    return phase.ravel(), centres


def grf_threshold(dims, corr_len, seed):
    """Thresholded Gaussian random field, volume fraction exactly 1/2."""
    n = int(np.prod(dims))
    noise = normal(seed, n).reshape(dims)
    spec = np.fft.rfftn(noise)
    del noise
    freqs = [np.fft.fftfreq(dims[a]) for a in range(len(dims) - 1)] + [np.fft.rfftfreq(dims[-1])]
    f2 = sum(np.meshgrid(*[f * f for f in freqs], indexing="ij", sparse=True))
    spec *= np.exp(-(2 * math.pi) ** 2 * f2 * corr_len ** 2 / 4.0)
    field_ = np.fft.irfftn(spec, s=dims, axes=tuple(range(len(dims)))).ravel()
    del spec
    med = np.partition(field_, n // 2)[n // 2]
    return (field_ >= med).astype(np.uint8)


@dataclass
class Config:
    name: str
    dims: tuple
    stencil: str
    thermal: bool
    materials: list            # per phase: ("kappa", k) or ("E_nu", E, nu)
    load: tuple
    reference: str             # "explicit" | "volume-mean" | "identity-scaled"
    reference_phase: int = 0   # explicit reference = this phase's tangent
    eta_cg: float = 1e-8
    eta_newton: float = 1e-5
    micro: dict = field(default_factory=dict)
    gpus: tuple = (1,)

    @property
    def dim(self):
        return len(self.dims)

    @property
    def components(self):
        return 1 if self.thermal else self.dim

    @property
    def num_pixels(self):
        return int(np.prod(self.dims))

    @property
    def dof(self):
        return self.components * self.num_pixels

    def tangents(self):
        out = []
        for mat in self.materials:
            if mat[0] == "kappa":
                out.append(mat[1] * np.eye(self.dim))
            else:
                K, G = youngs_to_bulk_shear(mat[1], mat[2])
                out.append(isotropic_stiffness(K, G, self.dim))
        return np.stack(out)

    def phases(self):
        kind = self.micro["kind"]
        seed = self.micro.get("seed", BASE_SEED)
        if kind == "balls":
            ph, _ = rsa_balls(self.dims, self.micro["radius"], seed, count=self.micro.get("count"),
                              fraction=self.micro.get("fraction"))
            return ph
        if kind == "grf":
            return grf_threshold(self.dims, self.micro["corr_len"], seed)
        raise ValueError(kind)

    def reference_matrix(self):
        return self.tangents()[self.reference_phase] if self.reference == "explicit" else None


SQRT2 = math.sqrt(2.0)


def config(name, n=None, contrast=None):
    """The BASELINE.json configurations c1..c5."""
    if name == "c1":
        return Config("c1", (256, 256), "two-triangles", True, [("kappa", 1.0), ("kappa", 10.0)], (1.0, 0.0),
                      "explicit", 0, 1e-8,
                      micro=dict(kind="balls", radius=12.0, count=20, seed=BASE_SEED + 1))
    if name == "c2":
        return Config("c2", (128, 128, 128), "trilinear-hex", True, [("kappa", 1.0), ("kappa", 100.0)],
                      (1.0, 0.0, 0.0), "volume-mean", 0, 1e-8,
                      micro=dict(kind="balls", radius=8.0, fraction=0.25, seed=BASE_SEED + 2))
    if name == "c3":
        n = n or 256
        return Config("c3", (n, n, n), "trilinear-hex", False, [("E_nu", 1.0, 0.3), ("E_nu", 1000.0, 0.2)],
                      (0, 0, 0, 0, 0, SQRT2 * 0.01), "explicit", 0, 1e-6,
                      micro=dict(kind="balls", radius=10.0 * n / 256, fraction=0.30, seed=BASE_SEED + 3),
                      gpus=(1, 2, 4, 8))
    if name == "c4":
        n = n or 512
        return Config("c4", (n, n, n), "trilinear-hex", False, [("E_nu", 1.0, 0.3), ("E_nu", 1e4, 0.2)],
                      (0, 0, 0, 0, 0, SQRT2 * 0.01), "explicit", 0, 1e-6,
                      micro=dict(kind="grf", corr_len=16.0 * n / 512, seed=BASE_SEED + 4), gpus=(2, 4, 8))
    if name == "c5":
        n = n or 1024
        contrast = contrast or 1e3
        return Config(f"c5", (n, n), "two-triangles", True, [("kappa", 1.0), ("kappa", float(contrast))],
                      (1.0, 0.0), "volume-mean", 0, 1e-8,
                      micro=dict(kind="balls", radius=12.0 * n / 256, fraction=0.30, seed=BASE_SEED + 5),
                      gpus=(1, 8))
    raise ValueError(name)
