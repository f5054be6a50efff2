"""Slab-decomposed solves over several GPUs of one node.

One process per GPU (torchrun / torch.distributed for the rendezvous only).
Rank r of G owns planes (2-D: rows) [r n0/G, (r+1) n0/G) of axis 0. The library's slab
context (homfe_gpu_create_dist) does the data-path exchanges itself with NCCL
over NVLink / NVSwitch:

  * K p: one halo plane (row) from each neighbour (ring), before every stencil;
  * M^-1 (3-D): pass 1 (per plane) -> all-to-all of k1 rows -> pass 2 (per
    axis-0 pencil, spectral solve) -> all-to-all back -> pass 3 (per plane);
  * M^-1 (2-D, c5): 1-D r2c along axis 1 of the owned rows -> all-to-all of
    half-spectrum column chunks (ceil(nh / G) each, the last padded) -> 1-D
    c2c along axis 0 + spectral solve on the owned columns -> back;
  * p.Ap, r.z, means and norms: all-reductions of per-rank fixed-order sums.

The exchange patterns and the transposed layouts are restated in numpy in
`slab_layout` so that the host-side logic is testable on CPU (gloo).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _check, _dp, _f64, _native, Grid, NonConvergedError, ValidationError, mandel_dim
from ._native import lib


def slab_range(n0, rank, world):
    if n0 % world:
        raise ValidationError("slab mode: dims[0] must be divisible by the number of ranks")
    nz = n0 // world
    return rank * nz, nz


def halo_planes(n0, rank, world):
    """Global plane indices of the lower / upper halo of a slab: the reference's
    periodic wrap (grid.cpp:278-288) of z0 - 1 and z0 + nz."""
    z0, nz = slab_range(n0, rank, world)
    return (z0 - 1) % n0, (z0 + nz) % n0


class slab_layout:
    """Index maps of the fused passes' exchanged spectra (csrc/fftfused.cu,
    TLayout), restated for host-side tests."""

    TB = 16  # T2 row pitch granule
    TG = 4   # T column group

    def __init__(self, c, n0, n1, world):
        self.c, self.n0, self.n1, self.world = c, n0, n1, world
        self.nzl = n0 // world
        self.n1l = n1 // world
        self.P = n1 // 2 + 1
        self.nb = (self.P + self.TB - 1) // self.TB
        self.ng = (self.P + self.TG - 1) // self.TG

    def chunk_t(self):
        return self.c * self.n1l * self.ng * self.nzl * self.TG

    def chunk_t2(self):
        return self.c * self.nzl * self.n1l * self.nb * self.TB

    def t(self, peer, comp, k1l, k2, i0l):
        return ((((peer * self.c + comp) * self.n1l + k1l) * self.ng + k2 // self.TG) * (self.nzl * self.TG)
                + i0l * self.TG + k2 % self.TG)

    def t2(self, peer, comp, i0l, k1l, k2):
        return (((peer * self.c + comp) * self.nzl + i0l) * self.n1l + k1l) * (self.nb * self.TB) + k2

    @staticmethod
    def pull_offset(me, q, chunk):
        """Peer pull (context.cu setup_peers): rank `me` reads source q's
        element t(q, ...) at q's own send buffer + (me - q) * chunk + t(q, ...),
        i.e. q's send-side chunk addressed to `me`."""
        return (me - q) * chunk


class slab_layout_2d:
    """2-D row slabs (csrc/context.cu, d == 2 slab spectra): the half
    spectrum's nh = n1/2 + 1 columns are split into G chunks of
    nhl = ceil(nh / G) (the last one zero-padded); S[c][i0l][k1 < G nhl] on the
    row owner, W[c][i0][k1l] on the column owner (k1 = owner * nhl + k1l)."""

    def __init__(self, c, n0, n1, world):
        self.c, self.n0, self.n1, self.world = c, n0, n1, world
        self.nzl = n0 // world
        self.nh = n1 // 2 + 1
        self.nhl = (self.nh + world - 1) // world

    def owner(self, k1):
        return k1 // self.nhl

    def s_index(self, comp, i0l, k1):
        return (comp * self.nzl + i0l) * (self.world * self.nhl) + k1

    def w_index(self, comp, i0, k1l):
        return (comp * self.n0 + i0) * self.nhl + k1l

    def valid(self, k1):
        return k1 < self.nh


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    _check(lib.homfe_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def sim_group_id(group):
    """Id blob selecting the in-process slab transport (host barriers and
    device-to-device copies between the W contexts of one process on one
    GPU): validates the multi-rank layouts without NCCL. Test use only."""
    return b"HBSIMGRP" + int(group).to_bytes(8, "little") + bytes(112)


class SlabContext:
    """Device context for one slab (wraps homfe_gpu_create_dist)."""

    def __init__(self, grid: Grid, components, rank, world, nccl_id: bytes, device=0):
        desc = _native.GridDesc()
        from . import STENCILS
        desc.dim = grid.dim
        desc.stencil = STENCILS[grid.stencil]
        for a in range(3):
            desc.dims[a] = grid.dims[a] if a < grid.dim else 1
            desc.lengths[a] = grid.lengths[a] if a < grid.dim else 1.0
        desc.components = components
        desc.device = device
        idb = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        _check(lib.homfe_gpu_create_dist(C.byref(desc), rank, world, C.cast(idb, C.c_void_p), C.byref(h)))
        self.h = h
        self.grid, self.c, self.rank, self.world = grid, components, rank, world
        self.m = grid.dim if components == 1 else mandel_dim(grid.dim)
        self.z0, self.nz = slab_range(grid.dims[0], rank, world)
        self.n_local = self.nz * int(np.prod(grid.dims[1:]))

    @property
    def transport(self):
        """'single', 'all_to_all' (NCCL exchanges) or 'peer_pull' (passes 2/3
        and the K halo read the peers' fields in place; HOMFE_P2P=0 disables)."""
        k = C.c_int32()
        _check(lib.homfe_gpu_slab_transport(self.h, C.byref(k)))
        return ("single", "all_to_all", "peer_pull")[k.value]

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib.homfe_gpu_destroy(h)
            self.h = None

    def set_material(self, cmats, local_phase):
        cm = _f64(np.asarray(cmats).reshape(-1, self.m, self.m).transpose(0, 2, 1))
        ph = np.ascontiguousarray(local_phase, dtype=np.uint8).ravel()
        if ph.size != self.n_local:
            raise ValidationError("slab mode: phase slab has the wrong size")
        _check(lib.homfe_gpu_set_material(self.h, cm.shape[0], _dp(cm), ph.ctypes.data_as(C.POINTER(C.c_uint8))))

    def apply_K(self, u_local):
        u = _f64(u_local).reshape(self.c, self.n_local)
        out = np.zeros_like(u)
        _check(lib.homfe_gpu_apply_K(self.h, _dp(u), _dp(out)))
        return out

    def set_reference(self, c_ref):
        cr = _f64(np.asarray(c_ref).T)
        _check(lib.homfe_gpu_set_reference(self.h, _dp(cr)))

    def apply_minv(self, r_local):
        r = _f64(r_local).reshape(self.c, self.n_local)
        out = np.zeros_like(r)
        _check(lib.homfe_gpu_apply_minv(self.h, _dp(r), _dp(out)))
        return out

    def solve(self, e, cfg, warm_local=None):
        e = _f64(e).ravel()
        u = np.zeros((self.c, self.n_local))
        avg = np.zeros(self.m)
        rep = _native.Report()
        warm = _f64(warm_local).reshape(self.c, self.n_local) if warm_local is not None else None
        code = lib.homfe_gpu_solve(self.h, _dp(e), C.byref(cfg), _dp(warm), _dp(u), _dp(avg), C.byref(rep))
        if code != _native.NONCONVERGED:
            _check(code)
        from . import _report_dict
        return dict(converged=bool(rep.converged), u=u, average_stress=avg, report=_report_dict(rep))
