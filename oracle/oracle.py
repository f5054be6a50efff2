"""ctypes wrapper of the CPU oracle (``oracle/_build/libhomfe_oracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs, never by the
product package. The oracle restates the reference hot path
(proj/src/{grid,operators,fields,precond,solver}.cpp) on the CPU; see
``oracle/homfe_oracle.cpp`` for the file:line map.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libhomfe_oracle.so")

STENCILS = {
    "bilinear-quad": 0,
    "two-triangles": 1,
    "four-triangles-two-node": 2,
    "trilinear-hex": 3,
}


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


class _Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("stencil", C.c_int32),
                ("dims", C.c_int64 * 3), ("lengths", C.c_double * 3)]


class _Cfg(C.Structure):
    _fields_ = [("eta_newton", C.c_double), ("eta_cg", C.c_double),
                ("max_newton", C.c_int32), ("max_cg", C.c_int32),
                ("reassembly_threshold", C.c_double), ("criterion", C.c_int32),
                ("policy", C.c_int32), ("policy_scale", C.c_double),
                ("policy_matrix", C.POINTER(C.c_double))]


class _Step(C.Structure):
    _fields_ = [("cg_iterations", C.c_int32), ("residual_initial", C.c_double),
                ("residual_final", C.c_double), ("increment_rel", C.c_double),
                ("precond_reassembled", C.c_int32)]


class _Report(C.Structure):
    _fields_ = [("n_steps", C.c_int32), ("steps", _Step * 32), ("cause", C.c_int32),
                ("converged", C.c_int32), ("assemblies", C.c_int32),
                ("seconds_cg", C.c_double), ("seconds_total", C.c_double),
                ("seconds_assembly", C.c_double)]


def build(force=False):
    """Compile the oracle with its Makefile (gcc only, no GPU)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(os.path.join(HERE, f)) for f in ("homfe_oracle.cpp", "homfe_oracle.h")):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
        _lib.or_precond_destroy.restype = None
    return _lib


def _ptr(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


def _check(code):
    if code != 0:
        raise OracleError(code, lib().or_last_error().decode())


class Grid:
    """Periodic grid descriptor (mirrors the reference ``Grid``/``GridLayout``)."""

    def __init__(self, dims, lengths, stencil):
        self.dims = tuple(int(d) for d in dims)
        self.lengths = tuple(float(x) for x in lengths)
        self.stencil = stencil
        self.dim = len(self.dims)
        g = _Grid()
        g.dim = self.dim
        g.stencil = STENCILS[stencil]
        for a in range(3):
            g.dims[a] = self.dims[a] if a < self.dim else 1
            g.lengths[a] = self.lengths[a] if a < self.dim else 1.0
        self._g = g
        npix = C.c_int64()
        npp = C.c_int32()
        qpp = C.c_int32()
        strides = (C.c_int64 * 3)()
        w = (C.c_double * 8)()
        _check(lib().or_layout_info(C.byref(g), C.byref(npix), C.byref(npp), C.byref(qpp), strides, w))
        self.num_pixels = npix.value
        self.nodes_per_pixel = npp.value
        self.quads_per_pixel = qpp.value
        self.num_nodes = self.num_pixels * self.nodes_per_pixel
        self.num_quads = self.num_pixels * self.quads_per_pixel
        self.strides = tuple(strides[a] for a in range(self.dim))
        self.weights = np.array([w[q] for q in range(self.quads_per_pixel)])
        self.cell_volume = float(np.prod(self.lengths))

    @property
    def ref(self):
        return C.byref(self._g)

    def m(self, c):
        return self.dim if c == 1 else self.dim * (self.dim + 1) // 2

    def quad_weights(self):
        return np.tile(self.weights, self.num_pixels)

    def neighbor_table(self):
        n_off = C.c_int32()
        _check(lib().or_neighbor_table(self.ref, None, C.byref(n_off)))
        out = np.zeros((self.num_pixels, n_off.value), dtype=np.int64)
        _check(lib().or_neighbor_table(self.ref, _ptr(out, C.c_int64), C.byref(n_off)))
        return out

    def stencil_table(self):
        ne = np.zeros(self.quads_per_pixel, dtype=np.int32)
        _check(lib().or_stencil_table(self.ref, _ptr(ne, C.c_int32), None, None, None))
        tot = int(ne.sum())
        offs = np.zeros(tot, dtype=np.int32)
        nodes = np.zeros(tot, dtype=np.int32)
        dphi = np.zeros((tot, 3))
        _check(lib().or_stencil_table(self.ref, _ptr(ne, C.c_int32), _ptr(offs, C.c_int32),
                                      _ptr(nodes, C.c_int32), _ptr(dphi)))
        return ne, offs, nodes, dphi


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def isotropic_stiffness(bulk, shear, d):
    m = 3 if d == 2 else 6
    out = np.zeros(m * m)
    _check(lib().or_isotropic_stiffness(C.c_double(bulk), C.c_double(shear), C.c_int32(d), _ptr(out)))
    return out.reshape(m, m).T.copy()  # col-major -> matrix


def gradient(g, c, u):
    u = _f64(u).ravel()
    out = np.zeros(g.num_quads * g.m(c))
    _check(lib().or_gradient(g.ref, C.c_int32(c), _ptr(u), _ptr(out)))
    return out.reshape(g.num_quads, g.m(c))


def divergence(g, c, s, weighted=True):
    s = _f64(s).ravel()
    out = np.zeros(c * g.num_nodes)
    _check(lib().or_divergence(g.ref, C.c_int32(c), _ptr(s), C.c_int32(int(weighted)), _ptr(out)))
    return out


def apply_tangent(g, c, tangent, u, weighted=True):
    """tangent: (num_quads, m, m) matrices (stored column-major as the reference)."""
    m = g.m(c)
    t = _f64(np.asarray(tangent).reshape(-1, m, m).transpose(0, 2, 1)).ravel()
    u = _f64(u).ravel()
    out = np.zeros(c * g.num_nodes)
    _check(lib().or_apply_tangent(g.ref, C.c_int32(c), _ptr(t), _ptr(u), C.c_int32(int(weighted)), _ptr(out)))
    return out


def _cmat(cmats, m):
    return _f64(np.asarray(cmats).reshape(-1, m, m).transpose(0, 2, 1)).ravel()


def apply_phase(g, c, cmats, phase, u, weighted=True):
    m = g.m(c)
    cm = _cmat(cmats, m)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    u = _f64(u).ravel()
    out = np.zeros(c * g.num_nodes)
    _check(lib().or_apply_phase(g.ref, C.c_int32(c), C.c_int32(cm.size // (m * m)), _ptr(cm),
                                _ptr(ph, C.c_uint8), _ptr(u), C.c_int32(int(weighted)), _ptr(out)))
    return out


def apply_reference(g, c, c_ref, u, weighted=True):
    m = g.m(c)
    cr = _cmat(c_ref, m)
    u = _f64(u).ravel()
    out = np.zeros(c * g.num_nodes)
    _check(lib().or_apply_reference(g.ref, C.c_int32(c), _ptr(cr), _ptr(u), C.c_int32(int(weighted)), _ptr(out)))
    return out


def fft_forward(x):
    x = _f64(x)
    dims = np.array(x.shape, dtype=np.int64)
    spec = list(x.shape)
    spec[-1] = spec[-1] // 2 + 1
    out = np.zeros(int(np.prod(spec)) * 2)
    _check(lib().or_fft_forward(C.c_int32(x.ndim), _ptr(dims, C.c_int64), _ptr(x), _ptr(out)))
    return out.view(np.complex128).reshape(spec)


def fft_inverse(X, shape):
    X = np.ascontiguousarray(X, dtype=np.complex128)
    dims = np.array(shape, dtype=np.int64)
    out = np.zeros(int(np.prod(shape)))
    _check(lib().or_fft_inverse(C.c_int32(len(shape)), _ptr(dims, C.c_int64),
                                _ptr(X.view(np.float64)), _ptr(out)))
    return out.reshape(shape)


class Preconditioner:
    """Impulse-probed, FFT-diagonalised, pseudo-inverted reference operator."""

    def __init__(self, g, c_ref, c, weighted=True, invert=True, symbol=None, exact=False):
        """exact=True: blocks from the long-double exact symbol
        (or_precond_exact) instead of the reference's impulse probing."""
        h = C.c_void_p()
        if exact:
            m = g.m(c)
            cr = _cmat(c_ref, m)
            _check(lib().or_precond_exact(g.ref, _ptr(cr), C.c_int32(c), C.c_int32(int(weighted)),
                                          C.c_int32(int(invert)), C.byref(h)))
        elif symbol is not None:
            sym = np.ascontiguousarray(symbol, dtype=np.complex128)
            _check(lib().or_precond_from_symbol(g.ref, C.c_int32(c), _ptr(sym.view(np.float64)),
                                                C.c_int32(int(weighted)), C.byref(h)))
        else:
            m = g.m(c)
            cr = _cmat(c_ref, m)
            _check(lib().or_precond_assemble(g.ref, _ptr(cr), C.c_int32(c), C.c_int32(int(weighted)),
                                             C.c_int32(int(invert)), C.byref(h)))
        self._h = h
        self.grid = g
        self.c = c

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().or_precond_destroy(self._h)
            self._h = None

    def blocks(self):
        nf = C.c_int64()
        bd = C.c_int32()
        _check(lib().or_precond_blocks(self._h, C.byref(nf), C.byref(bd), None))
        out = np.zeros(nf.value * bd.value * bd.value * 2)
        _check(lib().or_precond_blocks(self._h, C.byref(nf), C.byref(bd), _ptr(out)))
        # (nf, col, row) -> (nf, row, col)
        return out.view(np.complex128).reshape(nf.value, bd.value, bd.value).transpose(0, 2, 1)

    def apply(self, r):
        r = _f64(r).ravel()
        out = np.zeros_like(r)
        _check(lib().or_precond_apply(self.grid.ref, self._h, _ptr(r), _ptr(out)))
        return out


def pcg(g, c, cmats, phase, precond, b, eta, it_max):
    m = g.m(c)
    cm = _cmat(cmats, m)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    b = _f64(b).ravel()
    x = np.zeros_like(b)
    it = C.c_int32()
    conv = C.c_int32()
    hist = np.zeros(it_max + 1)
    _check(lib().or_pcg(g.ref, C.c_int32(c), C.c_int32(cm.size // (m * m)), _ptr(cm), _ptr(ph, C.c_uint8),
                        precond._h, _ptr(b), C.c_double(eta), C.c_int32(it_max), _ptr(x),
                        C.byref(it), _ptr(hist), C.byref(conv)))
    return dict(x=x, iterations=it.value, history=hist[: it.value + 1], converged=bool(conv.value))


def pcg_timed(g, c, cmats, phase, precond, b, iterations):
    """Fixed-iteration PCG returning (x, per-iteration seconds) (timing only)."""
    m = g.m(c)
    cm = _cmat(cmats, m)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    b = _f64(b).ravel()
    x = np.zeros_like(b)
    t = np.zeros(iterations)
    _check(lib().or_pcg_timed(g.ref, C.c_int32(c), C.c_int32(cm.size // (m * m)), _ptr(cm), _ptr(ph, C.c_uint8),
                              precond._h, _ptr(b), C.c_int32(iterations), _ptr(x), _ptr(t)))
    return x, t


def uniform_source():
    """The oracle's or_uniform as a C function pointer with argtypes (same
    stream as the product's homfe_random_uniform)."""
    fn = lib().or_uniform
    fn.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, C.POINTER(C.c_double)]
    fn.restype = C.c_int
    return fn


POLICIES = {"identity": 0, "identity-scaled": 0, "volume-mean": 1, "explicit": 2}


def newton_solve(g, thermal, cmats, phase, e, eta_newton=1e-5, eta_cg=1e-5, max_newton=25,
                 max_cg=20000, reassembly_threshold=0.1, criterion="strain", reference="volume-mean",
                 reference_scale=1.0, reference_matrix=None, warm_u=None):
    d = g.dim
    c = 1 if thermal else d
    m = g.m(c)
    cm = _cmat(cmats, m)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    e = _f64(e).ravel()
    cfg = _Cfg()
    cfg.eta_newton, cfg.eta_cg = eta_newton, eta_cg
    cfg.max_newton, cfg.max_cg = max_newton, max_cg
    cfg.reassembly_threshold = reassembly_threshold
    cfg.criterion = 0 if criterion == "strain" else 1
    cfg.policy = POLICIES[reference]
    cfg.policy_scale = reference_scale
    pm = None
    if reference_matrix is not None:
        pm = _cmat(reference_matrix, m)
        cfg.policy_matrix = _ptr(pm)
    u = np.zeros(c * g.num_nodes)
    avg = np.zeros(m)
    rep = _Report()
    wu = _f64(warm_u).ravel() if warm_u is not None else None
    code = lib().or_newton_solve(g.ref, C.c_int32(int(thermal)), C.c_int32(cm.size // (m * m)), _ptr(cm),
                                 _ptr(ph, C.c_uint8), _ptr(e), C.byref(cfg), _ptr(wu), _ptr(u), _ptr(avg),
                                 C.byref(rep))
    if code not in (0, 3):
        _check(code)
    steps = [dict(cg_iterations=rep.steps[i].cg_iterations, residual_initial=rep.steps[i].residual_initial,
                  residual_final=rep.steps[i].residual_final, increment_rel=rep.steps[i].increment_rel,
                  precond_reassembled=bool(rep.steps[i].precond_reassembled))
             for i in range(min(rep.n_steps, 32))]
    return dict(u=u, average_stress=avg, converged=bool(rep.converged),
                cause=["converged", "cg-stall", "newton-cap"][rep.cause], steps=steps,
                assemblies=rep.assemblies, seconds_cg=rep.seconds_cg, seconds_total=rep.seconds_total)


class _Material(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tangent", C.c_double * 36), ("bulk", C.c_double), ("shear", C.c_double),
                ("yield_stress", C.c_double), ("hardening", C.c_double)]


def material(kind, tangent=None, bulk=0.0, shear=0.0, yield_stress=0.0, hardening=0.0):
    """Catalog entry: kind "linear" (m x m tangent) or "j2" (material.cpp:37-101)."""
    mt = _Material()
    mt.kind = 0 if kind == "linear" else 1
    if tangent is not None:
        t = np.asarray(tangent, dtype=np.float64)
        flat = t.T.ravel()  # column-major
        for i, v in enumerate(flat):
            mt.tangent[i] = v
    mt.bulk, mt.shear, mt.yield_stress, mt.hardening = bulk, shear, yield_stress, hardening
    return mt


def j2_evaluate(d, bulk, shear, yield_stress, hardening, eps, g):
    """MaterialModel::evaluate for J2 (material.cpp:122-226): (sigma, tangent, g_new)."""
    m = 6 if d == 3 else 3
    eps = _f64(eps).ravel()
    g = _f64(g).ravel()
    sig = np.zeros(m)
    tan = np.zeros(m * m)
    gn = np.zeros(7)
    _check(lib().or_j2_evaluate(C.c_int32(d), C.c_double(bulk), C.c_double(shear), C.c_double(yield_stress),
                                C.c_double(hardening), _ptr(eps), _ptr(g), _ptr(sig), _ptr(tan), _ptr(gn)))
    return sig, tan.reshape(m, m).T.copy(), gn


class PrecondManager:
    """PrecondManager (solver.hpp:105-129) shared by the steps of a load
    program (solver.cpp:306-318)."""

    def __init__(self):
        lib().or_manager_create.restype = C.c_void_p
        self._h = C.c_void_p(lib().or_manager_create())

    def __del__(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().or_manager_destroy.argtypes = [C.c_void_p]
            lib().or_manager_destroy.restype = None
            lib().or_manager_destroy(self._h)
            self._h = None

    @property
    def assemblies(self):
        lib().or_manager_assemblies.argtypes = [C.c_void_p]
        return lib().or_manager_assemblies(self._h)


def newton_solve_models(g, thermal, models, phase, e, g0=None, eta_newton=1e-5, eta_cg=1e-5, max_newton=25,
                        max_cg=20000, reassembly_threshold=0.1, criterion="strain", reference="volume-mean",
                        reference_scale=1.0, reference_matrix=None, warm_u=None, manager=None):
    """Newton solve for a general (linear + J2) catalog with internal state;
    `manager`: a PrecondManager kept across calls (None: one per solve)."""
    d = g.dim
    c = 1 if thermal else d
    m = g.m(c)
    arr = (_Material * len(models))(*models)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    e = _f64(e).ravel()
    cfg = _Cfg()
    cfg.eta_newton, cfg.eta_cg = eta_newton, eta_cg
    cfg.max_newton, cfg.max_cg = max_newton, max_cg
    cfg.reassembly_threshold = reassembly_threshold
    cfg.criterion = 0 if criterion == "strain" else 1
    cfg.policy = POLICIES[reference]
    cfg.policy_scale = reference_scale
    pm = None
    if reference_matrix is not None:
        pm = _cmat(reference_matrix, m)
        cfg.policy_matrix = _ptr(pm)
    nq = g.quads_per_pixel * g.num_pixels
    width = 7 if any(mm.kind == 1 for mm in models) else 0
    g0a = _f64(g0).ravel() if g0 is not None else None
    gout = np.zeros(width * nq)
    u = np.zeros(c * g.num_nodes)
    avg = np.zeros(m)
    rep = _Report()
    wu = _f64(warm_u).ravel() if warm_u is not None else None
    args = (g.ref, C.c_int32(int(thermal)), C.c_int32(len(models)), arr, _ptr(ph, C.c_uint8), _ptr(g0a), _ptr(e),
            C.byref(cfg), _ptr(wu), _ptr(u), _ptr(gout) if width else None, _ptr(avg), C.byref(rep))
    if manager is None:
        code = lib().or_newton_solve_models(*args)
    else:
        code = lib().or_newton_solve_managed(*args, manager._h)
    if code not in (0, 3):
        _check(code)
    steps = [dict(cg_iterations=rep.steps[i].cg_iterations, residual_initial=rep.steps[i].residual_initial,
                  residual_final=rep.steps[i].residual_final, increment_rel=rep.steps[i].increment_rel,
                  precond_reassembled=bool(rep.steps[i].precond_reassembled))
             for i in range(min(rep.n_steps, 32))]
    return dict(u=u, average_stress=avg, internal=gout, converged=bool(rep.converged),
                cause=["converged", "cg-stall", "newton-cap"][rep.cause], steps=steps,
                assemblies=rep.assemblies)


def gamma_apply(g, c_ref, c, s):
    """projection.cpp:22-41: Gamma s with the unweighted reference blocks."""
    m = g.m(c)
    s = _f64(s).ravel()
    out = np.zeros(g.num_quads * m)
    cr = _cmat(c_ref, m)
    _check(lib().or_gamma_apply(g.ref, _ptr(cr), C.c_int32(c), _ptr(s), _ptr(out)))
    return out.reshape(g.num_quads, m)


def sb_newton_solve_models(g, thermal, models, phase, e, c_ref, g0=None, warm_strain=None, eta_newton=1e-5,
                           eta_cg=1e-5, max_newton=25, max_cg=20000):
    """sb_newton_solve (projection.cpp:93-185)."""
    d = g.dim
    c = 1 if thermal else d
    m = g.m(c)
    arr = (_Material * len(models))(*models)
    ph = np.ascontiguousarray(phase, dtype=np.uint8).ravel()
    e = _f64(e).ravel()
    cfg = _Cfg()
    cfg.eta_newton, cfg.eta_cg = eta_newton, eta_cg
    cfg.max_newton, cfg.max_cg = max_newton, max_cg
    cfg.reassembly_threshold = 0.1
    cr = _cmat(c_ref, m)
    nq = g.num_quads
    width = 7 if any(mm.kind == 1 for mm in models) else 0
    g0a = _f64(g0).ravel() if g0 is not None else None
    ws = _f64(warm_strain).ravel() if warm_strain is not None else None
    gout = np.zeros(width * nq)
    strain = np.zeros(nq * m)
    avg = np.zeros(m)
    rep = _Report()
    code = lib().or_sb_newton_solve(g.ref, C.c_int32(int(thermal)), C.c_int32(len(models)), arr,
                                    _ptr(ph, C.c_uint8), _ptr(g0a), _ptr(e), C.byref(cfg), _ptr(cr), _ptr(ws),
                                    _ptr(strain), _ptr(gout) if width else None, _ptr(avg), C.byref(rep))
    if code not in (0, 3):
        _check(code)
    steps = [dict(cg_iterations=rep.steps[i].cg_iterations, residual_initial=rep.steps[i].residual_initial,
                  residual_final=rep.steps[i].residual_final, increment_rel=rep.steps[i].increment_rel)
             for i in range(min(rep.n_steps, 32))]
    return dict(strain=strain.reshape(nq, m), internal=gout, average_stress=avg, converged=bool(rep.converged),
                cause=["converged", "cg-stall", "newton-cap"][rep.cause], steps=steps)


def eigenvalue_bounds(g, tangent, c_ref, c, pixel_constant=False):
    """eigenvalue_bounds + condition_estimate (spectral.cpp:33-127)."""
    m = g.m(c)
    t = np.ascontiguousarray(np.asarray(tangent, dtype=np.float64).transpose(0, 2, 1)).ravel()
    cr = _cmat(c_ref, m)
    lo = np.zeros(c * g.num_nodes)
    hi = np.zeros(c * g.num_nodes)
    cond = C.c_double()
    _check(lib().or_eigenvalue_bounds(g.ref, _ptr(t), C.c_int32(int(pixel_constant)), _ptr(cr), C.c_int32(c),
                                      _ptr(lo), _ptr(hi), C.byref(cond)))
    return lo, hi, cond.value


def volume_average(g, s):
    s = _f64(s)
    m = s.shape[-1]
    out = np.zeros(m)
    _check(lib().or_volume_average(g.ref, C.c_int32(m), _ptr(s.ravel()), _ptr(out)))
    return out


def weighted_dot(g, a, b):
    a = _f64(a)
    b = _f64(b)
    out = C.c_double()
    _check(lib().or_weighted_dot(g.ref, C.c_int32(a.shape[-1]), _ptr(a.ravel()), _ptr(b.ravel()), C.byref(out)))
    return out.value


def uniform(seed, n, lo=-1.0, hi=1.0):
    out = np.zeros(int(n))
    _check(lib().or_uniform(C.c_uint64(seed), C.c_int64(int(n)), C.c_double(lo), C.c_double(hi), _ptr(out)))
    return out


def set_threads(n):
    """Worker threads of the oracle's timing variant (1 = the reference's
    serial loop order, the default; bench.py --impl reference uses all host
    cores). Returns the previous setting."""
    global _threads
    prev = _threads
    lib().or_set_threads(C.c_int32(int(n)))
    _threads = int(n)
    return prev


_threads = 1
