"""B200-native PCG hot path of the FFT-preconditioned matrix-free FE
homogenization scheme (arXiv 2203.02962).

Python mirror of the reference module ``homfe._core``
(proj/src/bindings/module.cpp:148-390): same names, array shapes and error
types, backed by the CUDA C ABI in ``include/homfe_gpu.h``. Arrays use the
reference's layouts: nodal fields ``(components, num_nodes)``, quadrature
fields ``(num_quads, m)``, tangents ``(num_quads, m, m)``, phase maps flat
``uint8`` of length ``num_pixels``.

Deviations forced by the GPU design (documented in DESIGN.md):
  * operators act on pixel-constant linear tangents (a phase map plus a
    catalog of at most 256 m x m matrices) instead of arbitrary per-point
    TangentFields; ``apply_operator`` converts a pixel-constant tangent array;
  * J2 plasticity runs on the device with compact per-point tangents; the
    FourTrianglesTwoNode stencil uses the impulse-probed complex blocks; the
    strain-based scheme and spectral bounds are on the device too
    (SURVEY.md section 8(f) rows f1, f3, f4).
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _native
from ._native import lib

__all__ = [
    "Grid", "Material", "Preconditioner", "ValidationError", "NumericalSolverError", "NonConvergedError",
    "apply_operator", "apply_preconditioner", "assemble_preconditioner", "divergence_apply", "from_mandel",
    "gradient_apply", "isotropic_stiffness", "mandel_dim", "mandel_identity", "newton_solve", "to_mandel",
    "volume_average", "Solver", "pcg_solve",
]


class ValidationError(ValueError):
    """Invalid input (proj/include/homfe/common.hpp:15-18)."""


class NumericalSolverError(RuntimeError):
    """Numerical breakdown (proj/include/homfe/common.hpp:22-25)."""


class NonConvergedError(RuntimeError):
    """CG stall or Newton cap (CLI exit code 3, proj/tools/homog.cpp:23-26)."""


class DeviceError(RuntimeError):
    """CUDA / cuFFT failure."""


def _check(code):
    if code == _native.OK:
        return
    msg = lib.homfe_gpu_last_error().decode()
    raise {_native.VALIDATION: ValidationError, _native.NUMERICAL: NumericalSolverError,
           _native.NONCONVERGED: NonConvergedError}.get(code, DeviceError)(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


STENCILS = {"bilinear-quad": 0, "two-triangles": 1, "four-triangles-two-node": 2, "trilinear-hex": 3}


def mandel_dim(dim):
    if dim not in (2, 3):
        raise ValidationError(f"mandel: dimension must be 2 or 3, got {dim}")
    return dim * (dim + 1) // 2


def mandel_identity(dim):
    return np.eye(mandel_dim(dim))


_PAIRS = {2: [(0, 0), (1, 1), (0, 1)], 3: [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]}


def to_mandel(tensor):
    """proj/src/mandel.cpp:33-47."""
    t = np.asarray(tensor, dtype=float)
    d = t.shape[0]
    sym = 0.5 * (t + t.T)
    return np.array([sym[i, j] if i == j else math.sqrt(2.0) * sym[i, j] for i, j in _PAIRS[d]])


def from_mandel(v):
    """proj/src/mandel.cpp:49-70."""
    v = np.asarray(v, dtype=float)
    d = {3: 2, 6: 3}.get(v.size)
    if d is None:
        raise ValidationError("from_mandel: vector length must be 3 or 6")
    t = np.zeros((d, d))
    for a, (i, j) in enumerate(_PAIRS[d]):
        if i == j:
            t[i, j] = v[a]
        else:
            t[i, j] = t[j, i] = v[a] / math.sqrt(2.0)
    return t


def isotropic_stiffness(bulk, shear, dim):
    """3K P_vol + 2G P_dev in Mandel notation (proj/src/mandel.cpp:114-134)."""
    m = mandel_dim(dim)
    out = np.zeros(m * m)
    _check(lib.homfe_isotropic_stiffness(float(bulk), float(shear), int(dim), _dp(out)))
    return out.reshape(m, m).T.copy()


class Material:
    """Constitutive models of proj/include/homfe/material.hpp:36-69: linear
    (elastic / conductivity) and J2 plasticity (material.cpp:78-101,122-226)."""

    def __init__(self, tangent, thermal, dim, j2=None):
        self.tangent = np.array(tangent, dtype=float)
        self.thermal = thermal
        self.dim = dim
        self.j2 = j2  # (bulk, shear, yield_stress, hardening) or None

    @staticmethod
    def linear_elastic(stiffness):
        c = np.asarray(stiffness, dtype=float)
        if c.shape not in ((3, 3), (6, 6)):
            raise ValidationError("linear_elastic: stiffness must be 3x3 or 6x6")
        _check_spd(c, "linear_elastic")
        return Material(c, False, 2 if c.shape[0] == 3 else 3)

    @staticmethod
    def isotropic_elastic(bulk, shear, dim):
        return Material.linear_elastic(isotropic_stiffness(bulk, shear, dim))

    @staticmethod
    def conductivity(matrix):
        a = np.asarray(matrix, dtype=float)
        if a.shape not in ((2, 2), (3, 3)):
            raise ValidationError("conductivity: matrix must be 2x2 or 3x3")
        _check_spd(a, "conductivity")
        return Material(a, True, a.shape[0])

    @staticmethod
    def isotropic_conductivity(kappa, dim):
        if not kappa > 0.0:
            raise ValidationError("conductivity: kappa must be > 0")
        return Material.conductivity(kappa * np.eye(dim))

    @staticmethod
    def j2_plastic(bulk, shear, yield_stress, hardening, dim):
        if not (bulk > 0.0 and shear > 0.0 and yield_stress > 0.0):
            raise ValidationError("j2_plastic: K, G and tau_y0 must be > 0")
        if hardening < 0.0:
            raise ValidationError("j2_plastic: H must be >= 0")
        if dim not in (2, 3):
            raise ValidationError("j2_plastic: dimension must be 2 or 3")
        return Material(isotropic_stiffness(bulk, shear, dim), False, dim,
                        j2=(float(bulk), float(shear), float(yield_stress), float(hardening)))

    @property
    def nonlinear(self):
        return self.j2 is not None

    @property
    def flux_components(self):
        return self.dim if self.thermal else mandel_dim(self.dim)

    @property
    def internal_width(self):
        return 7 if self.j2 is not None else 0

    def model(self):
        """homfe_material catalog entry for the C ABI."""
        mm = _native.MaterialModel()
        if self.j2 is None:
            mm.kind = 0
            for i, v in enumerate(self.tangent.T.ravel()):
                mm.tangent[i] = v
        else:
            mm.kind = 1
            mm.bulk, mm.shear, mm.yield_stress, mm.hardening = self.j2
        return mm

    def evaluate(self, strain, internal=None):
        eps = np.asarray(strain, dtype=float)
        if eps.size != self.flux_components:
            raise ValidationError("evaluate: strain has wrong length")
        if not np.all(np.isfinite(eps)):
            raise NumericalSolverError("evaluate: non-finite strain input")
        if self.j2 is not None:
            raise ValidationError("evaluate: J2 is evaluated on the device inside the Newton solve")
        return self.tangent @ eps, self.tangent.copy(), np.zeros(0)


def _check_spd(a, what):
    scale = np.abs(a).max()
    if np.abs(a - a.T).max() > 1e-10 * scale:
        raise ValidationError(f"{what}: non-symmetric tangent rejected")
    try:
        np.linalg.cholesky(a)
    except np.linalg.LinAlgError:
        raise ValidationError(f"{what}: matrix must be positive definite") from None


class _Context:
    """One device context (grid + component count), owning device buffers."""

    def __init__(self, grid, components, device=0):
        desc = _native.GridDesc()
        n_gpus = getattr(grid, "n_gpus", 1)
        desc.dim = grid.dim
        desc.stencil = STENCILS[grid.stencil]
        for a in range(3):
            desc.dims[a] = grid.dims[a] if a < grid.dim else 1
            desc.lengths[a] = grid.lengths[a] if a < grid.dim else 1.0
        desc.components = components
        desc.device = device
        h = C.c_void_p()
        if n_gpus > 1:
            _check(lib.homfe_gpu_create_multi(C.byref(desc), int(n_gpus), C.byref(h)))
        else:
            _check(lib.homfe_gpu_create(C.byref(desc), C.byref(h)))
        self.h = h
        self.grid = grid
        self.c = components
        self.m = grid.dim if components == 1 else mandel_dim(grid.dim)
        self._material_key = None
        self._reference_key = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            lib.homfe_gpu_destroy(h)
            self.h = None

    def path(self):
        """Names of the kernels this context runs (homfe_gpu_path_info)."""
        f = C.c_int32()
        _check(lib.homfe_gpu_path_info(self.h, C.byref(f)))
        return {k for k, bit in _native.PATH_FLAGS.items() if f.value & bit}

    def set_material(self, cmats, phases):
        cm = _f64(np.asarray(cmats).reshape(-1, self.m, self.m).transpose(0, 2, 1))
        ph = np.ascontiguousarray(phases, dtype=np.uint8).ravel()
        key = (cm.tobytes(), ph.tobytes()) if ph.size <= 1 << 16 else None
        if key is not None and key == self._material_key:
            return
        self._material_key = None  # a failed upload leaves the context without a material
        _check(lib.homfe_gpu_set_material(self.h, cm.shape[0], _dp(cm),
                                          ph.ctypes.data_as(C.POINTER(C.c_uint8))))
        self._material_key = key

    def set_models(self, materials, phases):
        """General catalog (linear + J2): homfe_gpu_set_material_models."""
        ph = np.ascontiguousarray(phases, dtype=np.uint8).ravel()
        arr = (_native.MaterialModel * len(materials))(*[m.model() for m in materials])
        self._material_key = None
        _check(lib.homfe_gpu_set_material_models(self.h, len(materials), arr,
                                                 ph.ctypes.data_as(C.POINTER(C.c_uint8))))

    def set_reference(self, c_ref):
        cr = _f64(np.asarray(c_ref).T)
        key = cr.tobytes()
        if key == self._reference_key:
            return
        _check(lib.homfe_gpu_set_reference(self.h, _dp(cr)))
        self._reference_key = key


class Grid:
    """Periodic grid (proj/include/homfe/grid.hpp:75-129)."""

    def __init__(self, dims, lengths, stencil, n_gpus=1):
        """n_gpus > 1: one context over that many devices of this process
        (slab decomposition along axis 0, homfe_gpu_create_multi); linear
        solves, K, M^-1 and PCG take and return global fields."""
        dims = [int(x) for x in dims]
        self.n_gpus = int(n_gpus)
        lengths = [float(x) for x in lengths]
        if len(dims) != len(lengths):
            raise ValidationError("cell: dims and lengths must have equal rank")
        if len(dims) not in (2, 3):
            raise ValidationError(f"cell: dimension must be 2 or 3, got {len(dims)}")
        for a, (n, l) in enumerate(zip(dims, lengths)):
            if n < 2:
                raise ValidationError(f"cell.dims[{a}]: must be >= 2, got {n}")
            if not l > 0.0:
                raise ValidationError(f"cell.lengths[{a}]: must be > 0")
        if stencil not in STENCILS:
            raise ValidationError(f"stencil: unknown kind '{stencil}'")
        want = 3 if stencil == "trilinear-hex" else 2
        if len(dims) != want:
            raise ValidationError(f"stencil: {stencil} requires a {want}d cell, got {len(dims)}d")
        self.dims, self.lengths, self.stencil = tuple(dims), tuple(lengths), stencil
        self.dim = len(dims)
        self.num_pixels = int(np.prod(dims))
        self.nodes_per_pixel = 2 if stencil == "four-triangles-two-node" else 1
        self.quads_per_pixel = {"bilinear-quad": 4, "two-triangles": 2, "four-triangles-two-node": 4,
                                "trilinear-hex": 8}[stencil]
        self.num_nodes = self.num_pixels * self.nodes_per_pixel
        self.num_quads = self.num_pixels * self.quads_per_pixel
        self.cell_volume = float(np.prod(lengths))
        self._ctx = {}

    def quad_weights(self):
        vp = self.cell_volume / self.num_pixels
        return np.full(self.num_quads, vp / self.quads_per_pixel)

    def context(self, components):
        if components not in (1, self.dim):
            raise ValidationError("nodal field shape does not match layout")
        if components not in self._ctx:
            self._ctx[components] = _Context(self, components)
        return self._ctx[components]

    def index_maps(self):
        ctx = self.context(1)
        strides = np.zeros(3, dtype=np.int64)
        n_off = C.c_int32()
        _check(lib.homfe_gpu_index_maps(ctx.h, strides.ctypes.data_as(C.POINTER(C.c_int64)), None,
                                        C.byref(n_off)))
        nbr = np.zeros((self.num_pixels, n_off.value), dtype=np.int64)
        _check(lib.homfe_gpu_index_maps(ctx.h, None, nbr.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n_off)))
        return strides[: self.dim], nbr


def _nodal(grid, u):
    u = _f64(u)
    if u.ndim != 2 or u.shape[1] != grid.num_nodes:
        raise ValidationError("expected a (components, num_nodes) array")
    return u


def _quad(grid, s):
    s = _f64(s)
    if s.ndim != 2 or s.shape[0] != grid.num_quads:
        raise ValidationError("expected a (num_quads, components) array")
    return s


def gradient_apply(grid, u):
    """Symmetrized (or scalar) gradient at every quadrature point (operators.hpp:20-21)."""
    u = _nodal(grid, u)
    ctx = grid.context(u.shape[0])
    out = np.zeros((grid.num_quads, ctx.m))
    _check(lib.homfe_gpu_gradient(ctx.h, _dp(u), _dp(out)))
    return out


def divergence_apply(grid, s, weighted=True):
    """Weighted divergence D^T W s (operators.hpp:23-25)."""
    s = _quad(grid, s)
    m = s.shape[1]
    if m == grid.dim:
        c = 1
    elif m == mandel_dim(grid.dim):
        c = grid.dim
    else:
        raise ValidationError("quadrature field shape does not match layout")
    ctx = grid.context(c)
    out = np.zeros((c, grid.num_nodes))
    _check(lib.homfe_gpu_divergence(ctx.h, _dp(s), int(bool(weighted)), _dp(out)))
    return out


def _phases_from_tangent(grid, tangent):
    t = _f64(tangent)
    if t.ndim != 3 or t.shape[0] != grid.num_quads or t.shape[1] != t.shape[2]:
        raise ValidationError("expected a (num_quads, m, m) array")
    nq = grid.quads_per_pixel
    per_pixel = t.reshape(grid.num_pixels, nq, t.shape[1], t.shape[2])
    if not np.all(per_pixel == per_pixel[:, :1]):
        raise ValidationError("GPU operator requires a pixel-constant tangent")
    blocks = per_pixel[:, 0].reshape(grid.num_pixels, -1)
    uniq, inverse = np.unique(blocks, axis=0, return_inverse=True)
    if uniq.shape[0] > 256:
        raise ValidationError("GPU operator supports at most 256 distinct tangents")
    return uniq.reshape(-1, t.shape[1], t.shape[2]), inverse.astype(np.uint8).ravel()


def apply_operator(grid, tangent, u):
    """Fused matrix-free K u = D^T W C D u (operators.hpp:31-33). A
    pixel-constant tangent with at most 256 distinct blocks runs the phase-
    indexed fused kernels; any other TangentField (per-quadrature-point,
    non-symmetric, more than 256 blocks) runs gradient -> C_q -> weighted
    divergence on the device (operators.cpp:247-257)."""
    u = _nodal(grid, u)
    ctx = grid.context(u.shape[0])
    out = np.zeros_like(u)
    try:
        cmats, phases = _phases_from_tangent(grid, tangent)
    except ValidationError:
        t = _f64(tangent)
        if t.ndim != 3 or t.shape[0] != grid.num_quads or t.shape[1] != t.shape[2]:
            raise
        if t.shape[1] != ctx.m:
            raise ValidationError("tangent dimension does not match layout")
        blocks = np.ascontiguousarray(t.transpose(0, 2, 1))  # column-major blocks (fields.hpp:64-82)
        _check(lib.homfe_gpu_apply_tangent_field(ctx.h, _dp(blocks), _dp(u), _dp(out)))
        return out
    if cmats.shape[1] != ctx.m:
        raise ValidationError("tangent dimension does not match layout")
    ctx.set_material(cmats, phases)
    _check(lib.homfe_gpu_apply_K(ctx.h, _dp(u), _dp(out)))
    return out


class Preconditioner:
    """Inverted Fourier blocks of the reference operator (precond.hpp:28-79)."""

    def __init__(self, grid, c_ref, components, weighted=True):
        # unweighted blocks (projection.cpp:22-27): with equal Gauss weights
        # (all one-node stencils here) they are the weighted ones / w
        self.weighted = bool(weighted)
        self.grid = grid
        self.components = components
        self.c_ref = np.array(c_ref, dtype=float)
        ctx = grid.context(components)
        if self.c_ref.shape != (ctx.m, ctx.m):
            raise ValidationError("reference tangent has wrong dimension")
        ctx.set_reference(self.c_ref)
        self.block_dim = components * grid.nodes_per_pixel
        spec = list(grid.dims)
        spec[-1] = spec[-1] // 2 + 1
        self.num_frequencies = int(np.prod(spec))
        self.inverted = True

    def symbol(self):
        """K_ref_hat(xi), (num_frequencies, c, c), before inversion."""
        ctx = self.grid.context(self.components)
        ctx.set_reference(self.c_ref)
        bd = self.block_dim
        out = np.zeros(self.num_frequencies * bd * bd * 2)
        _check(lib.homfe_gpu_reference_blocks(ctx.h, _dp(out)))
        # column-major blocks (precond.hpp:38-45) -> (frequency, row, col)
        blocks = out.view(np.complex128).reshape(self.num_frequencies, bd, bd).transpose(0, 2, 1)
        return blocks if self.weighted else blocks / self.grid.quad_weights()[0]


def assemble_preconditioner(grid, c_ref, components, weighted=True):
    """assemble_reference + invert_blocks (precond.hpp:90-102)."""
    return Preconditioner(grid, c_ref, components, weighted)


def apply_preconditioner(grid, preconditioner, r):
    """M^-1 r (precond.hpp:104-106)."""
    r = _nodal(grid, r)
    if r.shape[0] != preconditioner.components:
        raise ValidationError("apply_preconditioner: field shape mismatch")
    ctx = grid.context(r.shape[0])
    ctx.set_reference(preconditioner.c_ref)
    out = np.zeros_like(r)
    _check(lib.homfe_gpu_apply_minv(ctx.h, _dp(r), _dp(out)))
    return out if preconditioner.weighted else out * grid.quad_weights()[0]


def gamma_apply(grid, preconditioner, s):
    """Compatibility projection D (D^T C_ref D)^+ D^T (projection.cpp:29-41,
    module.cpp:270-277); the blocks must be assembled unweighted."""
    if preconditioner.weighted:
        raise ValidationError("gamma_apply: blocks must be assembled without the weight fusion")
    s = _quad(grid, s)
    ctx = grid.context(preconditioner.components)
    if s.shape[1] != ctx.m:
        raise ValidationError("gamma_apply: field shape mismatch")
    ctx.set_reference(preconditioner.c_ref)
    out = np.zeros_like(s)
    _check(lib.homfe_gpu_gamma_apply(ctx.h, _dp(s), _dp(out)))
    return out


def eigenvalue_bounds(grid, tangent, c_ref, components, pixel_constant=False):
    """Sorted two-sided eigenvalue bounds and the condition estimate
    (spectral.cpp:33-127, module.cpp:286-297)."""
    ctx = grid.context(components)
    m = ctx.m
    t = np.asarray(tangent, dtype=float)
    if t.shape != (grid.num_quads, m, m):
        raise ValidationError("eigenvalue_bounds: tangent does not match layout")
    cr = np.asarray(c_ref, dtype=float)
    if cr.shape != (m, m):
        raise ValidationError("eigenvalue_bounds: reference has wrong size")
    tc = _f64(t.transpose(0, 2, 1))
    crc = _f64(cr.T)
    lo = np.zeros(components * grid.num_nodes)
    hi = np.zeros(components * grid.num_nodes)
    cond = C.c_double()
    _check(lib.homfe_gpu_eigenvalue_bounds(ctx.h, _dp(tc), int(pixel_constant), _dp(crc), _dp(lo), _dp(hi),
                                           C.byref(cond)))
    return lo, hi, cond.value


def volume_average(grid, s):
    """(1/|Y|) sum_Q w^Q s(Q) (fields.hpp:94-95)."""
    s = _quad(grid, s)
    m = s.shape[1]
    c = 1 if m == grid.dim else grid.dim
    ctx = grid.context(c)
    out = np.zeros(m)
    _check(lib.homfe_gpu_volume_average(ctx.h, _dp(s), _dp(out)))
    return out


def pcg_solve(grid, materials, phases, preconditioner, b, eta, it_max):
    """pcg_solve (solver.hpp:75-78) with A = K(materials, phases) and M^-1 =
    ``preconditioner``; returns dict(x, iterations, history, converged)."""
    b = _nodal(grid, b)
    ctx = grid.context(b.shape[0])
    ctx.set_material(np.stack([m.tangent for m in materials]), phases)
    ctx.set_reference(preconditioner.c_ref)
    x = np.zeros_like(b)
    it = C.c_int32()
    conv = C.c_int32()
    hist = np.zeros(int(it_max) + 1)
    _check(lib.homfe_gpu_pcg(ctx.h, _dp(b), float(eta), int(it_max), _dp(x), C.byref(it), _dp(hist),
                             C.byref(conv)))
    return dict(x=x, iterations=it.value, history=hist[: it.value + 1], converged=bool(conv.value))


_CAUSES = ("converged", "cg-stall", "newton-cap")
_POLICIES = {"identity-scaled": 0, "volume-mean": 1, "explicit": 2}


def _report_dict(rep):
    steps = [dict(cg_iterations=rep.steps[i].cg_iterations, residual_initial=rep.steps[i].residual_initial,
                  residual_final=rep.steps[i].residual_final, increment_rel=rep.steps[i].increment_rel,
                  precond_reassembled=bool(rep.steps[i].precond_reassembled))
             for i in range(min(rep.n_steps, 32))]
    return dict(cause=_CAUSES[rep.cause], newton_steps=rep.n_steps, cg_total=rep.total_cg, steps=steps,
                seconds_total=rep.seconds_total, seconds_cg=rep.seconds_cg, seconds_assembly=rep.seconds_assembly,
                seconds_constitutive=rep.seconds_constitutive,
                cg_device_ms=rep.cg_device_ms, assemblies=rep.assemblies, kernel_launches=rep.kernel_launches)


class Solver:
    """A reusable solve context: grid + material map on the device, then any
    number of ``solve(e)`` calls (warm-startable), mirroring
    run_load_program (proj/src/solver.cpp:298-319)."""

    def __init__(self, grid, materials, phases, eta_newton=1e-5, eta_cg=1e-5, max_newton=25, max_cg=20000,
                 reassembly_threshold=0.1, reference="volume-mean", reference_scale=1.0, reference_matrix=None,
                 criterion="strain"):
        if not materials:
            raise ValidationError("materials: catalog is empty")
        thermal = {m.thermal for m in materials}
        if len(thermal) != 1:
            raise ValidationError("materials: mixed thermal and mechanical models")
        if any(m.dim != grid.dim for m in materials):
            raise ValidationError("materials: model dimension mismatch")
        ph = np.ascontiguousarray(phases, dtype=np.uint8)
        if ph.ndim != 1 or ph.shape[0] != grid.num_pixels:
            raise ValidationError("expected a flat (num_pixels,) uint8 phase map")
        self.grid = grid
        self.c = 1 if thermal.pop() else grid.dim
        self.ctx = grid.context(self.c)
        self.nonlinear = any(m.nonlinear for m in materials)
        if self.nonlinear:
            self.ctx.set_models(materials, ph)
        else:
            self.ctx.set_material(np.stack([m.tangent for m in materials]), ph)
        self.width = 7 if self.nonlinear else 0
        # a Solver is one PrecondManager (solver.hpp:105-129) over its solves
        _check(lib.homfe_gpu_precond_reset(self.ctx.h))
        self.cfg = _native.SolveCfg()
        self.cfg.eta_newton, self.cfg.eta_cg = eta_newton, eta_cg
        self.cfg.max_newton, self.cfg.max_cg = max_newton, max_cg
        self.cfg.reassembly_threshold = reassembly_threshold
        self.cfg.criterion = 0 if criterion == "strain" else 1
        if reference not in _POLICIES:
            raise ValidationError("reference policy must be 'volume-mean', 'identity-scaled' or 'explicit'")
        self.cfg.reference_policy = _POLICIES[reference]
        self.cfg.reference_scale = reference_scale
        self._refmat = None
        if reference_matrix is not None:
            self._refmat = _f64(np.asarray(reference_matrix).T)
            self.cfg.reference_matrix = _dp(self._refmat)

    def solve(self, e, warm_start=None, raise_on_nonconvergence=False, internal=None, stress=False):
        """newton_solve (solver.cpp:171-296). ``internal``: committed state
        (num_quads x 7) for J2 catalogs; the result holds the outgoing state
        (trial state on convergence, the input otherwise)."""
        m = self.ctx.m
        e = _f64(e).ravel()
        if e.size != m:
            raise ValidationError(f"load vector has {e.size} components, expected {m}")
        u = np.zeros((self.c, self.grid.num_nodes))
        avg = np.zeros(m)
        rep = _native.Report()
        warm = _nodal(self.grid, warm_start) if warm_start is not None else None
        out = {}
        if self.nonlinear:
            nq = self.grid.num_quads
            g0 = None
            if internal is not None:
                g0 = _f64(internal).reshape(-1)
                if g0.size != nq * 7:
                    raise ValidationError("internal state does not match layout and catalog")
            g_out = np.zeros((nq, 7))
            code = lib.homfe_gpu_solve_state(self.ctx.h, _dp(e), C.byref(self.cfg), _dp(warm), _dp(g0), _dp(u),
                                             _dp(g_out), _dp(avg), C.byref(rep))
            out["internal"] = g_out
        else:
            code = lib.homfe_gpu_solve(self.ctx.h, _dp(e), C.byref(self.cfg), _dp(warm), _dp(u), _dp(avg),
                                       C.byref(rep))
        if code != _native.NONCONVERGED or raise_on_nonconvergence:
            _check(code)
        out.update(converged=bool(rep.converged), u=u, average_stress=avg, report=_report_dict(rep))
        if stress:
            sig = np.zeros((self.grid.num_quads, m))
            _check(lib.homfe_gpu_stress_field(self.ctx.h, _dp(sig)))
            out["stress"] = sig
        return out


def _solver_sb_solve(self, e, c_ref, internal=None, warm_strain=None, raise_on_nonconvergence=False):
    m = self.ctx.m
    e = _f64(e).ravel()
    if e.size != m:
        raise ValidationError(f"load vector has {e.size} components, expected {m}")
    nq = self.grid.num_quads
    cr = _f64(np.asarray(c_ref, dtype=float).T)
    if cr.size != m * m:
        raise ValidationError("reference: explicit matrix has wrong size")
    ws = _f64(warm_strain).reshape(-1) if warm_strain is not None else None
    if ws is not None and ws.size != nq * m:
        raise ValidationError("sb warm start has wrong shape")
    g0 = _f64(internal).reshape(-1) if (internal is not None and self.nonlinear) else None
    strain = np.zeros((nq, m))
    g_out = np.zeros((nq, 7)) if self.nonlinear else None
    avg = np.zeros(m)
    rep = _native.Report()
    code = lib.homfe_gpu_sb_solve(self.ctx.h, _dp(e), C.byref(self.cfg), _dp(cr), _dp(ws), _dp(g0), _dp(strain),
                                  _dp(g_out), _dp(avg), C.byref(rep))
    if code != _native.NONCONVERGED or raise_on_nonconvergence:
        _check(code)
    out = dict(converged=bool(rep.converged), strain=strain, average_stress=avg, report=_report_dict(rep))
    if self.nonlinear:
        out["internal"] = g_out
    return out


Solver.sb_solve = _solver_sb_solve


def newton_solve(grid, materials, phases, e, eta_newton=1e-5, eta_cg=1e-5, max_newton=25, max_cg=20000,
                 reassembly_threshold=0.1, reference="volume-mean", reference_scale=1.0, reference_matrix=None,
                 criterion="strain"):
    """One Newton-PCG solve at macroscopic strain e (solver.hpp:163-166;
    Python signature of proj/src/bindings/module.cpp:299-328)."""
    s = Solver(grid, materials, phases, eta_newton, eta_cg, max_newton, max_cg, reassembly_threshold, reference,
               reference_scale, reference_matrix, criterion)
    return s.solve(e, stress=True)


def sb_newton_solve(grid, materials, phases, e, c_ref, internal=None, warm_strain=None, eta_newton=1e-5,
                    eta_cg=1e-5, max_newton=25, max_cg=20000):
    """Strain-based scheme (projection.cpp:93-185): Newton on the
    fluctuating strain with Gamma-projected CG at a fixed reference."""
    s = Solver(grid, materials, phases, eta_newton, eta_cg, max_newton, max_cg)
    return s.sb_solve(e, c_ref, internal=internal, warm_strain=warm_strain)


def compare_db_sb(grid, materials, phases, loads, c_ref, eta_newton=1e-5, eta_cg=1e-5, max_newton=25,
                  max_cg=20000, reassembly_threshold=0.1):
    """DbSbComparison (projection.cpp:216-262): both schemes on one load
    program at matched tolerances and the same reference tangent."""
    s = Solver(grid, materials, phases, eta_newton, eta_cg, max_newton, max_cg, reassembly_threshold,
               reference="explicit", reference_matrix=c_ref)
    out = dict(db_reports=[], sb_reports=[], db_average_stress=[], sb_average_stress=[], strain_discrepancy=[],
               converged=True)
    g_db = g_sb = None
    w_db = w_sb = None
    db_u = []
    for e in loads:
        r = s.solve(e, warm_start=w_db, internal=g_db)
        out["converged"] &= r["converged"]
        if r["converged"] and s.nonlinear:
            g_db = r["internal"]
        out["db_reports"].append(r["report"])
        out["db_average_stress"].append(r["average_stress"])
        db_u.append(r["u"])
        w_db = r["u"]
    for i, e in enumerate(loads):
        r = s.sb_solve(e, c_ref, internal=g_sb, warm_strain=w_sb)
        out["converged"] &= r["converged"]
        if r["converged"] and s.nonlinear:
            g_sb = r["internal"]
        out["sb_reports"].append(r["report"])
        out["sb_average_stress"].append(r["average_stress"])
        w_sb = r["strain"]
        db_strain = gradient_apply(grid, db_u[i])
        scale = np.abs(db_strain).max()
        diff = np.abs(r["strain"] - db_strain).max()
        out["strain_discrepancy"].append(diff / scale if scale > 0 else diff)
    return out


def run_load_program(grid, materials, phases, loads, eta_newton=1e-5, eta_cg=1e-5, max_newton=25, max_cg=20000,
                     reassembly_threshold=0.1, reference="volume-mean", reference_scale=1.0, reference_matrix=None,
                     criterion="strain"):
    """run_load_program (proj/src/solver.cpp:298-319): load steps with warm
    starts; the internal state is committed after each converged step and the
    program stops at the first non-converged step."""
    if not len(loads):
        raise ValidationError("loading: at least one load step is required")
    s = Solver(grid, materials, phases, eta_newton, eta_cg, max_newton, max_cg, reassembly_threshold, reference,
               reference_scale, reference_matrix, criterion)
    results = []
    g = np.zeros((grid.num_quads, 7)) if s.nonlinear else None
    warm = None
    for e in loads:
        out = s.solve(e, warm_start=warm, internal=g, stress=True)
        if out["converged"] and s.nonlinear:
            g = out["internal"]
        results.append(dict(load=np.asarray(e, dtype=float), **out))
        if not out["converged"]:
            break
        warm = out["u"]
    return results
