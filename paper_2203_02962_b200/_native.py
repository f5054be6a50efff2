"""ctypes binding of the C ABI in ``include/homfe_gpu.h``.

The library is built in-tree by ``paper_2203_02962_b200/build.py`` into
``paper_2203_02962_b200/_lib/libhomfe_gpu.so``. There is no CPU fallback: if
the library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HOMFE_LIB") or os.path.join(HERE, "_lib", "libhomfe_gpu.so")

OK, VALIDATION, NONCONVERGED, NUMERICAL, DEVICE = 0, 2, 3, 4, 5


class GridDesc(C.Structure):
    _fields_ = [("dim", C.c_int32), ("stencil", C.c_int32), ("dims", C.c_int64 * 3),
                ("lengths", C.c_double * 3), ("components", C.c_int32), ("device", C.c_int32)]


class SolveCfg(C.Structure):
    _fields_ = [("eta_newton", C.c_double), ("eta_cg", C.c_double), ("max_newton", C.c_int32),
                ("max_cg", C.c_int32), ("reassembly_threshold", C.c_double), ("criterion", C.c_int32),
                ("reference_policy", C.c_int32), ("reference_scale", C.c_double),
                ("reference_matrix", C.POINTER(C.c_double))]


class NewtonStep(C.Structure):
    _fields_ = [("cg_iterations", C.c_int32), ("residual_initial", C.c_double),
                ("residual_final", C.c_double), ("increment_rel", C.c_double),
                ("precond_reassembled", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("n_steps", C.c_int32), ("steps", NewtonStep * 32), ("cause", C.c_int32),
                ("converged", C.c_int32), ("assemblies", C.c_int32), ("total_cg", C.c_int32),
                ("seconds_constitutive", C.c_double), ("seconds_cg", C.c_double),
                ("seconds_assembly", C.c_double), ("seconds_total", C.c_double),
                ("cg_device_ms", C.c_double), ("kernel_launches", C.c_int64)]


class MaterialModel(C.Structure):
    """homfe_material (include/homfe_gpu.h)."""
    _fields_ = [("kind", C.c_int32), ("tangent", C.c_double * 36), ("bulk", C.c_double), ("shear", C.c_double),
                ("yield_stress", C.c_double), ("hardening", C.c_double)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_double))


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2203_02962_b200.build` "
            "(nvcc, sm_100a). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    d, i32, i64, vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p
    sig = {
        "homfe_gpu_last_error": (C.c_char_p, []),
        "homfe_isotropic_stiffness": (C.c_int, [d, d, i32, P(d)]),
        "homfe_gpu_create": (C.c_int, [P(GridDesc), P(vp)]),
        "homfe_gpu_destroy": (C.c_int, [vp]),
        "homfe_gpu_set_material": (C.c_int, [vp, i32, P(d), P(C.c_uint8)]),
        "homfe_gpu_set_material_device": (C.c_int, [vp, i32, P(d), vp]),
        "homfe_gpu_solve": (C.c_int, [vp, P(d), P(SolveCfg), P(d), P(d), P(d), P(Report)]),
        "homfe_gpu_solve_device": (C.c_int, [vp, P(d), P(SolveCfg), vp, vp, P(d), P(Report)]),
        "homfe_gpu_apply_K": (C.c_int, [vp, P(d), P(d)]),
        "homfe_gpu_set_reference": (C.c_int, [vp, P(d)]),
        "homfe_gpu_apply_minv": (C.c_int, [vp, P(d), P(d)]),
        "homfe_gpu_reference_blocks": (C.c_int, [vp, P(d)]),
        "homfe_gpu_gradient": (C.c_int, [vp, P(d), P(d)]),
        "homfe_gpu_divergence": (C.c_int, [vp, P(d), i32, P(d)]),
        "homfe_gpu_apply_tangent_field": (C.c_int, [vp, P(d), P(d), P(d)]),
        "homfe_gpu_volume_average": (C.c_int, [vp, P(d), P(d)]),
        "homfe_gpu_pcg": (C.c_int, [vp, P(d), d, i32, P(d), P(i32), P(d), P(i32)]),
        "homfe_gpu_index_maps": (C.c_int, [vp, P(i64), P(i64), P(i32)]),
        "homfe_gpu_sizes": (C.c_int, [vp, P(i64), P(i64), P(i32), P(i64)]),
        "homfe_random_uniform": (C.c_int, [C.c_uint64, i64, d, d, P(d)]),
        "homfe_gpu_kernel_times": (C.c_int, [vp, i32, P(d)]),
        "homfe_nccl_unique_id": (C.c_int, [vp]),
        "homfe_gpu_create_dist": (C.c_int, [P(GridDesc), i32, i32, vp, P(vp)]),
        "homfe_gpu_slab_transport": (C.c_int, [vp, P(i32)]),
        "homfe_random_normal": (C.c_int, [C.c_uint64, i64, P(d)]),
        "homfe_gpu_set_material_models": (C.c_int, [vp, i32, P(MaterialModel), P(C.c_uint8)]),
        "homfe_gpu_internal_width": (C.c_int, [vp, P(i32), P(i64)]),
        "homfe_gpu_solve_state": (C.c_int, [vp, P(d), P(SolveCfg), P(d), P(d), P(d), P(d), P(d), P(Report)]),
        "homfe_gpu_stress_field": (C.c_int, [vp, P(d)]),
        "homfe_gpu_gamma_apply": (C.c_int, [vp, P(d), P(d)]),
        "homfe_gpu_sb_solve": (C.c_int, [vp, P(d), P(SolveCfg), P(d), P(d), P(d), P(d), P(d), P(d), P(Report)]),
        "homfe_gpu_eigenvalue_bounds": (C.c_int, [vp, P(d), i32, P(d), P(d), P(d), P(d)]),
        "homfe_gpu_path_info": (C.c_int, [vp, P(i32)]),
        "homfe_gpu_precond_reset": (C.c_int, [vp]),
        "homfe_gpu_create_multi": (C.c_int, [P(GridDesc), i32, P(vp)]),
        "homfe_gpu_weighted_dot": (C.c_int, [vp, P(d), P(d), P(d)]),
        "homfe_gpu_pcg_observed": (C.c_int, [vp, P(d), d, i32, P(d), P(i32), P(d), P(i32), OBSERVER, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

EXPORTED = ("homfe_gpu_last_error", "homfe_isotropic_stiffness", "homfe_gpu_create", "homfe_gpu_destroy",
            "homfe_gpu_set_material", "homfe_gpu_set_material_device", "homfe_gpu_solve",
            "homfe_gpu_solve_device", "homfe_gpu_apply_K", "homfe_gpu_set_reference", "homfe_gpu_apply_minv",
            "homfe_gpu_reference_blocks", "homfe_gpu_gradient", "homfe_gpu_divergence",
            "homfe_gpu_volume_average", "homfe_gpu_pcg", "homfe_gpu_index_maps", "homfe_gpu_sizes",
            "homfe_random_uniform", "homfe_random_normal", "homfe_gpu_kernel_times",
            "homfe_nccl_unique_id", "homfe_gpu_create_dist", "homfe_gpu_slab_transport", "homfe_gpu_set_material_models",
            "homfe_gpu_internal_width", "homfe_gpu_solve_state", "homfe_gpu_stress_field",
            "homfe_gpu_gamma_apply", "homfe_gpu_sb_solve", "homfe_gpu_eigenvalue_bounds", "homfe_gpu_path_info",
            "homfe_gpu_precond_reset", "homfe_gpu_weighted_dot", "homfe_gpu_pcg_observed",
            "homfe_gpu_create_multi", "homfe_gpu_apply_tangent_field")

PATH_FLAGS = {"fused_fft": 1, "hex_modal": 2, "while_graph": 4, "slab_spectra": 8, "slab": 16, "peer_pull": 32,
              "elem2d": 64, "multi": 128, "small2d": 256}
