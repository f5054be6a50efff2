"""Result bundle of a load program: the files
``homog solve`` writes (proj/tools/homog.cpp:69-166, proj/src/io.cpp:14-34,
98-120, layouts in proj/README.md "Result bundle"), produced from the GPU
solves of ``run_load_program``:

  u_step<i>.f64 / strain_step<i>.f64 / stress_step<i>.f64 (elasticity) or
  gradient_step<i>.f64 / flux_step<i>.f64 (thermal) with .meta.json sidecars,
  averages.csv, report.csv, solve.json, phases.u8.

The averages are re-computed on the host from the dumped field with the
reference's sequential weighted sum (fields.cpp:42-50), so reloading the
dumps and re-averaging reproduces averages.csv bitwise, as the reference
documents.
"""
from __future__ import annotations

import json
import os

import numpy as np

from . import ValidationError, gradient_apply


def _fmt(v):
    return "%.17g" % float(v)


def write_field(base, data, shape, layout, component_order, units):
    """write_field (io.cpp:14-34): raw little-endian float64 + JSON sidecar."""
    arr = np.ascontiguousarray(data, dtype="<f8").ravel()
    arr.tofile(base + ".f64")
    side = dict(dtype="float64", byte_order="little", count=int(arr.size), shape=[int(s) for s in shape],
                layout=layout, component_order=component_order, units=units)
    with open(base + ".meta.json", "w") as f:
        f.write(json.dumps(side, indent=2) + "\n")


def read_field(base):
    """read_field (io.cpp:36-62): (data reshaped to meta["shape"], meta)."""
    try:
        meta = json.load(open(base + ".meta.json"))
    except OSError:
        raise ValidationError(f"cannot open '{base}.meta.json'")
    data = np.fromfile(base + ".f64", dtype="<f8")
    if data.size != meta["count"]:
        raise ValidationError(f"field dump '{base}.f64' truncated")
    return data.reshape(meta["shape"]), meta


def _volume_average(grid, s):
    """fields.cpp:42-50 in the reference's loop order (sequential)."""
    w = grid.quad_weights()
    nq = grid.quads_per_pixel
    acc = np.zeros(s.shape[1])
    for q in range(s.shape[0]):
        acc = acc + w[q % nq] * s[q]
    return acc / grid.cell_volume


def write_result_bundle(out_dir, grid, phases, thermal, results, seed=None):
    """Write the bundle of ``run_load_program`` results (each with ``u``,
    ``stress``, ``load``, ``report``, ``converged``) into ``out_dir``."""
    os.makedirs(out_dir, exist_ok=True)
    np.ascontiguousarray(phases, dtype=np.uint8).tofile(os.path.join(out_dir, "phases.u8"))
    primal, dual = ("gradient", "flux") if thermal else ("strain", "stress")
    avg_rows, report_rows, status = [], [], []
    m = None
    for i, step in enumerate(results):
        tag = f"_step{i}"
        u = np.asarray(step["u"])
        write_field(os.path.join(out_dir, "u" + tag), u, [u.shape[0], u.shape[1]], "node-planar",
                    "temperature" if thermal else "displacement components", "temperature" if thermal else "length")
        e = np.asarray(step["load"], dtype=float)
        strain = gradient_apply(grid, u) + e[None, :]
        m = strain.shape[1]
        write_field(os.path.join(out_dir, primal + tag), strain, [strain.shape[0], m], "quad-interleaved",
                    "gradient components" if thermal else "mandel strain components", "dimensionless")
        stress = step.get("stress")
        if stress is None:
            raise ValidationError("result bundle: the solve did not return the stress field")
        write_field(os.path.join(out_dir, dual + tag), stress, [stress.shape[0], stress.shape[1]],
                    "quad-interleaved", "flux components" if thermal else "mandel stress components", "pressure")
        avg = _volume_average(grid, np.asarray(stress))
        avg_rows.append([str(i)] + [_fmt(v) for v in e] + [_fmt(v) for v in avg])
        rep = step["report"]
        for s, ns in enumerate(rep["steps"]):
            report_rows.append([str(i), str(s), str(ns["cg_iterations"]), _fmt(ns["residual_initial"]),
                                _fmt(ns["residual_final"]), _fmt(ns["increment_rel"]),
                                "1" if ns["precond_reassembled"] else "0"])
        status.append(dict(load_step=i, cause=rep["cause"], converged=bool(step["converged"]),
                           newton_steps=rep["newton_steps"], cg_total=rep["cg_total"],
                           seconds_total=rep["seconds_total"], seconds_cg=rep["seconds_cg"],
                           seconds_constitutive=rep.get("seconds_constitutive", 0.0),
                           seconds_assembly=rep["seconds_assembly"]))

    def write_csv(name, header, rows):
        with open(os.path.join(out_dir, name), "w") as f:
            f.write(",".join(header) + "\n")
            for r in rows:
                f.write(",".join(r) + "\n")

    write_csv("averages.csv", ["step"] + [f"e_{k}" for k in range(m)] + [f"avg_{dual}_{k}" for k in range(m)],
              avg_rows)
    write_csv("report.csv", ["load_step", "newton_step", "cg_iterations", "residual_initial", "residual_final",
                             "increment_rel", "precond_reassembled"], report_rows)
    with open(os.path.join(out_dir, "solve.json"), "w") as f:
        f.write(json.dumps(dict(steps=status, seed=seed), indent=2) + "\n")
