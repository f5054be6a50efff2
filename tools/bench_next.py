"""Measurements of the SURVEY 8(f) rows built beyond the hot path (one GPU):
f1 J2 Newton-PCG (displacement scheme) and f4 strain-based scheme + bounds.
Prints one JSON line per case. Per-iteration algorithmic bytes of the J2
tangent operator (generic two-pass path): p (8c) + phase (1) + compact
tangent (8 nq x 8) + sigma_q written and read (2 x 8 m nq) + Ap (8c) per
voxel, against MEASURED_PEAKS.json hbm_gbs."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs


def hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 7672.0


def j2_case(n):
    dims = (n, n, n)
    ph, _ = inputs.rsa_balls(dims, radius=10.0 * n / 256, seed=2203003, fraction=0.30)
    g = hb.Grid(dims, [1.0] * 3, "trilinear-hex")
    mats = [hb.Material.isotropic_elastic(1.0 / 1.2, 1.0 / 2.6, 3), hb.Material.j2_plastic(10.0 / 1.2, 10.0 / 2.6, 4e-3, 0.1, 3)]
    s = hb.Solver(g, mats, ph, eta_cg=1e-6, eta_newton=1e-5, reference="volume-mean")
    e = np.array([0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01])
    s.solve(e)
    t0 = time.perf_counter()
    out = s.solve(e)
    wall = time.perf_counter() - t0
    r = out["report"]
    dof = 3 * g.num_pixels
    it_ms = r["cg_device_ms"] / max(r["cg_total"], 1)
    b_iter_k = g.num_pixels * (24 + 1 + 8 * 8 * 8 + 2 * 8 * 6 * 8 + 24)
    return dict(case=f"f1 J2 DB Newton-PCG {dims} (elastic matrix + J2 spheres f=0.30, volume-mean reference)",
                converged=out["converged"], newton_steps=r["newton_steps"], cg_total=r["cg_total"],
                value=dof * r["cg_total"] / (r["cg_device_ms"] / 1e3), unit="DOF*it/s", iteration_ms=it_ms,
                time_to_solution_s=wall, max_ep_acc=float(out["internal"][:, 6].max()),
                k_bytes_per_apply=b_iter_k, k_apply_floor_ms=b_iter_k / (hbm() * 1e9) * 1e3)


def sb_case(n):
    dims = (n, n)
    ph, _ = inputs.rsa_balls(dims, radius=12.0 * n / 256, seed=2203005, fraction=0.30)
    g = hb.Grid(dims, [1.0, 1.0], "two-triangles")
    c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(12.0, 7.0, 2)
    mats = [hb.Material.linear_elastic(c0), hb.Material.linear_elastic(c1)]
    e = np.array([0.01, 0.0, 0.0])
    t0 = time.perf_counter()
    cmp = hb.compare_db_sb(g, mats, ph, [e], np.eye(3), eta_newton=1e-8, eta_cg=1e-8)
    wall = time.perf_counter() - t0
    db, sb = cmp["db_reports"][0], cmp["sb_reports"][0]
    return dict(case=f"f4 DB/SB comparison {dims} two triangles, 2-phase elastic, C_ref = I",
                converged=cmp["converged"], db_cg=db["cg_total"], sb_cg=sb["cg_total"],
                db_newton=db["newton_steps"], sb_newton=sb["newton_steps"],
                strain_discrepancy=cmp["strain_discrepancy"][0], sb_seconds_cg=sb["seconds_cg"],
                db_seconds_cg=db["seconds_cg"], wall_s=wall)


def bounds_case(n):
    dims = (n, n, n)
    g = hb.Grid(dims, [1.0] * 3, "trilinear-hex")
    ph, _ = inputs.rsa_balls(dims, radius=10.0 * n / 256, seed=2203003, fraction=0.30)
    c0, c1 = hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)
    t = np.where(np.repeat(ph.astype(bool), 8)[:, None, None], c1[None], c0[None])
    t0 = time.perf_counter()
    lo, hi, cond = hb.eigenvalue_bounds(g, t, c0, 3, pixel_constant=True)
    return dict(case=f"f4 eigenvalue bounds {dims} hex, c3 materials, C_ref = matrix", condition_estimate=cond,
                seconds=time.perf_counter() - t0, num_bounds=int(lo.size))


def twonode_case(n):
    dims = (n, n)
    ph, _ = inputs.rsa_balls(dims, radius=12.0 * n / 256, seed=2203005, fraction=0.30)
    g = hb.Grid(dims, [1.0, 1.0], "four-triangles-two-node")
    c0, c1 = hb.isotropic_stiffness(1.0, 0.5, 2), hb.isotropic_stiffness(12.0, 7.0, 2)
    s = hb.Solver(g, [hb.Material.linear_elastic(c0), hb.Material.linear_elastic(c1)], ph, eta_cg=1e-8)
    e = np.array([0.01, 0.0, 0.0])
    s.solve(e)
    t0 = time.perf_counter()
    out = s.solve(e)
    wall = time.perf_counter() - t0
    r = out["report"]
    dof = 2 * g.num_nodes
    return dict(case=f"f3 FourTrianglesTwoNode {dims} 2-phase elastic (probed complex blocks, volume-mean reference)",
                converged=out["converged"], cg_total=r["cg_total"], value=dof * r["cg_total"] / (r["cg_device_ms"] / 1e3),
                unit="DOF*it/s", iteration_ms=r["cg_device_ms"] / max(r["cg_total"], 1), time_to_solution_s=wall)


if __name__ == "__main__":
    for fn, arg in ((j2_case, 128), (sb_case, 1024), (bounds_case, 64), (twonode_case, 1024)):
        print(json.dumps(fn(arg)), flush=True)
