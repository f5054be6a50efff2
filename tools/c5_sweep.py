"""BASELINE config c5: 2-D scalar conductivity resolution / contrast sweep,
N in {1024, 2048, 4096, 8192} x contrast in {1e1, 1e3, 1e5} (seeded circular
inclusions at area fraction 0.3, same physical geometry at every N).
Per case: PCG iterations, DOF*it/s (CUDA-event PCG time), ms per iteration,
fraction of the HBM roofline (B_iter = 113 B/pixel) and time to
solution. One JSON line per case on stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
    HBM = float(json.load(f)["hbm_gbs"])

ns = [int(a) for a in os.environ.get("C5_N", "1024,2048,4096,8192").split(",")]
contrasts = [float(a) for a in os.environ.get("C5_CONTRAST", "1e1,1e3,1e5").split(",")]
for n in ns:
    for k in contrasts:
        cfg = inputs.config("c5", n=n, contrast=k)
        ph = cfg.phases()
        g = hb.Grid(cfg.dims, [1.0, 1.0], cfg.stencil)
        mats = [hb.Material(t, True, 2) for t in cfg.tangents()]
        s = hb.Solver(g, mats, ph, eta_cg=cfg.eta_cg, reference=cfg.reference)
        e = np.asarray(cfg.load, dtype=float)
        s.solve(e)  # warm-up (graph capture, plans)
        t0 = time.perf_counter()
        out = s.solve(e)
        wall = time.perf_counter() - t0
        rep = out["report"]
        it = rep["cg_total"]
        ms_it = rep["cg_device_ms"] / max(it, 1)
        dof = cfg.dof
        print(json.dumps({"config": "c5", "n": n, "contrast": k, "dof": dof, "pcg_iterations": it,
                          "converged": out["converged"], "dof_it_per_s": dof * it / (rep["cg_device_ms"] / 1e3),
                          "iteration_ms": ms_it,
                          "iteration_roofline_frac": 113.0 * n * n / (ms_it / 1e3) / 1e9 / HBM,
                          "time_to_solution_s": wall, "k_eff_xx": float(out["average_stress"][0])}), flush=True)
        del s
