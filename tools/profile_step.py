"""One c3 solve + per-stage kernel timing; the target of ncu captures."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import _native, inputs

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = inputs.config(name, n=int(os.environ["N"])) if os.environ.get("N") else inputs.config(name)
g = hb.Grid(cfg.dims, [1.0] * cfg.dim, cfg.stencil)
mats = [hb.Material(t, cfg.thermal, cfg.dim) for t in cfg.tangents()]
s = hb.Solver(g, mats, cfg.phases(), eta_cg=cfg.eta_cg, reference=cfg.reference,
              reference_matrix=cfg.reference_matrix(), max_cg=int(os.environ.get("MAX_CG", "20000")))
out = s.solve(cfg.load)
reps = int(os.environ.get("SOLVES", "1"))
for _ in range(reps - 1):
    out = s.solve(cfg.load)
rep = out["report"]
print(name, "iteration_ms", rep["cg_device_ms"] / max(rep["cg_total"], 1), "cg", rep["cg_total"])
ms = np.zeros(8)
hb._check(_native.lib.homfe_gpu_kernel_times(s.ctx.h, int(os.environ.get("REPS", "3")), ms.ctypes.data_as(C.POINTER(C.c_double))))
print(name, out["report"]["cg_total"], ms.round(4).tolist())
