import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs
cfg = inputs.config("c5", n=8192)
g = hb.Grid(cfg.dims, [1.0] * cfg.dim, cfg.stencil)
mats = [hb.Material(t, cfg.thermal, cfg.dim) for t in cfg.tangents()]
s = hb.Solver(g, mats, cfg.phases(), eta_cg=cfg.eta_cg, reference=cfg.reference, reference_matrix=cfg.reference_matrix(), max_cg=5)
try:
    s.solve(cfg.load)
except Exception as e:
    print(e)
