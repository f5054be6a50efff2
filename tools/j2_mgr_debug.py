"""Debug: shared PrecondManager J2 load program, GPU vs oracle per step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from oracle import oracle as o
params = [(1.0, 0.5, 1e-3, 0.05), (10.0, 5.0, 2e-3, 0.5)]
gpu = [hb.Material.j2_plastic(*p, 2) for p in params]
orc = [o.material("j2", bulk=p[0], shear=p[1], yield_stress=p[2], hardening=p[3]) for p in params]
ph = np.zeros(256, np.uint8)
ph.reshape(16, 16)[4:12, 4:12] = 1
loads = [np.array([1e-3, 0.0, 0.5e-3]) * s for s in (1.0, 2.0, 3.0, 4.0)]
kw = dict(eta_newton=1e-9, eta_cg=1e-10, reference="volume-mean", reassembly_threshold=0.05)
res = hb.run_load_program(hb.Grid((16, 16), (1.0, 1.0), "two-triangles"), gpu, ph, loads, **kw)
og = o.Grid((16, 16), (1.0, 1.0), "two-triangles")
mgr = o.PrecondManager()
g = warm = None
for step, e in enumerate(loads):
    ref = o.newton_solve_models(og, False, orc, ph, e, g0=g, warm_u=warm, manager=mgr, **kw)
    got = res[step] if step < len(res) else None
    print("step", step, "oracle", ref["converged"], ref["cause"], [(s["cg_iterations"], s["precond_reassembled"], round(s["increment_rel"], 14)) for s in ref["steps"]], ref["assemblies"])
    if got:
        print("        gpu", got["converged"], got["report"]["cause"], [(s["cg_iterations"], s["precond_reassembled"], round(s["increment_rel"], 14)) for s in got["report"]["steps"]], got["report"]["assemblies"])
    g, warm = ref["internal"], ref["u"]
