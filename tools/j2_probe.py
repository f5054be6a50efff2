"""J2 Newton-PCG on the GPU at a given size: Newton steps, CG iterations,
per-iteration device time (SURVEY 8(f) f1 measurement)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dims = (n, n, n)
ph, _ = inputs.rsa_balls(dims, radius=10.0 * n / 256, seed=2203003, fraction=0.30)
g = hb.Grid(dims, [1.0] * 3, "trilinear-hex")
mats = [hb.Material.isotropic_elastic(1.0 / (3 * (1 - 0.6)), 1.0 / 2.6, 3),
        hb.Material.j2_plastic(10.0 / (3 * (1 - 0.6)), 10.0 / 2.6, 4e-3, 0.1, 3)]
s = hb.Solver(g, mats, ph, eta_cg=1e-6, eta_newton=1e-5, reference="volume-mean")
e = np.array([0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01])
for rep in range(2):
    t0 = time.perf_counter()
    out = s.solve(e)
    t = time.perf_counter() - t0
r = out["report"]
dof = 3 * np.prod(dims)
print(f"J2 {dims}: converged {out['converged']} newton {r['newton_steps']} cg {r['cg_total']} "
      f"steps {[x['cg_iterations'] for x in r['steps']]} time {t:.3f}s cg_device {r['cg_device_ms']:.1f}ms "
      f"-> {dof * r['cg_total'] / (r['cg_device_ms'] / 1e3):.3e} DOF*it/s, max ep_acc {out['internal'][:, 6].max():.3e}")
