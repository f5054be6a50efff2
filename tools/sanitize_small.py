"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck): fused 3-pass path + modal hex K (elastic and scalar), 2-D
pixel stencils on the cuFFT path, a J2 Newton step and the two-node stencil."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def run(dims, stencil, thermal, eta=1e-6, max_cg=30):
    d = len(dims)
    ph, _ = inputs.rsa_balls(dims, radius=dims[0] / 6.0, seed=3, fraction=0.25)
    if thermal:
        cm = np.stack([np.eye(d), 50.0 * np.eye(d)])
        e = np.zeros(d)
        e[0] = 1.0
    else:
        cm = np.stack([hb.isotropic_stiffness(0.83, 0.38, d), hb.isotropic_stiffness(55.5, 41.7, d)])
        e = np.zeros(d * (d + 1) // 2)
        e[-1] = 0.01
    g = hb.Grid(dims, [1.0] * d, stencil)
    mats = [hb.Material(t, thermal, d) for t in cm]
    out = hb.newton_solve(g, mats, ph, e, eta_cg=eta, max_cg=max_cg, reference="explicit", reference_matrix=cm[0])
    print(dims, stencil, thermal, out["report"]["cg_total"], flush=True)


if which in ("all", "fused"):
    run((64, 128, 128), "trilinear-hex", False)   # fused passes (128^2 planes), modal K
    run((64, 128, 128), "trilinear-hex", True)
if which in ("all", "cufft"):
    run((16, 24, 40), "trilinear-hex", False)     # cuFFT path, generic element K
    run((96, 64), "two-triangles", True)          # 2-D warp-strip K
    run((48, 40), "bilinear-quad", False)
if which in ("all", "twonode"):
    run((12, 16), "four-triangles-two-node", False)
if which in ("all", "j2"):
    g = hb.Grid((32, 32, 32), [1.0] * 3, "trilinear-hex")
    ph, _ = inputs.rsa_balls((32, 32, 32), radius=5.0, seed=5, fraction=0.3)
    mats = [hb.Material.isotropic_elastic(0.83, 0.38, 3), hb.Material.j2_plastic(0.83, 0.38, 0.004, 0.01, 3)]
    out = hb.newton_solve(g, mats, ph, [0, 0, 0, 0, 0, 0.02], eta_cg=1e-6, max_cg=40)
    print("j2", out["report"]["cg_total"], flush=True)
