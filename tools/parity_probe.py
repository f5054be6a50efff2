"""Diagnostic: GPU vs oracle PCG iterate difference as a function of k, next
to the oracle-vs-oracle noise floor (1e-16 input perturbation)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import inputs
from oracle import oracle

dims = (24, 24, 24)
ph, _ = inputs.rsa_balls(dims, radius=3.0, seed=7, fraction=0.25)
cm = np.stack([np.eye(3), 100 * np.eye(3)])
og = oracle.Grid(dims, [1.0] * 3, "trilinear-hex")
g = hb.Grid(dims, [1.0] * 3, "trilinear-hex")
e = np.array([1.0, 0, 0])
sig = np.repeat(cm[ph], 8, axis=0) @ e
b = -oracle.divergence(og, 1, sig)
mats = [hb.Material(t, True, 3) for t in cm]
for cref in (np.eye(3),):
    pre = oracle.Preconditioner(og, cref, 1)
    gp = hb.assemble_preconditioner(g, cref, 1)
    for k in (10, 30, 56, 76, 100):
        xo = oracle.pcg(og, 1, cm, ph, pre, b, 0.0, k)
        xg = hb.pcg_solve(g, mats, ph, gp, b.reshape(1, -1), 0.0, k)
        rng = np.random.default_rng(0)
        xp = oracle.pcg(og, 1, cm, ph, pre, b * (1 + 1e-16 * rng.standard_normal(b.size)), 0.0, k)
        n = np.linalg.norm(xo["x"])
        print(k, "gpu-oracle", np.linalg.norm(xg["x"].ravel() - xo["x"]) / n, "oracle-noise",
              np.linalg.norm(xp["x"] - xo["x"]) / n, "hist", xo["history"][-1] / xo["history"][0])
    # operator-level differences
    u = oracle.uniform(3, g.num_nodes)
    ko = oracle.apply_phase(og, 1, cm, ph, u)
    kg = hb.apply_operator(g, cm[np.repeat(ph, 8)], u.reshape(1, -1)).ravel()
    print("K rel", np.abs(kg - ko).max() / np.abs(ko).max())
    r = u - u.mean()
    zo = pre.apply(r)
    zg = hb.apply_preconditioner(g, gp, r.reshape(1, -1)).ravel()
    print("Minv rel", np.abs(zg - zo).max() / np.abs(zo).max())
