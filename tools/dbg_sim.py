"""Debug helper: W slab contexts on one GPU (in-process transport) against
the single-device operators. usage: dbg_sim.py WORLD C [N0 N1]"""
import sys, threading
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import dist, inputs
world, c = int(sys.argv[1]), int(sys.argv[2])
n0 = int(sys.argv[3]) if len(sys.argv) > 3 else 64
n1 = int(sys.argv[4]) if len(sys.argv) > 4 else 128
dims = (n0, n1, n1)
ph, _ = inputs.rsa_balls(dims, radius=6.0, seed=5, fraction=0.25)
if c == 1:
    cm = np.stack([np.eye(3), 100.0 * np.eye(3)])
    e = [1.0, 0.0, 0.0]
else:
    cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)])
    e = [0, 0, 0, 0, 0, np.sqrt(2.0) * 0.01]
g = hb.Grid(dims, [1.0, 1.0, 1.0], "trilinear-hex")
rng = np.random.default_rng(2)
u = rng.uniform(-1, 1, (c, g.num_nodes))
ku_ref = hb.apply_operator(g, cm[np.repeat(ph, 8)], u)
r = u - u.mean(axis=1, keepdims=True)
z_ref = hb.apply_preconditioner(g, hb.assemble_preconditioner(g, cm[0], c), r)
plane = dims[1] * dims[2]
res = [None] * world
def rank_main(rank):
    sc = dist.SlabContext(g, c, rank, world, dist.sim_group_id(77 + world))
    print("rank", rank, sc.transport, flush=True)
    sl = slice(sc.z0 * plane, (sc.z0 + sc.nz) * plane)
    sc.set_material(cm, ph[sl])
    ku = sc.apply_K(u[:, sl])
    sc.set_reference(cm[0])
    z = sc.apply_minv(r[:, sl])
    res[rank] = (sl, ku, z)
ts = [threading.Thread(target=rank_main, args=(k,)) for k in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
print("expect u0", u[0,0], "u31", u[0,31*plane], "u32", u[0,32*plane], "u63", u[0,63*plane])
ku = np.zeros_like(u); z = np.zeros_like(u)
for sl, kl, zl in res: ku[:, sl] = kl; z[:, sl] = zl
for name, a, b in (("K", ku, ku_ref), ("Minv", z, z_ref)):
    d = np.abs(a - b).reshape(c, dims[0], plane).max(axis=2) / np.abs(b).max()
    for k in range(c):
        bad = np.nonzero(d[k] > 1e-12)[0]
        print(name, "comp", k, "bad planes", bad[:20], len(bad))
