import sys, threading
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import dist, inputs
world, c = int(sys.argv[1]), int(sys.argv[2])
dims = (64, 128, 128)
ph, _ = inputs.rsa_balls(dims, radius=6.0, seed=5, fraction=0.25)
if c == 1:
    cm = np.stack([np.eye(3), 100.0 * np.eye(3)])
else:
    cm = np.stack([hb.isotropic_stiffness(0.8333, 0.3846, 3), hb.isotropic_stiffness(555.5, 416.7, 3)])
g = hb.Grid(dims, [1.0, 1.0, 1.0], "trilinear-hex")
rng = np.random.default_rng(2)
u = rng.uniform(-1, 1, (c, g.num_nodes))
ku_ref = hb.apply_operator(g, cm[np.repeat(ph, 8)], u)
plane = dims[1] * dims[2]
res = [None] * world
def rank_main(rank):
    sc = dist.SlabContext(g, c, rank, world, dist.sim_group_id(77 + world))
    sl = slice(sc.z0 * plane, (sc.z0 + sc.nz) * plane)
    sc.set_material(cm, ph[sl])
    res[rank] = (sl, sc.apply_K(u[:, sl]))
ts = [threading.Thread(target=rank_main, args=(k,)) for k in range(world)]
[t.start() for t in ts]; [t.join() for t in ts]
print("expect u0", u[0,0], "u31", u[0,31*plane], "u32", u[0,32*plane], "u63", u[0,63*plane])
ku = np.zeros_like(u)
for sl, kl in res: ku[:, sl] = kl
d = np.abs(ku - ku_ref).reshape(c, dims[0], plane).max(axis=2)
for k in range(c):
    bad = np.nonzero(d[k] > 1e-12)[0]
    print("comp", k, "bad planes", bad[:20], len(bad))
# impulse test: only global plane P set
for P in (63, 32, 31, 0):
    u2 = np.zeros_like(u)
    u2[0].reshape(dims[0], plane)[P] = 1.0
    kr = hb.apply_operator(g, cm[np.repeat(ph, 8)], u2)
    res2 = [None] * world
    def rm(rank):
        sc = dist.SlabContext(g, c, rank, world, dist.sim_group_id(900 + P))
        sl = slice(sc.z0 * plane, (sc.z0 + sc.nz) * plane)
        sc.set_material(cm, ph[sl])
        res2[rank] = (sl, sc.apply_K(u2[:, sl]))
    ts = [threading.Thread(target=rm, args=(k,)) for k in range(world)]
    [t.start() for t in ts]; [t.join() for t in ts]
    kd = np.zeros_like(u2)
    for sl, kl in res2: kd[:, sl] = kl
    nzr = np.nonzero(np.abs(kr).reshape(c, dims[0], plane).max(axis=(0, 2)) > 0)[0]
    nzd = np.nonzero(np.abs(kd).reshape(c, dims[0], plane).max(axis=(0, 2)) > 0)[0]
    print("P", P, "ref planes", nzr, "dist planes", nzd)
