"""A/B timing of library builds: for every libhomfe_gpu.so given (or
variants/*/libhomfe_gpu.so plus the in-tree one), one c3 solve and the
per-stage CUDA-event times of the PCG iteration, plus K applied to a fixed
random field (checksum against the first library: every variant must
compute the same operator to rounding)."""
import ctypes as C
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import ctypes as C, json, os, sys
import numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2203_02962_b200 as hb
from paper_2203_02962_b200 import _native, inputs
name = os.environ.get("CFG", "c3")
cfg = inputs.config(name)
lengths = [1.0] * cfg.dim
g = hb.Grid(cfg.dims, lengths, cfg.stencil)
mats = [hb.Material(t, cfg.thermal, cfg.dim) for t in cfg.tangents()]
ph = cfg.phases()
s = hb.Solver(g, mats, ph, eta_cg=cfg.eta_cg, reference=cfg.reference, reference_matrix=cfg.reference_matrix())
out = s.solve(cfg.load)
out = s.solve(cfg.load)
rep = out["report"]
ms = np.zeros(8)
hb._check(_native.lib.homfe_gpu_kernel_times(s.ctx.h, 20, ms.ctypes.data_as(C.POINTER(C.c_double))))
rng = np.random.default_rng(5)
u = rng.uniform(-1, 1, (cfg.components, g.num_nodes))
ku = hb.apply_operator(g, cfg.tangents()[np.repeat(ph, g.quads_per_pixel)], u)
np.save(os.environ["KU_OUT"], ku)
print(json.dumps(dict(cg=rep["cg_total"], iter_ms=rep["cg_device_ms"] / rep["cg_total"], stages=ms.round(4).tolist(),
                      avg=out["average_stress"].tolist())))
'''


def main():
    libs = sys.argv[1:] or (sorted(glob.glob(os.path.join(ROOT, "variants", "*", "libhomfe_gpu.so"))) +
                            [os.path.join(ROOT, "paper_2203_02962_b200", "_lib", "libhomfe_gpu.so")])
    ref = None
    for lib in libs:
        kuf = "/tmp/ku_%d.npy" % abs(hash(lib))
        env = dict(os.environ, HOMFE_LIB=lib, ROOT=ROOT, KU_OUT=kuf)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-2000:]
        try:
            d = json.loads(line)
        except Exception:
            print(lib, "FAILED", line)
            continue
        import numpy as np
        ku = np.load(kuf)
        if ref is None:
            ref = ku
        d["ku_rel_vs_first"] = float(np.linalg.norm(ku - ref) / np.linalg.norm(ref))
        d["lib"] = os.path.relpath(lib, ROOT)
        print(json.dumps(d))


if __name__ == "__main__":
    main()
