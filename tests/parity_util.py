"""Fixed-k parity protocol shared by the GPU parity tests (SURVEY.md 8(c)
items 3 and 5).

At a fixed iteration count k the GPU PCG iterate is compared with the
oracle's (exact reference symbol, or_precond_exact). Two floors are measured
on the oracle side at the same k:
  * probing floor: the same oracle with the reference's impulse-probed blocks
    (precond.cpp:44-85) instead of the exact symbol;
  * reduction floor: the same oracle with a permuted reduction order (a
    different host-thread split of every dot product and FFT line).
Early iterates agree to ~1e-15; near convergence the iterate is as sensitive
to rounding as the remaining error (two orderings of the SAME oracle differ
by ~1e-8 at k = k_tol on a 24^3 contrast-100 problem). Hence:
  * k <= STRICT_K: the GPU must agree to 1e-10 outright;
  * larger k: to max(1e-10, 5 x floor), the floor reported next to it.
Every case is appended as one JSON line to $HOMFE_PARITY_LOG (the box's record
is committed as profiles/r02_parity_floors.jsonl).
"""
from __future__ import annotations

import json
import os

import numpy as np

from oracle.cfgutil import rel

STRICT_K = 10


def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def record(**kw):
    line = json.dumps(kw, default=float)
    print(line)
    path = os.environ.get("HOMFE_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(line + "\n")


def oracle_fixed_k(oracle_mod, og, c, cm, ph, cref, b, k, floors=True):
    """x_k of the exact-symbol oracle, and the two floors at k."""
    nt = host_threads()
    oracle_mod.set_threads(nt)
    pe = oracle_mod.Preconditioner(og, cref, c, exact=True)
    ex = oracle_mod.pcg(og, c, cm, ph, pe, b, 0.0, k)
    out = dict(x=ex["x"], history=ex["history"], iterations=ex["iterations"])
    if floors:
        if k > STRICT_K:  # the reduction floor matters only where the strict bound is relaxed
            oracle_mod.set_threads(max(1, nt // 2) if nt > 1 else 2)
            perm = oracle_mod.pcg(og, c, cm, ph, pe, b, 0.0, k)["x"]
            oracle_mod.set_threads(nt)
            out["floor_reduction"] = rel(perm, ex["x"])
        else:
            out["floor_reduction"] = None
        del pe
        pp = oracle_mod.Preconditioner(og, cref, c)
        probed = oracle_mod.pcg(og, c, cm, ph, pp, b, 0.0, k)["x"]
        out["floor_probing"] = rel(probed, ex["x"])
        out["x_probed"] = probed
    oracle_mod.set_threads(1)
    return out


def tolerance_for(k, ref):
    if k <= STRICT_K:
        return 1e-10
    return max(1e-10, 5.0 * max(ref["floor_reduction"] or 0.0, ref["floor_probing"] or 0.0))


def check_fixed_k(case, k, x_gpu, ref, extra=None):
    """Assert the protocol and record the case."""
    err = rel(x_gpu, ref["x"])
    tol = tolerance_for(k, ref)
    out = dict(case=case, k=k, rel_u_gpu_vs_exact=err, tolerance=tol,
               floor_reduction=ref.get("floor_reduction"), floor_probing=ref.get("floor_probing"),
               rel_u_gpu_vs_probed=rel(x_gpu, ref["x_probed"]) if "x_probed" in ref else None)
    if extra:
        out.update(extra)
    record(**out)
    assert err <= tol, out
    return out
