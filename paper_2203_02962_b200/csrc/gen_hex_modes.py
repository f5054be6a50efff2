#!/usr/bin/env python3
"""Generates hex_modes.inc: straight-line per-quad-mode code for the modal
hex kernel (hexfast.cu), so that every modal coefficient stays in a register.

Quad modes (per axis s = symmetric, a = antisymmetric over the two Gauss
points): sss, ass, sas, ssa, aas, asa, saa (aaa carries no gradient).
Modal coefficient index v = alpha*4 + beta*2 + gamma (axis 0, 1, 2; 0 = S,
1 = D). The incidence below maps modal coefficients to raw strain rows
(elastic, Mandel order 11 22 33 23 13 12 with the sqrt(2)/2 shear factor
folded into the material table) or to gradient directions (scalar).

Run: python gen_hex_modes.py  (rewrites hex_modes.inc next to this file)
"""
import os

MODES = ["sss", "ass", "sas", "ssa", "aas", "asa", "saa"]
CLASS = [0, 1, 1, 1, 2, 2, 2]
# elastic incidence: (strain row e, component k, modal v)
INC3 = [
    [(0, 0, 4), (1, 1, 2), (2, 2, 1), (3, 1, 1), (3, 2, 2), (4, 0, 1), (4, 2, 4), (5, 0, 2), (5, 1, 4)],
    [(1, 1, 6), (2, 2, 5), (3, 1, 5), (3, 2, 6), (4, 0, 5), (5, 0, 6)],
    [(0, 0, 6), (2, 2, 3), (3, 1, 3), (4, 0, 3), (4, 2, 6), (5, 1, 6)],
    [(0, 0, 5), (1, 1, 3), (3, 2, 3), (4, 2, 5), (5, 0, 3), (5, 1, 5)],
    [(2, 2, 7), (3, 1, 7), (4, 0, 7)],
    [(1, 1, 7), (3, 2, 7), (5, 0, 7)],
    [(0, 0, 7), (4, 2, 7), (5, 1, 7)],
]
# scalar incidence: (direction j, modal v)
INCS = [[(0, 4), (1, 2), (2, 1)], [(1, 6), (2, 5)], [(0, 6), (2, 3)], [(0, 5), (1, 3)], [(2, 7)], [(1, 7)],
        [(0, 7)]]


def gen_elastic(iso):
    out = []
    for md, inc in enumerate(INC3):
        cls = CLASS[md]
        rows = sorted({e for e, _, _ in inc})
        out.append(f"  {{  /* mode {MODES[md]} */")
        for e in rows:
            terms = [f"V[{k}][{v}]" for (ee, k, v) in inc if ee == e]
            out.append(f"    const double e{e} = {' + '.join(terms)};")
        if iso:
            out.append(f"    const double fl = mat[{cls * 3}], f2m = mat[{cls * 3 + 1}], fm = mat[{cls * 3 + 2}];")
            normals = [e for e in rows if e < 3]
            if normals:
                out.append(f"    const double lt = fl * ({' + '.join(f'e{e}' for e in normals)});")
            for e in rows:
                if e < 3:
                    out.append(f"    const double t{e} = fma(f2m, e{e}, lt);")
                else:
                    out.append(f"    const double t{e} = fm * e{e};")
        else:
            for i in rows:
                acc = None
                for j in rows:
                    term = f"mat[{cls * 36 + i * 6 + j}]"
                    acc = f"{term} * e{j}" if acc is None else f"fma({term}, e{j}, {acc})"
                out.append(f"    const double t{i} = {acc};")
        for (e, k, v) in inc:
            out.append(f"    HB_ACC({k}, {v}, t{e});")
        out.append("  }")
    return "\n".join(out)


def gen_scalar(iso):
    out = []
    for md, inc in enumerate(INCS):
        cls = CLASS[md]
        dirs = [j for j, _ in inc]
        out.append(f"  {{  /* mode {MODES[md]} */")
        for j, v in inc:
            out.append(f"    const double g{j} = V[0][{v}];")
        if iso:
            for j, v in inc:
                out.append(f"    HB_ACC(0, {v}, mat[{cls}] * g{j});")
        else:
            for j, v in inc:
                acc = None
                for jj in dirs:
                    term = f"mat[{cls * 9 + j * 3 + jj}]"
                    acc = f"{term} * g{jj}" if acc is None else f"fma({term}, g{jj}, {acc})"
                out.append(f"    HB_ACC(0, {v}, {acc});")
        out.append("  }")
    return "\n".join(out)


def gen_fold(elastic, iso, modal=False):
    """Mode code for the z-march kernel with the residual folded into the
    z-adjoint: contribution t to modal slot (k, v) adds +-t to A[k][v % 4]
    (lower face, minus for v >= 4) and t to B[k][v % 4] (upper face). A is
    seeded by the caller; B is assigned on its first contribution. Scaled
    rows (isotropic shear, scalar) go straight into FMAs.

    modal=True: the contributions accumulate into the modal residual
    R[k][v] instead (one operation per contribution, assigned on the first;
    slots without contributions are zeroed at the end) and the caller forms
    A = seed + R[m] - R[m + 4], B = R[m] + R[m + 4]: 36 -> 21 + 10 per
    component fewer accumulations for elasticity."""
    out = []
    seen = set()

    def acc(k, v, t=None, scale=None, e=None):
        if modal:
            first = (k, v) not in seen
            seen.add((k, v))
            if t is not None:
                out.append(f"    R[{k}][{v}] {'=' if first else '+='} {t};")
            elif first:
                out.append(f"    R[{k}][{v}] = {scale} * {e};")
            else:
                out.append(f"    R[{k}][{v}] = fma({scale}, {e}, R[{k}][{v}]);")
            return
        m = v % 4
        sgn = "-" if v >= 4 else ""
        first = (k, m) not in seen
        seen.add((k, m))
        if t is not None:
            out.append(f"    A[{k}][{m}] {'-' if v >= 4 else '+'}= {t};")
            out.append(f"    B[{k}][{m}] {'=' if first else '+='} {t};")
        else:
            out.append(f"    A[{k}][{m}] = fma({sgn}{scale}, {e}, A[{k}][{m}]);")
            if first:
                out.append(f"    B[{k}][{m}] = {scale} * {e};")
            else:
                out.append(f"    B[{k}][{m}] = fma({scale}, {e}, B[{k}][{m}]);")

    if elastic:
        for md, inc in enumerate(INC3):
            cls = CLASS[md]
            if iso and modal and cls == 2:
                # the three doubly-antisymmetric modes only see V[k][7] (one
                # normal + two shear rows each, same class factor), so their
                # sum is R[k][7] = f (lambda + 2mu + 2 mu) V[k][7] = mat[9] V[k][7]
                if md == 4:
                    out.append("  {  /* modes aas + asa + saa */")
                    out.append("    const double c7 = mat[9];")
                    for k in range(3):
                        acc(k, 7, scale="c7", e=f"V[{k}][7]")
                    out.append("  }")
                continue
            rows = sorted({e for e, _, _ in inc})
            out.append(f"  {{  /* mode {MODES[md]} */")
            for e in rows:
                terms = [f"V[{k}][{v}]" for (ee, k, v) in inc if ee == e]
                out.append(f"    const double e{e} = {' + '.join(terms)};")
            if iso:
                out.append(f"    const double fl = mat[{cls * 3}], f2m = mat[{cls * 3 + 1}], fm = mat[{cls * 3 + 2}];")
                normals = [e for e in rows if e < 3]
                if normals:
                    out.append(f"    const double lt = fl * ({' + '.join(f'e{e}' for e in normals)});")
                for e in rows:
                    if e < 3:
                        out.append(f"    const double t{e} = fma(f2m, e{e}, lt);")
                for (e, k, v) in inc:
                    if e < 3:
                        acc(k, v, t=f"t{e}")
                    else:
                        acc(k, v, scale="fm", e=f"e{e}")
            else:
                for i in rows:
                    a = None
                    for j in rows:
                        term = f"mat[{cls * 36 + i * 6 + j}]"
                        a = f"{term} * e{j}" if a is None else f"fma({term}, e{j}, {a})"
                    out.append(f"    const double t{i} = {a};")
                for (e, k, v) in inc:
                    acc(k, v, t=f"t{e}")
            out.append("  }")
    else:
        for md, inc in enumerate(INCS):
            cls = CLASS[md]
            dirs = [j for j, _ in inc]
            out.append(f"  {{  /* mode {MODES[md]} */")
            for j, v in inc:
                out.append(f"    const double g{j} = V[0][{v}];")
            if iso:
                out.append(f"    const double kk = mat[{cls}];")
                for j, v in inc:
                    acc(0, v, scale="kk", e=f"g{j}")
            else:
                for j, v in inc:
                    a = None
                    for jj in dirs:
                        term = f"mat[{cls * 9 + j * 3 + jj}]"
                        a = f"{term} * g{jj}" if a is None else f"fma({term}, g{jj}, {a})"
                    out.append(f"    const double q{j} = {a};")
                    acc(0, v, t=f"q{j}")
            out.append("  }")
    if modal:
        for k in range(3 if elastic else 1):
            for v in range(1, 8):
                if (k, v) not in seen:
                    out.append(f"  R[{k}][{v}] = 0.0;")
    return "\n".join(out)


def gen_qt():
    """Per-Gauss-point tangents (J2 consistent tangents, compact form
    C_q = 3k V + 2G a Dev - b n n^T): modal strain rows -> strain at the 8
    Gauss points (sign patterns of the quad modes) -> stress -> projected
    back onto the modes -> residual contributions (same incidence as the
    linear mode code). Inputs V[k][v], qs[6] (mode scale x Mandel factor),
    qw[6] (= w qs), kq, gq (phase bulk / shear), lin (no per-point tangent),
    tq (8 x 8 compact tangents of this element)."""
    out = []
    terms = {}  # (md, row) -> raw expression
    for md, inc in enumerate(INC3):
        for e in sorted({e for e, _, _ in inc}):
            terms[(md, e)] = " + ".join(f"V[{k}][{v}]" for (ee, k, v) in inc if ee == e)
    out.append("  {")
    for (md, e), expr in terms.items():
        idx = CLASS[md] * 2 + (1 if e >= 3 else 0)
        out.append(f"    const double E{md}_{e} = qs[{idx}] * ({expr});")
    for (md, e) in terms:
        out.append(f"    double S{md}_{e} = 0.0;")
    # quad sign patterns: mode name letters per axis (0, 1, 2)
    for q in range(8):
        i, j, k = (q >> 2) & 1, (q >> 1) & 1, q & 1
        sg = [1 if i else -1, 1 if j else -1, 1 if k else -1]

        def phi(md):
            v = 1
            for a, ch in enumerate(MODES[md]):
                if ch == "a":
                    v *= sg[a]
            return v
        out.append(f"    {{  /* Gauss point ({i},{j},{k}) */")
        for r in range(6):
            parts = []
            for (md, e) in terms:
                if e != r:
                    continue
                parts.append(("+" if phi(md) > 0 else "-") + f" E{md}_{e}")
            expr = " ".join(parts).lstrip("+ ").strip()
            if expr.startswith("- "):
                expr = "-" + expr[2:]
            out.append(f"      const double ep{r} = {expr if expr else '0.0'};")
        out.append("      double ca = 1.0, cb = 0.0, n0 = 0.0, n1 = 0.0, n2 = 0.0, n3 = 0.0, n4 = 0.0, n5 = 0.0;")
        out.append(f"      if (!lin) {{ const double* t = tq + {q * 8}; ca = t[0]; cb = t[1]; n0 = t[2]; n1 = t[3]; "
                   "n2 = t[4]; n3 = t[5]; n4 = t[6]; n5 = t[7]; }")
        out.append("      const double tr = ep0 + ep1 + ep2, t3 = tr * (1.0 / 3.0);")
        out.append("      const double ne = n0 * ep0 + n1 * ep1 + n2 * ep2 + n3 * ep3 + n4 * ep4 + n5 * ep5;")
        out.append("      const double g2 = 2.0 * gq * ca, kt = kq * tr, bn = cb * ne;")
        for r in range(6):
            if r < 3:
                out.append(f"      const double sg{r} = fma(g2, ep{r} - t3, kt) - bn * n{r};")
            else:
                out.append(f"      const double sg{r} = fma(g2, ep{r}, -bn * n{r});")
        for (md, e) in terms:
            out.append(f"      S{md}_{e} {'+' if phi(md) > 0 else '-'}= sg{e};")
        out.append("    }")
    for (md, e) in terms:
        idx = CLASS[md] * 2 + (1 if e >= 3 else 0)
        out.append(f"    {{ const double tt = qw[{idx}] * S{md}_{e};")
        for (ee, k, v) in INC3[md]:
            if ee == e:
                out.append(f"      HB_ACC({k}, {v}, tt);")
        out.append("    }")
    out.append("  }")
    return "\n".join(out)


def gen_norm(elastic):
    """sum_q |eps_q + E|^2 / (8 w) over the quad modes (orthogonal patterns):
    mode m contributes sum_rows (sc * e_row (+ E_row for sss))^2, with
    sc[2 cls + shear] = per-class mode scale (x sqrt(2)/2 on Mandel shear rows)."""
    out = []
    tables = INC3 if elastic else [[(j, 0, v) for (j, v) in inc] for inc in INCS]
    for md, inc in enumerate(tables):
        cls = CLASS[md]
        rows = sorted({e for e, _, _ in inc})
        out.append(f"  {{  /* mode {MODES[md]} */")
        for e in rows:
            terms = [f"V[{k}][{v}]" for (ee, k, v) in inc if ee == e]
            idx = cls * 2 + (1 if (elastic and e >= 3) else 0)
            base = f"fma(sc[{idx}], {' + '.join(terms)}, E[{e}])" if md == 0 else f"sc[{idx}] * ({' + '.join(terms)})"
            out.append(f"    {{ const double t = {base}; nacc = fma(t, t, nacc); }}")
        out.append("  }")
    return "\n".join(out)


def gen_sss(elastic):
    """Mandel strain of the constant quad mode plus E (= the element's quad average)."""
    out = []
    inc = INC3[0] if elastic else [(j, 0, v) for (j, v) in INCS[0]]
    for e in sorted({e for e, _, _ in inc}):
        terms = [f"V[{k}][{v}]" for (ee, k, v) in inc if ee == e]
        idx = 1 if (elastic and e >= 3) else 0
        out.append(f"  es[{e}] = fma(sc[{idx}], {' + '.join(terms)}, E[{e}]);")
    return "\n".join(out)


def main():
    here = os.path.dirname(os.path.abspath(__file__))
    parts = ["// GENERATED by gen_hex_modes.py -- do not edit.",
             "// Per-quad-mode strain, material contraction and adjoint of the modal",
             "// hex kernel. Inputs V[k][v], table `mat`; HB_ACC(k, v, t) accumulates",
             "// t into modal residual (k, v) (defined by the including kernel).",
             "#define HB_HEX_MODES_ELASTIC_ISO \\"]
    for name, body in (("ELASTIC_ISO", gen_elastic(True)), ("ELASTIC_GEN", gen_elastic(False)),
                       ("SCALAR_ISO", gen_scalar(True)), ("SCALAR_GEN", gen_scalar(False)),
                       ("FOLD_ELASTIC_ISO", gen_fold(True, True)), ("FOLD_ELASTIC_GEN", gen_fold(True, False)),
                       ("FOLD_SCALAR_ISO", gen_fold(False, True)), ("FOLD_SCALAR_GEN", gen_fold(False, False)),
                       ("RFOLD_ELASTIC_ISO", gen_fold(True, True, True)),
                       ("RFOLD_SCALAR_ISO", gen_fold(False, True, True)),
                       ("QT_ELASTIC", gen_qt()),
                       ("NRM_ELASTIC", gen_norm(True)), ("NRM_SCALAR", gen_norm(False)),
                       ("SSS_ELASTIC", gen_sss(True)), ("SSS_SCALAR", gen_sss(False))):
        if name != "ELASTIC_ISO":
            parts.append(f"#define HB_HEX_MODES_{name} \\")
        lines = body.split("\n")
        parts.extend(line + " \\" for line in lines[:-1])
        parts.append(lines[-1])
        parts.append("")
    with open(os.path.join(here, "hex_modes.inc"), "w") as f:
        f.write("\n".join(parts))


if __name__ == "__main__":
    main()
