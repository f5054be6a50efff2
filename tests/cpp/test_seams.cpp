// Operator-level seams of include/homfe/gpu.hpp against dense oracles built
// through the same API, restating the reference's own test cases:
//   * "fused operator equals the dense triple product"
//     (proj/tests/test_operators.cpp:168-193): K u == D^T W C D u (1e-12),
//     identity tangent == divergence(gradient(u)) (1e-13);
//   * "preconditioner application" (proj/tests/test_precond.cpp:201-252):
//     zero in / zero out, translations annihilated, M^-1 == pinv(K_ref) on a
//     zero-mean r (1e-10), K_ref M^-1 b == b for b = -D^T W s (1e-10),
//     symmetry and positive semi-definiteness;
//   * pcg_solve with an IterateObserver (solver.cpp:50-97): one observer call
//     per iteration, last observed iterate == x before mean removal;
//   * weighted_norm / volume_average of a constant field;
//   * FourTrianglesTwoNode newton_solve through the shim (nodes = 2 N_p: the
//     u buffer is sized by GridLayout::num_nodes).
// Prints "OK <name>" per case; exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

#include "homfe/gpu.hpp"

using namespace homfe;

namespace {

std::mt19937_64 gen(20230302);
double uni() { return (double)(gen() >> 11) * 0x1.0p-53 * 2.0 - 1.0; }

int fails = 0;
void check(bool ok, const char* what, double v) {
  if (!ok) {
    std::printf("FAIL %s (%.3e)\n", what, v);
    ++fails;
  }
}

double maxabs(const std::vector<double>& a) {
  double m = 0.0;
  for (double v : a) m = std::fmax(m, std::fabs(v));
  return m;
}

std::vector<double> spd(int m) {
  std::vector<double> a(m * m), c(m * m, 0.0);
  for (double& v : a) v = uni();
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      for (int k = 0; k < m; ++k) c[j * m + i] += a[k * m + i] * a[k * m + j];
      if (i == j) c[j * m + i] += 0.5;
    }
  return c;
}

// dense m x n matrix of a linear map by unit vectors
template <class F>
std::vector<double> dense(int rows, int cols, F&& apply) {
  std::vector<double> out(static_cast<std::size_t>(rows) * cols), e(cols, 0.0), col;
  for (int j = 0; j < cols; ++j) {
    std::fill(e.begin(), e.end(), 0.0);
    e[j] = 1.0;
    col = apply(e);
    for (int i = 0; i < rows; ++i) out[static_cast<std::size_t>(i) * cols + j] = col[i];
  }
  return out;
}

// (A + V V^T)^-1 - V V^T: pinv of a symmetric PSD A whose kernel is spanned
// by the orthonormal columns of V (the c component translations)
std::vector<double> pinv_translations(std::vector<double> a, int n, int c, Index nodes) {
  std::vector<double> vvt(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      if (i / nodes == j / nodes) vvt[static_cast<std::size_t>(i) * n + j] = 1.0 / (double)nodes;
  (void)c;
  for (std::size_t i = 0; i < a.size(); ++i) a[i] += vvt[i];
  std::vector<double> inv(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) inv[static_cast<std::size_t>(i) * n + i] = 1.0;
  for (int col = 0; col < n; ++col) {  // Gauss-Jordan, partial pivoting
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(a[(std::size_t)r * n + col]) > std::fabs(a[(std::size_t)piv * n + col])) piv = r;
    for (int k = 0; k < n; ++k) {
      std::swap(a[(std::size_t)col * n + k], a[(std::size_t)piv * n + k]);
      std::swap(inv[(std::size_t)col * n + k], inv[(std::size_t)piv * n + k]);
    }
    const double d = a[(std::size_t)col * n + col];
    for (int k = 0; k < n; ++k) {
      a[(std::size_t)col * n + k] /= d;
      inv[(std::size_t)col * n + k] /= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double f = a[(std::size_t)r * n + col];
      if (f == 0.0) continue;
      for (int k = 0; k < n; ++k) {
        a[(std::size_t)r * n + k] -= f * a[(std::size_t)col * n + k];
        inv[(std::size_t)r * n + k] -= f * inv[(std::size_t)col * n + k];
      }
    }
  }
  for (std::size_t i = 0; i < inv.size(); ++i) inv[i] -= vvt[i];
  return inv;
}

std::vector<double> matvec(const std::vector<double>& a, const std::vector<double>& x) {
  const std::size_t n = x.size();
  std::vector<double> y(a.size() / n, 0.0);
  for (std::size_t i = 0; i < y.size(); ++i)
    for (std::size_t j = 0; j < n; ++j) y[i] += a[i * n + j] * x[j];
  return y;
}

void operators_and_precond(const GridLayout& g, int c) {
  const int d = g.dim(), m = c == 1 ? d : d * (d + 1) / 2;
  const Index nodes = g.num_nodes(), nq = g.num_quads();
  const int n = c * (int)nodes, nqm = (int)nq * m;
  // two-phase linear map (pixel-constant tangents)
  MaterialMap map;
  const std::vector<double> c0 = spd(m), c1 = spd(m);
  const bool thermal = c == 1;
  map.catalog = {thermal ? MaterialModel::conductivity(c0, d) : MaterialModel::linear_elastic(c0, d),
                 thermal ? MaterialModel::conductivity(c1, d) : MaterialModel::linear_elastic(c1, d)};
  map.phase.resize(static_cast<std::size_t>(g.num_pixels()));
  for (std::size_t p = 0; p < map.phase.size(); ++p) map.phase[p] = (p * 7 + 3) % 5 < 2 ? 1 : 0;
  // dense D (nq m x n) and W
  const std::vector<double> D = dense(nqm, n, [&](const std::vector<double>& e) {
    NodalField u(c, nodes);
    u.data = e;
    return gradient_apply(g, u).data;
  });
  const double w = g.cell().cell_volume() / (double)g.num_pixels() / g.quads_per_pixel();
  NodalField u(c, nodes);
  for (double& v : u.data) v = uni();
  // K u vs D^T W C D u
  const std::vector<double> du = matvec(D, u.data);
  std::vector<double> s(du.size());
  for (Index q = 0; q < nq; ++q) {
    const std::vector<double>& cm = map.phase[q / g.quads_per_pixel()] ? c1 : c0;
    for (int i = 0; i < m; ++i) {
      double acc = 0.0;
      for (int j = 0; j < m; ++j) acc += cm[j * m + i] * du[q * m + j];
      s[q * m + i] = w * acc;
    }
  }
  std::vector<double> kd(n, 0.0);
  for (int i = 0; i < nqm; ++i)
    for (int j = 0; j < n; ++j) kd[j] += D[(std::size_t)i * n + j] * s[i];
  const NodalField ku = apply_tangent_operator(g, map, u);
  double err = 0.0;
  for (int i = 0; i < n; ++i) err = std::fmax(err, std::fabs(ku.data[i] - kd[i]));
  check(err < 1e-12 * std::fmax(1.0, maxabs(kd)), "K == D^T W C D", err);
  // a general per-quadrature TangentField (random, non-symmetric block at every
  // point, test_operators.cpp:168-193): fused operator == D^T W C_q D u
  {
    TangentField tf(m, nq);
    for (double& v : tf.data) v = uni();
    std::vector<double> sq(du.size());
    for (Index q = 0; q < nq; ++q)
      for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int j = 0; j < m; ++j) acc += tf.block(q)[j * m + i] * du[q * m + j];
        sq[q * m + i] = w * acc;
      }
    std::vector<double> kq(n, 0.0);
    for (int i = 0; i < nqm; ++i)
      for (int j = 0; j < n; ++j) kq[j] += D[(std::size_t)i * n + j] * sq[i];
    const NodalField kt = apply_tangent_operator(g, tf, u);
    double e2 = 0.0;
    for (int i = 0; i < n; ++i) e2 = std::fmax(e2, std::fabs(kt.data[i] - kq[i]));
    check(e2 < 1e-12 * std::fmax(1.0, maxabs(kq)), "general TangentField: K == D^T W C_q D", e2);
  }
  // identity tangent: fused == divergence(gradient(u))
  std::vector<double> id(m * m, 0.0);
  for (int i = 0; i < m; ++i) id[i * m + i] = 1.0;
  MaterialMap idmap;
  idmap.catalog = {thermal ? MaterialModel::conductivity(id, d) : MaterialModel::linear_elastic(id, d)};
  idmap.phase.assign(static_cast<std::size_t>(g.num_pixels()), 0);
  const NodalField a = apply_tangent_operator(g, idmap, u);
  const NodalField b = divergence_apply(g, gradient_apply(g, u));
  err = 0.0;
  for (int i = 0; i < n; ++i) err = std::fmax(err, std::fabs(a.data[i] - b.data[i]));
  check(err < 1e-13 * std::fmax(1.0, maxabs(b.data)), "identity tangent == div(grad)", err);

  // preconditioner
  const std::vector<double> cref = spd(m);
  const FrequencyBlockDiag inv = invert_blocks(assemble_reference(g, cref, c));
  NodalField zero(c, nodes);
  check(maxabs(apply_preconditioner(g, inv, zero).data) == 0.0, "zero in, zero out", 0.0);
  NodalField tr(c, nodes);
  for (int k = 0; k < c; ++k)
    for (Index i = 0; i < nodes; ++i) tr(k, i) = 1.0 + 0.5 * k;
  const double mt = maxabs(apply_preconditioner(g, inv, tr).data);
  check(mt < 1e-12, "translations annihilated", mt);
  // dense K_ref and its pseudo-inverse
  MaterialMap refmap;
  refmap.catalog = {thermal ? MaterialModel::conductivity(cref, d) : MaterialModel::linear_elastic(cref, d)};
  refmap.phase.assign(static_cast<std::size_t>(g.num_pixels()), 0);
  const std::vector<double> kref = dense(n, n, [&](const std::vector<double>& e) {
    NodalField v(c, nodes);
    v.data = e;
    return apply_tangent_operator(g, refmap, v).data;
  });
  const std::vector<double> pinv = pinv_translations(kref, n, c, nodes);
  NodalField r(c, nodes);
  for (double& v : r.data) v = uni();
  for (int k = 0; k < c; ++k) {
    double mean = 0.0;
    for (Index i = 0; i < nodes; ++i) mean += r(k, i);
    mean /= (double)nodes;
    for (Index i = 0; i < nodes; ++i) r(k, i) -= mean;
  }
  const NodalField z = apply_preconditioner(g, inv, r);
  const std::vector<double> zd = matvec(pinv, r.data);
  err = 0.0;
  for (int i = 0; i < n; ++i) err = std::fmax(err, std::fabs(z.data[i] - zd[i]));
  check(err < 1e-10 * std::fmax(1.0, maxabs(zd)), "M^-1 == pinv(K_ref)", err);
  // K_ref M^-1 b == b for b = -D^T W s
  QuadField sq(nq, m);
  for (double& v : sq.data) v = uni();
  NodalField bb = divergence_apply(g, sq);
  for (double& v : bb.data) v = -v;
  const NodalField kmb = apply_tangent_operator(g, refmap, apply_preconditioner(g, inv, bb));
  err = 0.0;
  for (int i = 0; i < n; ++i) err = std::fmax(err, std::fabs(kmb.data[i] - bb.data[i]));
  check(err < 1e-10 * maxabs(bb.data), "K_ref M^-1 b == b", err);
  // symmetry, PSD
  NodalField x(c, nodes), y(c, nodes);
  for (double& v : x.data) v = uni();
  for (double& v : y.data) v = uni();
  const NodalField mx = apply_preconditioner(g, inv, x), my = apply_preconditioner(g, inv, y);
  double xy = 0.0, yx = 0.0, xx = 0.0;
  for (int i = 0; i < n; ++i) {
    xy += x.data[i] * my.data[i];
    yx += y.data[i] * mx.data[i];
    xx += x.data[i] * mx.data[i];
  }
  check(std::fabs(xy - yx) < 1e-12 * (std::fabs(xy) + 1.0), "M^-1 symmetric", std::fabs(xy - yx));
  check(xx >= -1e-13, "M^-1 positive semi-definite", xx);
  // block(k) is the assembled symbol: block(0) vanishes (translations)
  const auto b0 = inv.block(0);
  double b0m = 0.0;
  for (const auto& v : b0) b0m = std::fmax(b0m, std::abs(v));
  check(b0m < 1e-12, "zero-frequency block vanishes", b0m);

  // pcg_solve with an observer
  int calls = 0;
  NodalField last;
  const PcgOutcome pc = pcg_solve(TangentOperator{&g, map}, inv, bb, 1e-10, 500, [&](const NodalField& xk) {
    ++calls;
    last = xk;
  });
  check(pc.converged, "pcg converged", (double)pc.iterations);
  check(calls == pc.iterations, "one observer call per iteration", (double)(calls - pc.iterations));
  check((int)pc.history.size() == pc.iterations + 1, "history length", (double)pc.history.size());
  const PcgOutcome plain = pcg_solve(TangentOperator{&g, map}, inv, bb, 1e-10, 500);
  err = 0.0;
  for (int i = 0; i < n; ++i) err = std::fmax(err, std::fabs(plain.x.data[i] - pc.x.data[i]));
  check(plain.iterations == pc.iterations && err == 0.0, "observed == plain PCG (bitwise)", err);
  // the last observed iterate is x before the final mean removal
  double dmean = 0.0;
  for (int k = 0; k < c; ++k) {
    double mo = 0.0, mx2 = 0.0;
    for (Index i = 0; i < nodes; ++i) {
      mo += last(k, i);
      mx2 += pc.x(k, i);
    }
    dmean = std::fmax(dmean, std::fabs(mx2) / (double)nodes);
    for (Index i = 0; i < nodes; ++i) {
      const double want = last(k, i) - mo / (double)nodes;
      err = std::fmax(err, std::fabs(pc.x(k, i) - want));
    }
  }
  check(err < 1e-13 * std::fmax(1.0, maxabs(pc.x.data)), "x == last observed iterate - mean", err);
  check(dmean < 1e-13 * std::fmax(1.0, maxabs(pc.x.data)), "x mean-free", dmean);

  // weighted_norm / volume_average of a constant field
  QuadField one(nq, m);
  for (Index q = 0; q < nq; ++q)
    for (int k = 0; k < m; ++k) one.vec(q)[k] = 1.0 + k;
  const double wn = weighted_norm(g, one);
  double want = 0.0;
  for (int k = 0; k < m; ++k) want += (1.0 + k) * (1.0 + k);
  want = std::sqrt(want * g.cell().cell_volume());
  check(std::fabs(wn - want) < 1e-13 * want, "weighted_norm", std::fabs(wn - want));
  const auto av = volume_average(g, one);
  double e2 = 0.0;
  for (int k = 0; k < m; ++k) e2 = std::fmax(e2, std::fabs(av[k] - (1.0 + k)));
  check(e2 < 1e-13, "volume_average", e2);
}

}  // namespace

int main() {
  try {
    {
      GridLayout g({{4, 3}, {1.0, 0.7}}, StencilKind::TwoTriangles);
      operators_and_precond(g, 1);
      operators_and_precond(g, 2);
      std::printf("OK two-triangles 4x3\n");
    }
    {
      GridLayout g({{3, 4}, {1.0, 1.3}}, StencilKind::BilinearQuad);
      operators_and_precond(g, 1);
      operators_and_precond(g, 2);
      std::printf("OK bilinear-quad 3x4\n");
    }
    {
      GridLayout g({{3, 2, 4}, {1.0, 0.8, 1.2}}, StencilKind::TrilinearHex);
      operators_and_precond(g, 1);
      operators_and_precond(g, 3);
      std::printf("OK trilinear-hex 3x2x4\n");
    }
    {
      // FourTrianglesTwoNode through newton_solve: u has 2 N_p nodes
      GridLayout g({{6, 8}, {1.0, 1.2}}, StencilKind::FourTrianglesTwoNode);
      MaterialMap map;
      map.catalog = {MaterialModel::isotropic_conductivity(1.0, 2), MaterialModel::isotropic_conductivity(20.0, 2)};
      map.phase.resize(48);
      for (std::size_t p = 0; p < 48; ++p) map.phase[p] = p % 3 == 1 ? 1 : 0;
      SolveConfig cfg;
      cfg.eta_cg = 1e-10;
      PrecondManager pm(ReferencePolicy::volume_mean(), 0.1, 1);
      const NewtonOutcome out = newton_solve(g, map, {1.0, 0.0}, cfg, pm);
      check(out.converged, "two-node newton converged", 0.0);
      check(out.u.nodes == 96 && out.u.data.size() == 96, "two-node u sized 2 N_p", (double)out.u.data.size());
      check(out.average_stress[0] > 1.0 && out.average_stress[0] < 20.0, "two-node <q> within bounds",
            out.average_stress[0]);
      check(pm.assemblies() == 1, "one assembly", (double)pm.assemblies());
      // a second solve with the same manager reuses the assembly (solver.cpp:120-142)
      const NewtonOutcome again = newton_solve(g, map, {0.0, 1.0}, cfg, pm);
      check(again.converged && pm.assemblies() == 1, "manager reused across solves", (double)pm.assemblies());
      std::printf("OK four-triangles-two-node newton_solve\n");
    }
  } catch (const std::exception& e) {
    std::printf("EXCEPTION %s\n", e.what());
    return 2;
  }
  if (fails) {
    std::printf("%d failures\n", fails);
    return 1;
  }
  std::printf("ALL OK\n");
  return 0;
}
