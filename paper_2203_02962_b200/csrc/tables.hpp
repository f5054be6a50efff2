// tables.hpp -- host-side setup: stencil tables, per-phase element data and
// the reference-tangent tensor used by the analytic Fourier symbol.
//
// Stencil tables restate proj/src/grid.cpp:81-145 (BilinearQuad,
// TwoTriangles) and 190-229 (TrilinearHex); the Mandel gradient rows restate
// proj/src/operators.cpp:16-53. FourTrianglesTwoNode (grid.cpp:147-188, two
// node types: corner and pixel centre) is kind 2 of make_stencil (SURVEY.md
// section 8(f), row f3; its preconditioner blocks are probed in probe.cu).
#pragma once

#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace hb {

inline StencilParams make_stencil(int kind, int d, const double* h) {
  StencilParams s;
  std::memset(&s, 0, sizeof(s));
  s.nn = 1;
  const double vp = d == 2 ? h[0] * h[1] : h[0] * h[1] * h[2];
  static const int quad_off[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {1, 1, 0}};
  static const int hex_off[8][3] = {{0, 0, 0}, {0, 0, 1}, {0, 1, 0}, {0, 1, 1},
                                    {1, 0, 0}, {1, 0, 1}, {1, 1, 0}, {1, 1, 1}};
  auto set_entry = [&](int q, int e, int off, double d0, double d1, double d2) {
    s.off[q][e] = off;
    s.dphi[q][e][0] = d0;
    s.dphi[q][e][1] = d1;
    s.dphi[q][e][2] = d2;
  };
  if (kind == 1) {  // TwoTriangles: centroid rule on two linear triangles
    if (d != 2) throw ValidationError("stencil: two-triangles requires a 2d cell");
    s.nq = 2;
    s.noff = 4;
    std::memcpy(s.offs, quad_off, sizeof(quad_off));
    s.ne[0] = s.ne[1] = 3;
    s.w[0] = s.w[1] = vp / 2.0;
    set_entry(0, 0, 0, -1.0 / h[0], -1.0 / h[1], 0.0);
    set_entry(0, 1, 1, 1.0 / h[0], 0.0, 0.0);
    set_entry(0, 2, 2, 0.0, 1.0 / h[1], 0.0);
    set_entry(1, 0, 3, 1.0 / h[0], 1.0 / h[1], 0.0);
    set_entry(1, 1, 2, -1.0 / h[0], 0.0, 0.0);
    set_entry(1, 2, 1, 0.0, -1.0 / h[1], 0.0);
    return s;
  }
  const double gq = 0.5 / std::sqrt(3.0);
  const double gp[2] = {0.5 - gq, 0.5 + gq};
  if (kind == 0) {  // BilinearQuad, 2x2 Gauss
    if (d != 2) throw ValidationError("stencil: bilinear-quad requires a 2d cell");
    s.nq = 4;
    s.noff = 4;
    std::memcpy(s.offs, quad_off, sizeof(quad_off));
    int q = 0;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j, ++q) {
        s.w[q] = vp / 4.0;
        s.ne[q] = 4;
        const double x = gp[i], y = gp[j];
        const double xi[2] = {1.0 - x, x}, dxi[2] = {-1.0 / h[0], 1.0 / h[0]};
        const double et[2] = {1.0 - y, y}, det[2] = {-1.0 / h[1], 1.0 / h[1]};
        int e = 0;
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b, ++e) set_entry(q, e, a + 2 * b, dxi[a] * et[b], xi[a] * det[b], 0.0);
      }
    return s;
  }
  if (kind == 3) {  // TrilinearHex, 2x2x2 Gauss
    if (d != 3) throw ValidationError("stencil: trilinear-hex requires a 3d cell");
    s.nq = 8;
    s.noff = 8;
    std::memcpy(s.offs, hex_off, sizeof(hex_off));
    int q = 0;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        for (int k = 0; k < 2; ++k, ++q) {
          s.w[q] = vp / 8.0;
          s.ne[q] = 8;
          const double x = gp[i], y = gp[j], z = gp[k];
          const double xi[2] = {1.0 - x, x}, dxi[2] = {-1.0 / h[0], 1.0 / h[0]};
          const double et[2] = {1.0 - y, y}, det[2] = {-1.0 / h[1], 1.0 / h[1]};
          const double ze[2] = {1.0 - z, z}, dze[2] = {-1.0 / h[2], 1.0 / h[2]};
          int e = 0;
          for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
              for (int c = 0; c < 2; ++c, ++e)
                set_entry(q, e, (a * 2 + b) * 2 + c, dxi[a] * et[b] * ze[c], xi[a] * det[b] * ze[c],
                          xi[a] * et[b] * dze[c]);
        }
    return s;
  }
  if (kind == 2) {  // FourTrianglesTwoNode: four triangles fanned around the centre node
    if (d != 2) throw ValidationError("stencil: four-triangles-two-node requires a 2d cell");
    s.nq = 4;
    s.noff = 4;
    s.nn = 2;
    std::memcpy(s.offs, quad_off, sizeof(quad_off));
    const double h0 = h[0], h1 = h[1];
    auto tri = [&](int q, int o0, double a0, double a1, int o1, double b0, double b1, double c0, double c1) {
      s.w[q] = vp / 4.0;
      s.ne[q] = 3;
      set_entry(q, 0, o0, a0, a1, 0.0);
      set_entry(q, 1, o1, b0, b1, 0.0);
      set_entry(q, 2, 0, c0, c1, 0.0);
      s.node[q][2] = 1;
    };
    tri(0, 0, -1.0 / h0, -1.0 / h1, 1, 1.0 / h0, -1.0 / h1, 0.0, 2.0 / h1);   // bottom
    tri(1, 1, 1.0 / h0, -1.0 / h1, 3, 1.0 / h0, 1.0 / h1, -2.0 / h0, 0.0);    // right
    tri(2, 3, 1.0 / h0, 1.0 / h1, 2, -1.0 / h0, 1.0 / h1, 0.0, -2.0 / h1);    // top
    tri(3, 2, -1.0 / h0, 1.0 / h1, 0, -1.0 / h0, -1.0 / h1, 2.0 / h0, 0.0);   // left
    return s;
  }
  throw ValidationError("stencil: invalid kind");
}

// Gradient-row matrix of one quadrature point: B[k][loc*c + comp], the linear
// map from element corner values to the m gradient rows (operators.cpp:16-32).
inline void quad_rows(const StencilParams& s, int q, int d, int c, std::vector<double>& B) {
  const int m = c == 1 ? d : mandel_dim(d);
  const int nloc = s.noff;
  const double s2 = std::sqrt(2.0) / 2.0;
  B.assign(m * nloc * c, 0.0);
  auto at = [&](int k, int loc, int comp) -> double& { return B[k * nloc * c + loc * c + comp]; };
  for (int e = 0; e < s.ne[q]; ++e) {
    const int loc = s.off[q][e];
    const double* dp = s.dphi[q][e];
    if (c == 1) {
      for (int a = 0; a < d; ++a) at(a, loc, 0) += dp[a];
    } else if (d == 2) {
      at(0, loc, 0) += dp[0];
      at(1, loc, 1) += dp[1];
      at(2, loc, 0) += s2 * dp[1];
      at(2, loc, 1) += s2 * dp[0];
    } else {
      at(0, loc, 0) += dp[0];
      at(1, loc, 1) += dp[1];
      at(2, loc, 2) += dp[2];
      at(3, loc, 1) += s2 * dp[2];
      at(3, loc, 2) += s2 * dp[1];
      at(4, loc, 0) += s2 * dp[2];
      at(4, loc, 2) += s2 * dp[0];
      at(5, loc, 0) += s2 * dp[1];
      at(5, loc, 1) += s2 * dp[0];
    }
  }
}

// Element stiffness K_e = sum_q w_q B_q^T C B_q (row-major NE x NE, NE = nloc*c)
// of one phase with column-major m x m tangent C.
inline void element_matrix(const StencilParams& s, int d, int c, const double* cm, double* ke) {
  const int m = c == 1 ? d : mandel_dim(d);
  const int ne = s.noff * c;
  std::vector<double> B, CB(m * ne);
  for (int i = 0; i < ne * ne; ++i) ke[i] = 0.0;
  for (int q = 0; q < s.nq; ++q) {
    quad_rows(s, q, d, c, B);
    for (int k = 0; k < m; ++k)
      for (int j = 0; j < ne; ++j) {
        double acc = 0.0;
        for (int l = 0; l < m; ++l) acc += cm[l * m + k] * B[l * ne + j];
        CB[k * ne + j] = acc;
      }
    for (int i = 0; i < ne; ++i)
      for (int j = 0; j < ne; ++j) {
        double acc = 0.0;
        for (int k = 0; k < m; ++k) acc += B[k * ne + i] * CB[k * ne + j];
        ke[i * ne + j] += s.w[q] * acc;
      }
  }
}

// Element load vector f_e = sum_q w_q B_q^T C e for a uniform macroscopic load.
inline void element_load(const StencilParams& s, int d, int c, const double* cm, const double* e,
                         double* fe) {
  const int m = c == 1 ? d : mandel_dim(d);
  const int ne = s.noff * c;
  std::vector<double> B;
  double ce[6];
  for (int i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int j = 0; j < m; ++j) acc += cm[j * m + i] * e[j];
    ce[i] = acc;
  }
  for (int i = 0; i < ne; ++i) fe[i] = 0.0;
  for (int q = 0; q < s.nq; ++q) {
    quad_rows(s, q, d, c, B);
    for (int i = 0; i < ne; ++i) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += B[k * ne + i] * ce[k];
      fe[i] += s.w[q] * acc;
    }
  }
}

// Fourth-order tensor A_ijkl (d^4, index ((i*d+j)*d+k)*d+l) of a Mandel
// stiffness (inverse of proj/src/mandel.cpp:49-72), for the Fourier symbol
// K_hat_ik = sum_jl A_ijkl M_jl.
inline void mandel_to_tensor(const double* cm, int d, double* A) {
  static const int p2[3][2] = {{0, 0}, {1, 1}, {0, 1}};
  static const int p3[6][2] = {{0, 0}, {1, 1}, {2, 2}, {1, 2}, {0, 2}, {0, 1}};
  const int m = mandel_dim(d);
  auto idx = [&](int i, int j) {
    for (int a = 0; a < m; ++a) {
      const int* pr = d == 2 ? p2[a] : p3[a];
      if ((pr[0] == i && pr[1] == j) || (pr[0] == j && pr[1] == i)) return a;
    }
    return -1;
  };
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      for (int k = 0; k < d; ++k)
        for (int l = 0; l < d; ++l) {
          const int a = idx(i, j), b = idx(k, l);
          const double sa = i == j ? 1.0 : std::sqrt(2.0);
          const double sb = k == l ? 1.0 : std::sqrt(2.0);
          A[((i * d + j) * d + k) * d + l] = cm[b * m + a] / (sa * sb);
        }
}

// isotropic_stiffness (proj/src/mandel.cpp:114-134): 3K P_vol + 2G P_dev,
// plane strain restriction (11, 22, 12) in 2-D. Column-major output.
inline void isotropic_stiffness(double K, double G, int d, double* out) {
  if (d != 2 && d != 3) throw ValidationError("mandel: dimension must be 2 or 3");
  if (!(K > 0.0) || !(G > 0.0)) throw ValidationError("isotropic_stiffness: moduli must be positive");
  double c3[36];
  const double tk = 3.0 * K, tg = 2.0 * G;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) {
      const double pv = (i < 3 ? 1.0 : 0.0) * (j < 3 ? 1.0 : 0.0) / 3.0;
      const double pd = (i == j ? 1.0 : 0.0) - pv;
      c3[j * 6 + i] = tk * pv + tg * pd;
    }
  if (d == 3) {
    std::memcpy(out, c3, sizeof(c3));
    return;
  }
  const int idx[3] = {0, 1, 5};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) out[b * 3 + a] = c3[idx[b] * 6 + idx[a]];
}

// Symmetric (1e-10 relative) and Cholesky-positive check
// (material.cpp:13-29, precond.cpp:13-24).
inline void check_spd(const double* a, int n, const char* what) {
  double scale = 0.0, asym = 0.0;
  for (int i = 0; i < n * n; ++i) scale = std::fmax(scale, std::fabs(a[i]));
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) asym = std::fmax(asym, std::fabs(a[j * n + i] - a[i * n + j]));
  if (asym > 1e-10 * scale) throw ValidationError(std::string(what) + ": non-symmetric tangent rejected");
  std::vector<double> l(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double dsum = a[j * n + j];
    for (int k = 0; k < j; ++k) dsum -= l[k * n + j] * l[k * n + j];
    if (!(dsum > 0.0)) throw ValidationError(std::string(what) + ": matrix must be positive definite");
    const double ljj = std::sqrt(dsum);
    l[j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = a[j * n + i];
      for (int k = 0; k < j; ++k) s -= l[k * n + i] * l[k * n + j];
      l[j * n + i] = s / ljj;
    }
  }
}

}  // namespace hb
