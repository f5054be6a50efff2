// spectral.cuh -- analytic Fourier symbol of the reference operator for the
// one-node stencils and its closed-form inverse (see spectral.cu header for
// the formulas and their derivation from precond.cpp:44-124).
#pragma once

#include "kernels.cuh"

namespace hb {
namespace spec {

template <int D>
__device__ __forceinline__ void freq_index(const SpecParams& p, int64_t k, int (&f)[3]) {
  if (p.nf < (int64_t(1) << 31)) {  // 32-bit index arithmetic (every single-GPU config)
    const unsigned kk = (unsigned)k, nh = (unsigned)p.nh;
    if (D == 3) {
      const unsigned t = kk / nh, n1r = (unsigned)p.n1r;
      f[2] = (int)(kk - t * nh);
      const unsigned t0 = t / n1r;
      f[1] = p.k1off + (int)(t - t0 * n1r);
      f[0] = (int)t0;
    } else {  // 2-D: k1off = the first column held (a slab rank's column chunk; 0 on one device)
      const unsigned t = kk / nh;
      f[1] = p.k1off + (int)(kk - t * nh);
      f[0] = (int)t;
      f[2] = 0;
    }
    return;
  }
  if (D == 3) {
    f[2] = (int)(k % p.nh);
    const int64_t t = k / p.nh;
    f[1] = p.k1off + (int)(t % p.n1r);
    f[0] = (int)(t / p.n1r);
  } else {
    f[1] = p.k1off + (int)(k % p.nh);
    f[0] = (int)(k / p.nh);
    f[2] = 0;
  }
}

// Symmetric gradient Gram matrix M(xi) (D x D, row-major).
template <int D>
__device__ __forceinline__ void gram(const SpecParams& p, const int (&f)[3], double (&M)[3][3]) {
  double sn[3], sh[3], ch[3], S2[3];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double4 t = p.tab[a][f[a]];
    sn[a] = t.x;
    sh[a] = t.z;
    ch[a] = t.w;
    S2[a] = 2.0 - (4.0 / 3.0) * sh[a] * sh[a];
  }
  // (host-precomputed factors: no divisions per frequency)
  if (p.kind == 3) {  // trilinear hex
    M[0][0] = p.cd[0] * sh[0] * sh[0] * S2[1] * S2[2];
    M[1][1] = p.cd[1] * sh[1] * sh[1] * S2[0] * S2[2];
    M[2][2] = p.cd[2] * sh[2] * sh[2] * S2[0] * S2[1];
    M[0][1] = M[1][0] = p.co[0][1] * sn[0] * sn[1] * S2[2];
    M[0][2] = M[2][0] = p.co[0][2] * sn[0] * sn[2] * S2[1];
    M[1][2] = M[2][1] = p.co[1][2] * sn[1] * sn[2] * S2[0];
  } else if (p.kind == 0) {  // bilinear quad
    M[0][0] = p.cd[0] * sh[0] * sh[0] * S2[1];
    M[1][1] = p.cd[1] * sh[1] * sh[1] * S2[0];
    M[0][1] = M[1][0] = p.co[0][1] * sn[0] * sn[1];
  } else {  // two triangles
    const double sd = sh[0] * ch[1] - ch[0] * sh[1];  // sin((t0 - t1)/2)
    M[0][0] = p.cd[0] * sh[0] * sh[0];
    M[1][1] = p.cd[1] * sh[1] * sh[1];
    M[0][1] = M[1][0] = p.co[0][1] * (sh[0] * sh[0] + sh[1] * sh[1] - sd * sd);
  }
}

// K_hat (C x C symmetric) from M and the reference tangent.
template <int D, int C>
__device__ __forceinline__ void symbol(const SpecParams& p, const double (&M)[3][3], double (&K)[3][3]) {
  if (p.iso) {
    // isotropic C_ref: A_ijkl = lam d_ij d_kl + mu (d_ik d_jl + d_il d_jk)
    double tr = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) tr += M[j][j];
    if (C == 1) {
      K[0][0] = p.mu * tr;
    } else {
      const double lm = p.lam + p.mu, mt = p.mu * tr;
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int k = 0; k < D; ++k) K[i][k] = lm * M[i][k] + (i == k ? mt : 0.0);
    }
    return;
  }
  if (C == 1) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j)
#pragma unroll
      for (int l = 0; l < D; ++l) s += p.A[j * D + l] * M[j][l];
    K[0][0] = s;
  } else {
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int k = i; k < D; ++k) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j)
#pragma unroll
          for (int l = 0; l < D; ++l) s += p.A[((i * D + j) * D + k) * D + l] * M[j][l];
        K[i][k] = s;
        K[k][i] = s;
      }
  }
}

// Inverse of a symmetric C x C matrix (adjugate / determinant).
template <int C>
__device__ __forceinline__ void sym_inverse(const double (&K)[3][3], double (&I)[3][3]) {
  if (C == 1) {
    I[0][0] = 1.0 / K[0][0];
  } else if (C == 2) {
    const double inv = 1.0 / (K[0][0] * K[1][1] - K[0][1] * K[0][1]);
    I[0][0] = K[1][1] * inv;
    I[1][1] = K[0][0] * inv;
    I[0][1] = I[1][0] = -K[0][1] * inv;
  } else {
    const double c00 = K[1][1] * K[2][2] - K[1][2] * K[1][2];
    const double c01 = K[0][2] * K[1][2] - K[0][1] * K[2][2];
    const double c02 = K[0][1] * K[1][2] - K[0][2] * K[1][1];
    const double c11 = K[0][0] * K[2][2] - K[0][2] * K[0][2];
    const double c12 = K[0][1] * K[0][2] - K[0][0] * K[1][2];
    const double c22 = K[0][0] * K[1][1] - K[0][1] * K[0][1];
    const double inv = 1.0 / (K[0][0] * c00 + K[0][1] * c01 + K[0][2] * c02);
    I[0][0] = c00 * inv;
    I[0][1] = I[1][0] = c01 * inv;
    I[0][2] = I[2][0] = c02 * inv;
    I[1][1] = c11 * inv;
    I[1][2] = I[2][1] = c12 * inv;
    I[2][2] = c22 * inv;
  }
}

// Eigenvalue range of a symmetric C x C matrix (closed forms).
template <int C>
__device__ __forceinline__ void sym_eig_range(const double (&K)[3][3], double& lmin, double& lmax) {
  if (C == 1) {
    lmin = lmax = K[0][0];
  } else if (C == 2) {
    const double m = 0.5 * (K[0][0] + K[1][1]);
    const double d = 0.5 * (K[0][0] - K[1][1]);
    const double r = sqrt(d * d + K[0][1] * K[0][1]);
    lmin = m - r;
    lmax = m + r;
  } else {
    const double p1 = K[0][1] * K[0][1] + K[0][2] * K[0][2] + K[1][2] * K[1][2];
    const double q = (K[0][0] + K[1][1] + K[2][2]) / 3.0;
    const double a0 = K[0][0] - q, a1 = K[1][1] - q, a2 = K[2][2] - q;
    const double p2 = a0 * a0 + a1 * a1 + a2 * a2 + 2.0 * p1;
    const double pp = sqrt(p2 / 6.0);
    if (pp == 0.0) {
      lmin = lmax = q;
      return;
    }
    const double b00 = a0 / pp, b11 = a1 / pp, b22 = a2 / pp;
    const double b01 = K[0][1] / pp, b02 = K[0][2] / pp, b12 = K[1][2] / pp;
    double r = 0.5 * (b00 * (b11 * b22 - b12 * b12) - b01 * (b01 * b22 - b12 * b02) + b02 * (b01 * b12 - b11 * b02));
    r = fmin(1.0, fmax(-1.0, r));
    const double phi = acos(r) / 3.0;
    lmax = q + 2.0 * pp * cos(phi);
    lmin = q + 2.0 * pp * cos(phi + 2.0943951023931954923);
  }
}

}  // namespace spec
}  // namespace hb
