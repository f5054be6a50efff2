// spectral.cu -- the Fourier-space half of M^-1 = F^-1 K_ref_hat^+ F.
//
// The reference assembles K_ref_hat(xi) by impulse probing (c*Nn operator
// sweeps plus (c*Nn)^2 FFTs, precond.cpp:44-85), inverts every block by a
// Hermitian eigendecomposition (precond.cpp:87-124) and stores c^2 complex
// numbers per frequency. For the one-node stencils on the GPU path the
// symbol is a closed form of the per-axis phases, real and symmetric:
//
//   K_hat_ik(xi) = sum_jl A_ijkl M_jl(xi),  M_jl = sum_q w_q conj(g_j(q)) g_l(q)
//
// with g(q) = sum_entries dphi e^{i theta . off} the gradient symbol of quad q.
// Per stencil (t_a = 2 pi k_a / N_a, s_a = sin(t_a/2), S2_a = 2 - 4/3 s_a^2):
//   TrilinearHex  M_aa = 8 w s_a^2/h_a^2 S2_b S2_c,  M_ab = 4 w sin t_a sin t_b/(h_a h_b) S2_c
//   BilinearQuad  M_aa = 8 w s_a^2/h_a^2 S2_b,       M_01 = 4 w sin t_0 sin t_1/(h_0 h_1)
//   TwoTriangles  M_aa = 8 w s_a^2/h_a^2,
//                 M_01 = 4 w (s_0^2 + s_1^2 - sin^2((t_0 - t_1)/2))/(h_0 h_1)
// so the preconditioner streams only r_hat in and z_hat out (no block reads),
// and the zero-frequency pseudo-inverse is exactly 0 (B_0 = 0, kernel = all
// translations). r.z is accumulated in the same pass by Parseval's identity.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void block_sum1(double v, double* out) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double s = lane < nw ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) *out = s;
  }
}

template <int D>
__device__ __forceinline__ void freq_index(const SpecParams& p, int64_t k, int (&f)[3]) {
  if (D == 3) {
    f[2] = (int)(k % p.nh);
    const int64_t t = k / p.nh;
    f[1] = (int)(t % p.n1);
    f[0] = (int)(t / p.n1);
  } else {
    f[1] = (int)(k % p.nh);
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
  const double w = p.w;
  if (p.kind == 3) {  // trilinear hex
    M[0][0] = 8.0 * w * sh[0] * sh[0] / (p.h[0] * p.h[0]) * S2[1] * S2[2];
    M[1][1] = 8.0 * w * sh[1] * sh[1] / (p.h[1] * p.h[1]) * S2[0] * S2[2];
    M[2][2] = 8.0 * w * sh[2] * sh[2] / (p.h[2] * p.h[2]) * S2[0] * S2[1];
    M[0][1] = M[1][0] = 4.0 * w * sn[0] * sn[1] / (p.h[0] * p.h[1]) * S2[2];
    M[0][2] = M[2][0] = 4.0 * w * sn[0] * sn[2] / (p.h[0] * p.h[2]) * S2[1];
    M[1][2] = M[2][1] = 4.0 * w * sn[1] * sn[2] / (p.h[1] * p.h[2]) * S2[0];
  } else if (p.kind == 0) {  // bilinear quad
    M[0][0] = 8.0 * w * sh[0] * sh[0] / (p.h[0] * p.h[0]) * S2[1];
    M[1][1] = 8.0 * w * sh[1] * sh[1] / (p.h[1] * p.h[1]) * S2[0];
    M[0][1] = M[1][0] = 4.0 * w * sn[0] * sn[1] / (p.h[0] * p.h[1]);
  } else {  // two triangles
    const double sd = sh[0] * ch[1] - ch[0] * sh[1];  // sin((t0 - t1)/2)
    M[0][0] = 8.0 * w * sh[0] * sh[0] / (p.h[0] * p.h[0]);
    M[1][1] = 8.0 * w * sh[1] * sh[1] / (p.h[1] * p.h[1]);
    M[0][1] = M[1][0] = 4.0 * w * (sh[0] * sh[0] + sh[1] * sh[1] - sd * sd) / (p.h[0] * p.h[1]);
  }
}

// K_hat (C x C symmetric) from M and the reference tangent.
template <int D, int C>
__device__ __forceinline__ void symbol(const SpecParams& p, const double (&M)[3][3], double (&K)[3][3]) {
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

template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_spectral(const __grid_constant__ SpecParams p, double2* __restrict__ spec,
                                                     const PcgState* st, double* partials) {
  if (st && st->done) return;
  const int64_t nf = p.nf;
  const int nl = D == 3 ? p.n2 : p.n1;
  double rz = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
    double2 r[C];
#pragma unroll
    for (int i = 0; i < C; ++i) r[i] = spec[i * nf + k];
    double2 z[C];
    if (k == 0) {
#pragma unroll
      for (int i = 0; i < C; ++i) z[i] = make_double2(0.0, 0.0);
    } else {
      int f[3];
      freq_index<D>(p, k, f);
      double M[3][3], K[3][3], I[3][3];
      gram<D>(p, f, M);
      symbol<D, C>(p, M, K);
      sym_inverse<C>(K, I);
#pragma unroll
      for (int i = 0; i < C; ++i) {
        double zr = 0.0, zi = 0.0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
          zr = fma(I[i][j], r[j].x, zr);
          zi = fma(I[i][j], r[j].y, zi);
        }
        z[i] = make_double2(zr * p.inv_np, zi * p.inv_np);
      }
      const int fl = D == 3 ? f[2] : f[1];
      const double wgt = (fl == 0 || (2 * fl == nl)) ? 1.0 : 2.0;
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < C; ++i) s += r[i].x * z[i].x + r[i].y * z[i].y;
      rz = fma(wgt, s, rz);
    }
#pragma unroll
    for (int i = 0; i < C; ++i) spec[i * nf + k] = z[i];
  }
  if (partials) block_sum1(rz, partials + blockIdx.x);
}

// Per block: max over frequencies k >= 1 of [lambda_min <= 1e-12 lambda_max]
// (precond.cpp:108-117) -- written as 1.0 / 0.0.
template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_symbol_check(const __grid_constant__ SpecParams p, double* partials) {
  double bad = 0.0;
  for (int64_t k = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.nf; k += (int64_t)gridDim.x * blockDim.x) {
    int f[3];
    freq_index<D>(p, k, f);
    double M[3][3], K[3][3];
    gram<D>(p, f, M);
    symbol<D, C>(p, M, K);
    double lmin, lmax;
    sym_eig_range<C>(K, lmin, lmax);
    if (!(lmin > 1e-12 * fabs(lmax))) bad = 1.0;
  }
  block_sum1(bad, partials + blockIdx.x);
}

template <int D, int C>
__global__ void k_symbol_dump(const __grid_constant__ SpecParams p, double2* blocks) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < p.nf; k += (int64_t)gridDim.x * blockDim.x) {
    int f[3];
    freq_index<D>(p, k, f);
    double M[3][3], K[3][3];
    gram<D>(p, f, M);
    symbol<D, C>(p, M, K);
#pragma unroll
    for (int i = 0; i < C; ++i)
#pragma unroll
      for (int j = 0; j < C; ++j) blocks[(k * C + i) * C + j] = make_double2(k == 0 ? 0.0 : K[i][j], 0.0);
  }
}

}  // namespace

#define HB_SPEC_DISPATCH(KERNEL, ...)                                                     \
  do {                                                                                    \
    if (p.d == 2 && p.c == 1) KERNEL<2, 1><<<kRedBlocks, kBlock, 0, s>>>(__VA_ARGS__);    \
    else if (p.d == 2 && p.c == 2) KERNEL<2, 2><<<kRedBlocks, kBlock, 0, s>>>(__VA_ARGS__); \
    else if (p.d == 3 && p.c == 1) KERNEL<3, 1><<<kRedBlocks, kBlock, 0, s>>>(__VA_ARGS__); \
    else if (p.d == 3 && p.c == 3) KERNEL<3, 3><<<kRedBlocks, kBlock, 0, s>>>(__VA_ARGS__); \
    else throw ValidationError("spectral: unsupported dimension/components");            \
    HB_CUDA(cudaGetLastError());                                                          \
  } while (0)

void launch_spectral(const SpecParams& p, double2* spec, const PcgState* st, double* partials, cudaStream_t s) {
  HB_SPEC_DISPATCH(k_spectral, p, spec, st, partials);
}

void launch_symbol_check(const SpecParams& p, double* partials, cudaStream_t s) {
  HB_SPEC_DISPATCH(k_symbol_check, p, partials);
}

void launch_symbol_dump(const SpecParams& p, double2* blocks, cudaStream_t s) {
  HB_SPEC_DISPATCH(k_symbol_dump, p, blocks);
}

}  // namespace hb
