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
#include "spectral.cuh"

namespace hb {

namespace {

using namespace spec;

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

template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_spectral(const __grid_constant__ SpecParams p, double2* __restrict__ spec,
                                                     const PcgState* st, double* partials) {
  if (st && !st->active) return;
  const int64_t nf = p.nf;
  const int nl = D == 3 ? p.n2 : p.n1;
  double rz = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
    double2 r[C];
#pragma unroll
    for (int i = 0; i < C; ++i) r[i] = spec[i * nf + k];
    double2 z[C];
    int f[3];
    freq_index<D>(p, k, f);
    if ((f[0] == 0 && f[1] == 0 && f[2] == 0) ||  // zero frequency (a slab rank may not hold it)
        f[D - 1] >= p.nhv) {                       // padding column of a 2-D slab chunk

#pragma unroll
      for (int i = 0; i < C; ++i) z[i] = make_double2(0.0, 0.0);
    } else {
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
