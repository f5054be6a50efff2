// j2.cu -- the nonlinear (J2 plasticity) Newton path on the GPU
// (SURVEY.md 8(f) row f1).
//
// The reference evaluates every Gauss point through MaterialModel::evaluate
// (proj/src/material.cpp:122-226: radial return in the 3-D Mandel space, the
// plane-strain embedding (11, 22, 12) -> slots (0, 1, 5) in 2-D) inside
// constitutive_sweep (proj/src/solver.cpp:144-169) and stores a full m x m
// TangentField per Gauss point (fields.hpp:64-82). Here:
//  * k_sweep: per pixel, gather the element corners, per Gauss point
//    eps = E + D u (operators.cpp:16-32 rows), evaluate the phase's model,
//    write the stress QuadField, the trial internal state (width 7, the
//    reference's InternalState layout) and a COMPACT consistent tangent
//    (a, b, n^): C = 3k V + 2G a D - b n^ n^T (material.cpp:163-170), 8
//    doubles per Gauss point instead of m^2; per-block partial sums of
//    sum_q w C_q (the volume-mean tangent of PrecondManager::ensure,
//    fields.cpp:52-61);
//  * k_tan_stress: the PCG operator's first half, sigma_q = C_q (D p)_q from
//    the compact tangent (linear phases: their catalog matrix); the second
//    half is the weighted divergence (operators.cpp:151-181).
// Fixed grids and fixed-order sums: deterministic.
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.cuh"

namespace hb {

namespace {

constexpr double kS32 = 1.2247448713915890491;  // sqrt(3/2)

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Mandel gradient rows at Gauss point q from the element corner values
// (operators.cpp:16-32 accumulate_rows).
template <int D, int C>
__device__ __forceinline__ void grad_rows(const StencilParams& sp, int q, const double (&uv)[8][3], double* gq) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  const double s2 = 0.70710678118654752440;
#pragma unroll
  for (int k = 0; k < M; ++k) gq[k] = 0.0;
  for (int en = 0; en < sp.ne[q]; ++en) {
    const double* dp = sp.dphi[q][en];
    const double* v = uv[sp.off[q][en]];
    if (C == 1) {
#pragma unroll
      for (int k = 0; k < D; ++k) gq[k] += dp[k] * v[0];
    } else if (D == 2) {
      gq[0] += dp[0] * v[0];
      gq[1] += dp[1] * v[1];
      gq[2] += s2 * (dp[1] * v[0] + dp[0] * v[1]);
    } else {
      gq[0] += dp[0] * v[0];
      gq[1] += dp[1] * v[1];
      gq[2] += dp[2] * v[2];
      gq[3] += s2 * (dp[2] * v[1] + dp[1] * v[2]);
      gq[4] += s2 * (dp[2] * v[0] + dp[0] * v[2]);
      gq[5] += s2 * (dp[1] * v[0] + dp[0] * v[1]);
    }
  }
}

template <int D>
__device__ __forceinline__ void embed6(const double* e, double* e6) {
  if (D == 3) {
#pragma unroll
    for (int i = 0; i < 6; ++i) e6[i] = e[i];
  } else {
    e6[0] = e[0];
    e6[1] = e[1];
    e6[2] = e6[3] = e6[4] = 0.0;
    e6[5] = e[2];
  }
}

template <int D>
__device__ __forceinline__ void extract(const double* s6, double* s) {
  if (D == 3) {
#pragma unroll
    for (int i = 0; i < 6; ++i) s[i] = s6[i];
  } else {
    s[0] = s6[0];
    s[1] = s6[1];
    s[2] = s6[5];
  }
}

// sigma6 = (3k V + 2G a Dev - b n n^T) e6   (V = m m^T / 3 with m = (1,1,1,0,0,0))
__device__ __forceinline__ void compact_apply(double k, double g, double a, double b, const double* n,
                                              const double* e6, double* s6) {
  const double tr = e6[0] + e6[1] + e6[2];
  double ne = 0.0;
#pragma unroll
  for (int i = 0; i < 6; ++i) ne = fma(n[i], e6[i], ne);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const double dev = e6[i] - (i < 3 ? tr / 3.0 : 0.0);
    s6[i] = (i < 3 ? k * tr : 0.0) + 2.0 * g * a * dev - b * n[i] * ne;
  }
}

template <int NV>
__device__ __forceinline__ void block_sum_store_nv(double (&v)[NV], double* out) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[i][warp] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NV; i += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[i][w];
    out[i] = s;
  }
}

template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_sweep(const Grid g, const __grid_constant__ StencilParams sp,
                                                   const NLArgs a) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  constexpr int NV = M * M;
  const int64_t np = g.np;
  double tacc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) tacc[i] = 0.0;
  double E[M];
#pragma unroll
  for (int k = 0; k < M; ++k) E[k] = a.e[k];
  int bad = 0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    int c0, c1, c2 = 0;
    if (D == 3) {
      c2 = (int)(p % g.n2);
      const int64_t t = p / g.n2;
      c1 = (int)(t % g.n1);
      c0 = (int)(t / g.n1);
    } else {
      c1 = (int)(p % g.n1);
      c0 = (int)(p / g.n1);
    }
    double uv[8][3];
    for (int o = 0; o < sp.noff; ++o) {
      const int i0 = wrapi(c0 + sp.offs[o][0], g.n0), i1 = wrapi(c1 + sp.offs[o][1], g.n1);
      const int i2 = D == 3 ? wrapi(c2 + sp.offs[o][2], g.n2) : 0;
      const int64_t nd = D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
#pragma unroll
      for (int k = 0; k < C; ++k) uv[o][k] = a.u ? a.u[k * np + nd] : 0.0;
    }
    const int ph = a.phase[p];
    const NLModel md = a.models[ph];
    for (int q = 0; q < sp.nq; ++q) {
      const int64_t qi = p * sp.nq + q;
      double eps[M];
      grad_rows<D, C>(sp, q, uv, eps);
#pragma unroll
      for (int k = 0; k < M; ++k) {
        eps[k] += E[k];
        if (!isfinite(eps[k])) bad = 1;
      }
      double sig[M];
      double Cq[NV];
      if (md.kind == 0) {
        const double* cm = a.cmat + (size_t)ph * NV;  // column-major
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < M; ++j) t = fma(cm[j * M + i], eps[j], t);
          sig[i] = t;
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) Cq[i] = cm[i];
        if (a.width) {
#pragma unroll
          for (int i = 0; i < 7; ++i) a.g_trial[qi * 7 + i] = 0.0;  // untouched slot (zeros)
        }
      } else {
        // radial return (material.cpp:122-171) from the committed state g0
        const double* gq = a.g0 + qi * 7;
        double e6[6], ee[6];
        embed6<D>(eps, e6);
#pragma unroll
        for (int i = 0; i < 6; ++i) ee[i] = e6[i] - gq[i];
        const double tr = ee[0] + ee[1] + ee[2];
        double st[6];
        double sn2 = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          st[i] = 2.0 * md.g * (ee[i] - (i < 3 ? tr / 3.0 : 0.0));
          sn2 = fma(st[i], st[i], sn2);
        }
        double s6[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) s6[i] = st[i] + (i < 3 ? md.k * tr : 0.0);
        const double s_norm = sqrt(sn2);
        const double q_tr = kS32 * s_norm;
        const double f = q_tr - (md.tau0 + md.hard * gq[6]);
        double ca = 1.0, cb = 0.0, nh[6] = {0, 0, 0, 0, 0, 0};
        double* gt = a.g_trial + qi * 7;
        if (f <= 0.0) {
#pragma unroll
          for (int i = 0; i < 7; ++i) gt[i] = gq[i];
        } else {
          const double dg = f / (3.0 * md.g + md.hard);
#pragma unroll
          for (int i = 0; i < 6; ++i) nh[i] = st[i] / s_norm;
#pragma unroll
          for (int i = 0; i < 6; ++i) s6[i] -= 2.0 * md.g * dg * kS32 * nh[i];
#pragma unroll
          for (int i = 0; i < 6; ++i) gt[i] = gq[i] + dg * kS32 * nh[i];
          gt[6] = gq[6] + dg;
          ca = 1.0 - 3.0 * md.g * dg / q_tr;
          cb = 6.0 * md.g * md.g * (1.0 / (3.0 * md.g + md.hard) - dg / q_tr);
        }
        extract<D>(s6, sig);
        double* tc = a.tanc + qi * 8;
        tc[0] = ca;
        tc[1] = cb;
#pragma unroll
        for (int i = 0; i < 6; ++i) tc[2 + i] = nh[i];
        // m x m block of the tangent (column-major) for the volume mean
        int idx[6];
        if (D == 3) {
#pragma unroll
          for (int i = 0; i < 6; ++i) idx[i] = i;
        } else {
          idx[0] = 0;
          idx[1] = 1;
          idx[2] = 5;
        }
#pragma unroll
        for (int jj = 0; jj < M; ++jj)
#pragma unroll
          for (int ii = 0; ii < M; ++ii) {
            const int i = idx[ii], j = idx[jj];
            const double vol = (i < 3 && j < 3) ? 1.0 / 3.0 : 0.0;
            const double dv = (i == j ? 1.0 : 0.0) - vol;
            Cq[jj * M + ii] = 3.0 * md.k * vol + 2.0 * md.g * ca * dv - cb * nh[i] * nh[j];
          }
      }
#pragma unroll
      for (int k = 0; k < M; ++k) a.sig[qi * M + k] = sig[k];
      const double w = sp.w[q];
#pragma unroll
      for (int i = 0; i < NV; ++i) tacc[i] = fma(w, Cq[i], tacc[i]);
    }
  }
  if (bad) a.status[0] = 1;
  block_sum_store_nv<NV>(tacc, a.partials + (size_t)blockIdx.x * NV);
}

template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_tan_stress(const Grid g, const __grid_constant__ StencilParams sp,
                                                        const NLArgs a, const PcgState* st) {
  if (st && st->done) return;
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  constexpr int NV = M * M;
  const int64_t np = g.np;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np; p += (int64_t)gridDim.x * blockDim.x) {
    int c0, c1, c2 = 0;
    if (D == 3) {
      c2 = (int)(p % g.n2);
      const int64_t t = p / g.n2;
      c1 = (int)(t % g.n1);
      c0 = (int)(t / g.n1);
    } else {
      c1 = (int)(p % g.n1);
      c0 = (int)(p / g.n1);
    }
    double uv[8][3];
    for (int o = 0; o < sp.noff; ++o) {
      const int i0 = wrapi(c0 + sp.offs[o][0], g.n0), i1 = wrapi(c1 + sp.offs[o][1], g.n1);
      const int i2 = D == 3 ? wrapi(c2 + sp.offs[o][2], g.n2) : 0;
      const int64_t nd = D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
#pragma unroll
      for (int k = 0; k < C; ++k) uv[o][k] = a.u[k * np + nd];
    }
    const int ph = a.phase[p];
    const NLModel md = a.models[ph];
    for (int q = 0; q < sp.nq; ++q) {
      const int64_t qi = p * sp.nq + q;
      double eps[M], sig[M];
      grad_rows<D, C>(sp, q, uv, eps);
      if (md.kind == 0) {
        const double* cm = a.cmat + (size_t)ph * NV;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < M; ++j) t = fma(cm[j * M + i], eps[j], t);
          sig[i] = t;
        }
      } else {
        const double* tc = a.tanc + qi * 8;
        double e6[6], s6[6];
        embed6<D>(eps, e6);
        compact_apply(md.k, md.g, tc[0], tc[1], tc + 2, e6, s6);
        extract<D>(s6, sig);
      }
#pragma unroll
      for (int k = 0; k < M; ++k) a.sig[qi * M + k] = sig[k];
    }
  }
}

}  // namespace

void launch_sweep(const Grid& g, const StencilParams& sp, const NLArgs& a, cudaStream_t s) {
  if (g.d == 2 && g.c == 2) k_sweep<2, 2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  else if (g.d == 3 && g.c == 3) k_sweep<3, 3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  else throw ValidationError("J2 path: mechanical grids only");
  HB_CUDA(cudaGetLastError());
}

void launch_tan_stress(const Grid& g, const StencilParams& sp, const NLArgs& a, const PcgState* st, cudaStream_t s) {
  if (g.d == 2 && g.c == 2) k_tan_stress<2, 2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  else if (g.d == 3 && g.c == 3) k_tan_stress<3, 3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  else throw ValidationError("J2 path: mechanical grids only");
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
