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

template <int M>
struct LinvM {
  double v[M * M];  // row-major L^-1 (C_ref = L L^T)
};

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// Mandel gradient rows at Gauss point q from the element corner values
// (operators.cpp:16-32 accumulate_rows).
template <int D, int C>
__device__ __forceinline__ void grad_rows(const StencilParams& sp, int q, const double (&uv)[9][3], double* gq) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  const double s2 = 0.70710678118654752440;
#pragma unroll
  for (int k = 0; k < M; ++k) gq[k] = 0.0;
  for (int en = 0; en < sp.ne[q]; ++en) {
    const double* dp = sp.dphi[q][en];
    const double* v = uv[sp.node[q][en] ? 8 : sp.off[q][en]];  // slot 8: centre node (type 1)
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
    double uv[9][3];
    if (!a.qeps) {
      const int64_t nodes = np * sp.nn;
      for (int o = 0; o < sp.noff; ++o) {
        const int i0 = wrapi(c0 + sp.offs[o][0], g.n0), i1 = wrapi(c1 + sp.offs[o][1], g.n1);
        const int i2 = D == 3 ? wrapi(c2 + sp.offs[o][2], g.n2) : 0;
        const int64_t nd = D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
#pragma unroll
        for (int k = 0; k < C; ++k) uv[o][k] = a.u ? a.u[k * nodes + nd] : 0.0;
      }
      if (sp.nn == 2) {
#pragma unroll
        for (int k = 0; k < C; ++k) uv[8][k] = a.u ? a.u[k * nodes + np + p] : 0.0;
      }
    }
    const int ph = a.phase[p];
    const NLModel md = a.models[ph];
    for (int q = 0; q < sp.nq; ++q) {
      const int64_t qi = p * sp.nq + q;
      double eps[M];
      if (a.qeps) {
#pragma unroll
        for (int k = 0; k < M; ++k) eps[k] = a.qeps[qi * M + k];
      } else {
        grad_rows<D, C>(sp, q, uv, eps);
      }
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
    double uv[9][3];
    const int64_t nodes = np * sp.nn;
    for (int o = 0; o < sp.noff; ++o) {
      const int i0 = wrapi(c0 + sp.offs[o][0], g.n0), i1 = wrapi(c1 + sp.offs[o][1], g.n1);
      const int i2 = D == 3 ? wrapi(c2 + sp.offs[o][2], g.n2) : 0;
      const int64_t nd = D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
#pragma unroll
      for (int k = 0; k < C; ++k) uv[o][k] = a.u[k * nodes + nd];
    }
    if (sp.nn == 2) {
#pragma unroll
      for (int k = 0; k < C; ++k) uv[8][k] = a.u[k * nodes + np + p];
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

template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_tan_mult(const Grid g, const __grid_constant__ StencilParams sp,
                                                      const NLArgs a, const double* __restrict__ x,
                                                      double* __restrict__ y) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  constexpr int NV = M * M;
  const int64_t nq = g.np * sp.nq;
  for (int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qi < nq; qi += (int64_t)gridDim.x * blockDim.x) {
    const int ph = a.phase[qi / sp.nq];
    const NLModel md = a.models[ph];
    double ev[M], sv[M];
#pragma unroll
    for (int k = 0; k < M; ++k) ev[k] = x[qi * M + k];
    if (md.kind == 0) {
      const double* cm = a.cmat + (size_t)ph * NV;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) t = fma(cm[j * M + i], ev[j], t);
        sv[i] = t;
      }
    } else {
      const double* tc = a.tanc + qi * 8;
      double e6[6], s6[6];
      embed6<D>(ev, e6);
      compact_apply(md.k, md.g, tc[0], tc[1], tc + 2, e6, s6);
      extract<D>(s6, sv);
    }
#pragma unroll
    for (int k = 0; k < M; ++k) y[qi * M + k] = sv[k];
  }
}

__global__ void __launch_bounds__(kBlock) k_qshift_norm2(const double* __restrict__ x, const double* __restrict__ e,
                                                          int64_t nq, int m, double* partials) {
  double acc = 0.0;
  for (int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qi < nq; qi += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < m; ++k) {
      const double v = x[qi * m + k] + (e ? e[k] : 0.0);
      acc = fma(v, v, acc);
    }
  double arr[1] = {acc};
  block_sum_store_nv<1>(arr, partials + blockIdx.x);
}

// per point: extreme generalized eigenvalues of (C_q, C_ref) via the
// reduced pencil L^-1 C L^-T (cyclic Jacobi, m <= 6)
template <int M>
__global__ void __launch_bounds__(kBlock) k_bounds_quad(const double* __restrict__ tan, int64_t nq, int nqp,
                                                         int pixel_constant, const __grid_constant__ LinvM<M> li,
                                                         double* qmin, double* qmax, int* status) {
  for (int64_t qi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; qi < nq; qi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = pixel_constant ? qi - qi % nqp : qi;
    const double* t = tan + src * M * M;  // column-major
    double tmp[M][M], a[M][M];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) acc = fma(li.v[i * M + k], t[j * M + k], acc);
        tmp[i][j] = acc;
      }
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < M; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) acc = fma(tmp[i][k], li.v[j * M + k], acc);
        a[i][j] = acc;
      }
    for (int sweep = 0; sweep < 60; ++sweep) {
      double off = 0.0;
#pragma unroll
      for (int i = 0; i < M; ++i)
#pragma unroll
        for (int j = i + 1; j < M; ++j) off += a[i][j] * a[i][j];
      if (off < 1e-300) break;
#pragma unroll
      for (int pp = 0; pp < M; ++pp)
#pragma unroll
        for (int qq = pp + 1; qq < M; ++qq) {
          const double apq = a[pp][qq];
          if (fabs(apq) < 1e-300) continue;
          const double th = 0.5 * (a[qq][qq] - a[pp][pp]) / apq;
          const double tt = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          const double cs = 1.0 / sqrt(tt * tt + 1.0), sn = tt * cs;
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const double akp = a[k][pp], akq = a[k][qq];
            a[k][pp] = cs * akp - sn * akq;
            a[k][qq] = sn * akp + cs * akq;
          }
#pragma unroll
          for (int k = 0; k < M; ++k) {
            const double apk = a[pp][k], aqk = a[qq][k];
            a[pp][k] = cs * apk - sn * aqk;
            a[qq][k] = sn * apk + cs * aqk;
          }
        }
    }
    double lo = a[0][0], hi = a[0][0];
#pragma unroll
    for (int i = 1; i < M; ++i) {
      lo = fmin(lo, a[i][i]);
      hi = fmax(hi, a[i][i]);
    }
    if (!(lo > 0.0)) status[0] = 2;
    qmin[qi] = lo;
    qmax[qi] = hi;
  }
}

// node min / max over the Gauss points whose basis supports the node
// (spectral.cpp:84-105), written c times per node (interleaved, i * c + k)
template <int D>
__global__ void __launch_bounds__(kBlock) k_bounds_nodes(const Grid g, const __grid_constant__ StencilParams sp,
                                                          const double* qmin, const double* qmax, int c,
                                                          double* lower, double* upper) {
  const int64_t np = g.np, nodes = np * sp.nn;
  for (int64_t nd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nd < nodes;
       nd += (int64_t)gridDim.x * blockDim.x) {
    const int type = (int)(nd / np);
    const int64_t n = nd - (int64_t)type * np;
    int c0, c1, c2 = 0;
    if (D == 3) {
      c2 = (int)(n % g.n2);
      const int64_t t = n / g.n2;
      c1 = (int)(t % g.n1);
      c0 = (int)(t / g.n1);
    } else {
      c1 = (int)(n % g.n1);
      c0 = (int)(n / g.n1);
    }
    double mn = INFINITY, mx = 0.0;
    for (int o = 0; o < (type ? 1 : sp.noff); ++o) {
      const int e0 = wrapi(c0 - sp.offs[o][0], g.n0), e1 = wrapi(c1 - sp.offs[o][1], g.n1);
      const int e2 = D == 3 ? wrapi(c2 - sp.offs[o][2], g.n2) : 0;
      const int64_t ep = D == 3 ? ((int64_t)e0 * g.n1 + e1) * g.n2 + e2 : (int64_t)e0 * g.n1 + e1;
      for (int q = 0; q < sp.nq; ++q) {
        bool sup = false;
        for (int en = 0; en < sp.ne[q]; ++en)
          if (sp.off[q][en] == o && sp.node[q][en] == type) sup = true;
        if (!sup) continue;
        mn = fmin(mn, qmin[ep * sp.nq + q]);
        mx = fmax(mx, qmax[ep * sp.nq + q]);
      }
    }
    for (int k = 0; k < c; ++k) {
      lower[nd * c + k] = mn;
      upper[nd * c + k] = mx;
    }
  }
}

}  // namespace

void launch_tan_mult(const Grid& g, const StencilParams& sp, const NLArgs& a, const double* x, double* y,
                     cudaStream_t s) {
  if (g.d == 2 && g.c == 2) k_tan_mult<2, 2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, x, y);
  else if (g.d == 3 && g.c == 3) k_tan_mult<3, 3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, x, y);
  else if (g.d == 2 && g.c == 1) k_tan_mult<2, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, x, y);
  else k_tan_mult<3, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, x, y);
  HB_CUDA(cudaGetLastError());
}

void launch_qshift_norm2(const double* x, const double* e, int64_t nq, int m, double* partials, cudaStream_t s) {
  k_qshift_norm2<<<kRedBlocks, kBlock, 0, s>>>(x, e, nq, m, partials);
  HB_CUDA(cudaGetLastError());
}

int bounds_device(const Grid& g, const StencilParams& sp, const double* d_tangent, int pixel_constant,
                  const double* linv, int c, double* d_lower, double* d_upper, cudaStream_t s) {
  const int64_t nq = g.np * sp.nq;
  double* qmin = nullptr;
  double* qmax = nullptr;
  int* status = nullptr;
  HB_CUDA(cudaMallocAsync(&qmin, nq * sizeof(double), s));
  HB_CUDA(cudaMallocAsync(&qmax, nq * sizeof(double), s));
  HB_CUDA(cudaMallocAsync(&status, sizeof(int), s));
  HB_CUDA(cudaMemsetAsync(status, 0, sizeof(int), s));
#define HB_BQ(M)                                                                          \
  do {                                                                                    \
    LinvM<M> li;                                                                          \
    for (int i = 0; i < M * M; ++i) li.v[i] = linv[i];                                    \
    k_bounds_quad<M><<<kRedBlocks, kBlock, 0, s>>>(d_tangent, nq, sp.nq, pixel_constant, li, qmin, qmax, status); \
  } while (0)
  switch (g.m) {
    case 2: HB_BQ(2); break;
    case 3: HB_BQ(3); break;
    default: HB_BQ(6); break;
  }
#undef HB_BQ
  HB_CUDA(cudaGetLastError());
  if (g.d == 2) k_bounds_nodes<2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, qmin, qmax, c, d_lower, d_upper);
  else k_bounds_nodes<3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, qmin, qmax, c, d_lower, d_upper);
  HB_CUDA(cudaGetLastError());
  int st = 0;
  HB_CUDA(cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, s));
  HB_CUDA(cudaStreamSynchronize(s));
  cudaFreeAsync(qmin, s);
  cudaFreeAsync(qmax, s);
  cudaFreeAsync(status, s);
  return st;
}

void launch_sweep(const Grid& g, const StencilParams& sp, const NLArgs& a, cudaStream_t s) {
  if (g.d == 2 && g.c == 2) k_sweep<2, 2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  else if (g.d == 3 && g.c == 3) k_sweep<3, 3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  else if (g.d == 2 && g.c == 1) k_sweep<2, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  else k_sweep<3, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a);
  HB_CUDA(cudaGetLastError());
}

void launch_tan_stress(const Grid& g, const StencilParams& sp, const NLArgs& a, const PcgState* st, cudaStream_t s) {
  if (g.d == 2 && g.c == 2) k_tan_stress<2, 2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  else if (g.d == 3 && g.c == 3) k_tan_stress<3, 3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  else if (g.d == 2 && g.c == 1) k_tan_stress<2, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  else k_tan_stress<3, 1><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, st);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
