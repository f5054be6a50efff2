// kernels.cu -- generic stencil, quadrature, reduction and PCG kernels.
//
// K u = D^T W C D u is evaluated with per-phase element matrices
// K_e = sum_q w_q B_q^T C B_q (algebraically identical to the reference's
// gather -> tangent contraction -> weighted scatter, operators.cpp:197-243,
// for pixel-constant linear tangents). The node-centric form below needs no
// atomics and sums each node's contributions in a fixed order, so results are
// bitwise reproducible.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum of NV values; thread 0 writes out[0..NV).
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* out) {
  __shared__ double red[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double s = warp_sum(v[i]);
    if (lane == 0) red[i][warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double s = lane < nw ? red[i][lane] : 0.0;
      s = warp_sum(s);
      if (lane == 0) out[i] = s;
    }
  }
}

__device__ __forceinline__ int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// ----------------------------------------------------------- element apply
template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_apply_elem(const Grid g, const ElemArgs a, int smem_ok) {
  if (a.st && a.st->done) return;
  constexpr int NL = 1 << D, NE = NL * C;
  extern __shared__ double ke_s[];
  const double* ke = a.ke;
  if (smem_ok) {
    const int tot = a.n_phases * NE * NE;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) ke_s[i] = a.ke[i];
    __syncthreads();
    ke = ke_s;
  }
  const int64_t np = g.np;
  double dotacc = 0.0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < np;
       n += (int64_t)gridDim.x * blockDim.x) {
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
    int w0[3], w1[3], w2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      w0[k] = wrap(c0 - 1 + k, g.n0);
      w1[k] = wrap(c1 - 1 + k, g.n1);
      w2[k] = D == 3 ? wrap(c2 - 1 + k, g.n2) : 0;
    }
    auto flat = [&](int i0, int i1, int i2) -> int64_t {
      return D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
    };
    double acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) acc[k] = 0.0;
#pragma unroll
    for (int e = 0; e < NL; ++e) {
      // this node is corner `e` (offset index) of the element below it
      int a0, a1, a2 = 0;
      if (D == 3) {
        a0 = (e >> 2) & 1; a1 = (e >> 1) & 1; a2 = e & 1;
      } else {
        a0 = e & 1; a1 = (e >> 1) & 1;
      }
      const int64_t eidx = flat(w0[1 - a0], w1[1 - a1], w2[1 - a2]);
      // slab mode: the element below plane (2-D: row) 0 lives on the previous rank
      const bool elo = g.dist && c0 - a0 < 0;
      const int ph = elo ? a.ph_lo[D == 3 ? (int64_t)w1[1 - a1] * g.n2 + w2[1 - a2] : (int64_t)w1[1 - a1]]
                         : a.phase[eidx];
      const double* row = ke + (size_t)ph * NE * NE + (size_t)(e * C) * NE;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        int b0, b1, b2 = 0;
        if (D == 3) {
          b0 = (j >> 2) & 1; b1 = (j >> 1) & 1; b2 = j & 1;
        } else {
          b0 = j & 1; b1 = (j >> 1) & 1;
        }
        const int64_t nidx = flat(w0[1 - a0 + b0], w1[1 - a1 + b1], w2[1 - a2 + b2]);
        // slab mode: node planes -1 / n0 come from the halo planes (exchanged, or a peer's field)
        const double* ub = a.u;
        int64_t cs = np, ni = nidx;
        if (g.dist) {
          const int z = c0 - a0 + b0;
          if (z < 0 || z >= g.n0) {
            ub = z < 0 ? a.halo_lo : a.halo_hi;
            cs = a.halo_cs ? a.halo_cs : (int64_t)g.n1 * g.n2;
            ni = D == 3 ? (int64_t)w1[1 - a1 + b1] * g.n2 + w2[1 - a2 + b2] : (int64_t)w1[1 - a1 + b1];
          }
        }
#pragma unroll
        for (int cj = 0; cj < C; ++cj) {
          const double v = __ldg(ub + cj * cs + ni);
#pragma unroll
          for (int ci = 0; ci < C; ++ci) acc[ci] = fma(row[ci * NE + j * C + cj], v, acc[ci]);
        }
      }
      if (a.fe) {
#pragma unroll
        for (int ci = 0; ci < C; ++ci) acc[ci] += a.fe[ph * NE + e * C + ci];
      }
    }
#pragma unroll
    for (int ci = 0; ci < C; ++ci) {
      const double v = a.scale * acc[ci];
      a.out[ci * np + n] = v;
      if (a.partials) dotacc = fma(__ldg(a.u + ci * np + n), v, dotacc);
    }
  }
  if (a.partials) {
    double v[1] = {dotacc};
    block_sum_store<1>(v, a.partials + blockIdx.x);
  }
}

// --------------------------------------------------------- quadrature loop
// One thread per pixel: gather the element corners, evaluate the Mandel
// gradient rows at every quadrature point (operators.cpp:16-32, 122-149).
// uv slots: corner offsets 0..noff-1 (node type 0), slot 8 = the pixel's
// centre node (type 1, FourTrianglesTwoNode)
__device__ __forceinline__ int uv_slot(const StencilParams& sp, int q, int en) {
  return sp.node[q][en] ? 8 : sp.off[q][en];
}

template <int D, int C>
__device__ __forceinline__ void quad_grad(const StencilParams& sp, int q, const double (&uv)[9][3],
                                          double* gq) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  const double s2 = 0.70710678118654752440;
#pragma unroll
  for (int k = 0; k < M; ++k) gq[k] = 0.0;
  for (int en = 0; en < sp.ne[q]; ++en) {
    const double* dp = sp.dphi[q][en];
    const double* v = uv[uv_slot(sp, q, en)];
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

template <int D, int C, int MODE>
__global__ void __launch_bounds__(kBlock) k_quad(const Grid g, const __grid_constant__ StencilParams sp,
                                                 const QuadArgs a) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  constexpr int NV = MODE == kQuadStress ? M : 1;
  const int64_t np = g.np;
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  double ev[M];
#pragma unroll
  for (int k = 0; k < M; ++k) ev[k] = a.e ? a.e[k] : 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x) {
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
    const int u0 = (c0 + 1 == g.n0 && !g.dist) ? 0 : c0 + 1;
    const int u1 = c1 + 1 == g.n1 ? 0 : c1 + 1;
    const int u2 = D == 3 ? (c2 + 1 == g.n2 ? 0 : c2 + 1) : 0;
    double uv[9][3];
    const int64_t nodes = np * sp.nn;
    for (int o = 0; o < sp.noff; ++o) {
      const int i0 = sp.offs[o][0] ? u0 : c0;
      const int i1 = sp.offs[o][1] ? u1 : c1;
      const int i2 = sp.offs[o][2] ? u2 : c2;
      if (g.dist && i0 == g.n0) {  // plane above the slab: halo
        const int64_t nd = (int64_t)i1 * g.n2 + i2;
        const int64_t pl = (int64_t)g.n1 * g.n2;
#pragma unroll
        for (int k = 0; k < C; ++k) uv[o][k] = a.u ? a.halo_hi[k * pl + nd] : 0.0;
        continue;
      }
      const int64_t nd = D == 3 ? ((int64_t)i0 * g.n1 + i1) * g.n2 + i2 : (int64_t)i0 * g.n1 + i1;
#pragma unroll
      for (int k = 0; k < C; ++k) uv[o][k] = a.u ? a.u[k * nodes + nd] : 0.0;
    }
    if (sp.nn == 2) {
#pragma unroll
      for (int k = 0; k < C; ++k) uv[8][k] = a.u ? a.u[k * nodes + np + p] : 0.0;
    }
    const double* cm = MODE == kQuadStress ? a.cmat + (size_t)a.phase[p] * M * M : nullptr;
    for (int q = 0; q < sp.nq; ++q) {
      double gq[M];
      quad_grad<D, C>(sp, q, uv, gq);
#pragma unroll
      for (int k = 0; k < M; ++k) gq[k] += ev[k];
      if (MODE == kQuadGrad) {
#pragma unroll
        for (int k = 0; k < M; ++k) a.gout[(p * sp.nq + q) * M + k] = gq[k];
      } else if (MODE == kQuadNorm2) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < M; ++k) s += gq[k] * gq[k];
        acc[0] += sp.w[q] * s;
      } else {
#pragma unroll
        for (int i = 0; i < M; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < M; ++j) s += cm[j * M + i] * gq[j];
          acc[i < NV ? i : 0] += sp.w[q] * s;
        }
      }
    }
  }
  if (MODE != kQuadGrad) block_sum_store<NV>(acc, a.partials + (size_t)blockIdx.x * NV);
}

// Node-centric weighted divergence D^T W s (operators.cpp:151-181).
template <int D, int C>
__global__ void __launch_bounds__(kBlock) k_divergence(const Grid g, const __grid_constant__ StencilParams sp,
                                                       const double* __restrict__ s, int weighted,
                                                       double* __restrict__ out) {
  constexpr int M = C == 1 ? D : (D == 2 ? 3 : 6);
  constexpr int NL = 1 << D;
  const double s2 = 0.70710678118654752440;
  const int64_t np = g.np, nodes = np * sp.nn;
  for (int64_t nd = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; nd < nodes;
       nd += (int64_t)gridDim.x * blockDim.x) {
    const int type = (int)(nd / np);  // node type (1 = pixel centre, FourTrianglesTwoNode)
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
    double acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) acc[k] = 0.0;
    for (int o = 0; o < (type ? 1 : NL); ++o) {
      // element whose corner `o` is this node (the centre node: its own pixel)
      const int e0 = wrap(c0 - sp.offs[o][0], g.n0);
      const int e1 = wrap(c1 - sp.offs[o][1], g.n1);
      const int e2 = D == 3 ? wrap(c2 - sp.offs[o][2], g.n2) : 0;
      const int64_t ep = D == 3 ? ((int64_t)e0 * g.n1 + e1) * g.n2 + e2 : (int64_t)e0 * g.n1 + e1;
      for (int q = 0; q < sp.nq; ++q) {
        const double w = weighted ? sp.w[q] : 1.0;
        const double* sv = s + (ep * sp.nq + q) * M;
        for (int en = 0; en < sp.ne[q]; ++en) {
          if (sp.off[q][en] != o || sp.node[q][en] != type) continue;
          const double* dp = sp.dphi[q][en];
          if (C == 1) {
            double t = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) t += dp[k] * sv[k];
            acc[0] += w * t;
          } else if (D == 2) {
            acc[0] += w * (dp[0] * sv[0] + s2 * dp[1] * sv[2]);
            acc[C > 1 ? 1 : 0] += w * (dp[1] * sv[1] + s2 * dp[0] * sv[2]);
          } else {
            acc[0] += w * (dp[0] * sv[0] + s2 * (dp[2] * sv[4] + dp[1] * sv[5]));
            acc[C > 1 ? 1 : 0] += w * (dp[1] * sv[1] + s2 * (dp[2] * sv[3] + dp[0] * sv[5]));
            acc[C > 2 ? 2 : 0] += w * (dp[2] * sv[2] + s2 * (dp[1] * sv[3] + dp[0] * sv[4]));
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < C; ++k) out[k * nodes + nd] = acc[k];
  }
}

// Weighted quadrature sum sum_q w_q s(q) of an interleaved quad field
// (fields.cpp:42-50), per-block partials of M values.
template <int M>
__global__ void __launch_bounds__(kBlock) k_quad_wsum(const Grid g, const __grid_constant__ StencilParams sp,
                                                      const double* __restrict__ s, double* partials) {
  double acc[M];
#pragma unroll
  for (int k = 0; k < M; ++k) acc[k] = 0.0;
  const int64_t nQ = g.np * sp.nq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nQ; q += (int64_t)gridDim.x * blockDim.x) {
    const double w = sp.w[q % sp.nq];
#pragma unroll
    for (int k = 0; k < M; ++k) acc[k] = fma(w, s[q * M + k], acc[k]);
  }
  block_sum_store<M>(acc, partials + (size_t)blockIdx.x * M);
}

// sum_q w_q a(q).b(q) over M-component quad fields (fields.cpp:19-35), one
// per-block partial (fixed grid: deterministic).
template <int M>
__global__ void __launch_bounds__(kBlock) k_quad_wdot(const Grid g, const __grid_constant__ StencilParams sp,
                                                      const double* __restrict__ a, const double* __restrict__ b,
                                                      double* partials) {
  double acc[1] = {0.0};
  const int64_t nQ = g.np * sp.nq;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nQ; q += (int64_t)gridDim.x * blockDim.x) {
    double d = 0.0;
#pragma unroll
    for (int k = 0; k < M; ++k) d = fma(a[q * M + k], b[q * M + k], d);
    acc[0] = fma(sp.w[q % sp.nq], d, acc[0]);
  }
  block_sum_store<1>(acc, partials + blockIdx.x);
}

__global__ void k_index_maps(const Grid g, const __grid_constant__ StencilParams sp, int64_t* nbr) {
  const int64_t np = g.np;
  const int64_t s0 = g.d == 3 ? (int64_t)g.n1 * g.n2 : g.n1;
  const int64_t s1 = g.d == 3 ? g.n2 : 1;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x) {
    int64_t t = p;
    const int c0 = (int)(t / s0);
    t -= c0 * s0;
    const int c1 = (int)(t / s1);
    const int c2 = (int)(t - c1 * s1);
    const int64_t cur[3] = {c0 * s0, c1 * s1, g.d == 3 ? (int64_t)c2 : 0};
    const int64_t nxt[3] = {(c0 + 1 == g.n0 ? 0 : c0 + 1) * s0, (c1 + 1 == g.n1 ? 0 : c1 + 1) * s1,
                            g.d == 3 ? (int64_t)(c2 + 1 == g.n2 ? 0 : c2 + 1) : 0};
    for (int o = 0; o < sp.noff; ++o) {
      int64_t f = 0;
      for (int ax = 0; ax < g.d; ++ax) f += sp.offs[o][ax] ? nxt[ax] : cur[ax];
      nbr[p * sp.noff + o] = f;
    }
  }
}

// ----------------------------------------------------------------- vectors
__global__ void k_dot_partials(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                               double* partials) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  double v[1] = {s};
  block_sum_store<1>(v, partials + blockIdx.x);
}

template <int C>
__global__ void k_comp_sums(const double* __restrict__ a, int64_t np, double* partials) {
  double s[C];
#pragma unroll
  for (int k = 0; k < C; ++k) s[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < C; ++k) s[k] += a[k * np + i];
  }
  block_sum_store<C>(s, partials + (size_t)blockIdx.x * C);
}

template <int C>
__global__ void k_sub_means(double* __restrict__ a, int64_t np, const double* __restrict__ sums, double count) {
  double mean[C];
#pragma unroll
  for (int k = 0; k < C; ++k) mean[k] = sums[k] / count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < np; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < C; ++k) a[k * np + i] -= mean[k];
  }
}

// Fixed-order final sum of per-block partials (nvals interleaved per block).
__global__ void k_final_sum(const double* __restrict__ partials, int nblocks, int nvals, double* out) {
  for (int v = 0; v < nvals; ++v) {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partials[(size_t)b * nvals + v];
    double arr[1] = {s};
    block_sum_store<1>(arr, out + v);
    __syncthreads();
  }
}

__global__ void k_axpy(double* __restrict__ y, double a, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], y[i]);
}

__global__ void k_scale(double* a, double sc, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] *= sc;
}

__device__ double block_total(const double* partials, int nblocks) {
  double s = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) s += partials[b];
  __shared__ double tot;
  double arr[1] = {s};
  block_sum_store<1>(arr, &tot);
  __syncthreads();
  return tot;
}

// r.z of r_0 and z_0 = M^-1 r_0 (solver.cpp:62-73).
__global__ void k_pcg_init(PcgState* st, const double* partials, int nblocks, double* hist) {
  const double s = block_total(partials, nblocks);
  if (threadIdx.x == 0) {
    const double rz = fmax(s, 0.0);
    st->rz = rz;
    st->norm0 = sqrt(rz);
    st->it = 0;
    st->status = 0;
    hist[0] = st->norm0;
    st->converged = st->norm0 == 0.0 ? 1 : 0;
    st->done = st->converged || st->it_max <= 0;
  }
}

// alpha = rz / p.Ap, abort on non-positive curvature (solver.cpp:74-80).
__global__ void k_pcg_alpha(PcgState* st, const double* partials, int nblocks) {
  if (st->done) {
    if (threadIdx.x == 0) st->active = 0;
    return;
  }
  const double pap = block_total(partials, nblocks);
  if (threadIdx.x == 0) {
    st->pap = pap;
    if (!(pap > 0.0)) {
      st->status = 4;
      st->done = 1;
      st->active = 0;
    } else {
      st->alpha = st->rz / pap;
      st->active = 1;
    }
  }
}

// r -= alpha Ap (solver.cpp:81-82; x is updated with p in k_update_xp, which
// reads p anyway: one vector pass fewer per iteration)
__global__ void k_update_r(double* __restrict__ r, const double* __restrict__ ap, int64_t n, const PcgState* st) {
  if (!st->active) return;
  const double alpha = st->alpha;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = fma(-alpha, ap[i], r[i]);
}

// rz_next, history, stopping test, beta (solver.cpp:84-93).
__global__ void k_pcg_beta(PcgState* st, const double* partials, int nblocks, double* hist) {
  if (!st->active) return;
  const double s = block_total(partials, nblocks);
  if (threadIdx.x == 0) {
    const double rzn = fmax(s, 0.0);
    const int it = st->it + 1;
    st->it = it;
    hist[it] = sqrt(rzn);
    if (sqrt(rzn) <= st->eta * st->norm0) {
      st->converged = 1;
      st->done = 1;
    } else {
      st->beta = rzn / st->rz;
      st->rz = rzn;
      if (it >= st->it_max) st->done = 1;
    }
  }
}

// beta kernel that also drives the device WHILE loop of the fused path.
__global__ void k_pcg_beta_cond(PcgState* st, const double* partials, int nblocks, double* hist,
                                cudaGraphConditionalHandle h) {
  if (!st->active) {
    if (threadIdx.x == 0) cudaGraphSetConditional(h, 0u);
    return;
  }
  const double s = block_total(partials, nblocks);
  if (threadIdx.x == 0) {
    const double rzn = fmax(s, 0.0);
    const int it = st->it + 1;
    st->it = it;
    hist[it] = sqrt(rzn);
    if (sqrt(rzn) <= st->eta * st->norm0) {
      st->converged = 1;
      st->done = 1;
    } else {
      st->beta = rzn / st->rz;
      st->rz = rzn;
      if (it >= st->it_max) st->done = 1;
    }
    cudaGraphSetConditional(h, st->done ? 0u : 1u);
  }
}

// x += alpha p (this iteration), p = z + beta p unless the loop just ended
// (solver.cpp:81, 93)
__global__ void k_update_xp(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ z, int64_t n,
                            const PcgState* st) {
  if (!st->active) return;
  const double alpha = st->alpha, beta = st->beta;
  const bool upd = !st->done;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[i];
    x[i] = fma(alpha, pv, x[i]);
    if (upd) p[i] = fma(beta, pv, z[i]);
  }
}

__global__ void k_set_while(cudaGraphConditionalHandle h, const PcgState* st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

__global__ void k_update_xp_cond(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ z,
                                 int64_t n, const PcgState* st, cudaGraphConditionalHandle h) {
  const int done = st->done;
  if (blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, done ? 0u : 1u);
  if (!st->active) return;
  const double alpha = st->alpha, beta = st->beta;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double pv = p[i];
    x[i] = fma(alpha, pv, x[i]);
    if (!done) p[i] = fma(beta, pv, z[i]);
  }
}

int grid_for(int64_t n) {
  const int64_t b = (n + kBlock - 1) / kBlock;
  return (int)(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}

}  // namespace

// ---------------------------------------------------------------- launchers
void launch_apply_elem(const Grid& g, const ElemArgs& a, cudaStream_t s) {
  const int nl = 1 << g.d, ne = nl * g.c;
  const size_t smem = (size_t)a.n_phases * ne * ne * sizeof(double);
  const int smem_ok = smem <= 160 * 1024;
  const size_t dyn = smem_ok ? smem : 0;
  const int blocks = kRedBlocks;
#define HB_ELEM(D, C)                                                                         \
  do {                                                                                        \
    if (dyn > 48 * 1024)                                                                      \
      HB_CUDA(cudaFuncSetAttribute(k_apply_elem<D, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn)); \
    k_apply_elem<D, C><<<blocks, kBlock, dyn, s>>>(g, a, smem_ok);                           \
  } while (0)
  if (g.d == 2 && g.c == 1) HB_ELEM(2, 1);
  else if (g.d == 2 && g.c == 2) HB_ELEM(2, 2);
  else if (g.d == 3 && g.c == 1) HB_ELEM(3, 1);
  else if (g.d == 3 && g.c == 3) HB_ELEM(3, 3);
  else throw ValidationError("apply: unsupported dimension/components");
#undef HB_ELEM
  HB_CUDA(cudaGetLastError());
}

void launch_quad(const Grid& g, const StencilParams& sp, int mode, const QuadArgs& a, cudaStream_t s) {
  const int blocks = kRedBlocks;
#define HB_Q(D, C)                                                                              \
  do {                                                                                          \
    if (mode == kQuadGrad) k_quad<D, C, kQuadGrad><<<blocks, kBlock, 0, s>>>(g, sp, a);         \
    else if (mode == kQuadNorm2) k_quad<D, C, kQuadNorm2><<<blocks, kBlock, 0, s>>>(g, sp, a);  \
    else k_quad<D, C, kQuadStress><<<blocks, kBlock, 0, s>>>(g, sp, a);                         \
  } while (0)
  if (g.d == 2 && g.c == 1) HB_Q(2, 1);
  else if (g.d == 2 && g.c == 2) HB_Q(2, 2);
  else if (g.d == 3 && g.c == 1) HB_Q(3, 1);
  else if (g.d == 3 && g.c == 3) HB_Q(3, 3);
  else throw ValidationError("quad: unsupported dimension/components");
#undef HB_Q
  HB_CUDA(cudaGetLastError());
}

void launch_divergence(const Grid& g, const StencilParams& sp, const double* sf, bool weighted, double* out,
                       cudaStream_t s) {
  const int blocks = grid_for(g.np * sp.nn);
  if (g.d == 2 && g.c == 1) k_divergence<2, 1><<<blocks, kBlock, 0, s>>>(g, sp, sf, weighted, out);
  else if (g.d == 2 && g.c == 2) k_divergence<2, 2><<<blocks, kBlock, 0, s>>>(g, sp, sf, weighted, out);
  else if (g.d == 3 && g.c == 1) k_divergence<3, 1><<<blocks, kBlock, 0, s>>>(g, sp, sf, weighted, out);
  else if (g.d == 3 && g.c == 3) k_divergence<3, 3><<<blocks, kBlock, 0, s>>>(g, sp, sf, weighted, out);
  else throw ValidationError("divergence: unsupported dimension/components");
  HB_CUDA(cudaGetLastError());
}

// sigma_q = C_q eps_q for a general TangentField (tangent_multiply,
// operators.cpp:183-192): column-major m x m block per quadrature point,
// one thread per point, in place on the quadrature field.
template <int M>
__global__ void __launch_bounds__(kBlock) k_tangent_field(int64_t nq, const double* __restrict__ t,
                                                         double* __restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    double e[M], sgm[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      e[j] = q[i * M + j];
      sgm[j] = 0.0;
    }
    const double* blk = t + i * M * M;
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int r = 0; r < M; ++r) sgm[r] = fma(blk[j * M + r], e[j], sgm[r]);
#pragma unroll
    for (int j = 0; j < M; ++j) q[i * M + j] = sgm[j];
  }
}

void launch_tangent_field(const Grid& g, const StencilParams& sp, const double* tangent, double* q, cudaStream_t s) {
  const int64_t nq = g.np * sp.nq;
  const int blocks = grid_for(nq);
  switch (g.m) {
    case 2: k_tangent_field<2><<<blocks, kBlock, 0, s>>>(nq, tangent, q); break;
    case 3: k_tangent_field<3><<<blocks, kBlock, 0, s>>>(nq, tangent, q); break;
    case 6: k_tangent_field<6><<<blocks, kBlock, 0, s>>>(nq, tangent, q); break;
    default: throw ValidationError("tangent field: unsupported strain dimension");
  }
  HB_CUDA(cudaGetLastError());
}

void launch_quad_wsum(const Grid& g, const StencilParams& sp, const double* sf, double* partials, cudaStream_t s) {
  switch (g.m) {
    case 2: k_quad_wsum<2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, sf, partials); break;
    case 3: k_quad_wsum<3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, sf, partials); break;
    case 6: k_quad_wsum<6><<<kRedBlocks, kBlock, 0, s>>>(g, sp, sf, partials); break;
    default: throw ValidationError("volume_average: unsupported component count");
  }
  HB_CUDA(cudaGetLastError());
}

void launch_quad_wdot(const Grid& g, const StencilParams& sp, const double* a, const double* b, double* partials,
                      cudaStream_t s) {
  switch (g.m) {
    case 2: k_quad_wdot<2><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, b, partials); break;
    case 3: k_quad_wdot<3><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, b, partials); break;
    case 6: k_quad_wdot<6><<<kRedBlocks, kBlock, 0, s>>>(g, sp, a, b, partials); break;
    default: throw ValidationError("weighted_dot: unsupported component count");
  }
  HB_CUDA(cudaGetLastError());
}

// per-phase voxel counts (MaterialMap::validate + volume-mean reference,
// material.cpp:252-277): shared-memory histogram, exact integer atomics
__global__ void __launch_bounds__(kBlock) k_phase_counts(const uint8_t* __restrict__ ph, int64_t n,
                                                          unsigned long long* __restrict__ counts) {
  __shared__ unsigned int hist[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
  __syncthreads();
  const int64_t n4 = n / 4;
  const uchar4* p4 = reinterpret_cast<const uchar4*>(ph);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const uchar4 v = p4[i];
    atomicAdd(&hist[v.x], 1u);
    atomicAdd(&hist[v.y], 1u);
    atomicAdd(&hist[v.z], 1u);
    atomicAdd(&hist[v.w], 1u);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&hist[ph[i]], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (hist[i]) atomicAdd(&counts[i], (unsigned long long)hist[i]);
}

void launch_phase_counts(const uint8_t* ph, int64_t n, unsigned long long* counts, cudaStream_t s) {
  HB_CUDA(cudaMemsetAsync(counts, 0, 256 * sizeof(unsigned long long), s));
  k_phase_counts<<<kRedBlocks / 4, kBlock, 0, s>>>(ph, n, counts);
  HB_CUDA(cudaGetLastError());
}

void launch_index_maps(const Grid& g, const StencilParams& sp, int64_t* nbr, cudaStream_t s) {
  k_index_maps<<<grid_for(g.np), kBlock, 0, s>>>(g, sp, nbr);
  HB_CUDA(cudaGetLastError());
}

void launch_dot_partials(const double* a, const double* b, int64_t n, double* partials, cudaStream_t s) {
  k_dot_partials<<<kRedBlocks, kBlock, 0, s>>>(a, b, n, partials);
  HB_CUDA(cudaGetLastError());
}

void launch_comp_sums(const double* a, int c, int64_t np, double* partials, cudaStream_t s) {
  if (c == 1) k_comp_sums<1><<<kRedBlocks, kBlock, 0, s>>>(a, np, partials);
  else if (c == 2) k_comp_sums<2><<<kRedBlocks, kBlock, 0, s>>>(a, np, partials);
  else k_comp_sums<3><<<kRedBlocks, kBlock, 0, s>>>(a, np, partials);
  HB_CUDA(cudaGetLastError());
}

void launch_sub_means(double* a, int c, int64_t np, const double* sums, cudaStream_t s, double count) {
  const int blocks = grid_for(np);
  if (count <= 0.0) count = (double)np;
  if (c == 1) k_sub_means<1><<<blocks, kBlock, 0, s>>>(a, np, sums, count);
  else if (c == 2) k_sub_means<2><<<blocks, kBlock, 0, s>>>(a, np, sums, count);
  else k_sub_means<3><<<blocks, kBlock, 0, s>>>(a, np, sums, count);
  HB_CUDA(cudaGetLastError());
}

void launch_final_sum(const double* partials, int nblocks, int nvals, double* out, cudaStream_t s) {
  k_final_sum<<<1, 1024, 0, s>>>(partials, nblocks, nvals, out);
  HB_CUDA(cudaGetLastError());
}

void launch_axpy(double* y, double a, const double* x, int64_t n, cudaStream_t s) {
  k_axpy<<<grid_for(n), kBlock, 0, s>>>(y, a, x, n);
  HB_CUDA(cudaGetLastError());
}

void launch_scale(double* a, double sc, int64_t n, cudaStream_t s) {
  k_scale<<<grid_for(n), kBlock, 0, s>>>(a, sc, n);
  HB_CUDA(cudaGetLastError());
}

void launch_pcg_init(PcgState* st, const double* partials, double* hist, cudaStream_t s, int nblocks) {
  k_pcg_init<<<1, 1024, 0, s>>>(st, partials, nblocks, hist);
  HB_CUDA(cudaGetLastError());
}
void launch_pcg_alpha(PcgState* st, const double* partials, cudaStream_t s, int nblocks) {
  k_pcg_alpha<<<1, 1024, 0, s>>>(st, partials, nblocks);
  HB_CUDA(cudaGetLastError());
}
void launch_update_r(double* r, const double* ap, int64_t n, const PcgState* st, cudaStream_t s) {
  k_update_r<<<grid_for(n), kBlock, 0, s>>>(r, ap, n, st);
  HB_CUDA(cudaGetLastError());
}
void launch_pcg_beta(PcgState* st, const double* partials, double* hist, cudaStream_t s, int nblocks) {
  k_pcg_beta<<<1, 1024, 0, s>>>(st, partials, nblocks, hist);
  HB_CUDA(cudaGetLastError());
}
void launch_pcg_beta_cond(PcgState* st, const double* partials, double* hist, cudaGraphConditionalHandle h,
                          cudaStream_t s) {
  k_pcg_beta_cond<<<1, 1024, 0, s>>>(st, partials, kRedBlocks, hist, h);
  HB_CUDA(cudaGetLastError());
}
void launch_update_xp(double* x, double* p, const double* z, int64_t n, const PcgState* st, cudaStream_t s) {
  k_update_xp<<<grid_for(n), kBlock, 0, s>>>(x, p, z, n, st);
  HB_CUDA(cudaGetLastError());
}
void launch_set_while(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s) {
  k_set_while<<<1, 32, 0, s>>>(h, st);
  HB_CUDA(cudaGetLastError());
}
void launch_update_xp_cond(double* x, double* p, const double* z, int64_t n, const PcgState* st,
                           cudaGraphConditionalHandle h, cudaStream_t s) {
  k_update_xp_cond<<<grid_for(n), kBlock, 0, s>>>(x, p, z, n, st, h);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
