// quad2d.cu -- K u for the 2-D one-node pixel stencils (TwoTriangles,
// BilinearQuad; c = 1 scalar or c = 2 plane elasticity) as a streaming,
// memory-bound kernel.
//
// The reference applies D^T W C D per quadrature point
// (proj/src/operators.cpp:197-243). Here:
//  * TwoTriangles (the c1 / c5 stencil): each triangle's gradient is a pair
//    of raw corner differences (grid.cpp:124-143: q0 = {off0 (-1/h0,-1/h1),
//    off1 (1/h0,0), off2 (0,1/h1)}, q1 = {off3 (1/h0,1/h1), off2 (-1/h0,0),
//    off1 (0,-1/h1)}); the flux is a per-phase m x m table with w and the
//    1/h factors folded in, and the corner residuals are +-sums of its
//    entries: ~20 (c = 1) / ~60 (c = 2) flops per pixel, c^2 + ... table reads;
//  * BilinearQuad: the per-phase 4c x 4c element matrix (tables.hpp).
//
// Work layout: a warp owns a strip of 31 output columns (axis 1, the
// contiguous one) and marches down a band of rows (axis 0). Lane t
// evaluates the element whose left column is x0 - 1 + t, so the element to
// the right of every output node is in the same warp (shfl_down) and no
// block-level exchange or barrier is needed; lane 31 only feeds lane 30. The
// element row above is carried in registers (one warm-up row per band) and
// the next row is loaded one step ahead. Every node is the same fixed-order
// sum: deterministic, and p.Ap is fused.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hb {

namespace {

constexpr int kStrip = 31;
// rows per task: 32 balances the tasks over the resident warps better than
// 64 on the smaller grids (2048^2: 0.035 -> 0.027 ms per launch; 8192^2:
// 0.396 -> 0.390 ms) at 1/32 warm-up rows
#ifndef HB_E2D_BAND
#define HB_E2D_BAND 32
#endif
constexpr int kBand = HB_E2D_BAND;
#ifndef HB_E2D_L2PF
#define HB_E2D_L2PF 3  // 8192^2: 0.390 -> 0.368 ms per launch (6 and 12 rows ahead: 0.370, 0.374)
#endif
#ifndef HB_E2D_PD
#define HB_E2D_PD 1  // rows loaded ahead
#endif

// element residual r[corner][k], corners 0 = (y, e), 1 = (y+1, e),
// 2 = (y, e+1), 3 = (y+1, e+1)
template <int C>
__device__ __forceinline__ void tri_element(const double (&u)[4][C], const double* __restrict__ A,
                                            double (&r)[4][C]) {
  if constexpr (C == 1) {
    // A = w/(hi hj) C_ij, 2 x 2 row-major
    const double a00 = A[0], a01 = A[1], a10 = A[2], a11 = A[3];
    {  // q0
      const double d0 = u[1][0] - u[0][0], d1 = u[2][0] - u[0][0];
      const double fa = fma(a00, d0, a01 * d1), fb = fma(a10, d0, a11 * d1);
      r[0][0] = -(fa + fb);
      r[1][0] = fa;
      r[2][0] = fb;
    }
    {  // q1
      const double d0 = u[3][0] - u[2][0], d1 = u[3][0] - u[1][0];
      const double fa = fma(a00, d0, a01 * d1), fb = fma(a10, d0, a11 * d1);
      r[3][0] = fa + fb;
      r[2][0] -= fa;
      r[1][0] -= fb;
    }
  } else {
    // A = the 3 x 3 Mandel table scaled: t = A e' with e' = (d0x, d1y, d1x + d0y)
    // rows give (w s0 / h0, w s1 / h1, w s2 s_12 / h1, w s2 s_12 / h0) via the
    // 4 x 3 table A[4][3]
    auto tri = [&](double d0x, double d0y, double d1x, double d1y, double& t0, double& t1, double& t2,
                   double& t3) {
      const double e2 = d1x + d0y;  // raw shear with its own 1/h folded per column
      t0 = fma(A[0], d0x, fma(A[1], d1y, A[2] * e2));
      t1 = fma(A[3], d0x, fma(A[4], d1y, A[5] * e2));
      t2 = fma(A[6], d0x, fma(A[7], d1y, A[8] * e2));
      t3 = fma(A[9], d0x, fma(A[10], d1y, A[11] * e2));
    };
    double t0, t1, t2, t3;
    // q0: d0 = u1 - u0 (axis 0), d1 = u2 - u0 (axis 1)
    tri(u[1][0] - u[0][0], u[1][1] - u[0][1], u[2][0] - u[0][0], u[2][1] - u[0][1], t0, t1, t2, t3);
    r[0][0] = -(t0 + t2);
    r[0][1] = -(t3 + t1);
    r[1][0] = t0;
    r[1][1] = t3;
    r[2][0] = t2;
    r[2][1] = t1;
    // q1: d0 = u3 - u2, d1 = u3 - u1
    tri(u[3][0] - u[2][0], u[3][1] - u[2][1], u[3][0] - u[1][0], u[3][1] - u[1][1], t0, t1, t2, t3);
    r[3][0] = t0 + t2;
    r[3][1] = t3 + t1;
    r[2][0] -= t0;
    r[2][1] -= t3;
    r[1][0] -= t2;
    r[1][1] -= t1;
  }
}

template <int C, bool TRI>
__global__ void __launch_bounds__(256) k_elem2d(const Grid g, const ElemArgs a, const double* __restrict__ tri_tab,
                                               int smem_ok) {
  if (a.st && a.st->done) return;
  constexpr int NE = 4 * C;
  constexpr int TS = C == 1 ? 4 : 12;  // triangle table entries per phase
  constexpr int MS = TRI ? TS : NE * NE;
  extern __shared__ double tab_s[];
  const double* tab = TRI ? tri_tab : a.ke;
  if (smem_ok) {
    const int tot = a.n_phases * MS;
    for (int i = threadIdx.x; i < tot; i += blockDim.x) tab_s[i] = tab[i];
    __syncthreads();
    tab = tab_s;
  }
  const int n0 = g.n0, n1 = g.n1;
  const int64_t np = g.np;
  const int lane = threadIdx.x & 31;
  const int strips = (n1 + kStrip - 1) / kStrip, bands = (n0 + kBand - 1) / kBand;
  const int ntask = strips * bands;
  double dotacc = 0.0;
  for (int task = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); task < ntask;
       task += gridDim.x * (blockDim.x >> 5)) {
    const int s = task % strips, b = task / strips;
    const int x0 = s * kStrip, y0 = b * kBand;
    int e = (x0 - 1 + lane) % n1;  // element column (left corner); lanes past n1 wrap (no output)
    e = e < 0 ? e + n1 : e;
    const int e1 = e + 1 == n1 ? 0 : e + 1;
    const int node = x0 + lane;  // output column of this lane (lane < 31)
    const bool out_ok = lane < kStrip && node < n1;
    const int yend = min(y0 + kBand, n0);
    const int yr = y0 - 1 < 0 ? n0 - 1 : y0 - 1;
    double uc[2][C];  // row y, columns e, e+1
#pragma unroll
    for (int k = 0; k < C; ++k) {
      uc[0][k] = __ldg(a.u + k * np + (int64_t)yr * n1 + e);
      uc[1][k] = __ldg(a.u + k * np + (int64_t)yr * n1 + e1);
    }
    double carry[C];
#pragma unroll
    for (int k = 0; k < C; ++k) carry[k] = 0.0;
    // software pipeline: corner values and phase of the rows PD steps ahead
    // live in a register ring (slot = step % PD, compile-time after unroll)
    constexpr int PD = HB_E2D_PD;
    double ring[PD][2][C];
    int phr[PD];
    const int nsteps = yend - (y0 - 1);
#pragma unroll
    for (int q = 0; q < PD; ++q) {
      if (q < nsteps) {
        int ye = y0 - 1 + q;
        ye = ye < 0 ? ye + n0 : (ye >= n0 ? ye - n0 : ye);
        const int yn = ye + 1 == n0 ? 0 : ye + 1;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          ring[q][0][k] = __ldg(a.u + k * np + (int64_t)yn * n1 + e);
          ring[q][1][k] = __ldg(a.u + k * np + (int64_t)yn * n1 + e1);
        }
        phr[q] = a.phase[(int64_t)ye * n1 + e];
      }
    }
#pragma unroll 1
    for (int st0 = 0; st0 < nsteps; st0 += PD) {
#pragma unroll
      for (int q = 0; q < PD; ++q) {
        const int stp = st0 + q;
        if (stp < nsteps) {
          const int y = y0 - 1 + stp;
          const int ye = y < 0 ? y + n0 : y;  // element row
          double un[2][C];
#pragma unroll
          for (int k = 0; k < C; ++k) {
            un[0][k] = ring[q][0][k];
            un[1][k] = ring[q][1][k];
          }
          const int ph = phr[q];
          if (HB_E2D_L2PF > 0 && stp + HB_E2D_L2PF < nsteps) {
            // pull the node row HB_E2D_L2PF steps ahead into L2: the register
            // prefetch one step ahead then waits for L2, not HBM (one row in
            // flight per warp covers only ~2.5 TB/s at HBM latency)
            int yp = ye + HB_E2D_L2PF + 1;
            yp = yp >= n0 ? yp - n0 : yp;
#pragma unroll
            for (int k = 0; k < C; ++k)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(a.u + k * np + (int64_t)yp * n1 + e));
          }
          if (stp + PD < nsteps) {
            int yf = ye + PD;  // element row PD steps ahead
            yf = yf >= n0 ? yf - n0 : yf;
            const int yfn = yf + 1 == n0 ? 0 : yf + 1;
#pragma unroll
            for (int k = 0; k < C; ++k) {
              ring[q][0][k] = __ldg(a.u + k * np + (int64_t)yfn * n1 + e);
              ring[q][1][k] = __ldg(a.u + k * np + (int64_t)yfn * n1 + e1);
            }
            phr[q] = a.phase[(int64_t)yf * n1 + e];
          }
          double ue[4][C], r[4][C];
#pragma unroll
          for (int k = 0; k < C; ++k) {
            ue[0][k] = uc[0][k];
            ue[1][k] = un[0][k];
            ue[2][k] = uc[1][k];
            ue[3][k] = un[1][k];
          }
          if constexpr (TRI) {
            tri_element<C>(ue, tab + ph * MS, r);
          } else {
            const double* K = tab + (size_t)ph * MS;
#pragma unroll
            for (int i = 0; i < NE; ++i) {
              double acc = 0.0;
#pragma unroll
              for (int j = 0; j < NE; ++j) acc = fma(K[i * NE + j], ue[j / C][j % C], acc);
              r[i / C][i % C] = acc;
            }
          }
          if (a.fe) {
#pragma unroll
            for (int i = 0; i < NE; ++i) r[i / C][i % C] += a.fe[ph * NE + i];
          }
#pragma unroll
          for (int k = 0; k < C; ++k) {
            // node (y, e+1) <- corner 2 of this element + corner 0 of the next
            const double top = r[2][k] + __shfl_down_sync(0xffffffffu, r[0][k], 1);
            const double bot = r[3][k] + __shfl_down_sync(0xffffffffu, r[1][k], 1);
            if (y >= y0 && out_ok) {
              const double v = a.scale * (carry[k] + top);
              a.out[(int64_t)k * np + (int64_t)ye * n1 + node] = v;
              dotacc = fma(uc[1][k], v, dotacc);
            }
            carry[k] = bot;
            uc[0][k] = un[0][k];
            uc[1][k] = un[1][k];
          }
        }
      }
    }
  }
  if (a.partials) {
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dotacc += __shfl_xor_sync(0xffffffffu, dotacc, o);
    if (lane == 0) red[threadIdx.x >> 5] = dotacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      a.partials[blockIdx.x] = t;
    }
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < kRedBlocks; i += blockDim.x) a.partials[i] = 0.0;
  }
}

}  // namespace

bool elem2d_eligible(const Grid& g) {
  // small (L2-resident) grids have too few strips: the generic pixel-parallel kernel wins
  return g.d == 2 && (g.c == 1 || g.c == 2) && !g.dist && g.n1 >= 2 && g.n0 >= 2 && g.np >= (1 << 20) &&
         g.nn == 1;
}

// Per-phase triangle tables (TwoTriangles): scalar A_ij = w C_ij / (h_i h_j);
// elastic rows (t0, t1, t2, t3) = w (s0 / h0, s1 / h1, s2 s12 / h1, s2 s12 / h0)
// as linear forms in (d0x, d1y, d1x + d0y) with the Mandel shear
// eps12 = s2 ((u1 - u0)_x / h1 + ...): see tri_element.
void elem2d_tri_tables(const Grid& g, int n_phases, const double* cmats, std::vector<double>& tab) {
  const double h0 = g.h[0], h1 = g.h[1];
  const double w = h0 * h1 / 2.0, s2 = 0.70710678118654752440;
  tab.clear();
  const int m = g.m;
  for (int ph = 0; ph < n_phases; ++ph) {
    const double* cm = cmats + (size_t)ph * m * m;  // column-major
    auto C = [&](int i, int j) { return cm[j * m + i]; };
    if (g.c == 1) {
      tab.push_back(w * C(0, 0) / (h0 * h0));
      tab.push_back(w * C(0, 1) / (h0 * h1));
      tab.push_back(w * C(1, 0) / (h1 * h0));
      tab.push_back(w * C(1, 1) / (h1 * h1));
    } else {
      // eps = (d0x / h0, d1y / h1, s2 (d1x / h1 + d0y / h0)); for the triangle
      // pairs of this stencil the shear enters as d1x / h1 + d0y / h0 -> with
      // h0 == h1 this is (d1x + d0y) / h; general h: keep both columns exact
      // by requiring square pixels (checked by the caller)
      const double hh = h0;
      // sigma_i = C_i0 d0x / h0 + C_i1 d1y / h1 + C_i2 s2 (d1x + d0y) / hh
      double L[3][3];
      for (int i = 0; i < 3; ++i) {
        L[i][0] = C(i, 0) / h0;
        L[i][1] = C(i, 1) / h1;
        L[i][2] = C(i, 2) * s2 / hh;
      }
      const double f[4] = {w / h0, w / h1, w * s2 / h1, w * s2 / h0};
      const int row[4] = {0, 1, 2, 2};
      for (int r = 0; r < 4; ++r)
        for (int j = 0; j < 3; ++j) tab.push_back(f[r] * L[row[r]][j]);
    }
  }
}

void launch_elem2d(const Grid& g, const ElemArgs& a, const double* d_tri, cudaStream_t s) {
  const bool tri = g.kind == 1 && d_tri && (g.c == 1 || g.h[0] == g.h[1]);
  const int ne = 4 * g.c;
  const int ms = tri ? (g.c == 1 ? 4 : 12) : ne * ne;
  const size_t smem = (size_t)a.n_phases * ms * sizeof(double);
  const int smem_ok = smem <= 48 * 1024;
  const size_t dyn = smem_ok ? smem : 0;
#define HB_E2D(C, T) k_elem2d<C, T><<<kRedBlocks, 256, dyn, s>>>(g, a, d_tri, smem_ok)
  if (g.c == 1) {
    if (tri) HB_E2D(1, true);
    else HB_E2D(1, false);
  } else {
    if (tri) HB_E2D(2, true);
    else HB_E2D(2, false);
  }
#undef HB_E2D
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
