// small2d.cu -- the whole PCG solve of a small 2-D scalar problem as ONE
// persistent thread-block cluster (c1: 256^2 pixels, TwoTriangles, c = 1).
//
// At 256^2 every vector is 512 KB: the multi-kernel iteration (K, alpha,
// r update, D2Z, symbol solve, beta, Z2D, x/p update: 8 launches) is launch
// and latency bound (~31 us per iteration for ~2 us of HBM traffic). Here a
// 16-CTA cluster (one CTA per SM, non-portable cluster size) keeps x, r, p
// and every intermediate in shared memory for the whole solve and runs the
// reference's loop (proj/src/solver.cpp:50-97) with cluster barriers instead
// of kernel boundaries:
//
//   CTA q owns pixel rows [16 q, 16 q + 16) of x, r, p (row-major, the
//   reference layout) and, in Fourier space, the half-spectrum columns
//   k1 in [8 q, 8 q + 8) (column 0 of CTA 0 packs the two real columns
//   k1 = 0 and k1 = 128 as one complex column, like the 3-D fused passes).
//
//   per iteration
//     K p        element rows march down the CTA's rows (two 256-thread
//                groups of 8 rows, one warm-up element row each); the
//                halo node rows -1 and 16 are read from the neighbouring
//                CTAs over DSMEM; x-neighbours via a shared exchange slot;
//                p.Ap partial per CTA
//     alpha      per-CTA partials stored into every CTA (DSMEM), cluster
//                barrier, fixed-order sum in every CTA (identical scalars)
//     r update + row r2c FFTs (two rows per complex 256-point transform)
//     gather     each CTA pulls its 8 columns from all 16 CTAs (DSMEM)
//     column FFT, z_hat = K_hat(xi)^-1 r_hat / N (spectral.cuh, the same
//                symbol as the cuFFT path), r.z by Parseval, inverse FFT
//     beta       cluster reduction as for alpha; stopping test of
//                solver.cpp:88-91 on every CTA
//     scatter    columns back into the owners' rows (DSMEM stores)
//     row c2r FFTs, x += alpha p, p = z + beta p
//
// Five cluster barriers per iteration, no HBM traffic inside the loop. The
// scalar protocol (PcgState, history) is the one of k_pcg_init / k_pcg_alpha
// / k_pcg_beta (kernels.cu), so the host side reads the same state.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "kernels.cuh"
#include "spectral.cuh"

namespace hb {

namespace {

namespace cg = cooperative_groups;

constexpr int kNX = 256;         // row length (axis 1, contiguous)
constexpr int kP = kNX / 2 + 1;  // half-spectrum length
constexpr int kR = 16;           // rows per CTA
constexpr int kCL = 16;          // CTAs per cluster (rows = kCL * kR = 256)
constexpr int kT = 512;          // threads per CTA
constexpr int kCols = kNX / 2 / kCL;  // column slots per CTA (8)
constexpr int kCP = kNX + 1;          // column buffer pitch (double2)

struct S2Args {
  double* x;
  double* r;  // in: b; out: final residual
  double* p;
  const uint8_t* phase;
  const double* tab;  // per-phase triangle tables, 4 doubles (elem2d_tri_tables)
  int n_phases;
  const double2* tw;  // W_256 four-step table (fft.cuh layout)
  PcgState* st;
  double* hist;
};

struct S2Smem {
  double* xs;     // [kR][kNX]
  double* rs;
  double* ps;
  double2* spec;  // [kR][kP] row spectra; aliased by Ap [kR][kNX] doubles
  double2* cb;    // [kCols][kCP] column buffers
  double2* tw4;   // [256] four-step twiddles
  double* tab;    // [n_phases][4]
  double* xch;    // [2][2][kNX][2] K x-exchange
  uint8_t* ph;    // [kR + 1][kNX] element rows -1 .. kR-1
};

__host__ __device__ constexpr size_t s2_smem_bytes(int n_phases) {
  return sizeof(double) * 3 * kR * kNX + sizeof(double2) * kR * kP + sizeof(double2) * kCols * kCP +
         sizeof(double2) * kNX + sizeof(double) * 4 * (size_t)n_phases + sizeof(double) * 2 * 2 * kNX * 2 +
         (size_t)(kR + 1) * kNX;
}

__device__ __forceinline__ S2Smem s2_layout(unsigned char* base, int n_phases) {
  S2Smem s;
  double* d = reinterpret_cast<double*>(base);
  s.xs = d;
  s.rs = d + kR * kNX;
  s.ps = d + 2 * kR * kNX;
  s.spec = reinterpret_cast<double2*>(d + 3 * kR * kNX);
  s.cb = s.spec + kR * kP;
  s.tw4 = s.cb + kCols * kCP;
  s.tab = reinterpret_cast<double*>(s.tw4 + kNX);
  s.xch = s.tab + 4 * n_phases;
  s.ph = reinterpret_cast<uint8_t*>(s.xch + 2 * 2 * kNX * 2);
  return s;
}

// Fixed-order sum of one value per thread over the CTA, then over the
// cluster: every CTA stores its total into slot [rank] of every CTA's `slots`
// and, after the cluster barrier, sums the kCL slots in rank order (all CTAs
// get the bitwise same scalar).
__device__ __forceinline__ double cluster_sum(double v, double* wred, double* slots, cg::cluster_group& cl,
                                              int rank) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) wred[warp] = v;
  __syncthreads();
  if (tid < kCL) {
    double s = 0.0;
    for (int w = 0; w < kT / 32; ++w) s += wred[w];
    double* dst = cl.map_shared_rank(slots, tid);
    dst[rank] = s;
  }
  cl.sync();
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < kCL; ++q) tot += slots[q];
  return tot;
}

// z = M^-1 r of the CTA's rows (row r2c, column transforms and the symbol
// solve, inverse), leaving z in the row-pair buffers of `spec` (.x = row 2g,
// .y = row 2g + 1, columns 0..255) and returning the cluster-wide r.z.
__device__ double precond(const SpecParams& sp, const S2Smem& s, cg::cluster_group& cl, int rank, double* wred,
                          double* slots) {
  const int tid = threadIdx.x;
  constexpr int TPF = 16;
  // ---- row r2c FFTs: group g (16 threads) transforms rows (2g, 2g+1) as
  // one complex sequence (four-step radix-16, fft.cuh), then splits the two
  // half spectra
  if (tid < (kR / 2) * TPF) {
    const int g = tid / TPF, t = tid % TPF;
    double2* buf = s.spec + (2 * g) * kP;
    double2 vr[16];
    const double* xa = s.rs + (2 * g) * kNX;
    const double* xb = xa + kNX;
#pragma unroll
    for (int i = 0; i < 16; ++i) vr[i] = make_double2(xa[t + i * TPF], xb[t + i * TPF]);
    fft::group_sync();
    fft::fft4step_regs<kNX, false>(vr, buf, t, s.tw4);
    constexpr int KN = (kP + TPF - 1) / TPF;
    double2 za[KN], zb[KN];
#pragma unroll
    for (int i = 0; i < KN; ++i) {
      const int k = t + i * TPF;
      if (k < kP) {
        const double2 zk = buf[k % kNX], zm = fft::conj(buf[(kNX - k) % kNX]);
        const double2 sm = fft::cadd(zk, zm), d = fft::csub(zk, zm);
        za[i] = make_double2(0.5 * sm.x, 0.5 * sm.y);
        zb[i] = make_double2(0.5 * d.y, -0.5 * d.x);  // -i/2 * d
      }
    }
    fft::group_sync();
#pragma unroll
    for (int i = 0; i < KN; ++i) {
      const int k = t + i * TPF;
      if (k < kP) {
        buf[k] = za[i];
        buf[kP + k] = zb[i];
      }
    }
  }
  cl.sync();  // every CTA's row spectra complete
  // ---- gather: warp w pulls rows of CTA w, this CTA's column slots
  {
    const int lane = tid & 31, w = tid >> 5;
    const int i = lane >> 1, half = lane & 1;
    const double2* src = cl.map_shared_rank(s.spec, w) + i * kP;
    double2 v[kCols / 2];  // all remote loads in flight before the first store
#pragma unroll
    for (int jj = 0; jj < kCols / 2; ++jj) {
      const int k1 = kCols * rank + half * (kCols / 2) + jj;
      if (k1 == 0) v[jj] = make_double2(src[0].x, src[kNX / 2].x);
      else v[jj] = src[k1];
    }
#pragma unroll
    for (int jj = 0; jj < kCols / 2; ++jj) s.cb[(half * (kCols / 2) + jj) * kCP + kR * w + i] = v[jj];
  }
  __syncthreads();
  // ---- column FFTs (axis 0)
  if (tid < kCols * TPF) fft::fft4step<kNX, false>(s.cb + (tid / TPF) * kCP, tid % TPF, s.tw4);
  __syncthreads();
  // ---- solve z_hat = K_hat^-1 r_hat / N_p, r.z (Parseval, solver.cpp:84)
  double rz = 0.0;
  auto zsolve = [&](double2 r, int k0, int k1, double wgt) -> double2 {
    if (k0 == 0 && k1 == 0) return make_double2(0.0, 0.0);
    const int f[3] = {k0, k1, 0};
    double M[3][3], K[3][3], I[3][3];
    spec::gram<2>(sp, f, M);
    spec::symbol<2, 1>(sp, M, K);
    spec::sym_inverse<1>(K, I);
    const double2 z = make_double2(I[0][0] * r.x * sp.inv_np, I[0][0] * r.y * sp.inv_np);
    rz = fma(wgt, r.x * z.x + r.y * z.y, rz);
    return z;
  };
  const int first = rank == 0 ? 1 : 0;  // CTA 0 slot 0: the packed real columns
  for (int e = first * kNX + tid; e < kCols * kNX; e += kT) {
    const int slot = e / kNX, k0 = e % kNX;
    double2* c = s.cb + slot * kCP + k0;
    *c = zsolve(*c, k0, kCols * rank + slot, 2.0);
  }
  if (rank == 0 && tid <= kNX / 2) {
    // X = A + i B (A: column k1 = 0, B: k1 = N/2, both Hermitian in k0):
    // each thread takes the pair (k0, -k0)
    const int k0 = tid, km = (kNX - k0) % kNX;
    const double2 X = s.cb[k0], Xm = fft::conj(s.cb[km]);
    const double2 sm = fft::cadd(X, Xm), d = fft::csub(X, Xm);
    const double2 A = make_double2(0.5 * sm.x, 0.5 * sm.y), B = make_double2(0.5 * d.y, -0.5 * d.x);
    const double2 zA = zsolve(A, k0, 0, 1.0), zB = zsolve(B, k0, kNX / 2, 1.0);
    if (km != k0) {  // the partner frequency: conjugates, same weight
      rz = fma(1.0, A.x * zA.x + A.y * zA.y, rz);
      rz = fma(1.0, B.x * zB.x + B.y * zB.y, rz);
    }
    __syncwarp(__activemask());
    // Z = zA + i zB at k0, conj(zA) + i conj(zB) at -k0
    s.cb[k0] = make_double2(zA.x - zB.y, zA.y + zB.x);
    if (km != k0) s.cb[km] = make_double2(zA.x + zB.y, zB.x - zA.y);
  }
  __syncthreads();
  if (tid < kCols * TPF) fft::fft4step<kNX, true>(s.cb + (tid / TPF) * kCP, tid % TPF, s.tw4);
  // cluster barrier inside: every gather done (row spectra free) and r.z known
  const double rz_tot = cluster_sum(rz, wred, slots, cl, rank);
  // ---- scatter the columns back into the owners' row spectra
  {
    const int lane = tid & 31, w = tid >> 5;
    const int i = lane >> 1, half = lane & 1;
    double2* dst = cl.map_shared_rank(s.spec, w) + i * kP;
#pragma unroll
    for (int jj = 0; jj < kCols / 2; ++jj) {
      const int slot = half * (kCols / 2) + jj;
      const int k1 = kCols * rank + slot;
      const double2 v = s.cb[slot * kCP + kR * w + i];
      if (k1 == 0) {
        dst[0] = make_double2(v.x, 0.0);
        dst[kNX / 2] = make_double2(v.y, 0.0);
      } else {
        dst[k1] = v;
      }
    }
  }
  cl.sync();
  // ---- row c2r: Z = A + i B of the row pair, z = IFFT(Z)
  if (tid < (kR / 2) * TPF) {
    const int g = tid / TPF, t = tid % TPF;
    double2* buf = s.spec + (2 * g) * kP;
    const double2* A = buf;
    const double2* B = buf + kP;
    double2 u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = t + i * TPF;
      const int k = n <= kNX / 2 ? n : kNX - n;
      double2 av = A[k], bv = B[k];
      if (k == 0 || k == kNX / 2) {
        av.y = 0.0;
        bv.y = 0.0;
      }
      u[i] = n <= kNX / 2 ? make_double2(av.x - bv.y, av.y + bv.x) : make_double2(av.x + bv.y, bv.x - av.y);
    }
    fft::group_sync();
    fft::fft4step_regs<kNX, true>(u, buf, t, s.tw4);
  }
  __syncthreads();
  return rz_tot;
}

// z of pixel (row y, column x) after precond()
__device__ __forceinline__ double z_at(const S2Smem& s, int y, int x) {
  const double2 v = s.spec[(y & ~1) * kP + x];
  return (y & 1) ? v.y : v.x;
}

__global__ void __launch_bounds__(kT, 1) k_pcg_small2d(const __grid_constant__ SpecParams sp, const S2Args a) {
  extern __shared__ __align__(16) unsigned char s2_raw[];
  __shared__ double wred[kT / 32];
  __shared__ double slots_a[kCL], slots_b[kCL];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const S2Smem s = s2_layout(s2_raw, a.n_phases);
  const int y0 = rank * kR;  // first global row of this CTA
  const int64_t base = (int64_t)y0 * kNX;
  // ---- load r = b, the phase rows (with the element row above), tables
  for (int i = tid; i < kR * kNX; i += kT) {
    s.rs[i] = a.r[base + i];
    s.xs[i] = 0.0;
  }
  for (int i = tid; i < (kR + 1) * kNX; i += kT) {
    int yy = y0 - 1 + i / kNX;
    yy = yy < 0 ? yy + kCL * kR : yy;
    s.ph[i] = a.phase[(int64_t)yy * kNX + i % kNX];
  }
  for (int i = tid; i < 4 * a.n_phases; i += kT) s.tab[i] = a.tab[i];
  for (int i = tid; i < kNX; i += kT) s.tw4[i] = a.tw[i];
  const double eta = a.st->eta;
  const int it_max = a.st->it_max;
  __syncthreads();
  cl.sync();  // every CTA's shared memory is initialised before any DSMEM access
  // ---- init (solver.cpp:62-73): z0 = M^-1 r0, rz0, p = z0
  double rz = fmax(precond(sp, s, cl, rank, wred, slots_b), 0.0);
  const double norm0 = sqrt(rz);
  for (int i = tid; i < kR * kNX; i += kT) s.ps[i] = z_at(s, i / kNX, i % kNX);
  int it = 0, status = 0, active = 0;
  bool converged = norm0 == 0.0;
  bool done = converged || it_max <= 0;
  double pap = 0.0, alpha = 0.0, beta = 0.0;
  if (rank == 0 && tid == 0) a.hist[0] = norm0;
  cl.sync();  // p complete everywhere (K reads the neighbours' rows)
  const int gy = tid / kNX, x = tid % kNX;
  const int xr = (x + 1) % kNX, xl = (x + kNX - 1) % kNX;
  const double* p_up = cl.map_shared_rank(s.ps, (rank + kCL - 1) % kCL) + (kR - 1) * kNX;  // row -1
  const double* p_dn = cl.map_shared_rank(s.ps, (rank + 1) % kCL);                          // row kR
  double* aps = reinterpret_cast<double*>(s.spec);
  while (!done) {
    // ---- K p (operators.cpp:197-243 for the TwoTriangles stencil), p.Ap
    double dot = 0.0;
    {
      const int e0 = gy * (kR / 2) - 1;  // first element row (warm-up)
      auto prow = [&](int y) -> const double* {
        return y < 0 ? p_up : (y >= kR ? p_dn : s.ps + y * kNX);
      };
      double uc0 = prow(e0)[x], uc1 = prow(e0)[xr];
      double carry = 0.0;
#pragma unroll 1
      for (int stp = 0; stp <= kR / 2; ++stp) {
        const int ye = e0 + stp;
        const double* pn = prow(ye + 1);
        const double un0 = pn[x], un1 = pn[xr];
        const double* A = s.tab + 4 * s.ph[(ye + 1) * kNX + x];
        // corners 0 = (ye, x), 1 = (ye+1, x), 2 = (ye, x+1), 3 = (ye+1, x+1)
        const double a00 = A[0], a01 = A[1], a10 = A[2], a11 = A[3];
        double r0, r1, r2, r3;
        {
          const double d0 = un0 - uc0, d1 = uc1 - uc0;
          const double fa = fma(a00, d0, a01 * d1), fb = fma(a10, d0, a11 * d1);
          r0 = -(fa + fb);
          r1 = fa;
          r2 = fb;
        }
        {
          const double d0 = un1 - uc1, d1 = un1 - un0;
          const double fa = fma(a00, d0, a01 * d1), fb = fma(a10, d0, a11 * d1);
          r3 = fa + fb;
          r2 -= fa;
          r1 -= fb;
        }
        double* xs = s.xch + (((stp & 1) * 2 + gy) * kNX) * 2;
        xs[2 * x] = r2;
        xs[2 * x + 1] = r3;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + gy), "r"(kNX) : "memory");
        const double q2 = xs[2 * xl], q3 = xs[2 * xl + 1];
        const double top = r0 + q2, bot = r1 + q3;
        if (stp > 0) {
          const double v = carry + top;
          aps[ye * kNX + x] = v;
          dot = fma(uc0, v, dot);
        }
        carry = bot;
        uc0 = un0;
        uc1 = un1;
      }
    }
    pap = cluster_sum(dot, wred, slots_a, cl, rank);
    // ---- alpha (solver.cpp:74-80)
    if (!(pap > 0.0)) {
      status = 4;
      done = true;
      active = 0;
      break;
    }
    active = 1;
    alpha = rz / pap;
    for (int i = tid; i < kR * kNX; i += kT) s.rs[i] = fma(-alpha, aps[i], s.rs[i]);
    __syncthreads();
    // ---- z = M^-1 r, beta, stopping test (solver.cpp:84-93)
    const double rzn = fmax(precond(sp, s, cl, rank, wred, slots_b), 0.0);
    it += 1;
    if (rank == 0 && tid == 0) a.hist[it] = sqrt(rzn);
    if (sqrt(rzn) <= eta * norm0) {
      converged = true;
      done = true;
    } else {
      beta = rzn / rz;
      rz = rzn;
      if (it >= it_max) done = true;
    }
    // ---- x += alpha p; p = z + beta p unless the loop ended (solver.cpp:81, 93)
    for (int i = tid; i < kR * kNX; i += kT) {
      const double pv = s.ps[i];
      s.xs[i] = fma(alpha, pv, s.xs[i]);
      if (!done) s.ps[i] = fma(beta, pv, z_at(s, i / kNX, i % kNX));
    }
    cl.sync();  // p complete everywhere before the next K
  }
  // ---- results
  for (int i = tid; i < kR * kNX; i += kT) {
    a.x[base + i] = s.xs[i];
    a.r[base + i] = s.rs[i];
    a.p[base + i] = s.ps[i];
  }
  if (rank == 0 && tid == 0) {
    PcgState* st = a.st;
    st->rz = rz;
    st->pap = pap;
    st->alpha = alpha;
    st->beta = beta;
    st->norm0 = norm0;
    st->it = it;
    st->done = 1;
    st->converged = converged ? 1 : 0;
    st->status = status;
    st->active = active;
  }
  cl.sync();  // no CTA exits while others may still read its shared memory
}

}  // namespace

bool small2d_eligible(const Grid& g, int n_phases) {
  return g.d == 2 && g.c == 1 && g.kind == 1 && g.nn == 1 && !g.dist && g.n0 == kCL * kR && g.n1 == kNX &&
         n_phases >= 1 && s2_smem_bytes(n_phases) <= 200 * 1024;
}

// Returns false (nothing launched) when the cluster cannot be scheduled on
// this device; the caller then runs the multi-kernel iteration.
bool launch_pcg_small2d(const SpecParams& sp, double* x, double* r, double* p, const uint8_t* phase,
                        const double* tri_tab, int n_phases, const double2* tw, PcgState* st, double* hist,
                        cudaStream_t s) {
  const size_t smem = s2_smem_bytes(n_phases);
  static int ok = -1;
  if (ok < 0) {
    ok = 0;
    if (cudaFuncSetAttribute(k_pcg_small2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024)) ==
            cudaSuccess &&
        cudaFuncSetAttribute(k_pcg_small2d, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(kCL);
      cfg.blockDim = dim3(kT);
      cfg.dynamicSmemBytes = 200 * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kCL;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, k_pcg_small2d, &cfg) == cudaSuccess && ncl >= 1) ok = 1;
    }
    cudaGetLastError();
  }
  if (!ok) return false;
  S2Args a;
  a.x = x;
  a.r = r;
  a.p = p;
  a.phase = phase;
  a.tab = tri_tab;
  a.n_phases = n_phases;
  a.tw = tw;
  a.st = st;
  a.hist = hist;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCL);
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  HB_CUDA(cudaLaunchKernelEx(&cfg, k_pcg_small2d, sp, a));
  return true;
}

}  // namespace hb
