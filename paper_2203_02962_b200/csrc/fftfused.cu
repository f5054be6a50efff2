// fftfused.cu -- the preconditioner M^-1 = F^-1 K_ref_hat^+ F of one PCG
// iteration as three streaming passes, fused with the PCG vector updates.
//
// The reference calls FFTW r2c/c2r per component and runs the per-frequency
// block multiply and the axpys as separate sweeps (precond.cpp:126-162,
// solver.cpp:80-92). cuFFT needs three HBM passes per 3-D transform; with the
// pointwise solve and the two update kernels that is 10 passes over c fields
// per iteration. Here:
//
//   pass 1  k_plane_fwd  one thread-block cluster per (component, x0-plane):
//           r <- r - alpha Ap (written back), 2-D r2c FFT of the plane
//           (row FFTs in each CTA's shared memory, column FFTs over DSMEM),
//           half spectrum T written once;
//   pass 2  k_pencil     per (k1, k2-tile): 1-D FFT along axis 0 for all c
//           components, z_hat = K_ref_hat(xi)^+ r_hat / N_p with the analytic
//           symbol, r.z by Parseval, inverse 1-D FFT, T written back;
//   pass 3  k_plane_inv  one cluster per (component, plane): inverse 2-D
//           c2r FFT, then x <- x + alpha p and p <- z + beta p (z is never
//           stored).
//
// Per component and voxel this moves 32 + 16 + 40 = 88 bytes, against 8
// streaming passes (~216 bytes) for cuFFT + separate kernels.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "fft.cuh"
#include "kernels.cuh"
#include "spectral.cuh"

namespace cg = cooperative_groups;

namespace hb {

namespace {

using fft::cadd;
using fft::cmul;
using fft::conj;
using fft::csub;

constexpr int kThreads = 256;

enum { kModePcg = 0, kModePlain = 1, kModeInit = 2, kModeZ = 3 };

// Intermediate spectra. Rank r of G owns planes [r nzl, (r+1) nzl) and, in
// pass 2, rows k1 in [r n1l, (r+1) n1l).
//   pass 1 -> 2: T[peer][c][k1l][k2 / 4][i0l][k2 % 4]   (tile-major)
//     written by the plane owner with peer = destination (k1 / n1l), read by
//     the pencil owner with peer = source (i0 / nzl); between the two an
//     all-to-all swaps peer chunks (G = 1: the same buffer, no exchange).
//     A pass-1 CTA stores 64-byte pieces; a pass-2 block's 4-column group
//     is one contiguous run per peer (one TMA bulk copy).
//   pass 2 -> 3: T2[peer][c][i0l][k1l][k2]   (plane-major, 16-aligned pitch)
//     written by the pencil owner with peer = destination (i0 / nzl), read
//     by the plane owner with peer = source (k1 / n1l).
// The scattered side of each transpose is a store (merged in L2).
constexpr int kTB = 16;  // T2 row pitch granule
constexpr int kTG = 4;   // T column group: a pencil block's TMA unit
__host__ __device__ constexpr int t_blocks(int np_plane) { return (np_plane / 2 + 1 + kTB - 1) / kTB; }
__host__ __device__ constexpr int t_groups(int np_plane) { return (np_plane / 2 + 1 + kTG - 1) / kTG; }
// Within a 64-byte [i0][4] row of T the column slot is XOR-swizzled by the
// plane index ((i0 >> 1) & 3, the pattern of CU_TENSOR_MAP_SWIZZLE_64B): a
// pencil thread's 16-byte reads of rows t, t+1, ... of ONE column then fall
// into 8 distinct bank groups (unswizzled: 2 -> 4-way conflicts on every
// stage read and re-layout write of pass 2).
__host__ __device__ constexpr int t_swz(int i0) { return (i0 >> 1) & 3; }
struct TLayout {
  int nc, n1l, nzl, nb, ng;  // ng: 4-column groups of T
  int sh1, shz;  // log2 n1l, log2 nzl (both powers of two)
  // global k1 / global i0 -> (peer, local) without divisions
  __device__ __forceinline__ int p1(int k1) const { return k1 >> sh1; }
  __device__ __forceinline__ int l1(int k1) const { return k1 & (n1l - 1); }
  __device__ __forceinline__ int pz(int i0) const { return i0 >> shz; }
  __device__ __forceinline__ int lz(int i0) const { return i0 & (nzl - 1); }
  // t(peer(k1), comp, k1l, k2, i0l) = (row1 * ng + k2 / 4) * nzl * 4 + i0l * 4 + k2 % 4
  __device__ __forceinline__ int row1(int comp, int k1) const { return comp * n1l + k1 + p1(k1) * (nc - 1) * n1l; }
  // t2(peer(k1), comp, i0l, k1l, k2) = row2 * (nb * 16) + k2
  __device__ __forceinline__ int row2(int comp, int i0l, int k1) const {
    const int q = p1(k1);
    return ((q * nc + comp) * nzl + i0l) * n1l + k1 - q * n1l;
  }
  __device__ __forceinline__ int64_t t(int peer, int comp, int k1l, int k2, int i0l) const {
    return ((((int64_t)peer * nc + comp) * n1l + k1l) * ng + (k2 / kTG)) * ((int64_t)nzl * kTG) +
           (int64_t)i0l * kTG + ((k2 % kTG) ^ t_swz(i0l));
  }
  __device__ __forceinline__ int64_t t2(int peer, int comp, int i0l, int k1l, int k2) const {
    return ((((int64_t)peer * nc + comp) * nzl + i0l) * n1l + k1l) * (int64_t)(nb * kTB) + k2;
  }
};


struct PlaneArgs {
  int n0;              // LOCAL planes per component (axis 0)
  int64_t np;          // LOCAL pixels per component
  TLayout L;
  double* r;           // pass 1 input (updated in PCG mode)
  const double* ap;    // pass 1, PCG mode
  double2* T;          // pass 1 output (TLayout::t)
  double2* T2;         // pass 3 input (TLayout::t2)
  double* p;           // pass 3
  double* x;           // pass 3, PCG mode
  double* z;           // pass 3, z mode
  const double2* tw;   // W_NP table
  const PcgState* st;  // PCG mode
  int mode;
  int dbg;             // profiling only: bit mask of skipped phases
  int ahead;           // L2 prefetch distance in clusters (0 = off): the inputs of cluster cid + ahead
  const double2* t2p[FusedFft::kMaxPeers];  // pass 3: chunk bases per source peer (FusedFft::t2pull)
};

template <int NP>
constexpr int tpf() {
  return NP / 16;
}

template <int NP>
constexpr int rows_slots() {
  constexpr int P = NP / 2 + 1;
  return 32 * P > 16 * (NP + 1) ? 32 * P : 16 * (NP + 1);
}

#ifndef HB_FWD_MINB
#define HB_FWD_MINB 3  // 80 registers, no spill of note: 48 instead of 33 resident clusters
#endif
template <int NP>
__global__ void __launch_bounds__(NP, HB_FWD_MINB) k_plane_fwd(const PlaneArgs a) {
  constexpr int P = NP / 2 + 1;
  constexpr int CL = NP / 32;
  constexpr int TPF = tpf<NP>();
  constexpr int H = NP / 2;
  constexpr int PT = 32 * H / NP;  // double2 per thread in the row block (= 16)
  if (a.mode == kModePcg && !a.st->active) return;
  extern __shared__ double2 sm[];
  double2* rows = sm;                      // 32 x P (row phase) / 16 x (NP+1) (column phase)
  double2* tws = rows + rows_slots<NP>();  // NP
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / CL;
  const int comp = cid / a.n0, i0 = cid % a.n0;
  const int tid = threadIdx.x, g = tid / TPF, t = tid % TPF;
  const int64_t plane = (int64_t)comp * a.np + (int64_t)i0 * NP * NP + (int64_t)rank * 32 * NP;
  constexpr uint32_t ROWB = NP * sizeof(double);
  const bool pcg = a.mode == kModePcg;
  if (tid == 0) {
    fft::mbar_init(&bar, 1);
    fft::fence_mbar_init();
  }
  __syncthreads();
  const bool noio = a.dbg & 128;  // profiling: no r / Ap traffic
  // PCG mode: r and Ap go straight from HBM into the row-FFT register layout
  // (thread t of group g: columns t + TPF i of rows 2g, 2g+1; each group
  // reads 2 x 128-byte row segments per step), r - alpha Ap is written back
  // from registers and fed to the FFT: no shared-memory staging of the rows
  // (measured: 128^2 planes 0.031 -> 0.026 ms; 256^2 planes 0.468 -> 0.505 ms,
  // there the TMA-staged rows win: HB_FWD_REGLOAD = largest plane size using it;
  // a hybrid -- r staged by TMA, Ap loaded in the FFT layout, update in the FFT
  // registers, no shared-memory update pass -- measured 0.460 -> 0.468 ms)
#ifndef HB_FWD_REGLOAD
#define HB_FWD_REGLOAD 128
#endif
  const bool regload = NP <= HB_FWD_REGLOAD && pcg && !noio;
  if (tid == 0 && !regload) {
    fft::mbar_expect_tx(&bar, noio ? 0 : 32 * ROWB);
    if (!noio)
      for (int y = 0; y < 32; ++y) fft::bulk_g2s(rows + y * P, a.r + plane + (int64_t)y * NP, ROWB, &bar);
  }
  for (int i = tid; i < NP; i += NP) tws[i] = a.tw[i];
  if (a.ahead > 0 && pcg && tid < 64 && cid + a.ahead < (int)(gridDim.x / CL)) {
    // L2 prefetch of the r and Ap rows of the cluster that will take this one's place
    const int cn = cid + a.ahead;
    const int64_t pl = (int64_t)(cn / a.n0) * a.np + (int64_t)(cn % a.n0) * NP * NP + (int64_t)rank * 32 * NP +
                       (int64_t)(tid & 31) * NP;
    const double* pf = (tid < 32 ? a.r : a.ap) + pl;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"((uint32_t)ROWB) : "memory");
  }
  double2 vr[16];  // row pair values in the FFT register layout
  if (regload) {
    const double alpha = a.st->alpha;
    double* ra = a.r + plane + (int64_t)(2 * g) * NP;
    double* rb = ra + NP;
    const double* pa = a.ap + plane + (int64_t)(2 * g) * NP;
    const double* pb = pa + NP;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = t + i * TPF;
      double x0 = ra[n], x1 = rb[n];
      x0 = fma(-alpha, __ldg(pa + n), x0);
      x1 = fma(-alpha, __ldg(pb + n), x1);
      ra[n] = x0;
      rb[n] = x1;
      vr[i] = make_double2(x0, x1);
    }
  } else {
    double2 apv[PT];
    if (pcg && !noio) {
      const double2* ap2 = reinterpret_cast<const double2*>(a.ap + plane);
#pragma unroll
      for (int i = 0; i < PT; ++i) apv[i] = ap2[tid + i * NP];
    }
    fft::mbar_wait(&bar, 0);
    if (pcg && !noio) {
      const double alpha = a.st->alpha;
#ifndef HB_FWD_RSTORE
#define HB_FWD_RSTORE 1  // r written back with plain stores from the update loop (0.468 -> 0.462 ms)
#endif
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int idx = tid + i * NP, row = idx / H, c2 = idx % H;
        double2 w = rows[row * P + c2];
        w.x = fma(-alpha, apv[i].x, w.x);
        w.y = fma(-alpha, apv[i].y, w.y);
        rows[row * P + c2] = w;
        if (HB_FWD_RSTORE) reinterpret_cast<double2*>(a.r + plane)[idx] = w;
      }
      __syncthreads();
      // (HB_FWD_RSTORE=0: r written back by TMA bulk stores instead, so that no
      // generic stores are in flight at the cluster barriers below)
      if (tid == 0 && !HB_FWD_RSTORE) {
        fft::fence_proxy_async();
        for (int y = 0; y < 32; ++y) fft::bulk_s2g(a.r + plane + (int64_t)y * NP, rows + y * P, ROWB);
        fft::bulk_commit();
        fft::bulk_wait_read();
      }
    }
  }
  if (!HB_FWD_RSTORE || !pcg || regload) __syncthreads();
  // row r2c: group g transforms the row pair (2g, 2g+1) in place
  if (!(a.dbg & 1)) {
    double2* buf = rows + (2 * g) * P;
    if (!regload) {
      const double* xa = reinterpret_cast<const double*>(rows + (2 * g) * P);
      const double* xb = reinterpret_cast<const double*>(rows + (2 * g + 1) * P);
#pragma unroll
      for (int i = 0; i < 16; ++i) vr[i] = make_double2(xa[t + i * TPF], xb[t + i * TPF]);
    }
    fft::group_sync();
    fft::fft4step_regs<NP, false>(vr, buf, t, tws);
    constexpr int KN = (P + TPF - 1) / TPF;
    double2 za[KN], zb[KN];
#pragma unroll
    for (int i = 0; i < KN; ++i) {
      const int k = t + i * TPF;
      if (k < P) {
        const double2 zk = buf[k % NP], zm = conj(buf[(NP - k) % NP]);
        const double2 s = cadd(zk, zm), d = csub(zk, zm);
        za[i] = make_double2(0.5 * s.x, 0.5 * s.y);
        zb[i] = make_double2(0.5 * d.y, -0.5 * d.x);  // -i/2 * d
      }
    }
    fft::group_sync();
#pragma unroll
    for (int i = 0; i < KN; ++i) {
      const int k = t + i * TPF;
      if (k < P) {
        buf[k] = za[i];
        buf[P + k] = zb[i];
      }
    }
  }
  cluster.sync();
  // gather this CTA's 16 column slots over DSMEM: warp w reads the rows of
  // CTA w, each half-warp one row's 16 contiguous columns (256 B)
  const int lane = tid & 31, warp = tid >> 5;
  const int jc = lane & 15, yo = lane >> 4;
  constexpr int NW = NP / 32;  // warps per CTA == CTAs per cluster
  static_assert(NW == CL, "one warp per remote CTA");
  double2 v[16];
  {
    const double2* src = (a.dbg & 2) ? rows : cluster.map_shared_rank(rows, warp);
    const int col = rank * 16 + jc;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2* row = src + (2 * i + yo) * P;
      if (col == 0) v[i] = make_double2(row[0].x, row[NP / 2].x);
      else v[i] = row[col];
    }
  }
  cluster.sync();  // every remote read done: local rows become column buffers
  // transpose into padded column buffers: slot jc, position y = 32 warp + 2 i + yo
#pragma unroll
  for (int i = 0; i < 16; ++i) rows[jc * (NP + 1) + 32 * warp + 2 * i + yo] = v[i];
  __syncthreads();
  double2* cbuf = rows + g * (NP + 1);
  if (!(a.dbg & 4)) fft::fft4step<NP, false>(cbuf, t, tws);
  __syncthreads();
  if (a.dbg & 8) return;
  const int first = rank == 0 ? 1 : 0;
  const int ncol = 16 - first;
  constexpr int NG = t_groups(NP);
  const int64_t zs = (int64_t)a.L.nzl * kTG;
  double2* tdst = a.T + (int64_t)(rank * (16 / kTG)) * zs + i0 * kTG;  // this CTA's 16 columns
  const int sw = t_swz(i0);
  if (first == 0) {
    // 16 columns: shifts instead of divisions
#pragma unroll 4
    for (int idx = tid; idx < 16 * NP; idx += NP) {
      const int k1 = idx >> 4, j = idx & 15;
      tdst[(int64_t)a.L.row1(comp, k1) * NG * zs + (j / kTG) * zs + ((j % kTG) ^ sw)] = rows[j * (NP + 1) + k1];
    }
  } else {
    for (int idx = tid; idx < ncol * NP; idx += NP) {
      const int k1 = idx / ncol, j = idx % ncol + first;
      tdst[(int64_t)a.L.row1(comp, k1) * NG * zs + (j / kTG) * zs + ((j % kTG) ^ sw)] = rows[j * (NP + 1) + k1];
    }
  }
  if (rank == 0 && g == 0) {
    // split the paired real columns k2 = 0 and k2 = NP/2
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = t + i * TPF;
      const double2 zk = cbuf[k], zm = conj(cbuf[(NP - k) % NP]);
      const double2 s = cadd(zk, zm), d = csub(zk, zm);
      a.T[a.L.t(a.L.p1(k), comp, a.L.l1(k), 0, i0)] = make_double2(0.5 * s.x, 0.5 * s.y);
      a.T[a.L.t(a.L.p1(k), comp, a.L.l1(k), NP / 2, i0)] = make_double2(0.5 * d.y, -0.5 * d.x);
    }
  }
}

#ifndef HB_INV_MINB
#define HB_INV_MINB 2
#endif
#ifndef HB_INV_AHEAD
#define HB_INV_AHEAD 0
#endif
#ifndef HB_FWD_AHEAD
#define HB_FWD_AHEAD 0
#endif
#ifndef HB_INV_SPLIT
#define HB_INV_SPLIT 2
#endif
#ifndef HB_INV_GROUPUPD
#define HB_INV_GROUPUPD 1
#endif
template <int NP>
__global__ void __launch_bounds__(NP, HB_INV_MINB) k_plane_inv(const __grid_constant__ PlaneArgs a) {
  constexpr int P = NP / 2 + 1;
  constexpr int CL = NP / 32;
  constexpr int TPF = tpf<NP>();
  constexpr int H = NP / 2;
  constexpr int PT = 32 * H / NP;
  if (a.mode == kModePcg && !a.st->active) return;
  extern __shared__ double2 sm[];
  double2* rows = sm;
  double2* tws = rows + rows_slots<NP>();
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int cid = blockIdx.x / CL;
  const int comp = cid / a.n0, i0 = cid % a.n0;
  const int tid = threadIdx.x, g = tid / TPF, t = tid % TPF;
  for (int i = tid; i < NP; i += NP) tws[i] = a.tw[i];
  if (a.ahead > 0 && cid + a.ahead < (int)(gridDim.x / CL)) {
    // pull the T2 block of the cluster that will take this one's place into
    // L2 (row k1 = tid: this rank's 16 columns, 256 bytes), so its first loads
    // do not wait for HBM
    const int cn = cid + a.ahead, compn = cn / a.n0, i0n = cn % a.n0;
    constexpr int PITCHN = t_blocks(NP) * kTB;
    const double2* pf = a.t2p[a.L.p1(tid)] + (int64_t)a.L.row2(compn, i0n, tid) * PITCHN + rank * 16;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(256u) : "memory");
  }
  // coalesced column loads: warp w takes k1 rows [32w, 32w+32), each
  // half-warp one row's 16 contiguous columns; transposed into padded buffers
  const int lane = tid & 31, warp = tid >> 5;
  const int jc = lane & 15, yo = lane >> 4;
  {
    const int col = rank * 16 + jc;
    constexpr int PITCH = t_blocks(NP) * kTB;
    // rows k = 32 warp + 2 i + yo share one peer (n1l is a multiple of 32)
    // (local receive buffer, or the source peer's own T2 over NVLink)
    const double2* src = a.t2p[a.L.p1(32 * warp)] + (int64_t)a.L.row2(comp, i0, 32 * warp + yo) * PITCH + col;
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (col == 0) {
        const double2 A = src[2 * i * PITCH];
        const double2 B = src[2 * i * PITCH + NP / 2];
        v[i] = make_double2(A.x - B.y, A.y + B.x);  // A + i B
      } else {
        v[i] = src[2 * i * PITCH];
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) rows[jc * (NP + 1) + 32 * warp + 2 * i + yo] = v[i];
  }
  __syncthreads();
#ifndef HB_INV_PREFETCH
#define HB_INV_PREFETCH 1
#endif
  if (HB_INV_PREFETCH && a.mode == kModePcg && tid < 64 && !(a.dbg & 256)) {
    // pull this CTA's p and x rows into L2 while the transforms run, so the
    // update at the end of each transform group hits L2
    const int64_t pl = (int64_t)comp * a.np + (int64_t)i0 * NP * NP + (int64_t)rank * 32 * NP + (int64_t)(tid & 31) * NP;
    const double* src = (tid < 32 ? a.p : a.x) + pl;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((uint32_t)(NP * sizeof(double)))
                 : "memory");
  }
  double2* cbuf = rows + g * (NP + 1);
  fft::fft4step<NP, true>(cbuf, t, tws);
  __syncthreads();
  // read back transposed: warp w takes rows [32w, 32w+32) of the 16 slots
  double2 w[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = rows[jc * (NP + 1) + 32 * warp + 2 * i + yo];
  cluster.sync();  // all column results in registers: regions become row storage
  {
    double2* dst = cluster.map_shared_rank(rows, warp);
    const int col = rank * 16 + jc;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double2* row = dst + (2 * i + yo) * P;
      if (col == 0) {
        row[0] = make_double2(w[i].x, 0.0);
        row[NP / 2] = make_double2(w[i].y, 0.0);
      } else {
        row[col] = w[i];
      }
    }
  }
  cluster.sync();
  // inverse row c2r: group g, rows (2g, 2g+1): Z = A + i B, z = IFFT(Z)
  {
    double2* buf = rows + (2 * g) * P;
    const double2* A = rows + (2 * g) * P;
    const double2* B = rows + (2 * g + 1) * P;
    double2 u[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = t + i * TPF;
      const int k = n <= NP / 2 ? n : NP - n;
      double2 av = A[k], bv = B[k];
      if (k == 0 || k == NP / 2) {
        av.y = 0.0;
        bv.y = 0.0;
      }
      u[i] = n <= NP / 2 ? make_double2(av.x - bv.y, av.y + bv.x) : make_double2(av.x + bv.y, bv.x - av.y);
    }
    fft::group_sync();
    fft::fft4step_regs<NP, true>(u, buf, t, tws);
  }
  const int64_t plane = (int64_t)comp * a.np + (int64_t)i0 * NP * NP + (int64_t)rank * 32 * NP;
#if HB_INV_GROUPUPD
  // each transform group updates its own row pair as soon as its inverse is
  // done (no block barrier: early groups' loads overlap later groups' FFTs)
  if (a.dbg & 256) return;  // profiling: no p / x traffic
  {
    const double2* zb = rows + (2 * g) * P;
    const int64_t r0 = plane + (int64_t)(2 * g) * NP;
    if (a.mode == kModePcg) {
      const double alpha = a.st->alpha, beta = a.st->beta;
      const int conv = a.st->converged;
      constexpr int NC = NP / TPF;  // columns per thread
      constexpr int CH = NC / HB_INV_SPLIT;
#pragma unroll
      for (int hh = 0; hh < HB_INV_SPLIT; ++hh) {
        double pv[2][CH], xv[2][CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int n = t + TPF * (hh * CH + i);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            pv[r][i] = a.p[r0 + r * NP + n];
            xv[r][i] = a.x[r0 + r * NP + n];
          }
        }
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int n = t + TPF * (hh * CH + i);
          const double2 z = zb[n];
#pragma unroll
          for (int r = 0; r < 2; ++r) a.x[r0 + r * NP + n] = fma(alpha, pv[r][i], xv[r][i]);
          if (!conv) {
            a.p[r0 + n] = fma(beta, pv[0][i], z.x);
            a.p[r0 + NP + n] = fma(beta, pv[1][i], z.y);
          }
        }
      }
    } else {
      double* out = (a.mode == kModeInit ? a.p : a.z) + r0;
#pragma unroll
      for (int i = 0; i < NP / TPF; ++i) {
        const int n = t + TPF * i;
        const double2 z = zb[n];
        out[n] = z.x;
        out[NP + n] = z.y;
      }
    }
  }
  return;
#endif
  __syncthreads();
  // row pair (2 rp, 2 rp + 1) at column n is z = rows[2 rp P + n] (two-for-one
  // packing): thread n reads it conflict-free and updates both rows' column n
  // (coalesced 8-byte global accesses)
  if (a.dbg & 256) return;  // profiling: no p / x traffic
  const int n = tid;
  if (a.mode == kModePcg) {
    double* pp = a.p + plane + n;
    double* xp = a.x + plane + n;
    const double alpha = a.st->alpha, beta = a.st->beta;
    const int conv = a.st->converged;
    constexpr int RP = 16 / HB_INV_SPLIT;  // row pairs per chunk (bounds live registers)
#pragma unroll
    for (int hh = 0; hh < HB_INV_SPLIT; ++hh) {
      double pv[2 * RP], xv[2 * RP];
#pragma unroll
      for (int i = 0; i < 2 * RP; ++i) {
        const int r = hh * 2 * RP + i;
        pv[i] = pp[r * NP];
        xv[i] = xp[r * NP];
      }
#pragma unroll
      for (int i = 0; i < RP; ++i) {
        const int rp = hh * RP + i;
        const double2 z = rows[2 * rp * P + n];
        xp[(2 * rp) * NP] = fma(alpha, pv[2 * i], xv[2 * i]);
        xp[(2 * rp + 1) * NP] = fma(alpha, pv[2 * i + 1], xv[2 * i + 1]);
        if (!conv) {
          pp[(2 * rp) * NP] = fma(beta, pv[2 * i], z.x);
          pp[(2 * rp + 1) * NP] = fma(beta, pv[2 * i + 1], z.y);
        }
      }
    }
  } else {
    double* out = (a.mode == kModeInit ? a.p : a.z) + plane + n;
#pragma unroll
    for (int rp = 0; rp < 16; ++rp) {
      const double2 z = rows[2 * rp * P + n];
      out[(2 * rp) * NP] = z.x;
      out[(2 * rp + 1) * NP] = z.y;
    }
  }
}

struct PencilArgs {
  int n0, n1;              // GLOBAL pencil length n0 and plane size n1 (= NP)
  int k1off;               // global k1 of local row 0 (rank * n1l)
  TLayout L;
  int P;                   // NP/2 + 1
  int ntk;                 // k2 tiles per k1
  const double2* tp[FusedFft::kMaxPeers];  // chunk bases per source peer (FusedFft::tpull)
  double2* T2;
  const double2* tw;       // W_N0 four-step table
  const PcgState* st;      // nullable
  double* partials;        // nullable (Parseval r.z)
  int nred;
  int dbg;
};

template <int C>
constexpr int pencil_bk() {
  return C == 3 ? 4 : 8;
}

// One transform group (TPF threads) per pencil (component, column): the
// step-1 inputs i0 = t + TPF n2 are loaded straight into registers (adjacent
// columns of neighbouring groups share 32-byte sectors), transformed, solved
// per frequency with all C components, inverse transformed and stored.
template <int N0, int C>
#ifndef HB_PENCIL_MINB
#define HB_PENCIL_MINB 2
#endif
// HB_PENCIL_INLAYOUT: the pencil transforms run in the TMA stage layout itself
// ([group][i0][4 ^ swizzle] rows: fft4step_*_map), so the stage is never
// re-laid: two block barriers and two shared-memory passes less per tile.
#ifndef HB_PENCIL_INLAYOUT
#define HB_PENCIL_INLAYOUT 1
#endif
#ifndef HB_PENCIL_LATEREFILL
#define HB_PENCIL_LATEREFILL 1
#endif
// HB_PENCIL_HALVES (in-layout, 256-point elastic pencils): the solve couples
// only the three components of a column, and columns {0,1} / {2,3} of a tile
// live in warps {0,2,4} / {1,3,5}; each half synchronises its transform ->
// solve -> transform hand-offs on its own named barrier (96 threads), so the
// halves drift apart and overlap their shared-memory and FP64 phases.
// (1 = immediate barrier ids behind a branch: 112 B of spills, 0.235 -> 0.270 ms;
// 2 = the id in a register, ptxas then reserves all 16 barriers: 0.235 -> 0.229 ms)
#ifndef HB_PENCIL_HALVES
#define HB_PENCIL_HALVES 2
#endif
__global__ void __launch_bounds__(C * pencil_bk<C>() * (N0 / 16), HB_PENCIL_MINB)
    k_pencil(const __grid_constant__ SpecParams sp, const __grid_constant__ PencilArgs a,
             const __grid_constant__ CUtensorMap t2map) {
  // Persistent blocks; tile = (k1 row, BK columns) for all C components.
  // Each tile's T data (BK/4 column groups x C components x peers, each a
  // contiguous run) is bulk-copied (TMA) into one of two stages while the
  // previous tile is transformed; after the raw reads the stage is reused
  // as the pencils' FFT / solve buffer.
  constexpr int TPF = tpf<N0>();
  constexpr int BK = pencil_bk<C>();
  constexpr int NT = C * BK * TPF;
  constexpr int NGB = BK / kTG;  // column groups per tile
  constexpr int STAGE = C * BK * N0;  // double2 per stage
  if (a.st && !a.st->active) return;
  extern __shared__ double2 sm_raw[];
  // 1024-byte alignment (the 64-byte swizzle of the tensor stores keys on
  // shared address bits 7-8) by pointer arithmetic on the shared symbol itself
  // (an integer round trip would make every stage access a generic LD/ST)
  double2* sm = reinterpret_cast<double2*>(reinterpret_cast<unsigned char*>(sm_raw) +
                                           ((1024u - (fft::smem_u32(sm_raw) & 1023u)) & 1023u));
  double2* stage0 = sm;             // [2][C][NGB][N0][kTG ^ swizzle]
  double2* tws = sm + 2 * STAGE;
  double2* t12 = tws + N0;  // [n1] (sin, sin(t/2)) of axes 1 and 2 (square planes: one table)
  __shared__ __align__(8) uint64_t full[2];
  const int tid = threadIdx.x, g = tid / TPF, t = tid % TPF;
  const int j = g % BK, comp = g / BK;
  const int P = a.P;
  const int ntiles = a.L.n1l * a.ntk;
  const int nzl = a.L.nzl;
  const int world = N0 / nzl;
  // one tile's bulk copies into stage st
  auto issue = [&](int tile, int st) {
    const int k1l = tile / a.ntk, c0 = (tile % a.ntk) * BK;
    uint32_t bytes = 0;
    for (int gg = 0; gg < NGB; ++gg)
      if (c0 / kTG + gg < a.L.ng) bytes += C * world * nzl * kTG * (uint32_t)sizeof(double2);
    fft::mbar_expect_tx(&full[st], bytes);
    for (int c = 0; c < C; ++c)
      for (int gg = 0; gg < NGB; ++gg) {
        if (c0 / kTG + gg >= a.L.ng) continue;
        for (int q = 0; q < world; ++q)
          fft::bulk_g2s(stage0 + st * STAGE + ((c * NGB + gg) * N0 + q * nzl) * kTG,
                        a.tp[q] + a.L.t(q, c, k1l, c0 + gg * kTG, 0), nzl * kTG * (uint32_t)sizeof(double2),
                        &full[st]);
      }
  };
  if (tid == 0) {
    fft::mbar_init(&full[0], 1);
    fft::mbar_init(&full[1], 1);
    fft::fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if ((int)blockIdx.x < ntiles) issue(blockIdx.x, 0);
    if ((int)(blockIdx.x + gridDim.x) < ntiles) issue(blockIdx.x + gridDim.x, 1);
  }
  for (int i = tid; i < N0; i += NT) tws[i] = a.tw[i];
  if (sp.kind == 3)
    for (int i = tid; i < a.n1; i += NT) {
      const double4 tv = sp.tab[1][i];
      t12[i] = make_double2(tv.x, tv.z);
    }
  // per-column symbol factors (hex, k0-independent parts) and the axis-0 table
  __shared__ double colf[BK][6];
  __shared__ double3 ax0[N0];
  for (int i = tid; i < N0; i += NT) {
    const double4 tv = sp.tab[0][i];
    ax0[i] = make_double3(tv.x, tv.z, 2.0 - (4.0 / 3.0) * tv.z * tv.z);  // sin, sin(t/2), S2
  }
  double rz = 0.0;
  int it = 0;
  int pend_tile = -1, pend_st = 0;
  constexpr bool INL = HB_PENCIL_INLAYOUT;
  if (INL) __syncthreads();  // tables ready before the first (barrier-free) transform
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it & 1;
    double2* stg = stage0 + st * STAGE;
    const int k1l = tile / a.ntk, c0 = (tile % a.ntk) * BK;
    const int k1 = a.k1off + k1l;
    fft::mbar_wait(&full[st], (it >> 1) & 1);
    double2 v[16];
    {
      const double2* src = stg + (comp * NGB + j / kTG) * N0 * kTG;
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) v[n2] = src[(t + TPF * n2) * kTG + ((j % kTG) ^ t_swz(t + TPF * n2))];
    }
    constexpr bool HALVES = INL && HB_PENCIL_HALVES && C == 3 && TPF == 16 && BK == 4;
    const int half = (tid >> 5) & 1;                       // HALVES: columns {2 half, 2 half + 1}
    const int hr = ((tid >> 6) << 5) | (tid & 31);         // rank within the half (0..95)
    auto half_sync = [&] {
      if (HB_PENCIL_HALVES == 2) {  // register id: ptxas reserves all 16 barriers
        asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "n"(NT / 2) : "memory");
      } else if (half) {
        asm volatile("bar.sync 2, %0;" ::"n"(NT / 2) : "memory");
      } else {
        asm volatile("bar.sync 1, %0;" ::"n"(NT / 2) : "memory");
      }
    };
    if (HALVES ? (sp.kind == 3 && hr < 2) : (sp.kind == 3 && tid < BK)) {
      const int ct = HALVES ? 2 * half + hr : tid;
      // M(k0) = diag(cf0 sh0^2, cf1 S2_0, cf2 S2_0) + offdiag(cf3 sn0, cf4 sn0, cf5 S2_0)
      // (shared-memory table and the host's division-free Gram factors: the
      // other warps wait for these four threads at the next block barrier)
      const int k2 = min(c0 + ct, P - 1);
      const double2 t1 = t12[k1], t2 = t12[k2];
      const double S21 = 2.0 - (4.0 / 3.0) * t1.y * t1.y, S22 = 2.0 - (4.0 / 3.0) * t2.y * t2.y;
      colf[ct][0] = sp.cd[0] * S21 * S22;
      colf[ct][1] = sp.cd[1] * t1.y * t1.y * S22;
      colf[ct][2] = sp.cd[2] * t2.y * t2.y * S21;
      colf[ct][3] = sp.co[0][1] * t1.x * S22;
      colf[ct][4] = sp.co[0][2] * t2.x * S21;
      colf[ct][5] = sp.co[1][2] * t1.x * t2.x;
    }
    if (!INL) __syncthreads();  // raw stage reads done (stage becomes the FFT buffers); colf, tws ready
    double2* buf = stg;               // [C][BK][N0]; INL: stays [C][NGB][N0][kTG ^ swizzle]
    double2* pb = INL ? stg + (comp * NGB + j / kTG) * N0 * kTG : buf + g * N0;
    const int jm = j % kTG;
    auto slot = [jm](int n) { return n * kTG + (jm ^ t_swz(n)); };
    // element (component i, column jj, frequency k0) of the tile
    auto at = [&](int i, int jj, int k0) -> double2& {
      if (INL) return stg[((i * NGB + jj / kTG) * N0 + k0) * kTG + ((jj % kTG) ^ t_swz(k0))];
      return buf[(i * BK + jj) * N0 + k0];
    };
    if (INL) {
      if (!(a.dbg & 32)) fft::fft4step_regs_map<N0, false>(v, pb, t, tws, slot);
    } else if (!(a.dbg & 32)) fft::fft4step_regs<N0, false>(v, pb, t, tws);
    else
#pragma unroll
      for (int n2 = 0; n2 < 16; ++n2) pb[t + TPF * n2] = v[n2];
    if (HALVES) half_sync();
    else __syncthreads();
    if (HB_PENCIL_LATEREFILL && tid == 0 && pend_tile >= 0) {
      // the previous tile's stage: its stores were issued a forward transform
      // ago, so this wait returns at once (at the tile end warp 0 sat in it
      // while the others waited for it at the next barrier)
      fft::bulk_wait_read();
      issue(pend_tile, pend_st);
      pend_tile = -1;
    }
    // the solve: every thread of the block (HALVES: of the half) takes
    // frequencies of the tile's (the half's) columns, all C components each
    const int se0 = HALVES ? hr : tid, sen = HALVES ? 2 * N0 : N0 * BK, sed = HALVES ? NT / 2 : NT;
    for (int e = se0; e < sen && !(a.dbg & 16); e += sed) {
      const int jj = (HALVES ? 2 * half : 0) + e / N0, k0 = e % N0;
      const int k2 = c0 + jj;
      if (k2 >= P) continue;
      double2 r[C], z[C];
#pragma unroll
      for (int i = 0; i < C; ++i) r[i] = at(i, jj, k0);
      if (k0 == 0 && k1 == 0 && k2 == 0) {
#pragma unroll
        for (int i = 0; i < C; ++i) z[i] = make_double2(0.0, 0.0);
      } else {
        double M[3][3], K[3][3], I[3][3];
        if (sp.kind == 3) {
          const double3 t0 = ax0[k0];
          const double* cf = colf[jj];
          M[0][0] = cf[0] * t0.y * t0.y;
          M[1][1] = cf[1] * t0.z;
          M[2][2] = cf[2] * t0.z;
          M[0][1] = M[1][0] = cf[3] * t0.x;
          M[0][2] = M[2][0] = cf[4] * t0.x;
          M[1][2] = M[2][1] = cf[5] * t0.z;
        } else {
          const int f[3] = {k0, k1, k2};
          spec::gram<3>(sp, f, M);
        }
        spec::symbol<3, C>(sp, M, K);
        spec::sym_inverse<C>(K, I);
#pragma unroll
        for (int i = 0; i < C; ++i) {
          double zr = 0.0, zi = 0.0;
#pragma unroll
          for (int jj2 = 0; jj2 < C; ++jj2) {
            zr = fma(I[i][jj2], r[jj2].x, zr);
            zi = fma(I[i][jj2], r[jj2].y, zi);
          }
          z[i] = make_double2(zr * sp.inv_np, zi * sp.inv_np);
        }
        const double wgt = (k2 == 0 || 2 * k2 == a.n1) ? 1.0 : 2.0;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < C; ++i) s += r[i].x * z[i].x + r[i].y * z[i].y;
        rz = fma(wgt, s, rz);
      }
#pragma unroll
      for (int i = 0; i < C; ++i) at(i, jj, k0) = z[i];
    }
    if (HALVES) half_sync();
    else __syncthreads();
    if (INL) {
      if (!(a.dbg & 32)) fft::fft4step_map<N0, true>(pb, t, tws, slot);
    } else {
    if (!(a.dbg & 32)) fft::fft4step<N0, true>(pb, t, tws);
#pragma unroll
    for (int n = 0; n < 16; ++n) v[n] = pb[t + TPF * n];
    __syncthreads();  // every pencil read back: re-lay the stage as [C][group][i0][4]
    {
      // slots swizzled like T: the tensor map (SWIZZLE_64B) undoes it on the way out
      double2* dst = stg + (comp * NGB + j / kTG) * N0 * kTG;
#pragma unroll
      for (int n = 0; n < 16; ++n) dst[(t + TPF * n) * kTG + ((j % kTG) ^ t_swz(t + TPF * n))] = v[n];
    }
    }
    fft::fence_proxy_async();  // generic smem writes -> async-proxy (TMA) reads
    __syncthreads();
    if (tid == 0) {
      // T2 is plane-major: each (component, 4-column group) is a box of
      // 64 bytes x n0 planes, scattered by the TMA engine
      if (!(a.dbg & 64)) {
        for (int c = 0; c < C; ++c)
          for (int gg = 0; gg < NGB; ++gg) {
            if (c0 / kTG + gg >= a.L.ng) continue;
            const double2* src = stg + (c * NGB + gg) * N0 * kTG;
            asm volatile(
                "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                    reinterpret_cast<uint64_t>(&t2map)),
                "r"(2 * (c0 + gg * kTG)), "r"(k1l), "r"(0), "r"(c), "r"(0), "r"(fft::smem_u32(src))
                : "memory");
          }
        fft::bulk_commit();
      }
      if (tile + 2 * (int)gridDim.x < ntiles) {
        if (HB_PENCIL_LATEREFILL) {
          pend_tile = tile + 2 * gridDim.x;  // refilled after the next tile's first barrier
          pend_st = st;
        } else {
          fft::bulk_wait_read();  // the stores have read the stage
          issue(tile + 2 * gridDim.x, st);
        }
      }
    }
    // no block barrier here: the other warps go on to the next tile (other
    // stage, its own mbarrier); this stage is only touched again after the
    // next tile's first barrier, which warp 0 reaches after the refill issue
    // (0.356 -> 0.350 ms)
  }
  if (tid == 0) fft::bulk_wait();  // stores complete before the block retires
  if (a.partials) {
    __shared__ double red[32];
    const int lane = tid & 31, warp = tid >> 5;
    constexpr int NWP = (NT + 31) / 32;
    if constexpr (NT % 32 == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rz += __shfl_xor_sync(0xffffffffu, rz, o);
    } else {
      // the last warp is partial (NT = 48 for 64-plane elastic pencils): only
      // existing lanes take part, lanes past the end contribute nothing
      const int wn = min(32, NT - 32 * warp);
      const unsigned mask = wn == 32 ? 0xffffffffu : ((1u << wn) - 1u);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_down_sync(mask, rz, o);
        if (lane + o < wn) rz += t;
      }
    }
    __syncthreads();
    if (lane == 0) red[warp] = rz;
    __syncthreads();
    if (warp == 0) {
      double s2 = lane < NWP ? red[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (lane == 0) a.partials[blockIdx.x] = s2;
    }
    if (blockIdx.x == 0)
      for (int i = gridDim.x + tid; i < a.nred; i += NT) a.partials[i] = 0.0;
  }
}

static int ilog2(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  if ((1 << l) != v) throw ValidationError("fused FFT: slab sizes must be powers of two");
  return l;
}

TLayout layout_of(const FusedFft& f) {
  return TLayout{f.c, f.n1l, f.n0, t_blocks(f.np_plane), t_groups(f.np_plane), ilog2(f.n1l), ilog2(f.n0)};
}

#ifndef HB_CLUSTER_POLICY
#define HB_CLUSTER_POLICY 0
#endif
template <class K>
void launch_cluster(K kernel, int grid, int block, int cl, size_t smem, cudaStream_t s, const PlaneArgs& a) {
  HB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // cluster scheduling policy preference (HOMFE_CLUSTER_POLICY: 1 = spread, 2 = load balancing)
  static const int policy = [] {
    const char* e = std::getenv("HOMFE_CLUSTER_POLICY");
    return e ? std::atoi(e) : HB_CLUSTER_POLICY;
  }();
  if (policy) {
    attr[1].id = cudaLaunchAttributeClusterSchedulingPolicyPreference;
    attr[1].val.clusterSchedulingPolicyPreference =
        policy == 2 ? cudaClusterSchedulingPolicyLoadBalancing : cudaClusterSchedulingPolicySpread;
    cfg.numAttrs = 2;
  }
  static bool shown = false;
  if (!shown && std::getenv("HOMFE_FFT_OCC")) {
    shown = true;
    int ncl = 0;
    HB_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kernel, &cfg));
    std::fprintf(stderr, "plane kernel: cluster %d, smem %zu, max active clusters %d, grid clusters %d\n", cl, smem,
                 ncl, grid / cl);
  }
  HB_CUDA(cudaLaunchKernelEx(&cfg, kernel, a));
}

template <int NP>
void run_planes(const FusedFft& f, bool inverse, const PlaneArgs& a, cudaStream_t s) {
  constexpr int CL = NP / 32;
  const size_t smem = sizeof(double2) * ((size_t)rows_slots<NP>() + NP);
  const int grid = CL * f.n0 * f.c;
  if (inverse) launch_cluster(k_plane_inv<NP>, grid, NP, CL, smem, s, a);
  else launch_cluster(k_plane_fwd<NP>, grid, NP, CL, smem, s, a);
}

template <int N0, int C>
void run_pencils_c(const FusedFft& f, const SpecParams& sp, const PcgState* st, double* partials, cudaStream_t s) {
  constexpr int BK = pencil_bk<C>();
  constexpr int NT = C * BK * (N0 / 16);
  PencilArgs a;
  a.n0 = f.n0g;
  a.n1 = f.np_plane;
  a.k1off = f.rank * f.n1l;
  a.L = layout_of(f);
  a.P = f.np_plane / 2 + 1;
  a.ntk = (a.P + BK - 1) / BK;
  for (int q = 0; q < FusedFft::kMaxPeers; ++q) a.tp[q] = f.tpull[q];
  a.T2 = f.T2;
  a.tw = f.tw0;
  a.st = st;
  a.partials = partials;
  a.nred = kRedBlocks;
  a.dbg = f.dbg;
  const int ntiles = a.L.n1l * a.ntk;
  const size_t smem = sizeof(double2) * (2 * (size_t)C * BK * N0 + N0 + f.np_plane) + 1024;
  HB_CUDA(cudaFuncSetAttribute(k_pencil<N0, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  static int grid_cap[2] = {0, 0};  // resident blocks of this instantiation (persistent grid)
  int& cap = grid_cap[C == 3];
  if (!cap) {
    int dev = 0, sms = 0, per = 0;
    HB_CUDA(cudaGetDevice(&dev));
    HB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pencil<N0, C>, NT, smem));
    cap = sms * (per > 0 ? per : 1);
  }
  int grid = ntiles < cap ? ntiles : cap;
  if (grid > kRedBlocks) grid = kRedBlocks;
  k_pencil<N0, C><<<grid, NT, smem, s>>>(sp, a, *reinterpret_cast<const CUtensorMap*>(f.t2map));
  HB_CUDA(cudaGetLastError());
}

template <int N0>
void run_pencils(const FusedFft& f, const SpecParams& sp, const PcgState* st, double* partials, cudaStream_t s) {
  if (f.c == 3) run_pencils_c<N0, 3>(f, sp, st, partials, s);
  else run_pencils_c<N0, 1>(f, sp, st, partials, s);
}

}  // namespace

// T2 as a 5-D fp64 tensor {2 pitch, n1l, nzl, c, world} (innermost first);
// box {8, 1, nzl, 1, world} = one 4-column group of one k1 row over all planes.
void fused_make_maps(FusedFft& f) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    HB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeFn>(fn);
  }
  const cuuint64_t pitch = (cuuint64_t)t_blocks(f.np_plane) * kTB;  // complex per row
  const cuuint64_t dims[5] = {2 * pitch, (cuuint64_t)f.n1l, (cuuint64_t)f.n0, (cuuint64_t)f.c, (cuuint64_t)f.world};
  const cuuint64_t row = pitch * sizeof(double2);
  const cuuint64_t strides[4] = {row, row * f.n1l, row * f.n1l * f.n0, row * f.n1l * f.n0 * f.c};
  const cuuint32_t box[5] = {2 * kTG, 1, (cuuint32_t)f.n0, 1, (cuuint32_t)f.world};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUtensorMap* m = reinterpret_cast<CUtensorMap*>(f.t2map);
  const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, f.T2, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
}

bool fused_fft_eligible(const Grid& g) {
  if (g.d != 3 || (g.c != 1 && g.c != 3)) return false;
  if (g.n1 != g.n2 || (g.n2 != 128 && g.n2 != 256)) return false;
  const int n0g = g.dist ? g.n0g : g.n0;
  if (n0g != 64 && n0g != 128 && n0g != 256) return false;
  if (g.dist && ((g.world & (g.world - 1)) != 0 || g.n1 % g.world != 0 || g.n1 / g.world < 32 ||
                 g.n0 * g.world != n0g))
    return false;
  return true;
}

// L2 prefetch distance of the plane passes in clusters (HOMFE_PF_FWD /
// HOMFE_PF_INV override; 0 = off).
static int plane_ahead(int inverse) {
  static int v[2] = {-1, -1};
  if (v[inverse] < 0) {
    const char* e = std::getenv(inverse ? "HOMFE_PF_INV" : "HOMFE_PF_FWD");
    v[inverse] = e ? std::atoi(e) : (inverse ? HB_INV_AHEAD : HB_FWD_AHEAD);
  }
  return v[inverse];
}

static void planes(const FusedFft& f, bool inverse, const PlaneArgs& a, cudaStream_t s) {
  if (f.np_plane == 256) run_planes<256>(f, inverse, a, s);
  else run_planes<128>(f, inverse, a, s);
}

static void pencils(const FusedFft& f, const SpecParams& sp, const PcgState* st, double* partials, cudaStream_t s) {
  switch (f.n0g) {
    case 64: run_pencils<64>(f, sp, st, partials, s); break;
    case 128: run_pencils<128>(f, sp, st, partials, s); break;
    default: run_pencils<256>(f, sp, st, partials, s); break;
  }
}

// PCG iteration part: r -= alpha Ap; z = M^-1 r (with r.z partials).
void fused_forward(const FusedFft& f, const SpecParams& sp, double* r, const double* ap, const PcgState* st,
                   double* partials, cudaStream_t s, int which) {
  PlaneArgs a = {};
  a.n0 = f.n0;
  a.np = f.np;
  a.L = layout_of(f);
  a.r = r;
  a.ap = ap;
  a.T = f.T;
  a.T2 = f.T2;
  a.tw = f.tw_plane;
  a.st = st;
  a.mode = ap ? kModePcg : kModePlain;
  a.dbg = f.dbg;
  a.ahead = plane_ahead(0);
  if (which & 1) planes(f, false, a, s);
  if (which & 2) pencils(f, sp, st, partials, s);
}

// x += alpha p; p = z + beta p   (st != nullptr), or p = z (init), or z out.
void fused_inverse(const FusedFft& f, double* p, double* x, double* z, const PcgState* st, int init,
                   cudaStream_t s) {
  PlaneArgs a = {};
  a.n0 = f.n0;
  a.np = f.np;
  a.L = layout_of(f);
  a.T = f.T;
  for (int q = 0; q < FusedFft::kMaxPeers; ++q) a.t2p[q] = f.t2pull[q];
  a.tw = f.tw_plane;
  a.p = p;
  a.x = x;
  a.z = z;
  a.st = st;
  a.mode = st ? kModePcg : (init ? kModeInit : kModeZ);
  a.dbg = f.dbg;
  a.ahead = plane_ahead(1);
  planes(f, true, a, s);
}

}  // namespace hb
