// hexfast.cu -- element-centric, flop-lean K u for trilinear hexahedra
// (2x2x2 Gauss) on cubic voxels.
//
// The reference evaluates K u = D^T W C D u per quadrature point
// (proj/src/operators.cpp:197-243): ~3.6 kflop per voxel for elasticity,
// which would make this kernel FP64-bound at ~10x the HBM time on a B200.
// Here each element is evaluated once, in a separable "modal" basis:
//
//  * per axis the two nodal values become (S, D) = (u0 + u1, u1 - u0); the
//    two Gauss points are symmetric about the element centre, so values at
//    the Gauss points are S/2 -+ g D (g = 1/(2 sqrt 3)) and derivatives D/h;
//  * the 8 quadrature points are recombined into 8 symmetric/antisymmetric
//    "quad modes" (Hadamard basis, orthogonal), in which every gradient
//    component is a single scaled modal coefficient and the mode (a,a,a)
//    vanishes; sum_q w e_q^T C e_q = 8 w sum_modes e_m^T C e_m;
//  * per mode only 6 / 5 / 3 strain rows are non-zero (modes with 0 / 1 / 2
//    antisymmetric axes), so the material contraction costs 36+3*25+3*9 FMA
//    for a general anisotropic C and ~40 flops for an isotropic one.
//
// The result is algebraically identical to the reference operator (same
// bilinear form); only the rounding differs. ~200 (isotropic) / ~300
// (anisotropic) DP ops per element instead of ~3600.
//
// Work layout: one block per (y-range, z-range) tile covering complete
// x-rows (blockDim.x = N2, lanes along the contiguous axis => coalesced).
// A thread marches its x column through TY rows (inner, y) and TZ planes
// (outer, z). Each element's 8 corner residuals are reduced without atomics:
// x-neighbours by warp shuffle (+ one smem hop between warps, which also
// closes the periodic wrap), y-neighbours by a register carry, z-neighbours
// by a per-thread shared-memory row buffer. The first row and plane of a
// tile are recomputed (warm-up) so that tiles are independent. Every output
// node is the same fixed-order sum => bitwise reproducible.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fft.cuh"
#include "kernels.cuh"

namespace hb {

namespace {


// Per-phase material table layout (doubles):
//   ISO:      [3 classes][3] = f*lambda, f*2mu, f*mu, then f_2*(lambda + 4mu)   (elastic)
//             [3 classes][1] = f*kappa                 (scalar)
//   general:  [3 classes][M*M] = f * (S C S)  (S = diag(1,1,1,s2,s2,s2))
template <int C, bool ISO>
constexpr int mat_stride() {
  return ISO ? (C == 3 ? 10 : 3) : (C == 3 ? 3 * 36 : 3 * 9);
}

// Forward separable (S, D) transform of 8 corner values x[a*4+b*2+c].
__device__ __forceinline__ void modal_fwd(const double (&x)[8], double (&v)[8]) {
  double t[8];
#pragma unroll
  for (int ab = 0; ab < 4; ++ab) {  // axis 2 (c)
    t[ab * 2 + 0] = x[ab * 2 + 0] + x[ab * 2 + 1];
    t[ab * 2 + 1] = x[ab * 2 + 1] - x[ab * 2 + 0];
  }
  double s[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)  // axis 1 (b)
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      s[a * 4 + 0 * 2 + g] = t[a * 4 + 0 * 2 + g] + t[a * 4 + 1 * 2 + g];
      s[a * 4 + 1 * 2 + g] = t[a * 4 + 1 * 2 + g] - t[a * 4 + 0 * 2 + g];
    }
#pragma unroll
  for (int bg = 0; bg < 4; ++bg) {  // axis 0 (a)
    v[0 * 4 + bg] = s[0 * 4 + bg] + s[1 * 4 + bg];
    v[1 * 4 + bg] = s[1 * 4 + bg] - s[0 * 4 + bg];
  }
}

// Adjoint of modal_fwd.
__device__ __forceinline__ void modal_adj(const double (&v)[8], double (&x)[8]) {
  double s[8];
#pragma unroll
  for (int bg = 0; bg < 4; ++bg) {
    s[0 * 4 + bg] = v[0 * 4 + bg] - v[1 * 4 + bg];
    s[1 * 4 + bg] = v[0 * 4 + bg] + v[1 * 4 + bg];
  }
  double t[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      t[a * 4 + 0 * 2 + g] = s[a * 4 + 0 * 2 + g] - s[a * 4 + 1 * 2 + g];
      t[a * 4 + 1 * 2 + g] = s[a * 4 + 0 * 2 + g] + s[a * 4 + 1 * 2 + g];
    }
#pragma unroll
  for (int ab = 0; ab < 4; ++ab) {
    x[ab * 2 + 0] = t[ab * 2 + 0] - t[ab * 2 + 1];
    x[ab * 2 + 1] = t[ab * 2 + 0] + t[ab * 2 + 1];
  }
}

// Element residual r = K_e u (corner-major, [corner][k]); the per-mode code
// is generated straight-line (gen_hex_modes.py -> hex_modes.inc).
#include "hex_modes.inc"

template <int C, bool ISO>
__device__ __forceinline__ void hex_element(const double (&u)[8][C], const double* __restrict__ mat,
                                            double (&r)[8][C]) {
  double V[C][8];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = u[i][k];
    modal_fwd(x, V[k]);
  }
  double R[C][8];
#pragma unroll
  for (int k = 0; k < C; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) R[k][i] = 0.0;
#define HB_ACC(k, v, t) R[k][v] += (t)
  if constexpr (C == 3) {
    if constexpr (ISO) {
      HB_HEX_MODES_ELASTIC_ISO
    } else {
      HB_HEX_MODES_ELASTIC_GEN
    }
  } else {
    if constexpr (ISO) {
      HB_HEX_MODES_SCALAR_ISO
    } else {
      HB_HEX_MODES_SCALAR_GEN
    }
  }
#undef HB_ACC
#pragma unroll
  for (int k = 0; k < C; ++k) {
    double x[8];
    modal_adj(R[k], x);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i][k] = x[i];
  }
}

struct HexArgs {
  const double* u;
  const double* halo_lo, *halo_hi;  // dist mode: neighbour planes [c][plane]
  const uint8_t* ph_lo;             // dist mode: phase plane z0-1
  int64_t halo_cs;                  // dist mode: component stride of the halo planes
  int dist;
  double* out;
  const uint8_t* phase;
  const double* mat;     // n_phases * mat_stride
  const double* fe;      // nullable: n_phases x 8C element loads (corner-major)
  int n_phases;
  double scale;
  double* partials;      // nullable
  int nred;              // number of partial slots to fill (kRedBlocks)
  const PcgState* st;
  int n0, n1, n2;
  int tiles_y, tiles_z;
  // per-Gauss-point tangents (J2 path): compact (a, b, n[6]) per point,
  // mat = per phase (linear flag, bulk, shear); qs / qw mode scales
  const double* tanc;
  double qs[6], qw[6];
};

template <int C, bool ISO, int kTY, int kTZ>
__global__ void __launch_bounds__(256, 2) k_hex_fast(const HexArgs a) {
  if (a.st && a.st->done) return;
  constexpr int MS = mat_stride<C, ISO>();
  extern __shared__ double smem[];
  const int nx = blockDim.x;           // == n2
  const int nw = nx >> 5;
  double* zbuf = smem;                                  // [kTY][C][nx]
  double* xbuf = zbuf + kTY * C * nx;                   // [2][nw][4*C]
  double* mat_s = xbuf + 2 * nw * 4 * C;                // [n_phases][MS]
  double* fe_s = mat_s + a.n_phases * MS;               // [n_phases][8C]
  for (int i = threadIdx.x; i < a.n_phases * MS; i += nx) mat_s[i] = a.mat[i];
  if (a.fe)
    for (int i = threadIdx.x; i < a.n_phases * 8 * C; i += nx) fe_s[i] = a.fe[i];
  __syncthreads();

  const int x = threadIdx.x;
  const int lane = x & 31, warp = x >> 5;
  const int xp = x + 1 == nx ? 0 : x + 1;
  const int64_t plane = (int64_t)a.n1 * nx;
  const int64_t np = plane * a.n0;
  double dotacc = 0.0;
  int step = 0;
  const int ntiles = a.tiles_y * a.tiles_z;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int y0 = (tile % a.tiles_y) * kTY;
    const int z0 = (tile / a.tiles_y) * kTZ;
    for (int zi = -1; zi < kTZ; ++zi) {
      int z = z0 + zi;
      int z1 = z + 1;
      // plane pointers + component strides: periodic wrap on one device,
      // halo planes at the slab ends in dist mode
      const double* up[2];
      int64_t cs[2];
      if (a.dist) {
        up[0] = z < 0 ? a.halo_lo : a.u + (int64_t)z * plane;
        cs[0] = z < 0 ? a.halo_cs : np;
        up[1] = z1 >= a.n0 ? a.halo_hi : a.u + (int64_t)z1 * plane;
        cs[1] = z1 >= a.n0 ? a.halo_cs : np;
      } else {
        z = z < 0 ? z + a.n0 : z;
        z1 = z + 1 == a.n0 ? 0 : z + 1;
        up[0] = a.u + (int64_t)z * plane;
        up[1] = a.u + (int64_t)z1 * plane;
        cs[0] = cs[1] = np;
      }
      const uint8_t* phz = (a.dist && z < 0) ? a.ph_lo : a.phase + (int64_t)z * plane;
      // row y0 - 1 at planes z, z+1: uc[a][c][k]
      double uc[2][2][C];
      {
        const int y = y0 == 0 ? a.n1 - 1 : y0 - 1;
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int k = 0; k < C; ++k) {
            uc[aa][0][k] = __ldg(up[aa] + k * cs[aa] + (int64_t)y * nx + x);
            uc[aa][1][k] = __ldg(up[aa] + k * cs[aa] + (int64_t)y * nx + xp);
          }
      }
      double ycarry[2][C];
#pragma unroll
      for (int aa = 0; aa < 2; ++aa)
#pragma unroll
        for (int k = 0; k < C; ++k) ycarry[aa][k] = 0.0;
#pragma unroll 1
      for (int yi = -1; yi < kTY; ++yi) {
        int y = y0 + yi;
        y = y < 0 ? y + a.n1 : y;
        const int y1 = y + 1 == a.n1 ? 0 : y + 1;
        double un[2][2][C];
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int k = 0; k < C; ++k) {
            un[aa][0][k] = __ldg(up[aa] + k * cs[aa] + (int64_t)y1 * nx + x);
            un[aa][1][k] = __ldg(up[aa] + k * cs[aa] + (int64_t)y1 * nx + xp);
          }
        // corners: loc = (aa*2 + b)*2 + c
        double ue[8][C];
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int k = 0; k < C; ++k) {
              ue[(aa * 2 + 0) * 2 + c][k] = uc[aa][c][k];
              ue[(aa * 2 + 1) * 2 + c][k] = un[aa][c][k];
            }
        const int ph = phz[(int64_t)y * nx + x];
        double r[8][C];
        hex_element<C, ISO>(ue, mat_s + ph * MS, r);
        if (a.fe) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int k = 0; k < C; ++k) r[i][k] += fe_s[ph * 8 * C + i * C + k];
        }
        // x exchange: c = 1 corners go to lane + 1
        double* xb = xbuf + (step & 1) * nw * 4 * C;
        if (lane == 31) {
#pragma unroll
          for (int ab = 0; ab < 4; ++ab)
#pragma unroll
            for (int k = 0; k < C; ++k) xb[warp * 4 * C + ab * C + k] = r[ab * 2 + 1][k];
        }
        __syncthreads();
        double R[4][C];  // [aa*2+b][k] at node column x
        const int src = warp == 0 ? nw - 1 : warp - 1;
#pragma unroll
        for (int ab = 0; ab < 4; ++ab)
#pragma unroll
          for (int k = 0; k < C; ++k) {
            double recv = __shfl_up_sync(0xffffffffu, r[ab * 2 + 1][k], 1);
            if (lane == 0) recv = xb[src * 4 * C + ab * C + k];
            R[ab][k] = r[ab * 2 + 0][k] + recv;
          }
        ++step;
        if (yi >= 0) {
          double* zb = zbuf + (yi * C) * nx + x;
#pragma unroll
          for (int k = 0; k < C; ++k) {
            const double v0 = R[0][k] + ycarry[0][k];  // plane z, row y
            if (zi >= 0) {
              const double val = a.scale * (v0 + zb[k * nx]);
              const int64_t o = k * np + (int64_t)z * plane + (int64_t)y * nx + x;
              a.out[o] = val;
              dotacc = fma(uc[0][0][k], val, dotacc);
            }
            zb[k * nx] = R[2][k] + ycarry[1][k];  // plane z+1, row y
          }
        }
#pragma unroll
        for (int k = 0; k < C; ++k) {
          ycarry[0][k] = R[1][k];
          ycarry[1][k] = R[3][k];
        }
#pragma unroll
        for (int aa = 0; aa < 2; ++aa)
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int k = 0; k < C; ++k) uc[aa][c][k] = un[aa][c][k];
      }
    }
  }
  if (a.partials) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dotacc += __shfl_xor_sync(0xffffffffu, dotacc, o);
    if (lane == 0) red[warp] = dotacc;
    __syncthreads();
    if (warp == 0) {
      double s = lane < nw ? red[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) a.partials[blockIdx.x] = s;
    }
    if (blockIdx.x == 0)
      for (int i = gridDim.x + threadIdx.x; i < a.nred; i += nx) a.partials[i] = 0.0;
  }
}


// ===========================================================================
// v2: z-march with TMA-staged rows and shared per-axis transforms.
//
// Each block owns a contiguous run of "element rows" r = zb * n1 + y (zb = a
// block of KZ element planes) and marches z inside a row:
//  * unit j of a row = plane pz = zb*KZ - 1 + j, node rows y and y+1, all
//    components (+ the element phase row), bulk-copied by one thread into a
//    D-deep shared-memory ring (cp.async.bulk + mbarrier);
//  * forward: the x- and y-stages of the (S, D) transform are done once per
//    plane and carried in registers to the next element (Lo), so an element
//    costs 16 instead of 24 adds per component;
//  * adjoint: z-stage with a register carry of the upper face (zc), then the
//    x-stage (warp shuffle + one shared-memory hop between warps), then the
//    y-stage; node row y+1's partial waits in a per-thread shared-memory
//    buffer (ybuf, KZ x C) for the next element row.
// The first row of a run and the first element plane of a row are warm-up
// (recomputed, not stored), so runs are independent and every node is the
// same fixed-order sum (bitwise reproducible). Runs are balanced over exactly
// (resident blocks) CTAs.
// ===========================================================================
constexpr int kZDepth = 3;
#ifndef HB_HEXZ_JUNROLL
#define HB_HEXZ_JUNROLL 2
#endif
constexpr int kJUnroll = HB_HEXZ_JUNROLL;  // z-steps per loop body (isotropic variants)
// HB_HEXZ_RFOLD: isotropic catalogs accumulate the modal residual before the
// z-adjoint (fewer DP operations per element than folding every
// contribution into both faces)
#ifndef HB_HEXZ_ISSUE
#define HB_HEXZ_ISSUE 2
#endif
#ifndef HB_HEXZ_RFOLD
#define HB_HEXZ_RFOLD 1
#endif
#ifndef HB_HEXZ_MINB3
#define HB_HEXZ_MINB3 2
#endif
#ifndef HB_HEXZ_KZ3
#define HB_HEXZ_KZ3 8
#endif
// z-block depth of 512-wide rows (one 512-thread block per SM; KZ = 8 at
// c = 3 needs ~221 KB of shared memory)
#ifndef HB_HEXZ_KZ512
#define HB_HEXZ_KZ512 8
#endif
// scalar z-block depth: 16, or 8 on small grids (fewer than ~8 element rows
// per resident block at 16: warm-up rows dominate); HB_HEXZ_KZ1 forces one
#ifndef HB_HEXZ_KZ1
#define HB_HEXZ_KZ1 0
#endif

template <int C>
__host__ __device__ constexpr int zslot_bytes(int nx) {
  return 2 * C * nx * 8 + nx;
}

template <int V>
__device__ __forceinline__ void acc_fold(double (&A)[4], double (&B)[4], double t) {
  if constexpr (V < 4) {
    A[V] += t;
    B[V] += t;
  } else {
    A[V - 4] -= t;
    B[V - 4] += t;
  }
}

struct ZRun {
  int rows_total;  // n1 * (n0 / KZ)
  int grid;
  int list_cap;
};

template <int C, int KZ>
__device__ __forceinline__ void z_issue(const HexArgs& a, const int* its, int u, unsigned char* slot,
                                        uint64_t* bar) {
  const int nx = a.n2;
  const int i = u / (KZ + 2), j = u - i * (KZ + 2);
  const int info = its[i];
  const int y = info & 0xffff, zb = (info >> 16) & 0x7fff;
  const int y1 = y + 1 == a.n1 ? 0 : y + 1;
  const int64_t plane = (int64_t)a.n1 * nx;
  const int64_t np = plane * a.n0;
  int pz = zb * KZ - 1 + j;
  const double* src;
  int64_t cs;
  if (a.dist) {
    src = pz < 0 ? a.halo_lo : (pz >= a.n0 ? a.halo_hi : a.u + (int64_t)pz * plane);
    cs = (pz < 0 || pz >= a.n0) ? a.halo_cs : np;  // exchanged planes or a peer's field
  } else {
    pz = pz < 0 ? pz + a.n0 : (pz >= a.n0 ? pz - a.n0 : pz);
    src = a.u + (int64_t)pz * plane;
    cs = np;
  }
  const uint32_t row_bytes = nx * 8;
  fft::mbar_expect_tx(bar, 2 * C * row_bytes + (j ? nx : 0));
  double* dst = reinterpret_cast<double*>(slot);
#pragma unroll
  for (int k = 0; k < C; ++k) {
    fft::bulk_g2s(dst + (0 * C + k) * nx, src + k * cs + (int64_t)y * nx, row_bytes, bar);
    fft::bulk_g2s(dst + (1 * C + k) * nx, src + k * cs + (int64_t)y1 * nx, row_bytes, bar);
  }
  if (j) {
    int zp = zb * KZ - 2 + j;  // element plane
    const uint8_t* ph;
    if (a.dist && zp < 0) ph = a.ph_lo;
    else {
      zp = zp < 0 ? zp + a.n0 : zp;
      ph = a.phase + (int64_t)zp * plane;
    }
    fft::bulk_g2s(slot + 2 * C * row_bytes, ph + (int64_t)y * nx, nx, bar);
  }
}

// One piece of unit u's copies: part 2k + r = row y + r of component k
// (r = 0, 1), part 2C = the element phase row; part 0 also registers the
// unit's byte count (arrive.expect_tx; the tx-count may go transiently
// negative when another part's copy lands first). Spreading the parts over
// the warps keeps any one warp from arriving late at the next barrier.
template <int C, int KZ>
__device__ __forceinline__ void z_issue_part(const HexArgs& a, const int* its, int u, unsigned char* slot,
                                             uint64_t* bar, int part) {
  const int nx = a.n2;
  const int i = u / (KZ + 2), j = u - i * (KZ + 2);
  const int info = its[i];
  const int y = info & 0xffff, zb = (info >> 16) & 0x7fff;
  const uint32_t row_bytes = nx * 8;
  if (part == 0) fft::mbar_expect_tx(bar, 2 * C * row_bytes + (j ? nx : 0));
  const int64_t plane = (int64_t)a.n1 * nx;
  if (part < 2 * C) {
    const int k = part >> 1, r = part & 1;
    const int yr = r ? (y + 1 == a.n1 ? 0 : y + 1) : y;
    int pz = zb * KZ - 1 + j;
    const double* src;
    int64_t cs;
    if (a.dist) {
      src = pz < 0 ? a.halo_lo : (pz >= a.n0 ? a.halo_hi : a.u + (int64_t)pz * plane);
      cs = (pz < 0 || pz >= a.n0) ? a.halo_cs : plane * a.n0;
    } else {
      pz = pz < 0 ? pz + a.n0 : (pz >= a.n0 ? pz - a.n0 : pz);
      src = a.u + (int64_t)pz * plane;
      cs = plane * a.n0;
    }
    fft::bulk_g2s(reinterpret_cast<double*>(slot) + (r * C + k) * nx, src + k * cs + (int64_t)yr * nx, row_bytes,
                  bar);
  } else if (j) {
    int zp = zb * KZ - 2 + j;  // element plane
    const uint8_t* ph;
    if (a.dist && zp < 0) ph = a.ph_lo;
    else {
      zp = zp < 0 ? zp + a.n0 : zp;
      ph = a.phase + (int64_t)zp * plane;
    }
    fft::bulk_g2s(slot + 2 * C * row_bytes, ph + (int64_t)y * nx, nx, bar);
  }
}

// The same for unit (i, j) given directly (no division of u) and a
// compile-time row length NXT (0 = a.n2).
template <int C, int KZ, int NXT>
__device__ __forceinline__ void z_issue_lane(const HexArgs& a, const int* its, int i, int j, unsigned char* slot,
                                             uint64_t* bar, int part) {
  const int nx = NXT ? NXT : a.n2;
  const int info = its[i];
  const int y = info & 0xffff, zb = (info >> 16) & 0x7fff;
  const uint32_t row_bytes = nx * 8;
  if (part == 0) fft::mbar_expect_tx(bar, 2 * C * row_bytes + (j ? nx : 0));
  const int plane = a.n1 * nx;  // < 2^31 (create checks c np < 2^31)
  // one straight-line path for the u rows (parts 0..2C-1) and the phase row
  // (part 2C, element plane = node plane - 1): the lanes differ only in
  // selected offsets, so the issuing warp does not run two divergent branches
  const bool isph = part == 2 * C;
  const int k = part >> 1, r = part & 1;
  const int yr = (r && !isph) ? (y + 1 == a.n1 ? 0 : y + 1) : y;
  int pz = zb * KZ - 1 + j - (isph ? 1 : 0);
  const unsigned char* src;
  if (a.dist) {
    if (isph) {
      src = pz < 0 ? a.ph_lo : a.phase + (int64_t)pz * plane;
    } else {
      const bool halo = pz < 0 || pz >= a.n0;
      const double* s8 = pz < 0 ? a.halo_lo : (pz >= a.n0 ? a.halo_hi : a.u + (int64_t)pz * plane);
      s8 += (int64_t)k * (halo ? a.halo_cs : (int64_t)plane * a.n0);
      src = reinterpret_cast<const unsigned char*>(s8);
    }
    src += (int64_t)yr * nx * (isph ? 1 : 8);
  } else {
    pz = pz < 0 ? pz + a.n0 : (pz >= a.n0 ? pz - a.n0 : pz);
    const int64_t off = (int64_t)((isph ? 0 : k * a.n0) + pz) * plane + yr * nx;  // elements
    src = isph ? a.phase + off : reinterpret_cast<const unsigned char*>(a.u + off);
  }
  const uint32_t dst_off = isph ? 2 * C * row_bytes : (uint32_t)(r * C + k) * row_bytes;
  if (!isph || j) fft::bulk_g2s(slot + dst_off, src, isph ? (uint32_t)nx : row_bytes, bar);
}

template <int C, bool ISO, int KZ, bool FE, int NXT, bool QT = false, bool MATS = true>
__global__ void __launch_bounds__(NXT == 512 ? 512 : 256, (NXT == 512 || QT) ? 1 : (C == 3 ? HB_HEXZ_MINB3 : 2))
    k_hex_z(const HexArgs a, const ZRun run) {
  if (a.st && a.st->done) return;
  constexpr int MS = QT ? 3 : mat_stride<C, ISO>();
  constexpr int D = kZDepth;
  extern __shared__ __align__(16) unsigned char zsm[];
  const int nx = NXT ? NXT : blockDim.x;  // == n2 (compile-time for the common sizes: immediate smem offsets)
  const int nw = nx >> 5;
  const int sb = zslot_bytes<C>(nx);
  unsigned char* ring = zsm;                                        // [D][sb]
  double* ybuf = reinterpret_cast<double*>(zsm + D * sb);            // [KZ][C][nx]
  double* lo_s = ybuf + KZ * C * nx;                                 // [C][4][nx]
  double* edge = lo_s + 4 * C * nx;                                  // [2][nw][C][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(edge + 2 * nw * C * 2);  // [D]
  int* its = reinterpret_cast<int*>(full + D);                       // [list_cap]
  double* mat_s = reinterpret_cast<double*>(its + ((run.list_cap + 1) & ~1));  // optional table copy

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  // this block's run of element rows and its y-iteration list
  const int r0 = (int)((int64_t)blockIdx.x * run.rows_total / run.grid);
  const int r1 = (int)((int64_t)(blockIdx.x + 1) * run.rows_total / run.grid);
  __shared__ int n_its_s;
  if (tid == 0) {
    int n = 0;
    for (int r = r0; r < r1; ++r) {
      const int zb = r / a.n1, y = r - zb * a.n1;
      if (r == r0 || y == 0) its[n++] = (y == 0 ? a.n1 - 1 : y - 1) | (zb << 16) | (1 << 31);
      its[n++] = y | (zb << 16);
    }
    n_its_s = n;
    for (int d = 0; d < D; ++d) fft::mbar_init(&full[d], 1);
    fft::fence_mbar_init();
  }
  // MATS: the per-phase table lives in shared memory (the common case; a
  // statically shared pointer keeps its loads LDS instead of generic LD)
  if (MATS)
    for (int i = tid; i < a.n_phases * MS; i += nx) mat_s[i] = a.mat[i];
  __syncthreads();
  const int n_its = n_its_s;
  const int nunits = n_its * (KZ + 2);
  if (tid == 0)
    for (int u = 0; u < D && u < nunits; ++u) z_issue<C, KZ>(a, its, u, ring + u * sb, &full[u]);

  const int x = tid;
  const int xp = x + 1 == nx ? 0 : x + 1;
  const int plane_i = a.n1 * nx;
  const int np_i = plane_i * a.n0;
  double dotacc = 0.0;
  double zc[C][4], uprev[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    uprev[k] = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) zc[k][m] = 0.0;
  }
  int u = 0;
  int slot = 0, par = 0;  // ring slot u % D and its phase (u / D) & 1
#pragma unroll 1
  for (int it = 0; it < n_its; ++it) {
    const int info = its[it];
    const int y = info & 0xffff, zb = (info >> 16) & 0x7fff;
    const bool warm = info < 0;
    // output node (x, y) of plane zb*KZ, component 0; + zi*plane + k*np
    // (32-bit: c np < 2^31 for every one-device grid, create checks it)
    const int orow = (zb * KZ * a.n1 + y) * nx + x;
    // two z-steps per loop body on the register-light variants: the
    // loop-carried faces alternate between register sets instead of being
    // copied (0.430 -> 0.414 ms at c3)
    constexpr int JU = (ISO && !QT && NXT != 512) ? kJUnroll : 1;
#pragma unroll JU
    for (int j = 0; j < KZ + 2; ++j, ++u) {
      unsigned char* sl = ring + slot * sb;
      fft::mbar_wait(&full[slot], par);
      const double* rows = reinterpret_cast<const double*>(sl);
      double Up[C][4], ucur[C];
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const double a0 = rows[(0 * C + k) * nx + x], a1 = rows[(0 * C + k) * nx + xp];
        const double b0 = rows[(1 * C + k) * nx + x], b1 = rows[(1 * C + k) * nx + xp];
        const double aS = a0 + a1, aD = a1 - a0, bS = b0 + b1, bD = b1 - b0;
        Up[k][0] = aS + bS;
        Up[k][1] = aD + bD;
        Up[k][2] = bS - aS;
        Up[k][3] = bD - aD;
        ucur[k] = a0;
      }
      const int ph = j ? sl[2 * C * nx * 8 + x] : 0;
      double nodev[C][2];
      if (j) {
        // lower plane's x/y-stage values (stored by the previous step)
        double V[C][8];
#pragma unroll
        for (int k = 0; k < C; ++k)
#pragma unroll
          for (int m = 0; m < 4; ++m) {
#ifdef HB_HEXZ_EXP_NOLO  // timing experiment only (wrong results): no lower-face round trip
            const double lo = 0.5 * Up[k][m] + zc[k][m];
#else
            const double lo = lo_s[(k * 4 + m) * nx + x];
#endif
            V[k][m] = lo + Up[k][m];
            V[k][4 + m] = Up[k][m] - lo;
          }
        // modal residual folded straight into the z-adjoint: A = lower face
        // (seeded with the previous element's upper face), B = upper face
        double A[C][4], B[C][4];  // B: assigned by its first contribution
        const double* mat = (MATS ? mat_s : a.mat) + ph * MS;
        if constexpr (HB_HEXZ_RFOLD && ISO && !QT) {
          // modal residual R[k][v] first (one operation per contribution),
          // then the z-adjoint: A = seed + R[m] - R[m+4], B = R[m] + R[m+4]
          // (R[k][0]: the constant mode carries no gradient)
          double R[C][8];
          if constexpr (C == 3) {
            HB_HEX_MODES_RFOLD_ELASTIC_ISO
          } else {
            HB_HEX_MODES_RFOLD_SCALAR_ISO
          }
#pragma unroll
          for (int k = 0; k < C; ++k) {
            A[k][0] = zc[k][0] - R[k][4];
            B[k][0] = R[k][4];
#pragma unroll
            for (int m = 1; m < 4; ++m) {
              A[k][m] = zc[k][m] + (R[k][m] - R[k][m + 4]);
              B[k][m] = R[k][m] + R[k][m + 4];
            }
          }
        } else {
#pragma unroll
        for (int k = 0; k < C; ++k)
#pragma unroll
          for (int m = 0; m < 4; ++m) A[k][m] = zc[k][m];
        if constexpr (QT && C == 3) {
#pragma unroll
          for (int k = 0; k < C; ++k)
#pragma unroll
            for (int m = 0; m < 4; ++m) B[k][m] = 0.0;
          const bool lin = mat[0] != 0.0;
          const double kq = mat[1], gq = mat[2];
          int ze = zb * KZ - 2 + j;
          ze = ze < 0 ? ze + a.n0 : ze;
          const double* tq = a.tanc + (((int64_t)ze * a.n1 + y) * nx + x) * 64;
          const double* qs = a.qs;
          const double* qw = a.qw;
#define HB_ACC(k, v, t) acc_fold<v>(A[k], B[k], (t))
          HB_HEX_MODES_QT_ELASTIC
#undef HB_ACC
        } else if constexpr (C == 3) {
          if constexpr (ISO) {
            HB_HEX_MODES_FOLD_ELASTIC_ISO
          } else {
            HB_HEX_MODES_FOLD_ELASTIC_GEN
          }
        } else {
          if constexpr (ISO) {
            HB_HEX_MODES_FOLD_SCALAR_ISO
          } else {
            HB_HEX_MODES_FOLD_SCALAR_GEN
          }
        }
        }
        if constexpr (FE) {  // element load, moved to the modal basis (fwd / 8)
#pragma unroll
          for (int k = 0; k < C; ++k) {
            double fx[8], fv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) fx[i] = __ldg(a.fe + ph * 8 * C + i * C + k);
            modal_fwd(fx, fv);
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              A[k][m] += 0.125 * (fv[m] - fv[4 + m]);
              B[k][m] += 0.125 * (fv[m] + fv[4 + m]);
            }
          }
        }
        double sp[C][2];
#pragma unroll
        for (int k = 0; k < C; ++k) {
#pragma unroll
          for (int m = 0; m < 4; ++m) zc[k][m] = B[k][m];
#pragma unroll
          for (int ym = 0; ym < 2; ++ym) {
            const double sm = A[k][ym * 2] - A[k][ym * 2 + 1];
            sp[k][ym] = A[k][ym * 2] + A[k][ym * 2 + 1];
            const double recv = __shfl_up_sync(0xffffffffu, sp[k][ym], 1);
            nodev[k][ym] = lane ? sm + recv : sm;
          }
        }
        if (lane == 31) {
          double* eg = edge + ((u & 1) * nw + warp) * C * 2;
#pragma unroll
          for (int k = 0; k < C; ++k) {
            eg[k * 2 + 0] = sp[k][0];
            eg[k * 2 + 1] = sp[k][1];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < C; ++k)
#pragma unroll
        for (int m = 0; m < 4; ++m) {
#ifndef HB_HEXZ_EXP_NOLO
          lo_s[(k * 4 + m) * nx + x] = Up[k][m];
#endif
        }
      __syncthreads();  // edges visible; ring slot fully read
      // refill this slot with unit u + D, one copy per warp
#if HB_HEXZ_ISSUE == 0
      if (lane == 0 && u + D < nunits)
        for (int part = warp; part <= 2 * C; part += nw) z_issue_part<C, KZ>(a, its, u + D, sl, &full[slot], part);
#else
      // the 2C + 1 copies of the unit are issued by lanes 0..2C of ONE warp in
      // the same instruction stream (the warp rotates with u): the other
      // warps skip the refill bookkeeping (16 % of the kernel's issued
      // instructions when every warp's lane 0 issued one copy)
      if (u + D < nunits && warp == (HB_HEXZ_ISSUE == 1 ? (u & (nw - 1)) : 0) && lane <= 2 * C) {
        int jn = j + D, in = it;
        if (jn >= KZ + 2) {
          jn -= KZ + 2;
          ++in;
        }
        z_issue_lane<C, KZ, NXT>(a, its, in, jn, sl, &full[slot], lane);
      }
#endif
      if (++slot == D) {
        slot = 0;
        par ^= 1;
      }
      if (j >= 2) {
        const int zi = j - 2;
        const double* eg = edge + ((u & 1) * nw + (warp == 0 ? nw - 1 : warp - 1)) * C * 2;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          double n0v = nodev[k][0], n1v = nodev[k][1];
          if (lane == 0) {
            n0v += eg[k * 2 + 0];
            n1v += eg[k * 2 + 1];
          }
          const double rowy = n0v - n1v, rowy1 = n0v + n1v;
          double* yb = ybuf + (zi * C + k) * nx + x;
          if (!warm) {
            // scale = 1 in every launch without element loads (PCG, apply_K)
            const double val = FE ? a.scale * (rowy + *yb) : rowy + *yb;
            a.out[k * np_i + orow + zi * plane_i] = val;
            dotacc = fma(uprev[k], val, dotacc);
          }
          *yb = rowy1;
        }
      }
#pragma unroll
      for (int k = 0; k < C; ++k) uprev[k] = ucur[k];
    }
  }
  if (a.partials) {
    __shared__ double red[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dotacc += __shfl_xor_sync(0xffffffffu, dotacc, o);
    if (lane == 0) red[warp] = dotacc;
    __syncthreads();
    if (warp == 0) {
      double t = lane < nw ? red[lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      if (lane == 0) a.partials[blockIdx.x] = t;
    }
    if (blockIdx.x == 0)
      for (int i = gridDim.x + tid; i < a.nred; i += nx) a.partials[i] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// Quadrature reductions of the Newton shell on the hex fast path
// (solver.cpp:216-263 norms, :321-324 average stress): in the modal basis the
// 8 Gauss-point patterns are orthogonal, so
//   sum_q w |eps_q + E|^2 = 8w sum_modes |s_m e_m (+ E for the constant mode)|^2
//   sum_q w C (eps_q + E)  = 8w C (s_0 e_sss + E)
// (s_m = 1/(4h), 1/(4 sqrt3 h), 1/(12h) by class; sqrt(2)/2 on Mandel shear).
// One element per thread, rows (y, z) strided over a fixed grid; per-block
// partials (deterministic). Sums are returned without the 8w = h^3 factor.
struct HexQArgs {
  const double* u;
  const double* halo_hi;  // dist: plane n0 of u
  int dist;
  const double* e;        // nullable macro strain (Mandel, m)
  const uint8_t* phase;
  const double* cmat;     // stress: n_phases x m x m column-major
  double* partials;       // per block: 1 (norm) or m (stress)
  double sc[6];
  int n0, n1, n2;
};

template <int C, bool STRESS>
__global__ void __launch_bounds__(256) k_hex_quad(const HexQArgs a) {
  constexpr int M = C == 3 ? 6 : 3;
  constexpr int NV = STRESS ? M : 1;
  const int nx = a.n2;
  const int64_t plane = (int64_t)a.n1 * nx, np = plane * a.n0;
  double E[M], sc[6];
#pragma unroll
  for (int k = 0; k < M; ++k) E[k] = a.e ? a.e[k] : 0.0;
#pragma unroll
  for (int k = 0; k < 6; ++k) sc[k] = a.sc[k];
  double acc[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) acc[i] = 0.0;
  const int nrows = a.n0 * a.n1;
  for (int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < nrows * (nx / 32);
       r += gridDim.x * (blockDim.x / 32)) {
    // warp-granular work item: (row, 32-column segment)
    const int row = r / (nx / 32), seg = r % (nx / 32);
    const int z = row / a.n1, y = row % a.n1;
    const int x = seg * 32 + (threadIdx.x & 31);
    const int xp = x + 1 == nx ? 0 : x + 1, y1 = y + 1 == a.n1 ? 0 : y + 1;
    const double* p0 = a.u + (int64_t)z * plane;
    const double* p1;
    int64_t cs1 = np;
    if (z + 1 < a.n0) p1 = p0 + plane;
    else if (a.dist) {
      p1 = a.halo_hi;
      cs1 = plane;
    } else p1 = a.u;
    double V[C][8];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      double xx[8];
      xx[0] = __ldg(p0 + k * np + (int64_t)y * nx + x);
      xx[1] = __ldg(p0 + k * np + (int64_t)y * nx + xp);
      xx[2] = __ldg(p0 + k * np + (int64_t)y1 * nx + x);
      xx[3] = __ldg(p0 + k * np + (int64_t)y1 * nx + xp);
      xx[4] = __ldg(p1 + k * cs1 + (int64_t)y * nx + x);
      xx[5] = __ldg(p1 + k * cs1 + (int64_t)y * nx + xp);
      xx[6] = __ldg(p1 + k * cs1 + (int64_t)y1 * nx + x);
      xx[7] = __ldg(p1 + k * cs1 + (int64_t)y1 * nx + xp);
      modal_fwd(xx, V[k]);
    }
    if constexpr (!STRESS) {
      double nacc = 0.0;
      if constexpr (C == 3) {
        HB_HEX_MODES_NRM_ELASTIC
      } else {
        HB_HEX_MODES_NRM_SCALAR
      }
      acc[0] += nacc;
    } else {
      double es[M];
      if constexpr (C == 3) {
        HB_HEX_MODES_SSS_ELASTIC
      } else {
        HB_HEX_MODES_SSS_SCALAR
      }
      const double* cm = a.cmat + (size_t)a.phase[(int64_t)z * plane + (int64_t)y * nx + x] * M * M;
#pragma unroll
      for (int i = 0; i < M; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) t = fma(__ldg(cm + j * M + i), es[j], t);
        acc[i] += t;
      }
    }
  }
  __shared__ double red[NV][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double v = acc[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[i][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    a.partials[(size_t)blockIdx.x * NV + threadIdx.x] = v;
  }
}
}  // namespace

// z-block depth: bounded by the per-thread row buffer (KZ x C x nx doubles)
static int hex_kz(const Grid& g) {
  if (g.n2 > 256) return g.c == 3 ? HB_HEXZ_KZ512 : 8;  // 512-wide rows: one 512-thread block per SM
  if (g.c == 3) return HB_HEXZ_KZ3;
  if (HB_HEXZ_KZ1) return HB_HEXZ_KZ1;
  return ((int64_t)g.n1 * (g.n0 / 16) >= 2048 && g.n0 % 16 == 0) ? 16 : 8;
}

static bool hex_v2(const Grid& g) {
  const char* e = std::getenv("HOMFE_HEX_V1");
  if (e && e[0] == '1') return false;
  return g.n0 % hex_kz(g) == 0;
}

// Tile (rows y per thread, planes z per tile): a larger tile recomputes
// fewer warm-up elements ((1 + 1/TY)(1 + 1/TZ)) but yields fewer blocks.
static void hex_tile(const Grid& g, int& ty, int& tz) {
  ty = 8;
  tz = 16;
  if (const char* e = std::getenv("HOMFE_HEX_TILE")) {
    int a = 0, b = 0;
    if (std::sscanf(e, "%dx%d", &a, &b) == 2) {
      ty = a;
      tz = b;
    }
  }
  (void)g;
}

bool hex_fast_eligible(const Grid& g) {
  if (g.d != 3 || g.kind != 3 || (g.c != 1 && g.c != 3)) return false;
  int ty, tz;
  hex_tile(g, ty, tz);
  if (g.n2 % 32 != 0 || g.n2 > 512 || (g.n2 > 256 && g.n2 != 512)) return false;
  if (g.n2 == 512 && !hex_v2(g)) return false;
  if (!hex_v2(g) && (g.n1 % ty != 0 || g.n0 % tz != 0)) return false;
  if (g.h[0] != g.h[1] || g.h[1] != g.h[2]) return false;
  return true;
}

// Per-phase material tables for the modal kernel. Returns false if the
// catalog is not isotropic (then the general table is produced).
bool hex_fast_tables(const Grid& g, int n_phases, const double* cmats, std::vector<double>& iso,
                     std::vector<double>& gen) {
  const int m = g.m;
  const double h = g.h[0];
  const double f[3] = {h / 16.0, h / 48.0, h / 144.0};  // 8 w s_mode^2 per class
  const double s2 = 0.70710678118654752440;
  bool all_iso = true;
  iso.clear();
  gen.clear();
  for (int ph = 0; ph < n_phases; ++ph) {
    const double* cm = cmats + (size_t)ph * m * m;  // column-major
    auto C = [&](int i, int j) { return cm[j * m + i]; };
    if (m == 6) {
      const double lam = C(0, 1), twomu = C(3, 3);
      const double tol = 8e-16 * (std::fabs(lam) + std::fabs(twomu));
      bool ok = true;
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          double want;
          if (i < 3 && j < 3) want = (i == j) ? lam + twomu : lam;
          else want = (i == j) ? twomu : 0.0;
          if (std::fabs(C(i, j) - want) > tol) ok = false;
        }
      all_iso = all_iso && ok;
      for (int c = 0; c < 3; ++c) {
        iso.push_back(f[c] * lam);
        iso.push_back(f[c] * twomu);
        iso.push_back(f[c] * 0.5 * twomu);  // mu: s2^2 * 2mu on the raw shear rows
      }
      iso.push_back(f[2] * (lam + 2.0 * twomu));  // modes aas + asa + saa merged (RFOLD)
      for (int c = 0; c < 3; ++c)
        for (int i = 0; i < 6; ++i)
          for (int j = 0; j < 6; ++j) {
            const double si = i < 3 ? 1.0 : s2, sj = j < 3 ? 1.0 : s2;
            gen.push_back(f[c] * si * C(i, j) * sj);
          }
    } else {
      const double k0 = C(0, 0);
      bool ok = true;
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          if (C(i, j) != (i == j ? k0 : 0.0)) ok = false;
      all_iso = all_iso && ok;
      for (int c = 0; c < 3; ++c) iso.push_back(f[c] * k0);
      for (int c = 0; c < 3; ++c)
        for (int i = 0; i < 3; ++i)
          for (int j = 0; j < 3; ++j) gen.push_back(f[c] * C(i, j));
    }
  }
  return all_iso;
}

template <int C, bool ISO, int KZ, bool FE, int NXT, bool QT = false, bool MATS = true>
static void launch_hex_z_nx_m(const Grid& g, const HexArgs& a, int n_phases, cudaStream_t s);

template <int C, bool ISO, int KZ, bool FE, int NXT, bool QT = false>
static void launch_hex_z_nx(const Grid& g, const HexArgs& a, int n_phases, cudaStream_t s) {
  constexpr int MS = QT ? 3 : mat_stride<C, ISO>();
  if (n_phases * MS <= 2048) launch_hex_z_nx_m<C, ISO, KZ, FE, NXT, QT, true>(g, a, n_phases, s);
  else launch_hex_z_nx_m<C, ISO, KZ, FE, NXT, QT, false>(g, a, n_phases, s);
}

template <int C, bool ISO, int KZ, bool FE, int NXT, bool QT, bool MATS>
static void launch_hex_z_nx_m(const Grid& g, const HexArgs& a, int n_phases, cudaStream_t s) {
  constexpr int MS = QT ? 3 : mat_stride<C, ISO>();
  const int nx = g.n2, nw = nx / 32;
  const int rows_total = g.n1 * (g.n0 / KZ);
  auto smem_for = [&](int grid) {
    const int per = (rows_total + grid - 1) / grid;
    const int cap = 2 * per + 4;
    size_t b = (size_t)kZDepth * zslot_bytes<C>(nx) + sizeof(double) * ((size_t)KZ * C * nx + 4 * C * nx + 2 * nw * C * 2) +
               sizeof(uint64_t) * kZDepth + sizeof(int) * ((cap + 1) & ~1);
    if (MATS) b += sizeof(double) * (size_t)n_phases * MS;
    return b;
  };
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    HB_CUDA(cudaGetDevice(&dev));
    HB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  size_t smem = smem_for(2 * sms);
  HB_CUDA(cudaFuncSetAttribute(k_hex_z<C, ISO, KZ, FE, NXT, QT, MATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hex_z<C, ISO, KZ, FE, NXT, QT, MATS>, nx, smem));
  if (per_sm < 1) per_sm = 1;
  int grid = per_sm * sms;
  if (grid > rows_total) grid = rows_total;
  if (grid > kRedBlocks) grid = kRedBlocks;
  smem = smem_for(grid);
  HB_CUDA(cudaFuncSetAttribute(k_hex_z<C, ISO, KZ, FE, NXT, QT, MATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ZRun run;
  run.rows_total = rows_total;
  run.grid = grid;
  run.list_cap = 2 * ((rows_total + grid - 1) / grid) + 4;
  k_hex_z<C, ISO, KZ, FE, NXT, QT, MATS><<<grid, nx, smem, s>>>(a, run);
}

template <int C, bool ISO, int KZ, bool FE>
static void launch_hex_z(const Grid& g, const HexArgs& a, int n_phases, cudaStream_t s) {
  if (g.n2 == 512) {
    launch_hex_z_nx<C, ISO, C == 3 ? HB_HEXZ_KZ512 : 8, FE, 512>(g, a, n_phases, s);
    return;
  }
  if (g.n2 == 256) launch_hex_z_nx<C, ISO, KZ, FE, 256>(g, a, n_phases, s);
  else if (g.n2 == 128) launch_hex_z_nx<C, ISO, KZ, FE, 128>(g, a, n_phases, s);
  else launch_hex_z_nx<C, ISO, KZ, FE, 0>(g, a, n_phases, s);
}

void launch_hex_fast(const Grid& g, const ElemArgs& ea, const double* d_mat, bool iso, cudaStream_t s) {
  HexArgs a;
  a.u = ea.u;
  a.halo_lo = ea.halo_lo;
  a.halo_hi = ea.halo_hi;
  a.ph_lo = ea.ph_lo;
  a.halo_cs = ea.halo_cs ? ea.halo_cs : (int64_t)g.n1 * g.n2;
  a.dist = g.dist;
  a.out = ea.out;
  a.phase = ea.phase;
  a.mat = d_mat;
  a.fe = ea.fe;
  a.n_phases = ea.n_phases;
  a.scale = ea.scale;
  a.partials = ea.partials;
  a.nred = kRedBlocks;
  a.st = ea.st;
  a.n0 = g.n0;
  a.n1 = g.n1;
  a.n2 = g.n2;
  if (hex_v2(g)) {
    if (!a.fe && a.scale != 1.0) throw ValidationError("hexfast: a scaled K without element loads is not supported");
#define HB_HEXZ(C, ISO, KZ)                                      \
  do {                                                           \
    if (a.fe) launch_hex_z<C, ISO, KZ, true>(g, a, ea.n_phases, s); \
    else launch_hex_z<C, ISO, KZ, false>(g, a, ea.n_phases, s);     \
  } while (0)
    if (g.c == 3) {
      if (iso) HB_HEXZ(3, true, HB_HEXZ_KZ3);
      else HB_HEXZ(3, false, HB_HEXZ_KZ3);
    } else {
      if (hex_kz(g) == 16) {
        if (iso) HB_HEXZ(1, true, 16);
        else HB_HEXZ(1, false, 16);
      } else {
        if (iso) HB_HEXZ(1, true, 8);
        else HB_HEXZ(1, false, 8);
      }
    }
#undef HB_HEXZ
    HB_CUDA(cudaGetLastError());
    return;
  }
  int kTY, kTZ;
  hex_tile(g, kTY, kTZ);
  a.tiles_y = g.n1 / kTY;
  a.tiles_z = g.n0 / kTZ;
  const int ntiles = a.tiles_y * a.tiles_z;
  const int grid = ntiles < kRedBlocks ? ntiles : kRedBlocks;
  const int nw = g.n2 / 32;
  const int ms = iso ? (g.c == 3 ? 9 : 3) : (g.c == 3 ? 108 : 27);
  const size_t smem = sizeof(double) * ((size_t)kTY * g.c * g.n2 + 2 * nw * 4 * g.c + (size_t)ea.n_phases * ms +
                                        (size_t)ea.n_phases * 8 * g.c);
#define HB_HEX_T(C, ISO, TY, TZ)                                                                    \
  do {                                                                                              \
    HB_CUDA(cudaFuncSetAttribute(k_hex_fast<C, ISO, TY, TZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k_hex_fast<C, ISO, TY, TZ><<<grid, g.n2, smem, s>>>(a);                                         \
  } while (0)
#define HB_HEX(C, ISO)                                                        \
  do {                                                                        \
    if (kTY == 8 && kTZ == 16) HB_HEX_T(C, ISO, 8, 16);                       \
    else if (kTY == 16 && kTZ == 16) HB_HEX_T(C, ISO, 16, 16);                \
    else if (kTY == 8 && kTZ == 32) HB_HEX_T(C, ISO, 8, 32);                  \
    else if (kTY == 16 && kTZ == 8) HB_HEX_T(C, ISO, 16, 8);                  \
    else if (kTY == 4 && kTZ == 32) HB_HEX_T(C, ISO, 4, 32);                  \
    else if (kTY == 32 && kTZ == 8) HB_HEX_T(C, ISO, 32, 8);                  \
    else throw ValidationError("hexfast: unsupported tile");                  \
  } while (0)
  if (g.c == 3) {
    if (iso) HB_HEX(3, true);
    else HB_HEX(3, false);
  } else {
    if (iso) HB_HEX(1, true);
    else HB_HEX(1, false);
  }
#undef HB_HEX
#undef HB_HEX_T
  HB_CUDA(cudaGetLastError());
}

// Newton-shell quadrature sums on the hex fast path; false if not eligible.
bool launch_hex_quad(const Grid& g, int mode, const double* u, const double* halo_hi, const double* e,
                     const uint8_t* phase, const double* cmat, double* partials, cudaStream_t s) {
  if (!hex_fast_eligible(g)) return false;
  HexQArgs a;
  a.u = u;
  a.halo_hi = halo_hi;
  a.dist = g.dist;
  a.e = e;
  a.phase = phase;
  a.cmat = cmat;
  a.partials = partials;
  const double h = g.h[0], r2 = 0.70710678118654752440;
  const double s0 = 1.0 / (4.0 * h), s1 = 1.0 / (4.0 * std::sqrt(3.0) * h), s2 = 1.0 / (12.0 * h);
  const double scv[6] = {s0, s0 * r2, s1, s1 * r2, s2, s2 * r2};
  for (int i = 0; i < 6; ++i) a.sc[i] = scv[i];
  a.n0 = g.n0;
  a.n1 = g.n1;
  a.n2 = g.n2;
  if (mode == 0) {
    if (g.c == 3) k_hex_quad<3, false><<<kRedBlocks, 256, 0, s>>>(a);
    else k_hex_quad<1, false><<<kRedBlocks, 256, 0, s>>>(a);
  } else {
    if (g.c == 3) k_hex_quad<3, true><<<kRedBlocks, 256, 0, s>>>(a);
    else k_hex_quad<1, true><<<kRedBlocks, 256, 0, s>>>(a);
  }
  HB_CUDA(cudaGetLastError());
  return true;
}

// K u with per-Gauss-point compact tangents (J2 Newton path, C = 3): the
// z-march kernel with the mode contraction replaced by strain at the 8 Gauss
// points, the compact consistent tangent and the projection back onto the
// modes. qtab: per phase (linear flag, bulk, shear).
bool launch_hex_fast_qt(const Grid& g, const ElemArgs& ea, const double* d_qtab, const double* d_tanc,
                        cudaStream_t s) {
  if (!hex_fast_eligible(g) || g.c != 3 || !hex_v2(g) || g.dist) return false;
  HexArgs a{};
  a.u = ea.u;
  a.dist = 0;
  a.out = ea.out;
  a.phase = ea.phase;
  a.mat = d_qtab;
  a.fe = nullptr;
  a.n_phases = ea.n_phases;
  a.scale = ea.scale;
  if (a.scale != 1.0) return false;  // the generic two-pass operator handles scaled applications
  a.partials = ea.partials;
  a.nred = kRedBlocks;
  a.st = ea.st;
  a.n0 = g.n0;
  a.n1 = g.n1;
  a.n2 = g.n2;
  a.tanc = d_tanc;
  const double h = g.h[0], r2 = 0.70710678118654752440, w = h * h * h / 8.0;
  const double s0 = 1.0 / (4.0 * h), s1 = 1.0 / (4.0 * std::sqrt(3.0) * h), s2 = 1.0 / (12.0 * h);
  const double qs[6] = {s0, s0 * r2, s1, s1 * r2, s2, s2 * r2};
  for (int i = 0; i < 6; ++i) {
    a.qs[i] = qs[i];
    a.qw[i] = w * qs[i];
  }
  if (g.n2 == 512) launch_hex_z_nx<3, true, 4, false, 512, true>(g, a, ea.n_phases, s);
  else if (g.n2 == 256) launch_hex_z_nx<3, true, HB_HEXZ_KZ3, false, 256, true>(g, a, ea.n_phases, s);
  else if (g.n2 == 128) launch_hex_z_nx<3, true, HB_HEXZ_KZ3, false, 128, true>(g, a, ea.n_phases, s);
  else launch_hex_z_nx<3, true, HB_HEXZ_KZ3, false, 0, true>(g, a, ea.n_phases, s);
  HB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace hb
