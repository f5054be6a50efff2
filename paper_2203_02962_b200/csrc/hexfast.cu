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

#include "kernels.cuh"

namespace hb {

namespace {


// Per-phase material table layout (doubles):
//   ISO:      [3 classes][3] = f*lambda, f*2mu, f*mu   (elastic)
//             [3 classes][1] = f*kappa                 (scalar)
//   general:  [3 classes][M*M] = f * (S C S)  (S = diag(1,1,1,s2,s2,s2))
template <int C, bool ISO>
constexpr int mat_stride() {
  return ISO ? (C == 3 ? 9 : 3) : (C == 3 ? 3 * 36 : 3 * 9);
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
        cs[0] = z < 0 ? plane : np;
        up[1] = z1 >= a.n0 ? a.halo_hi : a.u + (int64_t)z1 * plane;
        cs[1] = z1 >= a.n0 ? plane : np;
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

}  // namespace

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
  if (g.n2 % 32 != 0 || g.n2 > 256 || g.n1 % ty != 0 || g.n0 % tz != 0) return false;
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

void launch_hex_fast(const Grid& g, const ElemArgs& ea, const double* d_mat, bool iso, cudaStream_t s) {
  HexArgs a;
  a.u = ea.u;
  a.halo_lo = ea.halo_lo;
  a.halo_hi = ea.halo_hi;
  a.ph_lo = ea.ph_lo;
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

}  // namespace hb
