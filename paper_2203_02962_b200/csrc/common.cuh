// common.cuh -- shared device/host definitions of the homfe B200 path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace hb {

// Error classes of proj/include/homfe/common.hpp:15-25, plus the CLI's
// non-convergence exit code (proj/tools/homog.cpp:23-26).
struct ValidationError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NonConverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define HB_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      throw ::hb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));  \
  } while (0)

constexpr int kMaxQuads = 8;
constexpr int kMaxEntries = 8;
constexpr int kMaxPhases = 256;

// Stencil table (grid.hpp:37-64) passed by value to kernels. Offsets are
// 0/1 per axis; `loc` numbers an element corner by its offset index.
struct StencilParams {
  int nq;                                  // quadrature points per pixel
  int ne[kMaxQuads];                       // entries per quad
  int off[kMaxQuads][kMaxEntries];         // offset index of each entry
  double dphi[kMaxQuads][kMaxEntries][3];  // shape-function derivatives
  double w[kMaxQuads];                     // quadrature weights
  int noff;                                // distinct offsets (4 or 8)
  int offs[8][3];                          // offset vectors (axis 0 slowest)
  int node[kMaxQuads][kMaxEntries];        // node type of each entry (0 corner, 1 centre)
  int nn;                                  // node types per pixel (1, or 2 for FourTrianglesTwoNode)
};

// Periodic grid geometry. 2-D grids use (n0, n1) with n2 = 1.
struct Grid {
  int d;        // 2 or 3
  int c;        // nodal components (1 or d)
  int m;        // gradient components (d or Mandel d(d+1)/2)
  int kind;     // StencilKind
  int n0, n1, n2;
  int64_t np;   // pixels (nodes = nn * np)
  double h[3];
  double cell_volume;
  // slab decomposition along axis 0 (dist = 1): n0 / np are the LOCAL plane
  // and pixel counts of this rank; the global grid has n0g planes.
  int dist;
  int n0g, z0, rank, world;
  int64_t npg;
  int nn;       // node types per pixel (grid.hpp nodes_per_pixel)
};

// PCG scalars resident on the device (solver.cpp:62-94).
struct PcgState {
  double rz;        // r.z of the current iterate
  double rz_new;
  double pap;       // p.Ap
  double alpha, beta;
  double norm0;     // |r_0|_{M^-1}
  double eta;
  int32_t it;       // completed iterations
  int32_t it_max;
  int32_t done;     // loop finished (converged, cap, or breakdown)
  int32_t converged;
  int32_t status;   // 0 ok, 4 non-positive curvature
  int32_t active;   // the current iteration computed alpha (not finished before it)
};

__host__ __device__ inline int mandel_dim(int d) { return d * (d + 1) / 2; }

}  // namespace hb
