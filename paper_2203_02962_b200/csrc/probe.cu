// probe.cu -- the reference's impulse-probed block preconditioner
// (proj/src/precond.cpp:44-162) for stencils with two node types per pixel
// (FourTrianglesTwoNode), where the Fourier blocks are
// complex Hermitian (c Nn) x (c Nn) matrices instead of a real closed-form
// symbol:
//  * assembly: one impulse per (component, node type) slice through the
//    reference operator, the response's slices D2Z-transformed, stored as
//    block columns (k_probe_store);
//  * inversion per frequency (k_probe_invert): k = 0 via the translation
//    kernel, (B0 + V V^T)^-1 - V V^T; k > 0 via the eigen-decomposition of the
//    real symmetric 2b x 2b embedding [[Re, -Im], [Im, Re]] (cyclic Jacobi),
//    refusing lambda_min <= 1e-12 lambda_max like invert_blocks;
//  * application (k_probe_apply): per-frequency block matvec between the
//    batched D2Z / Z2D of all slices, 1/N_p folded in.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace hb {

namespace {

constexpr int kMaxB = 4;  // c * Nn <= 2 * 2

__global__ void k_probe_store(const double2* __restrict__ spec, int b, int64_t nf, int col, double2* blocks) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x)
    for (int row = 0; row < b; ++row) blocks[k * b * b + (int64_t)col * b + row] = spec[(int64_t)row * nf + k];
}

// Gauss-Jordan inverse of an n x n complex matrix (column-major), n <= 4
__device__ bool cinv(int n, double2 (&a)[kMaxB * kMaxB], double2 (&inv)[kMaxB * kMaxB]) {
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) inv[j * n + i] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  for (int col = 0; col < n; ++col) {
    int piv = col;
    double best = -1.0;
    for (int r = col; r < n; ++r) {
      const double2 v = a[col * n + r];
      const double mag = v.x * v.x + v.y * v.y;
      if (mag > best) {
        best = mag;
        piv = r;
      }
    }
    if (!(best > 0.0)) return false;
    if (piv != col)
      for (int j = 0; j < n; ++j) {
        double2 t = a[j * n + col];
        a[j * n + col] = a[j * n + piv];
        a[j * n + piv] = t;
        t = inv[j * n + col];
        inv[j * n + col] = inv[j * n + piv];
        inv[j * n + piv] = t;
      }
    const double2 p = a[col * n + col];
    const double den = p.x * p.x + p.y * p.y;
    const double2 pinv = make_double2(p.x / den, -p.y / den);
    for (int j = 0; j < n; ++j) {
      const double2 v = a[j * n + col], w = inv[j * n + col];
      a[j * n + col] = make_double2(v.x * pinv.x - v.y * pinv.y, v.x * pinv.y + v.y * pinv.x);
      inv[j * n + col] = make_double2(w.x * pinv.x - w.y * pinv.y, w.x * pinv.y + w.y * pinv.x);
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      const double2 f = a[col * n + r];
      for (int j = 0; j < n; ++j) {
        const double2 v = a[j * n + col], w = inv[j * n + col];
        a[j * n + r].x -= f.x * v.x - f.y * v.y;
        a[j * n + r].y -= f.x * v.y + f.y * v.x;
        inv[j * n + r].x -= f.x * w.x - f.y * w.y;
        inv[j * n + r].y -= f.x * w.y + f.y * w.x;
      }
    }
  }
  return true;
}

__global__ void k_probe_invert(double2* blocks, int64_t nf, int b, int nn, int* status) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
    double2* blk = blocks + k * b * b;
    if (k == 0) {
      // translation kernel V(c Nn + n, c) = 1/sqrt(Nn): (V V^T)_ij = 1/Nn within a component
      double2 a[kMaxB * kMaxB], inv[kMaxB * kMaxB];
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) {
          const double vv = (i / nn == j / nn) ? 1.0 / nn : 0.0;
          a[j * b + i] = make_double2(blk[j * b + i].x + vv, blk[j * b + i].y);
        }
      if (!cinv(b, a, inv)) {
        status[0] = 1;
        continue;
      }
      for (int j = 0; j < b; ++j)
        for (int i = 0; i < b; ++i) {
          const double vv = (i / nn == j / nn) ? 1.0 / nn : 0.0;
          blk[j * b + i] = make_double2(inv[j * b + i].x - vv, inv[j * b + i].y);
        }
      continue;
    }
    // real symmetric embedding E = [[Re, -Im], [Im, Re]] (2b x 2b)
    const int n2 = 2 * b;
    double e[2 * kMaxB][2 * kMaxB], v[2 * kMaxB][2 * kMaxB];
    for (int i = 0; i < b; ++i)
      for (int j = 0; j < b; ++j) {
        const double2 z = blk[j * b + i];
        e[i][j] = z.x;
        e[i][j + b] = -z.y;
        e[i + b][j] = z.y;
        e[i + b][j + b] = z.x;
      }
    for (int i = 0; i < n2; ++i)
      for (int j = 0; j < n2; ++j) v[i][j] = i == j ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 60; ++sweep) {
      double off = 0.0;
      for (int i = 0; i < n2; ++i)
        for (int j = i + 1; j < n2; ++j) off += e[i][j] * e[i][j];
      if (off < 1e-300) break;
      for (int p = 0; p < n2; ++p)
        for (int q = p + 1; q < n2; ++q) {
          const double apq = e[p][q];
          if (fabs(apq) < 1e-300) continue;
          const double th = 0.5 * (e[q][q] - e[p][p]) / apq;
          const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
          const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
          for (int r = 0; r < n2; ++r) {
            const double arp = e[r][p], arq = e[r][q];
            e[r][p] = cs * arp - sn * arq;
            e[r][q] = sn * arp + cs * arq;
          }
          for (int r = 0; r < n2; ++r) {
            const double apr = e[p][r], aqr = e[q][r];
            e[p][r] = cs * apr - sn * aqr;
            e[q][r] = sn * apr + cs * aqr;
          }
          for (int r = 0; r < n2; ++r) {
            const double vrp = v[r][p], vrq = v[r][q];
            v[r][p] = cs * vrp - sn * vrq;
            v[r][q] = sn * vrp + cs * vrq;
          }
        }
    }
    double lmin = e[0][0], lmax = fabs(e[0][0]);
    for (int i = 1; i < n2; ++i) {
      lmin = fmin(lmin, e[i][i]);
      lmax = fmax(lmax, fabs(e[i][i]));
    }
    if (lmin <= 1e-12 * lmax) {
      status[0] = 2;
      continue;
    }
    // inverse of the embedding = V diag(1/lambda) V^T; its blocks are (Re, Im)
    for (int i = 0; i < b; ++i)
      for (int j = 0; j < b; ++j) {
        double re = 0.0, im = 0.0;
        for (int l = 0; l < n2; ++l) {
          const double il = 1.0 / e[l][l];
          re += v[i][l] * il * v[j][l];
          im += v[i + b][l] * il * v[j][l];
        }
        blk[j * b + i] = make_double2(re, im);
      }
  }
}

__global__ void k_probe_apply(double2* spec, const double2* __restrict__ blocks, int64_t nf, int b, double scale) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nf; k += (int64_t)gridDim.x * blockDim.x) {
    double2 x[kMaxB];
    for (int s = 0; s < b; ++s) x[s] = spec[(int64_t)s * nf + k];
    const double2* blk = blocks + k * b * b;
    for (int r = 0; r < b; ++r) {
      double re = 0.0, im = 0.0;
      for (int s = 0; s < b; ++s) {
        const double2 m = blk[s * b + r];
        re += m.x * x[s].x - m.y * x[s].y;
        im += m.x * x[s].y + m.y * x[s].x;
      }
      spec[(int64_t)r * nf + k] = make_double2(re * scale, im * scale);
    }
  }
}

int grid_of(int64_t n) {
  const int64_t b = (n + 255) / 256;
  return (int)(b < 4096 ? (b < 1 ? 1 : b) : 4096);
}

}  // namespace

void launch_probe_store(const double2* spec, int b, int64_t nf, int col, double2* blocks, cudaStream_t s) {
  k_probe_store<<<grid_of(nf), 256, 0, s>>>(spec, b, nf, col, blocks);
  HB_CUDA(cudaGetLastError());
}

void launch_probe_invert(double2* blocks, int64_t nf, int b, int nn, int* status, cudaStream_t s) {
  if (b > kMaxB) throw ValidationError("preconditioner: block dimension too large");
  k_probe_invert<<<grid_of(nf), 128, 0, s>>>(blocks, nf, b, nn, status);
  HB_CUDA(cudaGetLastError());
}

void launch_probe_apply(double2* spec, const double2* blocks, int64_t nf, int b, double scale, cudaStream_t s) {
  k_probe_apply<<<grid_of(nf), 256, 0, s>>>(spec, blocks, nf, b, scale);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
