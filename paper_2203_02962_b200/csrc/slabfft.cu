// slabfft.cu -- the transposes of the slab-decomposed spectrum for plane
// sizes the fused passes do not cover (e.g. c4's 512^2 planes).
//
// The reference transforms the whole periodic cell with FFTW r2c/c2r
// (fft.cpp:23-79, precond.cpp:126-162). With the cell split into slabs of
// n0l = n0/W planes, each rank runs the 2-D r2c of its planes (cuFFT),
// ships every k1-row block to the rank owning those rows, runs the 1-D
// transform along axis 0 on its rows (cuFFT), solves, and reverses the path:
//
//   S [c][i0l][k1][k2]  --pack_fwd-->  W_q [c][i0 = me n0l + i0l][k1l][k2]
//   W [c][i0][k1l][k2]  --pack_inv-->  S_q [c][i0l][k1 = me n1l + k1l][k2]
//
// push = 1 stores straight into the destination rank's W / S (peer pointers,
// NVLink), push = 0 into per-peer send chunks [q][c][i0l][k1l][k2] for an
// all-to-all, followed by the matching unpack. Pure permutations: the
// element order of every (c, i0, k1, k2) is fixed, so results are bitwise
// those of the all-to-all path.
#include "kernels.cuh"

namespace hb {

namespace {

constexpr int kPeers = 8;

struct PeerPtrs {
  double2* p[kPeers];
};

__global__ void __launch_bounds__(kBlock) k_pack_fwd(const SlabDims d, const double2* __restrict__ S,
                                                     const PeerPtrs dst, int push) {
  const int64_t n = (int64_t)d.c * d.n0l * d.n1 * d.nh;
  const int dn0 = push ? d.n0 : d.n0l, i0base = push ? d.me * d.n0l : 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(idx % d.nh);
    int64_t t = idx / d.nh;
    const int k1 = (int)(t % d.n1);
    t /= d.n1;
    const int i0l = (int)(t % d.n0l), comp = (int)(t / d.n0l);
    const int q = k1 / d.n1l, k1l = k1 - q * d.n1l;
    dst.p[q][(((int64_t)comp * dn0 + i0base + i0l) * d.n1l + k1l) * d.nh + k2] = S[idx];
  }
}

__global__ void __launch_bounds__(kBlock) k_unpack_fwd(const SlabDims d, const double2* __restrict__ recv,
                                                       double2* __restrict__ W) {
  const int64_t n = (int64_t)d.c * d.n0 * d.n1l * d.nh;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(idx % d.nh);
    int64_t t = idx / d.nh;
    const int k1l = (int)(t % d.n1l);
    t /= d.n1l;
    const int i0 = (int)(t % d.n0), comp = (int)(t / d.n0);
    const int q = i0 / d.n0l, i0l = i0 - q * d.n0l;
    W[idx] = recv[q * d.chunk() + (((int64_t)comp * d.n0l + i0l) * d.n1l + k1l) * d.nh + k2];
  }
}

__global__ void __launch_bounds__(kBlock) k_pack_inv(const SlabDims d, const double2* __restrict__ W,
                                                     const PeerPtrs dst, int push) {
  const int64_t n = (int64_t)d.c * d.n0 * d.n1l * d.nh;
  const int drow = push ? d.n1 : d.n1l, k1base = push ? d.me * d.n1l : 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(idx % d.nh);
    int64_t t = idx / d.nh;
    const int k1l = (int)(t % d.n1l);
    t /= d.n1l;
    const int i0 = (int)(t % d.n0), comp = (int)(t / d.n0);
    const int q = i0 / d.n0l, i0l = i0 - q * d.n0l;
    dst.p[q][(((int64_t)comp * d.n0l + i0l) * drow + k1base + k1l) * d.nh + k2] = W[idx];
  }
}

__global__ void __launch_bounds__(kBlock) k_unpack_inv(const SlabDims d, const double2* __restrict__ recv,
                                                       double2* __restrict__ S) {
  const int64_t n = (int64_t)d.c * d.n0l * d.n1 * d.nh;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int k2 = (int)(idx % d.nh);
    int64_t t = idx / d.nh;
    const int k1 = (int)(t % d.n1);
    t /= d.n1;
    const int i0l = (int)(t % d.n0l), comp = (int)(t / d.n0l);
    const int q = k1 / d.n1l, k1l = k1 - q * d.n1l;
    S[idx] = recv[q * d.chunk() + (((int64_t)comp * d.n0l + i0l) * d.n1l + k1l) * d.nh + k2];
  }
}

PeerPtrs peers(const SlabDims& d, double2* const* dst) {
  PeerPtrs p{};
  for (int q = 0; q < kPeers; ++q) p.p[q] = dst[q < d.world ? q : 0];
  return p;
}

int grid_for(int64_t n) {
  const int64_t b = (n + kBlock - 1) / kBlock;
  return (int)(b < 4 * kRedBlocks ? b : 4 * kRedBlocks);
}

}  // namespace

void launch_slab_pack_fwd(const SlabDims& d, const double2* S, double2* const* dst, int push, cudaStream_t s) {
  k_pack_fwd<<<grid_for(d.chunk() * d.world), kBlock, 0, s>>>(d, S, peers(d, dst), push);
  HB_CUDA(cudaGetLastError());
}

void launch_slab_unpack_fwd(const SlabDims& d, const double2* recv, double2* W, cudaStream_t s) {
  k_unpack_fwd<<<grid_for(d.chunk() * d.world), kBlock, 0, s>>>(d, recv, W);
  HB_CUDA(cudaGetLastError());
}

void launch_slab_pack_inv(const SlabDims& d, const double2* W, double2* const* dst, int push, cudaStream_t s) {
  k_pack_inv<<<grid_for(d.chunk() * d.world), kBlock, 0, s>>>(d, W, peers(d, dst), push);
  HB_CUDA(cudaGetLastError());
}

void launch_slab_unpack_inv(const SlabDims& d, const double2* recv, double2* S, cudaStream_t s) {
  k_unpack_inv<<<grid_for(d.chunk() * d.world), kBlock, 0, s>>>(d, recv, S);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
