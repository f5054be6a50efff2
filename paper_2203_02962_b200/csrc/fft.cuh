// fft.cuh -- shared-memory fp64 FFT building blocks (Stockham autosort,
// radix 8 / 16 in registers) for the fused preconditioner passes.
//
// An N-point transform is done by a group of TPF = N / 16 threads that hold
// 16 values each per stage; stages for N = 128: 16 x 8, 256: 16 x 16,
// 512: 8 x 8 x 8. Stage (Ns, R), butterfly j:
//   v[r] = x[j + r N/R] * W_{Ns R}^{r (j mod Ns)},  v = DFT_R(v),
//   y[(j / Ns) Ns R + (j mod Ns) + r Ns] = v[r]
// (Govindaraju et al., SC'08), in place: a group barrier separates the
// loads of a stage from its stores. Transforms are unnormalised; INV uses
// conjugate twiddles (FFTW/cuFFT sign conventions).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hb {
namespace fft {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 conj(double2 a) { return make_double2(a.x, -a.y); }
// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  const double2 b0 = cadd(a0, a2), b1 = csub(a0, a2);
  const double2 b2 = cadd(a1, a3), b3 = mul_mi<INV>(csub(a1, a3));
  a0 = cadd(b0, b2);
  a2 = csub(b0, b2);
  a1 = cadd(b1, b3);
  a3 = csub(b1, b3);
}

// W_8^k constants
template <bool INV>
__device__ __forceinline__ double2 w8(int k) {
  const double h = 0.70710678118654752440;
  switch (k & 7) {
    case 0: return make_double2(1.0, 0.0);
    case 1: return make_double2(h, INV ? h : -h);
    case 2: return make_double2(0.0, INV ? 1.0 : -1.0);
    case 3: return make_double2(-h, INV ? h : -h);
    case 4: return make_double2(-1.0, 0.0);
    case 5: return make_double2(-h, INV ? -h : h);
    case 6: return make_double2(0.0, INV ? -1.0 : 1.0);
    default: return make_double2(h, INV ? -h : h);
  }
}

// W_16^k constants
template <bool INV>
__device__ __forceinline__ double2 w16(int k) {
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  const double h = 0.70710678118654752440;
  double cs, sn;
  switch (k & 15) {
    case 0: cs = 1.0; sn = 0.0; break;
    case 1: cs = c1; sn = s1; break;
    case 2: cs = h; sn = h; break;
    case 3: cs = s1; sn = c1; break;
    case 4: cs = 0.0; sn = 1.0; break;
    case 5: cs = -s1; sn = c1; break;
    case 6: cs = -h; sn = h; break;
    case 7: cs = -c1; sn = s1; break;
    case 8: cs = -1.0; sn = 0.0; break;
    case 9: cs = -c1; sn = -s1; break;
    case 10: cs = -h; sn = -h; break;
    case 11: cs = -s1; sn = -c1; break;
    case 12: cs = 0.0; sn = -1.0; break;
    case 13: cs = s1; sn = -c1; break;
    case 14: cs = h; sn = -h; break;
    default: cs = c1; sn = -s1; break;
  }
  // forward: exp(-i 2 pi k / 16) = (cos, -sin)
  return make_double2(cs, INV ? sn : -sn);
}

// In-register DFT of size 8: n = n1 + 2 n2, X[k2 + 4 k1].
template <bool INV>
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = cmul(o1, w8<INV>(1));
  o2 = mul_mi<INV>(o2);
  o3 = cmul(o3, w8<INV>(3));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, o1);
  v[5] = csub(e1, o1);
  v[2] = cadd(e2, o2);
  v[6] = csub(e2, o2);
  v[3] = cadd(e3, o3);
  v[7] = csub(e3, o3);
}

// In-register DFT of size 16: n = n1 + 4 n2 -> X[k2 + 4 k1].
template <bool INV>
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
  double2 y[4][4];
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {
    double2 a0 = v[n1], a1 = v[n1 + 4], a2 = v[n1 + 8], a3 = v[n1 + 12];
    dft4<INV>(a0, a1, a2, a3);
    y[n1][0] = a0;
    y[n1][1] = a1;
    y[n1][2] = a2;
    y[n1][3] = a3;
  }
#pragma unroll
  for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
    for (int k2 = 1; k2 < 4; ++k2) y[n1][k2] = cmul(y[n1][k2], w16<INV>(n1 * k2));
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    double2 a0 = y[0][k2], a1 = y[1][k2], a2 = y[2][k2], a3 = y[3][k2];
    dft4<INV>(a0, a1, a2, a3);
    v[k2] = a0;
    v[k2 + 4] = a1;
    v[k2 + 8] = a2;
    v[k2 + 12] = a3;
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dftR(double2 (&v)[R]) {
  if constexpr (R == 16) dft16<INV>(v);
  else dft8<INV>(v);
}

// ---- TMA bulk copies (cp.async.bulk) with mbarrier completion -------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// order preceding generic-proxy shared accesses before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// wait until the smem sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// bounded wait: a protocol bug traps (launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (done) return;
    if (n > (1u << 20)) __trap();
  }
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Barrier over the TPF threads of one transform (TPF <= 32 divides the warp
// into aligned groups, so a warp barrier suffices).
__device__ __forceinline__ void group_sync() { __syncwarp(); }

// One Stockham stage on buf[0..N) by the TPF threads of a group.
// tw: table W_N^k = exp(-2 pi i k / N), k < N.
template <int N, int R, int NS, bool INV, int TPF>
__device__ __forceinline__ void stage(double2* buf, int t, const double2* __restrict__ tw) {
  constexpr int NB = N / R;
  constexpr int PER = NB / TPF;  // butterflies per thread
  double2 v[PER][R];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = t + b * TPF;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = buf[j + r * NB];
  }
  group_sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = t + b * TPF;
    const int k = j % NS;
    if (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const double2 w = tw[(r * k * (N / (NS * R))) % N];
        v[b][r] = cmul(v[b][r], INV ? conj(w) : w);
      }
    }
    dftR<R, INV>(v[b]);
    const int base = (j / NS) * NS * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) buf[base + r * NS] = v[b][r];
  }
  group_sync();
}

// Four-step transform for N = A x 16 (A = N/16 = TPF threads, N <= 256):
// x[n1 + A n2] -> DFT16 over n2 -> twiddle W_N^{n1 k2} -> Y[n1][k2] stored
// XOR-swizzled at n1*16 + (k2 ^ n1) (conflict-free both ways) -> DFT_A over
// n1 -> X[k2 + 16 k1]. tw4 is laid out [k2][n1] (conflict-free reads).
template <int N, bool INV>
__device__ __forceinline__ void fft4step(double2* buf, int t, const double2* __restrict__ tw4) {
  constexpr int A = N / 16;
  double2 v[16];
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = buf[t + A * n2];
  dft16<INV>(v);
  if (t > 0) {
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) {
      const double2 w = tw4[k2 * A + t];
      v[k2] = cmul(v[k2], INV ? conj(w) : w);
    }
  }
  group_sync();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[t * 16 + (k2 ^ (t & 15))] = v[k2];
  group_sync();
  constexpr int PER = 16 / A;  // step-2 transforms per thread
  double2 u[PER][A];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) u[b][n1] = buf[n1 * 16 + (k2 ^ n1)];
    if constexpr (A == 16) dft16<INV>(u[b]);
    else if constexpr (A == 8) dft8<INV>(u[b]);
    else dft4<INV>(u[b][0], u[b][1], u[b][2], u[b][3]);
  }
  group_sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) buf[k2 + 16 * k1] = u[b][k1];
  }
  group_sync();
}

// Same transform with the step-1 inputs x[t + A n2] (n2 < 16) already in
// registers; buf (N slots) only holds the intermediate and the output.
template <int N, bool INV>
__device__ __forceinline__ void fft4step_regs(double2 (&v)[16], double2* buf, int t,
                                              const double2* __restrict__ tw4) {
  constexpr int A = N / 16;
  dft16<INV>(v);
  if (t > 0) {
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) {
      const double2 w = tw4[k2 * A + t];
      v[k2] = cmul(v[k2], INV ? conj(w) : w);
    }
  }
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[t * 16 + (k2 ^ (t & 15))] = v[k2];
  group_sync();
  constexpr int PER = 16 / A;
  double2 u[PER][A];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) u[b][n1] = buf[n1 * 16 + (k2 ^ n1)];
    if constexpr (A == 16) dft16<INV>(u[b]);
    else if constexpr (A == 8) dft8<INV>(u[b]);
    else dft4<INV>(u[b][0], u[b][1], u[b][2], u[b][3]);
  }
  group_sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) buf[k2 + 16 * k1] = u[b][k1];
  }
  group_sync();
}

// The same two transforms on a pencil whose element n lives at buf[F(n)] (F a
// bijection onto the pencil's own slots, e.g. the interleaved, XOR-swizzled
// [i0][4] rows of pass 2's TMA stage): the transform runs in the layout the
// TMA engine loads and stores, so no re-layout pass and no block barrier is
// needed around it (only the group's own threads touch these slots).
template <int N, bool INV, class IDX>
__device__ __forceinline__ void fft4step_map(double2* buf, int t, const double2* __restrict__ tw4, IDX F) {
  constexpr int A = N / 16;
  double2 v[16];
#pragma unroll
  for (int n2 = 0; n2 < 16; ++n2) v[n2] = buf[F(t + A * n2)];
  dft16<INV>(v);
  if (t > 0) {
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) {
      const double2 w = tw4[k2 * A + t];
      v[k2] = cmul(v[k2], INV ? conj(w) : w);
    }
  }
  group_sync();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[F(t * 16 + (k2 ^ (t & 15)))] = v[k2];
  group_sync();
  constexpr int PER = 16 / A;
  double2 u[PER][A];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) u[b][n1] = buf[F(n1 * 16 + (k2 ^ n1))];
    if constexpr (A == 16) dft16<INV>(u[b]);
    else if constexpr (A == 8) dft8<INV>(u[b]);
    else dft4<INV>(u[b][0], u[b][1], u[b][2], u[b][3]);
  }
  group_sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) buf[F(k2 + 16 * k1)] = u[b][k1];
  }
  group_sync();
}

// v: the step-1 inputs x[t + A n2], read by the caller from buf[F(.)] itself
// (hence the group barrier before the first write).
template <int N, bool INV, class IDX>
__device__ __forceinline__ void fft4step_regs_map(double2 (&v)[16], double2* buf, int t,
                                                  const double2* __restrict__ tw4, IDX F) {
  constexpr int A = N / 16;
  dft16<INV>(v);
  if (t > 0) {
#pragma unroll
    for (int k2 = 1; k2 < 16; ++k2) {
      const double2 w = tw4[k2 * A + t];
      v[k2] = cmul(v[k2], INV ? conj(w) : w);
    }
  }
  group_sync();
#pragma unroll
  for (int k2 = 0; k2 < 16; ++k2) buf[F(t * 16 + (k2 ^ (t & 15)))] = v[k2];
  group_sync();
  constexpr int PER = 16 / A;
  double2 u[PER][A];
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) u[b][n1] = buf[F(n1 * 16 + (k2 ^ n1))];
    if constexpr (A == 16) dft16<INV>(u[b]);
    else if constexpr (A == 8) dft8<INV>(u[b]);
    else dft4<INV>(u[b][0], u[b][1], u[b][2], u[b][3]);
  }
  group_sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int k2 = t + b * A;
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) buf[F(k2 + 16 * k1)] = u[b][k1];
  }
  group_sync();
}

// Full N-point transform of buf (in shared memory) by TPF = N/16 threads.
// N <= 256: four-step (table layout tw4); N = 512: Stockham (plain W_N).
template <int N, bool INV>
__device__ __forceinline__ void fft(double2* buf, int t, const double2* __restrict__ tw) {
  constexpr int TPF = N / 16;
  if constexpr (N <= 256) {
    fft4step<N, INV>(buf, t, tw);
  } else {
    static_assert(N == 512, "unsupported FFT size");
    stage<512, 8, 1, INV, TPF>(buf, t, tw);
    stage<512, 8, 8, INV, TPF>(buf, t, tw);
    stage<512, 8, 64, INV, TPF>(buf, t, tw);
  }
}

}  // namespace fft
}  // namespace hb
