// context.cu -- C ABI (include/homfe_gpu.h): device context, material setup,
// preconditioner setup, the device-resident PCG loop and the linear Newton
// shell. Host code follows the reference control flow:
//   pcg_solve          proj/src/solver.cpp:50-97
//   PrecondManager     proj/src/solver.cpp:99-142
//   newton_solve       proj/src/solver.cpp:171-296
// The PCG iteration runs as one CUDA graph whose conditional WHILE node loops
// on the device until the stopping test of solver.cpp:88-91 fires, so the
// host never synchronises inside a solve.
#include <cufft.h>
#include <nccl.h>
#include <cub/cub.cuh>
#include <atomic>
#include <condition_variable>
#include <thread>
#include <mutex>
#include <map>

#include <algorithm>
#include <random>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/homfe_gpu.h"
#include "kernels.cuh"
#include "tables.hpp"

using namespace hb;

namespace {

thread_local std::string g_err;

struct CufftError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define HB_NCCL(expr)                                                                   \
  do {                                                                                  \
    ncclResult_t _r = (expr);                                                           \
    if (_r != ncclSuccess) throw CudaError(std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

#define HB_CUFFT(expr)                                                                  \
  do {                                                                                  \
    cufftResult _r = (expr);                                                            \
    if (_r != CUFFT_SUCCESS) throw CufftError(std::string(#expr) + " failed: " + std::to_string((int)_r)); \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return HOMFE_OK;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return HOMFE_VALIDATION;
  } catch (const NonConverged& e) {
    g_err = e.what();
    return HOMFE_NONCONVERGED;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return HOMFE_NUMERICAL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return HOMFE_DEVICE;
  } catch (const CufftError& e) {
    g_err = e.what();
    return HOMFE_DEVICE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HOMFE_DEVICE;
  }
}

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  HB_CUDA(cudaMalloc(&p, n * sizeof(T) + 16));
  return static_cast<T*>(p);
}

// Scratch device buffers of one call, freed on every exit path (exceptions
// included).
struct Scratch {
  std::vector<void*> bufs;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch() {
    for (void* p : bufs) cudaFree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    T* p = dalloc<T>(n > 0 ? n : 1);
    bufs.push_back(p);
    return p;
  }
};

}  // namespace

struct SimGroup {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0, generation = 0;
  std::vector<const void*> ptr;      // per rank: published buffer
  std::vector<double> red;           // per rank: reduction staging (<= 256 values)
  std::vector<uint64_t> ured;
};
struct homfe_ctx {
  int device = 0;
  Grid g{};
  StencilParams sp{};
  int nl = 0, ne = 0;
  int64_t nf = 0;
  cudaStream_t stream = nullptr, stream2 = nullptr;
  cufftHandle fwd = 0, inv = 0;
  // material
  int n_phases = 0;
  std::vector<double> catalog;      // n_phases x m x m col-major
  std::vector<int64_t> counts;      // pixels per phase
  uint8_t* d_phase = nullptr;
  double* d_ke = nullptr;
  double* d_fe = nullptr;
  double* d_cmat = nullptr;
  double* d_hexmat = nullptr;       // modal-basis material table (hexfast.cu)
  bool no_fast2d = false;           // HOMFE_FAST2D=0: generic 2-D element kernel
  double* d_tri = nullptr;          // TwoTriangles flux tables (quad2d.cu)
  // nonlinear (J2) path, j2.cu
  bool nonlinear = false;           // the catalog holds a J2 phase
  bool nl_op = false;               // apply_K is the tangent operator (inside newton_nl)
  bool graphs_nl = false;           // captured graphs hold the tangent operator
  std::vector<NLModel> models;
  NLModel* d_models = nullptr;
  double *d_g0 = nullptr, *d_gtr = nullptr, *d_tanc = nullptr, *d_sig = nullptr, *d_qs = nullptr,
         *d_tpart = nullptr;
  int* d_status = nullptr;
  bool sig_valid = false;           // d_sig holds the last solve's stress
  bool qt_ok = false;               // J2 operator on the modal hex kernel (all phases iso or J2)
  double* d_qtab = nullptr;         // per phase (linear flag, bulk, shear)
  // impulse-probed block preconditioner (probe.cu), node types per pixel > 1
  double2* d_blocks = nullptr;      // inverted blocks (nf x b x b)
  double2* d_blocks_raw = nullptr;  // K_ref_hat before inversion (reference_blocks hook)
  uint8_t* d_phase0 = nullptr;      // zero phase map for the reference operator
  NLModel* d_model0 = nullptr;
  double* d_cref = nullptr;
  // strain-based scheme (projection.cpp): quad-space unknown and CG vectors
  double *d_strain = nullptr, *d_sx = nullptr, *d_sr = nullptr, *d_sp = nullptr, *d_sap = nullptr,
         *d_scp = nullptr;
  bool hex_fast = false, hex_iso = false;
  // vectors
  double *d_x = nullptr, *d_r = nullptr, *d_p = nullptr, *d_ap = nullptr, *d_z = nullptr, *d_u = nullptr;
  double2* d_spec = nullptr;
  double* d_quad = nullptr;         // lazily allocated quad field (parity hooks)
  double4* d_tab[3] = {nullptr, nullptr, nullptr};
  // fused three-pass preconditioner (fftfused.cu)
  bool fused = false;
  FusedFft ff{};
  double2* d_tw = nullptr;          // W_{n1} then W_{n0}
  double2* d_spec2 = nullptr;       // second spectrum buffer of the fused passes
  // reference
  SpecParams spp{};
  bool have_ref = false;
  std::vector<double> c_ref;
  // PrecondManager state (solver.hpp:105-129): the context is the caller's
  // manager; it persists across solves (load steps) until
  // homfe_gpu_precond_reset (a new PrecondManager)
  bool pm_valid = false;
  std::vector<double> pm_mean;      // volume-averaged tangent at the last assembly
  std::vector<double> pm_cref;      // reference used by the last assembly
  // scalars
  PcgState* d_st = nullptr;
  PcgState* h_st = nullptr;         // pinned
  double* d_partials = nullptr;
  double* d_scal = nullptr;         // small scratch (final sums)
  double* h_scal = nullptr;         // pinned
  double* d_hist = nullptr;
  int hist_cap = 0;
  double* d_e = nullptr;
  // graph of the whole PCG (init + device WHILE loop + mean removal)
  cudaGraphExec_t pcg_exec = nullptr;
  double graph_eta = -1.0;
  int graph_itmax = -1;
  bool use_while = true;
  bool small2d = false;            // persistent one-cluster PCG (small2d.cu) allowed
  double2* d_tw256 = nullptr;      // its W_256 four-step table
  bool body_eager = false;
  cudaGraphExec_t body_exec = nullptr;  // fallback: one iteration per launch
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches = 0;
  // slab decomposition (homfe_gpu_create_dist): NCCL communicator, halo planes
  bool dist = false;
  ncclComm_t comm = nullptr;
  SimGroup* sim = nullptr;          // in-process slab transport (tests on one GPU), see sim_*
  double* d_hlo = nullptr;          // plane z0-1 of the vector being stenciled, [c][plane]
  double* d_hhi = nullptr;          // plane z0+nz
  uint8_t* d_ph_lo = nullptr;       // phase plane z0-1
  double* d_red = nullptr;          // globally reduced scalars
  double2* d_spec_r = nullptr;      // all-to-all receive buffers of the fused passes
  double2* d_spec2_r = nullptr;
  // peer pull (slab mode over NVLink): passes 2 / 3 and the K halo planes read
  // the peers' fields in place (IPC mappings, or the in-process transport's
  // own pointers); the all-to-alls and halo sends become stream barriers
  bool peer = false;
  double* peer_p[FusedFft::kMaxPeers] = {};  // every rank's p (d_p)
  void* peer_a[FusedFft::kMaxPeers] = {};    // every rank's T (fused) / W (slab spectra)
  void* peer_b[FusedFft::kMaxPeers] = {};    // every rank's T2 (fused) / S (slab spectra)
  // slab spectra for plane sizes outside the fused passes (slabfft.cu)
  bool slab_fft = false;
  SlabDims sd{};
  cufftHandle p2f = 0, p2i = 0, p1 = 0;      // 2-D D2Z / Z2D of the local planes; 1-D Z2Z along axis 0
  double2* d_S = nullptr;                    // [c][n0l][n1][nh]
  double2* d_W = nullptr;                    // [c][n0][n1l][nh]
  double2* d_send = nullptr;                 // all-to-all chunks (push == 0)
  double2* d_recv = nullptr;
  std::vector<void*> ipc_open;               // IPC mappings to close
  double* d_bar = nullptr;                   // barrier all-reduce scratch

  // single-process multi-GPU context (homfe_gpu_create_multi): the rank
  // contexts of the slab decomposition, one host thread each per call
  std::vector<homfe_ctx*> ranks;
  int64_t mp_np = 0, mp_nq = 0, mp_nf = 0;  // global sizes
  int mp_c = 0, mp_m = 0;

  int64_t nvec() const { return (int64_t)g.c * g.nn * g.np; }
  int64_t nodes() const { return (int64_t)g.nn * g.np; }
};

namespace {

void destroy_graphs(homfe_ctx* c) {
  if (c->pcg_exec) cudaGraphExecDestroy(c->pcg_exec);
  if (c->body_exec) cudaGraphExecDestroy(c->body_exec);
  c->pcg_exec = nullptr;
  c->body_exec = nullptr;
  c->graph_eta = -1.0;
  c->graph_itmax = -1;
}

void sync(homfe_ctx* c) { HB_CUDA(cudaStreamSynchronize(c->stream)); }

// ---- in-process slab transport (tests) ------------------------------------
// W contexts of one process on one device, driven by W host threads, with the
// collectives done as device-to-device copies between host barriers. The
// kernels never wait on each other on the device (all waiting is on the
// host), so this validates the slab layouts, halos and reduction order of
// the multi-GPU path on one GPU. Selected by an id blob starting "HBSIMGRP".
static std::mutex g_sim_mu;
static std::map<uint64_t, std::shared_ptr<SimGroup>> g_sim;

void sim_barrier(SimGroup* g) {
  std::unique_lock<std::mutex> lk(g->m);
  const int gen = g->generation;
  if (++g->arrived == g->world) {
    g->arrived = 0;
    ++g->generation;
    g->cv.notify_all();
  } else {
    g->cv.wait(lk, [&] { return g->generation != gen; });
  }
}

// publish my pointer, wait for everyone, run `body` (pulls from peers), wait again
template <class F>
void sim_exchange(homfe_ctx* c, const void* mine, F body) {
  SimGroup* G = c->sim;
  HB_CUDA(cudaStreamSynchronize(c->stream));
  G->ptr[c->g.rank] = mine;
  sim_barrier(G);
  body(G);
  HB_CUDA(cudaStreamSynchronize(c->stream));
  sim_barrier(G);
}

void sim_halo(homfe_ctx* c, const void* v, size_t elem, int comps, int64_t comp_stride, void* lo, void* hi) {
  const Grid& g = c->g;
  const int prev = (g.rank - 1 + g.world) % g.world, next = (g.rank + 1) % g.world;
  const size_t plane = (size_t)g.n1 * g.n2;
  sim_exchange(c, v, [&](SimGroup* G) {
    for (int k = 0; k < comps; ++k) {
      const char* pv = static_cast<const char*>(G->ptr[prev]) + (size_t)k * comp_stride * elem;
      const char* nx = static_cast<const char*>(G->ptr[next]) + (size_t)k * comp_stride * elem;
      if (lo)
        HB_CUDA(cudaMemcpyAsync(static_cast<char*>(lo) + k * plane * elem, pv + (size_t)(g.n0 - 1) * plane * elem,
                                plane * elem, cudaMemcpyDeviceToDevice, c->stream));
      if (hi)
        HB_CUDA(cudaMemcpyAsync(static_cast<char*>(hi) + k * plane * elem, nx, plane * elem,
                                cudaMemcpyDeviceToDevice, c->stream));
    }
  });
}

void sim_all_to_all(homfe_ctx* c, const double2* send, double2* recv, int64_t chunk) {
  sim_exchange(c, send, [&](SimGroup* G) {
    for (int q = 0; q < c->g.world; ++q)
      HB_CUDA(cudaMemcpyAsync(recv + q * chunk, static_cast<const double2*>(G->ptr[q]) + (int64_t)c->g.rank * chunk,
                              chunk * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  });
}

// sum over ranks in rank order (a fixed order, like NCCL's for a given communicator)
template <class T>
void sim_allreduce(homfe_ctx* c, T* dptr, int n) {
  SimGroup* G = c->sim;
  std::vector<T> mine(n);
  HB_CUDA(cudaMemcpyAsync(mine.data(), dptr, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
  {
    std::lock_guard<std::mutex> lk(G->m);
    for (int i = 0; i < n; ++i) {
      if constexpr (std::is_same<T, double>::value) G->red[(size_t)c->g.rank * 256 + i] = mine[i];
      else G->ured[(size_t)c->g.rank * 256 + i] = mine[i];
    }
  }
  sim_barrier(G);
  std::vector<T> tot(n, T(0));
  for (int r = 0; r < G->world; ++r)
    for (int i = 0; i < n; ++i) {
      if constexpr (std::is_same<T, double>::value) tot[i] += G->red[(size_t)r * 256 + i];
      else tot[i] += G->ured[(size_t)r * 256 + i];
    }
  sim_barrier(G);
  HB_CUDA(cudaMemcpyAsync(dptr, tot.data(), n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  HB_CUDA(cudaStreamSynchronize(c->stream));
}

// ---- slab-mode exchanges (NCCL over NVLink / NVSwitch) --------------------
// halo planes of a component-planar vector: my first plane goes to the
// previous rank (its upper halo), my last plane to the next rank (its lower
// halo); periodic ring, so world == 1 exchanges with itself.
void exchange_halo(homfe_ctx* c, const double* v, cudaStream_t s) {
  const Grid& g = c->g;
  if (c->sim) {
    sim_halo(c, v, sizeof(double), g.c, g.np, c->d_hlo, c->d_hhi);
    return;
  }
  const int prev = (g.rank - 1 + g.world) % g.world, next = (g.rank + 1) % g.world;
  const size_t plane = (size_t)g.n1 * g.n2;
  HB_NCCL(ncclGroupStart());
  for (int k = 0; k < g.c; ++k) {
    const double* base = v + (int64_t)k * g.np;
    HB_NCCL(ncclSend(base, plane, ncclDouble, prev, c->comm, s));
    HB_NCCL(ncclSend(base + (int64_t)(g.n0 - 1) * plane, plane, ncclDouble, next, c->comm, s));
    HB_NCCL(ncclRecv(c->d_hhi + k * plane, plane, ncclDouble, next, c->comm, s));
    HB_NCCL(ncclRecv(c->d_hlo + k * plane, plane, ncclDouble, prev, c->comm, s));
  }
  HB_NCCL(ncclGroupEnd());
}

// swap peer chunks of a fused-pass spectrum (planes <-> k1 rows)
void all_to_all(homfe_ctx* c, const double2* send, double2* recv, int64_t chunk, cudaStream_t s) {
  if (c->g.world == 1) {
    if (send != recv)
      HB_CUDA(cudaMemcpyAsync(recv, send, chunk * sizeof(double2), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (c->sim) {
    sim_all_to_all(c, send, recv, chunk);
    return;
  }
  HB_NCCL(ncclGroupStart());
  for (int q = 0; q < c->g.world; ++q) {
    HB_NCCL(ncclSend(send + q * chunk, 2 * chunk, ncclDouble, q, c->comm, s));
    HB_NCCL(ncclRecv(recv + q * chunk, 2 * chunk, ncclDouble, q, c->comm, s));
  }
  HB_NCCL(ncclGroupEnd());
}

// Stream barrier over the slab ranks: on return (in stream order) every
// rank's preceding work is complete. NCCL: a 1-element all-reduce (its
// completion needs every rank's contribution, queued after that rank's
// preceding kernels); in-process: host barrier after a stream drain.
void peer_barrier(homfe_ctx* c, cudaStream_t s) {
  if (c->sim) {
    HB_CUDA(cudaStreamSynchronize(s));
    sim_barrier(c->sim);
    return;
  }
  HB_NCCL(ncclAllReduce(c->d_bar, c->d_bar, 1, ncclDouble, ncclSum, c->comm, s));
}

// pass 1 -> pass 2: all-to-all of T, or (peer pull) a barrier after which
// pass 2 reads every peer's T chunk for this rank over NVLink
void xfer_t(homfe_ctx* c, cudaStream_t s) {
  if (c->peer) peer_barrier(c, s);
  else all_to_all(c, c->ff.T, c->ff.Trecv, c->ff.chunk_t(), s);
}
// pass 2 -> pass 3; `synced`: an all-reduce was queued after pass 2 already
void xfer_t2(homfe_ctx* c, cudaStream_t s, bool synced) {
  if (c->peer) {
    if (!synced) peer_barrier(c, s);
  } else {
    all_to_all(c, c->ff.T2, c->ff.T2recv, c->ff.chunk_t2(), s);
  }
}

// partials -> d_red[slot..slot+n): fixed-order local sum, then a sum over
// ranks (NCCL's fixed ring/tree order: identical on every rank and run).
double* reduce_global(homfe_ctx* c, int nvals, int slot, cudaStream_t s) {
  launch_final_sum(c->d_partials, kRedBlocks, nvals, c->d_red + slot, s);
  if (c->sim) sim_allreduce<double>(c, c->d_red + slot, nvals);
  else HB_NCCL(ncclAllReduce(c->d_red + slot, c->d_red + slot, nvals, ncclDouble, ncclSum, c->comm, s));
  return c->d_red + slot;
}

// Deterministic reduction of kRedBlocks partials (nvals each) to host.
void reduce_to_host(homfe_ctx* c, int nvals, double* out) {
  if (c->dist) {
    reduce_global(c, nvals, 0, c->stream);
    HB_CUDA(cudaMemcpyAsync(c->h_scal, c->d_red, nvals * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    std::memcpy(out, c->h_scal, nvals * sizeof(double));
    return;
  }
  launch_final_sum(c->d_partials, kRedBlocks, nvals, c->d_scal, c->stream);
  HB_CUDA(cudaMemcpyAsync(c->h_scal, c->d_scal, nvals * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  std::memcpy(out, c->h_scal, nvals * sizeof(double));
}

void fft_forward(homfe_ctx* c, const double* in, cudaStream_t s) {
  HB_CUFFT(cufftSetStream(c->fwd, s));
  HB_CUFFT(cufftExecD2Z(c->fwd, const_cast<double*>(in), reinterpret_cast<cufftDoubleComplex*>(c->d_spec)));
}

void fft_inverse(homfe_ctx* c, double* out, cudaStream_t s) {
  HB_CUFFT(cufftSetStream(c->inv, s));
  HB_CUFFT(cufftExecZ2D(c->inv, reinterpret_cast<cufftDoubleComplex*>(c->d_spec), out));
}

// ---- slab spectra for any plane size (slabfft.cu) ------------------------
// forward: 2-D r2c of the local planes, transpose to k1 rows (pushed into the
// owners' W, or all-to-all), 1-D transform along axis 0 per component
void slab_forward(homfe_ctx* c, const double* in, cudaStream_t s) {
  const SlabDims& d = c->sd;
  HB_CUFFT(cufftSetStream(c->p2f, s));
  HB_CUFFT(cufftExecD2Z(c->p2f, const_cast<double*>(in), reinterpret_cast<cufftDoubleComplex*>(c->d_S)));
  double2* dst[FusedFft::kMaxPeers];
  if (c->peer || d.world == 1) {  // world 1: the "transpose" lands in the own W
    for (int q = 0; q < d.world; ++q) dst[q] = static_cast<double2*>(c->peer_a[q]);
    launch_slab_pack_fwd(d, c->d_S, dst, 1, s);
    if (c->peer) peer_barrier(c, s);
  } else {
    for (int q = 0; q < d.world; ++q) dst[q] = c->d_send + q * d.chunk();
    launch_slab_pack_fwd(d, c->d_S, dst, 0, s);
    all_to_all(c, c->d_send, c->d_recv, d.chunk(), s);
    launch_slab_unpack_fwd(d, c->d_recv, c->d_W, s);
  }
  HB_CUFFT(cufftSetStream(c->p1, s));
  const int64_t per = (int64_t)d.n0 * d.n1l * d.nh;
  for (int k = 0; k < d.c; ++k) {
    auto* w = reinterpret_cast<cufftDoubleComplex*>(c->d_W + k * per);
    HB_CUFFT(cufftExecZ2Z(c->p1, w, w, CUFFT_FORWARD));
  }
  c->launches += 3 + d.c;
}

// z_hat = K_ref_hat^+ r_hat / N_p on this rank's k1 rows (global frequencies)
void slab_solve(homfe_ctx* c, const PcgState* st, double* partials, cudaStream_t s) {
  SpecParams p = c->spp;
  p.nf = (int64_t)c->sd.n0 * c->sd.n1l * c->sd.nh;
  p.n1r = c->sd.n1l;
  p.k1off = c->sd.me * c->sd.n1l;
  if (c->g.d == 2) p.nh = c->sd.n1l;  // frequencies (i0, k1off + k1l), columns >= nhv are padding
  launch_spectral(p, c->d_W, st, partials, s);
  c->launches += 1;
}

// inverse: 1-D along axis 0, transpose back to planes, 2-D c2r
void slab_inverse(homfe_ctx* c, double* out, cudaStream_t s) {
  const SlabDims& d = c->sd;
  HB_CUFFT(cufftSetStream(c->p1, s));
  const int64_t per = (int64_t)d.n0 * d.n1l * d.nh;
  for (int k = 0; k < d.c; ++k) {
    auto* w = reinterpret_cast<cufftDoubleComplex*>(c->d_W + k * per);
    HB_CUFFT(cufftExecZ2Z(c->p1, w, w, CUFFT_INVERSE));
  }
  double2* dst[FusedFft::kMaxPeers];
  if (c->peer || d.world == 1) {
    // peers finished reading their S (their pack_fwd) before the forward barrier
    for (int q = 0; q < d.world; ++q) dst[q] = static_cast<double2*>(c->peer_b[q]);
    launch_slab_pack_inv(d, c->d_W, dst, 1, s);
    if (c->peer) peer_barrier(c, s);
  } else {
    for (int q = 0; q < d.world; ++q) dst[q] = c->d_send + q * d.chunk();
    launch_slab_pack_inv(d, c->d_W, dst, 0, s);
    all_to_all(c, c->d_send, c->d_recv, d.chunk(), s);
    launch_slab_unpack_inv(d, c->d_recv, c->d_S, s);
  }
  HB_CUFFT(cufftSetStream(c->p2i, s));
  HB_CUFFT(cufftExecZ2D(c->p2i, reinterpret_cast<cufftDoubleComplex*>(c->d_S), out));
  c->launches += 3 + d.c;
}

// z = M^-1 r; optional Parseval r.z partials.
void precond_apply(homfe_ctx* c, const double* r, double* z, const PcgState* st, double* partials,
                   cudaStream_t s) {
  if (c->g.nn > 1) {
    // apply_preconditioner (precond.cpp:126-162): all slices D2Z, block
    // matvec per frequency (1/N_p folded in), all slices Z2D
    fft_forward(c, r, s);
    launch_probe_apply(c->d_spec, c->d_blocks, c->nf, c->g.c * c->g.nn, 1.0 / (double)c->g.np, s);
    fft_inverse(c, z, s);
    if (partials) launch_dot_partials(r, z, c->nvec(), partials, s);
    c->launches += 4;
    return;
  }
  if (c->slab_fft) {
    slab_forward(c, r, s);
    slab_solve(c, st, partials, s);
    slab_inverse(c, z, s);
    return;
  }
  if (c->fused) {
    fused_forward(c->ff, c->spp, const_cast<double*>(r), nullptr, nullptr, partials, s, 1);
    xfer_t(c, s);
    fused_forward(c->ff, c->spp, const_cast<double*>(r), nullptr, nullptr, partials, s, 2);
    xfer_t2(c, s, false);
    fused_inverse(c->ff, nullptr, nullptr, z, nullptr, 0, s);
    c->launches += 3;
    return;
  }
  fft_forward(c, r, s);
  launch_spectral(c->spp, c->d_spec, st, partials, s);
  fft_inverse(c, z, s);
  c->launches += 3;
}

NLArgs nl_args(homfe_ctx* c, const double* u) {
  NLArgs a{};
  a.u = u;
  a.e = c->d_e;
  a.phase = c->d_phase;
  a.models = c->d_models;
  a.cmat = c->d_cmat;
  a.g0 = c->d_g0;
  a.g_trial = c->d_gtr;
  a.tanc = c->d_tanc;
  a.sig = c->d_sig;
  a.partials = c->d_tpart;
  a.status = c->d_status;
  a.width = c->nonlinear ? 7 : 0;
  return a;
}

void apply_K(homfe_ctx* c, const double* u, double* out, const double* fe, double scale, double* partials,
             const PcgState* st, cudaStream_t s) {
  if (c->nl_op && c->qt_ok && c->hex_fast) {
    // J2 tangent operator on the modal hex kernel (per-Gauss-point compact tangents)
    ElemArgs ea{u, nullptr, nullptr, nullptr, out, c->d_phase, c->d_ke, c->n_phases, nullptr, scale, partials, st};
    if (launch_hex_fast_qt(c->g, ea, c->d_qtab, c->d_tanc, s)) {
      c->launches += 1;
      return;
    }
  }
  if (c->nl_op || c->g.nn > 1) {  // two node types: the quadrature-point path
    // tangent operator of the current Newton state: sigma_q = C_q (D u)_q,
    // then the weighted divergence (operators.cpp:197-257 in two passes)
    NLArgs a = nl_args(c, u);
    a.sig = c->d_qs;
    launch_tan_stress(c->g, c->sp, a, st, s);
    launch_divergence(c->g, c->sp, c->d_qs, true, out, s);
    const int64_t n = c->nvec();
    if (scale != 1.0) launch_scale(out, scale, n, s);
    if (partials) launch_dot_partials(u, out, n, partials, s);
    c->launches += 3;
    return;
  }
  ElemArgs a{u, c->d_hlo, c->d_hhi, c->d_ph_lo, out, c->d_phase, c->d_ke, c->n_phases, fe, scale, partials, st};
  if (c->peer && u == c->d_p) {
    // halo planes read in place from the neighbours' p (after a barrier: their
    // last write of p, pass 3 or an upload, is complete)
    const Grid& g = c->g;
    const int prev = (g.rank - 1 + g.world) % g.world, next = (g.rank + 1) % g.world;
    peer_barrier(c, s);
    a.halo_lo = c->peer_p[prev] + (int64_t)(g.n0 - 1) * g.n1 * g.n2;
    a.halo_hi = c->peer_p[next];
    a.halo_cs = g.np;
  } else if (c->dist) {
    exchange_halo(c, u, s);
  }
  if (c->hex_fast) launch_hex_fast(c->g, a, c->d_hexmat, c->hex_iso, s);
  else if (elem2d_eligible(c->g) && !c->no_fast2d) launch_elem2d(c->g, a, c->d_tri, s);
  else launch_apply_elem(c->g, a, s);
  c->launches += 1;
}

void require_material(homfe_ctx* c) {
  if (c->n_phases <= 0) throw ValidationError("materials: no material map set");
}
void require_reference(homfe_ctx* c) {
  if (!c->have_ref) throw ValidationError("apply_preconditioner: blocks are not inverted");
}

// assemble_reference + invert_blocks (precond.cpp:44-124) for the analytic
// symbol: validate C_ref, load the tensor, run the singularity test.
void ensure_nl_buffers(homfe_ctx* c);

// assemble_reference + invert_blocks (precond.cpp:44-124) by impulse probing,
// for stencils with two node types (complex Hermitian blocks, probe.cu).
void probe_assemble(homfe_ctx* c, const double* cref) {
  const int m = c->g.m, b = c->g.c * c->g.nn;
  const int64_t np = c->g.np, nv = c->nvec();
  ensure_nl_buffers(c);
  if (!c->d_blocks) {
    c->d_blocks = dalloc<double2>((size_t)c->nf * b * b);
    c->d_blocks_raw = dalloc<double2>((size_t)c->nf * b * b);
    c->d_phase0 = dalloc<uint8_t>(np);
    HB_CUDA(cudaMemset(c->d_phase0, 0, np));
    c->d_model0 = reinterpret_cast<NLModel*>(dalloc<double>(sizeof(NLModel) / sizeof(double) + 1));
    const NLModel lin{0, 0.0, 0.0, 0.0, 0.0};
    HB_CUDA(cudaMemcpy(c->d_model0, &lin, sizeof(NLModel), cudaMemcpyHostToDevice));
    c->d_cref = dalloc<double>(36);
  }
  HB_CUDA(cudaMemcpyAsync(c->d_cref, cref, (size_t)m * m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  NLArgs a{};
  a.u = c->d_p;
  a.phase = c->d_phase0;
  a.models = c->d_model0;
  a.cmat = c->d_cref;
  a.sig = c->d_qs;
  const double one = 1.0;
  for (int col = 0; col < b; ++col) {
    // one impulse per (component, node type) slice -> one block column
    HB_CUDA(cudaMemsetAsync(c->d_p, 0, nv * sizeof(double), c->stream));
    HB_CUDA(cudaMemcpyAsync(c->d_p + (int64_t)col * np, &one, sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch_tan_stress(c->g, c->sp, a, nullptr, c->stream);
    launch_divergence(c->g, c->sp, c->d_qs, true, c->d_ap, c->stream);
    fft_forward(c, c->d_ap, c->stream);
    launch_probe_store(c->d_spec, b, c->nf, col, c->d_blocks_raw, c->stream);
  }
  HB_CUDA(cudaMemcpyAsync(c->d_blocks, c->d_blocks_raw, (size_t)c->nf * b * b * sizeof(double2),
                          cudaMemcpyDeviceToDevice, c->stream));
  HB_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(int), c->stream));
  launch_probe_invert(c->d_blocks, c->nf, b, c->g.nn, c->d_status, c->stream);
  int st = 0;
  HB_CUDA(cudaMemcpyAsync(&st, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (st == 1) throw NumericalError("invert_blocks: singular zero-frequency block");
  if (st == 2) throw NumericalError("invert_blocks: singular non-zero-frequency block");
}

void set_reference(homfe_ctx* c, const double* cref) {
  const int m = c->g.m, d = c->g.d;
  check_spd(cref, m, "reference tangent");
  if (c->g.nn > 1) {
    c->have_ref = false;
    destroy_graphs(c);
    probe_assemble(c, cref);
    c->c_ref.assign(cref, cref + m * m);
    c->have_ref = true;
    return;
  }
  SpecParams& p = c->spp;
  if (c->g.c == 1) {
    for (int j = 0; j < d; ++j)
      for (int l = 0; l < d; ++l) p.A[j * d + l] = cref[l * d + j];
  } else {
    mandel_to_tensor(cref, d, p.A);
  }
  // isotropic reference: closed-form symbol (spectral.cuh)
  {
    p.iso = 0;
    auto C = [&](int i, int j) { return cref[j * m + i]; };
    if (c->g.c == 1) {
      bool ok = true;
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
          if (C(i, j) != (i == j ? C(0, 0) : 0.0)) ok = false;
      if (ok) {
        p.iso = 1;
        p.mu = C(0, 0);
      }
    } else {
      const double lam = C(0, 1), twomu = m == 6 ? C(3, 3) : C(2, 2);
      const double tol = 8e-16 * (std::fabs(lam) + std::fabs(twomu));
      bool ok = true;
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
          const bool nn = i < d && j < d;
          const double want = nn ? (i == j ? lam + twomu : lam) : (i == j ? twomu : 0.0);
          if (std::fabs(C(i, j) - want) > tol) ok = false;
        }
      if (ok) {
        p.iso = 1;
        p.lam = lam;
        p.mu = 0.5 * twomu;
      }
    }
    if (const char* e = std::getenv("HOMFE_ISO_SYMBOL")) if (e[0] == '0') p.iso = 0;
  }
  c->c_ref.assign(cref, cref + m * m);
  destroy_graphs(c);  // spectral kernel nodes hold the symbol parameters by value
  launch_symbol_check(p, c->d_partials, c->stream);
  double bad = 0.0;
  reduce_to_host(c, 1, &bad);
  if (bad != 0.0) {
    c->have_ref = false;
    throw NumericalError("invert_blocks: singular non-zero-frequency block");
  }
  c->have_ref = true;
}

// ---------------------------------------------------------------- PCG graph
void capture_init(homfe_ctx* c, cudaStream_t s) {
  const int64_t n = c->nvec();
  HB_CUDA(cudaMemsetAsync(c->d_x, 0, n * sizeof(double), s));
  if (c->fused) {
    fused_forward(c->ff, c->spp, c->d_r, nullptr, nullptr, c->d_partials, s, 1);
    xfer_t(c, s);
    fused_forward(c->ff, c->spp, c->d_r, nullptr, nullptr, c->d_partials, s, 2);
    if (c->dist) launch_pcg_init(c->d_st, reduce_global(c, 1, 1, s), c->d_hist, s, 1);
    else launch_pcg_init(c->d_st, c->d_partials, c->d_hist, s);
    xfer_t2(c, s, c->dist);
    fused_inverse(c->ff, c->d_p, nullptr, nullptr, nullptr, 1, s);  // p = z_0
    return;
  }
  precond_apply(c, c->d_r, c->d_z, nullptr, c->d_partials, s);
  if (c->dist) launch_pcg_init(c->d_st, reduce_global(c, 1, 1, s), c->d_hist, s, 1);
  else launch_pcg_init(c->d_st, c->d_partials, c->d_hist, s);
  HB_CUDA(cudaMemcpyAsync(c->d_p, c->d_z, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

void remove_means_on(homfe_ctx* c, double* v, cudaStream_t s) {
  const int64_t nodes = c->nodes();
  launch_comp_sums(v, c->g.c, nodes, c->d_partials, s);
  if (c->dist) {
    launch_sub_means(v, c->g.c, nodes, reduce_global(c, c->g.c, 4, s), s, (double)c->g.npg);
  } else {
    launch_final_sum(c->d_partials, kRedBlocks, c->g.c, c->d_scal, s);
    launch_sub_means(v, c->g.c, nodes, c->d_scal, s);
  }
}

void capture_tail(homfe_ctx* c, cudaStream_t s) {
  // x.remove_component_means() (solver.cpp:95)
  remove_means_on(c, c->d_x, s);
}

void body_sequence(homfe_ctx* c, cudaStream_t s, bool cond, cudaGraphConditionalHandle h) {
  const int64_t n = c->nvec();
  if (c->fused) {
    // K p (+ p.Ap) -> alpha -> [r -= alpha Ap, F_planes r] -> a2a -> [F_0, K^-1,
    // F_0^-1, r.z] -> beta -> a2a -> [F_planes^-1, x += alpha p, p = z + beta p]
    apply_K(c, c->d_p, c->d_ap, nullptr, 1.0, c->d_partials, c->d_st, s);
    if (c->dist) launch_pcg_alpha(c->d_st, reduce_global(c, 1, 2, s), s, 1);
    else launch_pcg_alpha(c->d_st, c->d_partials, s);
    fused_forward(c->ff, c->spp, c->d_r, c->d_ap, c->d_st, c->d_partials, s, 1);
    xfer_t(c, s);
    fused_forward(c->ff, c->spp, c->d_r, c->d_ap, c->d_st, c->d_partials, s, 2);
    if (c->dist) launch_pcg_beta(c->d_st, reduce_global(c, 1, 3, s), c->d_hist, s, 1);
    else if (cond) launch_pcg_beta_cond(c->d_st, c->d_partials, c->d_hist, h, s);
    else launch_pcg_beta(c->d_st, c->d_partials, c->d_hist, s);
    xfer_t2(c, s, c->dist);
    fused_inverse(c->ff, c->d_p, c->d_x, nullptr, c->d_st, 0, s);
    return;
  }
  if (c->slab_fft) {
    // slab spectra for other plane sizes: the cuFFT-path sequence with the
    // scalars reduced over the ranks
    apply_K(c, c->d_p, c->d_ap, nullptr, 1.0, c->d_partials, c->d_st, s);
    launch_pcg_alpha(c->d_st, reduce_global(c, 1, 2, s), s, 1);
    launch_update_r(c->d_r, c->d_ap, n, c->d_st, s);
    slab_forward(c, c->d_r, s);
    slab_solve(c, c->d_st, c->d_partials, s);
    launch_pcg_beta(c->d_st, reduce_global(c, 1, 3, s), c->d_hist, s, 1);
    slab_inverse(c, c->d_z, s);
    launch_update_xp(c->d_x, c->d_p, c->d_z, n, c->d_st, s);
    return;
  }
  apply_K(c, c->d_p, c->d_ap, nullptr, 1.0, c->d_partials, c->d_st, s);
  launch_pcg_alpha(c->d_st, c->d_partials, s);
  launch_update_r(c->d_r, c->d_ap, n, c->d_st, s);
  if (c->g.nn > 1) {
    // probed blocks: z = M^-1 r, then r.z in real space
    precond_apply(c, c->d_r, c->d_z, c->d_st, c->d_partials, s);
    launch_pcg_beta(c->d_st, c->d_partials, c->d_hist, s);
  } else {
    fft_forward(c, c->d_r, s);
    launch_spectral(c->spp, c->d_spec, c->d_st, c->d_partials, s);
    launch_pcg_beta(c->d_st, c->d_partials, c->d_hist, s);
    fft_inverse(c, c->d_z, s);
  }
  if (cond) launch_update_xp_cond(c->d_x, c->d_p, c->d_z, n, c->d_st, h, s);
  else launch_update_xp(c->d_x, c->d_p, c->d_z, n, c->d_st, s);
}

void write_state(homfe_ctx* c, double eta, int it_max, int active = 0) {
  std::memset(c->h_st, 0, sizeof(PcgState));
  c->h_st->eta = eta;
  c->h_st->it_max = it_max;
  c->h_st->active = active;
  HB_CUDA(cudaMemcpyAsync(c->d_st, c->h_st, sizeof(PcgState), cudaMemcpyHostToDevice, c->stream));
}

bool build_while_graph(homfe_ctx* c) {
  cudaStream_t s = c->stream;
  cudaGraph_t graph = nullptr;
  HB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  bool ok = true;
  try {
    capture_init(c, s);
    cudaStreamCaptureStatus status;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    HB_CUDA(cudaStreamGetCaptureInfo(s, &status, nullptr, &cg, &deps, &ndeps));
    cudaGraphConditionalHandle h;
    HB_CUDA(cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault));
    launch_set_while(h, c->d_st, s);
    HB_CUDA(cudaStreamGetCaptureInfo(s, &status, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    HB_CUDA(cudaGraphAddNode(&cnode, cg, deps, ndeps, &cp));
    HB_CUDA(cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    HB_CUDA(cudaStreamBeginCaptureToGraph(c->stream2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    try {
      body_sequence(c, c->stream2, true, h);
    } catch (...) {
      cudaGraph_t tmp;
      cudaStreamEndCapture(c->stream2, &tmp);
      throw;
    }
    cudaGraph_t body_out;
    HB_CUDA(cudaStreamEndCapture(c->stream2, &body_out));
    capture_tail(c, s);
  } catch (const std::exception& e) {
    g_err = e.what();
    ok = false;
  }
  cudaError_t end = cudaStreamEndCapture(s, &graph);
  if (!ok || end != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return false;
  }
  cudaError_t inst = cudaGraphInstantiate(&c->pcg_exec, graph, 0);
  cudaGraphDestroy(graph);
  if (inst != cudaSuccess) {
    cudaGetLastError();
    c->pcg_exec = nullptr;
    return false;
  }
  return true;
}

void build_body_graph(homfe_ctx* c) {
  cudaStream_t s = c->stream;
  cudaGraph_t graph = nullptr;
  HB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    body_sequence(c, s, false, 0);
  } catch (...) {
    cudaStreamEndCapture(s, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  HB_CUDA(cudaStreamEndCapture(s, &graph));
  HB_CUDA(cudaGraphInstantiate(&c->body_exec, graph, 0));
  cudaGraphDestroy(graph);
}

struct PcgResult {
  int iterations = 0;
  bool converged = false;
  double device_ms = 0.0;
  double last_history = 0.0;
};

// pcg_solve with r = b already in d_r; x lands in d_x (mean-free).
// obs (nullable): IterateObserver of pcg_solve (solver.cpp:87), called with
// a host copy of x_k after every iteration; forces the host-driven loop of
// one-iteration graphs (a debugging / inspection mode, not the fast path).
PcgResult run_pcg(homfe_ctx* c, double eta, int it_max, double* h_history,
                  homfe_iterate_observer obs = nullptr, void* obs_user = nullptr) {
  if (it_max + 1 > c->hist_cap) {
    destroy_graphs(c);  // graphs capture the history pointer
    if (c->d_hist) cudaFree(c->d_hist);
    c->hist_cap = it_max + 1;
    c->d_hist = dalloc<double>(c->hist_cap);
  }
  write_state(c, eta, it_max);
  HB_CUDA(cudaEventRecord(c->ev0, c->stream));
  bool ran = false;
  if (c->small2d && !obs && !c->nl_op && c->have_ref && small2d_eligible(c->g, c->n_phases)) {
    // the whole loop (init, iterations) in one persistent cluster
    ran = launch_pcg_small2d(c->spp, c->d_x, c->d_r, c->d_p, c->d_phase, c->d_tri, c->n_phases, c->d_tw256,
                             c->d_st, c->d_hist, c->stream);
    if (ran) {
      capture_tail(c, c->stream);
      c->launches += 4;
    } else {
      c->small2d = false;
    }
  }
  if (ran) {
  } else if (c->use_while) {
    if (!c->pcg_exec) {
      if (!build_while_graph(c)) {
        c->use_while = false;  // fall back to a host-driven loop of one-iteration graphs
      }
    }
  }
  if (ran) {
  } else if (c->use_while && !obs) {
    HB_CUDA(cudaGraphLaunch(c->pcg_exec, c->stream));
  } else {
    capture_init(c, c->stream);
    if (!c->body_exec && !c->body_eager) {
      try {
        build_body_graph(c);
      } catch (const std::exception&) {
        c->body_eager = true;  // e.g. collectives that cannot be captured
        cudaGetLastError();
      }
    }
    HB_CUDA(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    int launched = 0;
    int batch = 1;
    std::vector<double> hx(obs ? c->nvec() : 0);
    while (!c->h_st->done && launched < it_max) {
      const int it_before = c->h_st->it;
      for (int i = 0; i < batch && launched < it_max; ++i, ++launched) {
        if (c->body_exec) HB_CUDA(cudaGraphLaunch(c->body_exec, c->stream));
        else body_sequence(c, c->stream, false, 0);
      }
      HB_CUDA(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
      if (obs) HB_CUDA(cudaMemcpyAsync(hx.data(), c->d_x, hx.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                       c->stream));
      sync(c);
      if (c->h_st->status == 4) break;
      if (obs && c->h_st->it > it_before) obs(obs_user, c->h_st->it, hx.data());
      batch = obs ? 1 : std::min(batch * 2, 16);
    }
    capture_tail(c, c->stream);
  }
  HB_CUDA(cudaEventRecord(c->ev1, c->stream));
  HB_CUDA(cudaMemcpyAsync(c->h_st, c->d_st, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  PcgResult res;
  float ms = 0.f;
  HB_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  res.device_ms = ms;
  res.iterations = c->h_st->it;
  res.converged = c->h_st->converged != 0;
  if (c->h_st->status == 4)
    throw NumericalError("pcg: non-positive curvature, operator is not positive definite");
  std::vector<double> hist(res.iterations + 1);
  HB_CUDA(cudaMemcpy(hist.data(), c->d_hist, hist.size() * sizeof(double), cudaMemcpyDeviceToHost));
  res.last_history = hist.back();
  if (h_history) std::copy(hist.begin(), hist.end(), h_history);
  const int body_kernels = c->fused ? 6 : 8;
  if (!ran) c->launches += (int64_t)res.iterations * body_kernels + 8;
  return res;
}

double quad_norm(homfe_ctx* c, const double* u, const double* d_e) {
  if (c->dist && u) exchange_halo(c, u, c->stream);
  double scale = 1.0;
  if (c->hex_fast && u &&
      launch_hex_quad(c->g, 0, u, c->d_hhi, d_e, c->d_phase, c->d_cmat, c->d_partials, c->stream)) {
    scale = c->g.h[0] * c->g.h[0] * c->g.h[0];  // 8 w
  } else {
    QuadArgs a{u, c->d_hhi, d_e, c->d_phase, c->d_cmat, nullptr, c->d_partials};
    launch_quad(c->g, c->sp, kQuadNorm2, a, c->stream);
  }
  c->launches += 2;
  double v = 0.0;
  reduce_to_host(c, 1, &v);
  return std::sqrt(v * scale);
}

double vec_dot(homfe_ctx* c, const double* a, const double* b) {
  launch_dot_partials(a, b, c->nvec(), c->d_partials, c->stream);
  c->launches += 2;
  double v = 0.0;
  reduce_to_host(c, 1, &v);
  return v;
}

void remove_means(homfe_ctx* c, double* v) {
  remove_means_on(c, v, c->stream);
  c->launches += 3;
}

void set_material(homfe_ctx* c, int n_phases, const double* tangents, const uint8_t* phase, bool device_phase) {
  const int m = c->g.m;
  c->sig_valid = false;
  if (n_phases < 1) throw ValidationError("materials: catalog is empty");
  if (n_phases > kMaxPhases) throw ValidationError("materials: at most 256 phases");
  for (int ph = 0; ph < n_phases; ++ph) check_spd(tangents + ph * m * m, m, "material");
  // phase map upload + per-phase voxel counts on the device (integer atomics:
  // exact, order-independent)
  if (device_phase) HB_CUDA(cudaMemcpyAsync(c->d_phase, phase, c->g.np, cudaMemcpyDeviceToDevice, c->stream));
  else HB_CUDA(cudaMemcpyAsync(c->d_phase, phase, c->g.np, cudaMemcpyHostToDevice, c->stream));
  launch_phase_counts(c->d_phase, c->g.np, reinterpret_cast<unsigned long long*>(c->d_red), c->stream);
  std::vector<int64_t> counts(256, 0);
  if (c->dist) {
    // global phase counts (volume-mean reference) over the slabs
    if (c->sim) sim_allreduce<uint64_t>(c, reinterpret_cast<uint64_t*>(c->d_red), 256);
    else HB_NCCL(ncclAllReduce(c->d_red, c->d_red, 256, ncclUint64, ncclSum, c->comm, c->stream));
  }
  HB_CUDA(cudaMemcpyAsync(counts.data(), c->d_red, 256 * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  for (int v = n_phases; v < 256; ++v)
    if (counts[v]) {
      c->n_phases = 0;  // the uploaded map is invalid: no material until the next valid call
      c->catalog.clear();
      throw ValidationError("materials: phase id " + std::to_string(v) + " missing from catalog");
    }
  counts.resize(n_phases);
  c->counts = counts;
  c->catalog.assign(tangents, tangents + n_phases * m * m);
  if (c->dist) {
    // phase plane z0-1 (previous rank's last plane), for the warm-up elements
    const Grid& g = c->g;
    const int prev = (g.rank - 1 + g.world) % g.world, next = (g.rank + 1) % g.world;
    const size_t plane = (size_t)g.n1 * g.n2;
    if (c->sim) {
      sim_halo(c, c->d_phase, 1, 1, 0, c->d_ph_lo, nullptr);
    } else {
      HB_NCCL(ncclGroupStart());
      HB_NCCL(ncclSend(c->d_phase + (int64_t)(g.n0 - 1) * plane, plane, ncclUint8, next, c->comm, c->stream));
      HB_NCCL(ncclRecv(c->d_ph_lo, plane, ncclUint8, prev, c->comm, c->stream));
      HB_NCCL(ncclGroupEnd());
    }
  }
  // per-phase tables in buffers sized for the full catalog (stable pointers:
  // captured graphs stay valid unless the kernel configuration changes)
  const int ne = c->ne;
  std::vector<double> ke((size_t)n_phases * ne * ne);
  for (int ph = 0; ph < n_phases; ++ph) element_matrix(c->sp, c->g.d, c->g.c, tangents + ph * m * m, &ke[(size_t)ph * ne * ne]);
  if (!c->d_ke) {
    c->d_ke = dalloc<double>((size_t)kMaxPhases * ne * ne);
    c->d_fe = dalloc<double>((size_t)kMaxPhases * ne);
    c->d_cmat = dalloc<double>((size_t)kMaxPhases * m * m);
    c->d_hexmat = dalloc<double>((size_t)kMaxPhases * (c->g.c == 3 ? 108 : 27));
  }
  HB_CUDA(cudaMemcpyAsync(c->d_ke, ke.data(), ke.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  HB_CUDA(cudaMemcpyAsync(c->d_cmat, tangents, (size_t)n_phases * m * m * sizeof(double), cudaMemcpyHostToDevice,
                          c->stream));
  if (c->g.d == 2 && c->g.kind == 1) {
    std::vector<double> tt;
    elem2d_tri_tables(c->g, n_phases, tangents, tt);
    if (!c->d_tri) c->d_tri = dalloc<double>((size_t)kMaxPhases * 12);
    HB_CUDA(cudaMemcpyAsync(c->d_tri, tt.data(), tt.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  }
  // modal-basis tables of the element-centric hex kernel
  bool hex_fast = false, hex_iso = false;
  const char* env = std::getenv("HOMFE_HEX_FAST");
  if (hex_fast_eligible(c->g) && (c->dist || !(env && env[0] == '0'))) {
    std::vector<double> iso, gen;
    hex_iso = hex_fast_tables(c->g, n_phases, tangents, iso, gen);
    const std::vector<double>& t = hex_iso ? iso : gen;
    HB_CUDA(cudaMemcpyAsync(c->d_hexmat, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    hex_fast = true;
  }
  if (c->g.nn > 1) {
    // two node types run on the quadrature-point path with linear models
    ensure_nl_buffers(c);
    c->models.assign(n_phases, NLModel{0, 0.0, 0.0, 0.0, 0.0});
    HB_CUDA(cudaMemcpyAsync(c->d_models, c->models.data(), c->models.size() * sizeof(NLModel),
                            cudaMemcpyHostToDevice, c->stream));
  }
  sync(c);
  if (hex_fast != c->hex_fast || hex_iso != c->hex_iso || n_phases != c->n_phases)
    destroy_graphs(c);  // graphs capture the kernel variant and the catalog size
  c->hex_fast = hex_fast;
  c->hex_iso = hex_iso;
  c->n_phases = n_phases;
}

// ReferencePolicy::resolve (solver.cpp:99-118); volume mean from phase counts.
std::vector<double> resolve_reference(homfe_ctx* c, const homfe_solve_cfg* cfg) {
  const int m = c->g.m;
  std::vector<double> cr(m * m, 0.0);
  if (cfg->reference_policy == HOMFE_REF_IDENTITY_SCALED) {
    if (!(cfg->reference_scale > 0.0)) throw ValidationError("reference: identity scale must be > 0");
    for (int i = 0; i < m; ++i) cr[i * m + i] = cfg->reference_scale;
  } else if (cfg->reference_policy == HOMFE_REF_VOLUME_MEAN) {
    const double wq = c->sp.w[0] * c->sp.nq;  // equal weights: pixel volume
    for (int ph = 0; ph < c->n_phases; ++ph) {
      const double f = (double)c->counts[ph] * wq;
      for (int i = 0; i < m * m; ++i) cr[i] += f * c->catalog[(size_t)ph * m * m + i];
    }
    for (int i = 0; i < m * m; ++i) cr[i] /= c->g.cell_volume;
  } else if (cfg->reference_policy == HOMFE_REF_EXPLICIT) {
    if (!cfg->reference_matrix) throw ValidationError("reference: explicit matrix has wrong size");
    std::copy(cfg->reference_matrix, cfg->reference_matrix + m * m, cr.begin());
  } else {
    throw ValidationError("reference: invalid policy");
  }
  return cr;
}

double frob(const std::vector<double>& a) {
  double s2 = 0.0;
  for (double v : a) s2 += v * v;
  return std::sqrt(s2);
}

// PrecondManager::ensure (solver.cpp:120-142) with the volume-averaged
// tangent `mean` of the current state: reassemble on first use, or when the
// mean drifted beyond the threshold AND the resolved reference changed.
// Returns whether it reassembled (one assembly counted).
bool precond_ensure(homfe_ctx* c, const homfe_solve_cfg* cfg, const std::vector<double>& mean, homfe_report* rep) {
  const int m = c->g.m;
  bool need = !c->pm_valid;
  if (!need) {
    std::vector<double> diff(m * m);
    for (int i = 0; i < m * m; ++i) diff[i] = mean[i] - c->pm_mean[i];
    need = frob(diff) > cfg->reassembly_threshold * frob(c->pm_mean);
  }
  if (need) {
    std::vector<double> cref;
    if (cfg->reference_policy == HOMFE_REF_VOLUME_MEAN) {
      cref = mean;
    } else {
      cref = resolve_reference(c, cfg);
    }
    if (!c->pm_valid || cref != c->pm_cref) {
      set_reference(c, cref.data());
      c->pm_cref = cref;
      c->pm_mean = mean;
      c->pm_valid = true;
      rep->assemblies += 1;
      return true;
    }
  }
  // the manager keeps its blocks: restore them on the device if a parity hook
  // (homfe_gpu_set_reference) replaced the context's reference since
  if (!c->have_ref || c->c_ref != c->pm_cref) set_reference(c, c->pm_cref.data());
  return false;
}

void validate_cfg(const homfe_solve_cfg* cfg) {
  if (!cfg) throw ValidationError("solver: null config");
  if (!(cfg->eta_newton > 0.0 && cfg->eta_newton < 1.0) || !(cfg->eta_cg > 0.0 && cfg->eta_cg < 1.0))
    throw ValidationError("solver: tolerances must lie in (0,1)");
  if (cfg->max_newton < 1 || cfg->max_cg < 1) throw ValidationError("solver: iteration caps must be >= 1");
  if (!(cfg->reassembly_threshold >= 0.0)) throw ValidationError("solver: reassembly threshold must be >= 0");
}

// newton_solve, linear branch (solver.cpp:171-296). u in/out lives in d_u.
void newton(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, double* avg_out, homfe_report* rep) {
  const auto t_total = Clock::now();
  validate_cfg(cfg);
  require_material(c);
  const int m = c->g.m, ne = c->ne;
  for (int k = 0; k < m; ++k)
    if (!std::isfinite(e[k])) throw ValidationError("load vector has non-finite entries");
  std::memset(rep, 0, sizeof(*rep));
  c->launches = 0;
  c->sig_valid = false;
  if (c->graphs_nl) {
    destroy_graphs(c);  // captured graphs hold the tangent operator
    c->graphs_nl = false;
  }
  HB_CUDA(cudaMemcpyAsync(c->d_e, e, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // element load vectors f_e = sum_q w B^T C e per phase
  std::vector<double> fe((size_t)c->n_phases * ne);
  for (int ph = 0; ph < c->n_phases; ++ph)
    element_load(c->sp, c->g.d, c->g.c, &c->catalog[(size_t)ph * m * m], e, &fe[(size_t)ph * ne]);
  HB_CUDA(cudaMemcpyAsync(c->d_fe, fe.data(), fe.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));

  // PrecondManager::ensure: a linear tangent's volume mean is the phase-count
  // average; it never drifts within a solve, so only step 0 can reassemble.
  auto t0 = Clock::now();
  homfe_solve_cfg vm = *cfg;
  vm.reference_policy = HOMFE_REF_VOLUME_MEAN;
  const bool reassembled = precond_ensure(c, cfg, resolve_reference(c, &vm), rep);
  rep->seconds_assembly += since(t0);

  double bnorm0 = 0.0, inc_rel = INFINITY;
  bool have_inc = false;
  const int64_t n = c->nvec();
  for (int step = 0;; ++step) {
    t0 = Clock::now();
    // b = -D^T W C (e + D u) = -(K u + f)
    apply_K(c, c->d_u, c->d_r, c->d_fe, -1.0, nullptr, nullptr, c->stream);
    sync(c);
    rep->seconds_constitutive += since(t0);
    // z = M^-1 b and b.z (Parseval) in one pass
    precond_apply(c, c->d_r, c->d_z, nullptr, c->d_partials, c->stream);
    double bz = 0.0;
    reduce_to_host(c, 1, &bz);
    const double bnorm = std::sqrt(std::max(0.0, bz));
    if (step == 0) bnorm0 = bnorm;
    const bool residual_ok = bnorm <= cfg->eta_newton * bnorm0;
    const bool increment_ok = have_inc && inc_rel <= cfg->eta_newton;
    if (step > 0 && (increment_ok || residual_ok)) {
      rep->cause = 0;
      rep->converged = 1;
      break;
    }
    if (step == cfg->max_newton) {
      rep->cause = 2;
      rep->converged = 0;
      break;
    }
    // zero-RHS test (only needed when the step is taken: the two strain norms
    // are not computed for the final convergence check)
    const double strain_scale = quad_norm(c, c->d_u, c->d_e);
    const bool b_is_zero = bnorm == 0.0 || quad_norm(c, c->d_z, nullptr) <= 1e-12 * strain_scale;
    t0 = Clock::now();
    PcgResult pr;
    if (b_is_zero) {
      HB_CUDA(cudaMemsetAsync(c->d_x, 0, n * sizeof(double), c->stream));
      pr.converged = true;
      pr.last_history = bnorm;
    } else {
      pr = run_pcg(c, cfg->eta_cg, cfg->max_cg, nullptr);  // r = b already in d_r
    }
    rep->seconds_cg += since(t0);
    rep->cg_device_ms += pr.device_ms;
    // u += x; u.remove_component_means()   (solver.cpp:262-263)
    launch_axpy(c->d_u, 1.0, c->d_x, n, c->stream);
    c->launches += 1;
    remove_means(c, c->d_u);
    if (cfg->criterion == 0) {
      const double num = quad_norm(c, c->d_x, nullptr);
      const double den = quad_norm(c, c->d_u, nullptr);
      inc_rel = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    } else {
      const double num = std::sqrt(vec_dot(c, c->d_x, c->d_x));
      const double den = std::sqrt(vec_dot(c, c->d_u, c->d_u));
      inc_rel = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    }
    have_inc = true;
    if (rep->n_steps < 32) {
      homfe_newton_step& s = rep->steps[rep->n_steps];
      s.cg_iterations = pr.iterations;
      s.residual_initial = bnorm;
      s.residual_final = pr.last_history;
      s.increment_rel = inc_rel;
      s.precond_reassembled = (step == 0 && reassembled) ? 1 : 0;
    }
    rep->n_steps += 1;
    rep->total_cg += pr.iterations;
    if (!pr.converged) {
      rep->cause = 1;
      rep->converged = 0;
      break;
    }
  }
  // <sigma> = (1/|Y|) sum_q w C (e + D u)   (solver.cpp:321-324)
  if (c->dist) exchange_halo(c, c->d_u, c->stream);
  double sscale = 1.0;
  if (c->hex_fast && launch_hex_quad(c->g, 1, c->d_u, c->d_hhi, c->d_e, c->d_phase, c->d_cmat, c->d_partials,
                                     c->stream)) {
    sscale = c->g.h[0] * c->g.h[0] * c->g.h[0];
  } else {
    QuadArgs qa{c->d_u, c->d_hhi, c->d_e, c->d_phase, c->d_cmat, nullptr, c->d_partials};
    launch_quad(c->g, c->sp, kQuadStress, qa, c->stream);
  }
  c->launches += 2;
  double avg[6];
  reduce_to_host(c, m, avg);
  for (int k = 0; k < m; ++k) avg_out[k] = avg[k] * sscale / c->g.cell_volume;
  rep->seconds_total = since(t_total);
  rep->kernel_launches = c->launches;
}


void ensure_nl_buffers(homfe_ctx* c) {
  if (c->d_sig) return;
  const size_t nq = (size_t)c->g.np * c->sp.nq;
  const int m = c->g.m;
  c->d_models = reinterpret_cast<NLModel*>(dalloc<double>(kMaxPhases * sizeof(NLModel) / sizeof(double) + 1));
  c->d_g0 = dalloc<double>(nq * 7);
  c->d_gtr = dalloc<double>(nq * 7);
  c->d_tanc = dalloc<double>(nq * 8);
  c->d_sig = dalloc<double>(nq * m);
  c->d_qs = dalloc<double>(nq * m);
  c->d_tpart = dalloc<double>((size_t)kRedBlocks * 36);
  c->d_status = reinterpret_cast<int*>(dalloc<double>(1));
}

// constitutive_sweep (solver.cpp:144-169) at d_u: stress, trial state,
// compact tangents; returns the volume-mean tangent (fields.cpp:52-61).
std::vector<double> nl_sweep(homfe_ctx* c) {
  const int m = c->g.m;
  HB_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(int), c->stream));
  launch_sweep(c->g, c->sp, nl_args(c, c->d_u), c->stream);
  c->launches += 1;
  std::vector<double> part((size_t)kRedBlocks * m * m);
  int bad = 0;
  HB_CUDA(cudaMemcpyAsync(part.data(), c->d_tpart, part.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  HB_CUDA(cudaMemcpyAsync(&bad, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  if (bad) throw NumericalError("evaluate: non-finite strain input");
  std::vector<double> mean(m * m, 0.0);
  for (int b = 0; b < kRedBlocks; ++b)
    for (int i = 0; i < m * m; ++i) mean[i] += part[(size_t)b * m * m + i];
  for (int i = 0; i < m * m; ++i) mean[i] /= c->g.cell_volume;
  c->sig_valid = true;
  return mean;
}


// newton_solve (solver.cpp:171-296) for a catalog with J2 phases: a
// constitutive sweep per Newton step, PrecondManager::ensure with the
// volume-mean tangent drift (solver.cpp:120-142), PCG on the tangent
// operator. d_g0 holds the committed state; on return d_gtr (converged) or
// d_g0 (otherwise) is the outgoing state.
bool newton_nl(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, double* avg_out, homfe_report* rep) {
  const auto t_total = Clock::now();
  validate_cfg(cfg);
  require_material(c);
  const int m = c->g.m;
  for (int k = 0; k < m; ++k)
    if (!std::isfinite(e[k])) throw ValidationError("load vector has non-finite entries");
  std::memset(rep, 0, sizeof(*rep));
  c->launches = 0;
  HB_CUDA(cudaMemcpyAsync(c->d_e, e, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  if (!c->graphs_nl) {
    destroy_graphs(c);  // captured operator changes
    c->graphs_nl = true;
  }
  double bnorm0 = 0.0, inc_rel = INFINITY;
  bool have_inc = false, converged_state = false;
  const int64_t n = c->nvec();
  for (int step = 0;; ++step) {
    auto t0 = Clock::now();
    const std::vector<double> mean = nl_sweep(c);
    // b = -D^T W sigma
    launch_divergence(c->g, c->sp, c->d_sig, true, c->d_r, c->stream);
    launch_scale(c->d_r, -1.0, n, c->stream);
    rep->seconds_constitutive += since(t0);
    // PrecondManager::ensure
    t0 = Clock::now();
    const bool reassembled = precond_ensure(c, cfg, mean, rep);
    rep->seconds_assembly += since(t0);
    // z = M^-1 b and b.z
    c->nl_op = false;
    precond_apply(c, c->d_r, c->d_z, nullptr, c->d_partials, c->stream);
    double bz = 0.0;
    reduce_to_host(c, 1, &bz);
    const double bnorm = std::sqrt(std::max(0.0, bz));
    if (step == 0) bnorm0 = bnorm;
    const double strain_scale = quad_norm(c, c->d_u, c->d_e);
    const bool b_is_zero = bnorm == 0.0 || quad_norm(c, c->d_z, nullptr) <= 1e-12 * strain_scale;
    const bool residual_ok = bnorm <= cfg->eta_newton * bnorm0;
    const bool increment_ok = have_inc && inc_rel <= cfg->eta_newton;
    if (step > 0 && (increment_ok || residual_ok)) {
      rep->cause = 0;
      rep->converged = 1;
      converged_state = true;
      break;
    }
    if (step == cfg->max_newton) {
      rep->cause = 2;
      rep->converged = 0;
      break;
    }
    t0 = Clock::now();
    PcgResult pr;
    if (b_is_zero) {
      HB_CUDA(cudaMemsetAsync(c->d_x, 0, n * sizeof(double), c->stream));
      pr.converged = true;
      pr.last_history = bnorm;
    } else {
      c->nl_op = true;
      try {
        pr = run_pcg(c, cfg->eta_cg, cfg->max_cg, nullptr);
      } catch (...) {
        c->nl_op = false;
        throw;
      }
      c->nl_op = false;
    }
    rep->seconds_cg += since(t0);
    rep->cg_device_ms += pr.device_ms;
    launch_axpy(c->d_u, 1.0, c->d_x, n, c->stream);
    c->launches += 1;
    remove_means(c, c->d_u);
    if (cfg->criterion == 0) {
      const double num = quad_norm(c, c->d_x, nullptr);
      const double den = quad_norm(c, c->d_u, nullptr);
      inc_rel = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    } else {
      const double num = std::sqrt(vec_dot(c, c->d_x, c->d_x));
      const double den = std::sqrt(vec_dot(c, c->d_u, c->d_u));
      inc_rel = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    }
    have_inc = true;
    if (rep->n_steps < 32) {
      homfe_newton_step& sr = rep->steps[rep->n_steps];
      sr.cg_iterations = pr.iterations;
      sr.residual_initial = bnorm;
      sr.residual_final = pr.last_history;
      sr.increment_rel = inc_rel;
      sr.precond_reassembled = reassembled ? 1 : 0;
    }
    rep->n_steps += 1;
    rep->total_cg += pr.iterations;
    if (!pr.converged) {
      rep->cause = 1;
      rep->converged = 0;
      nl_sweep(c);  // stress at the returned iterate (solver.cpp:281-290)
      break;
    }
  }
  // <sigma> = volume average of the state's stress (solver.cpp:321-324)
  launch_quad_wsum(c->g, c->sp, c->d_sig, c->d_partials, c->stream);
  c->launches += 2;
  double avg[6];
  reduce_to_host(c, m, avg);
  for (int k = 0; k < m; ++k) avg_out[k] = avg[k] / c->g.cell_volume;
  rep->seconds_total = since(t_total);
  rep->kernel_launches = c->launches;
  return converged_state;
}


// newton_solve dispatch: the linear branch (phase-indexed tangents), or the
// general one (J2 catalogs; two-node stencils, whose operator runs on the
// quadrature-point path) from a zero committed state.
void solve_dispatch(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, double* avg_out, homfe_report* r) {
  if (c->nonlinear || c->g.nn > 1) {
    ensure_nl_buffers(c);
    HB_CUDA(cudaMemsetAsync(c->d_g0, 0, (size_t)c->g.np * c->sp.nq * 7 * sizeof(double), c->stream));
    newton_nl(c, e, cfg, avg_out, r);
  } else {
    newton(c, e, cfg, avg_out, r);
  }
}

void ensure_sb_buffers(homfe_ctx* c) {
  if (c->d_strain) return;
  const size_t n = (size_t)c->g.np * c->sp.nq * c->g.m;
  c->d_strain = dalloc<double>(n);
  c->d_sx = dalloc<double>(n);
  c->d_sr = dalloc<double>(n);
  c->d_sp = dalloc<double>(n);
  c->d_sap = dalloc<double>(n);
  c->d_scp = dalloc<double>(n);
}

// Gamma s = D (D^T C_ref D)^+ D^T s (projection.cpp:29-41). With equal
// Gauss weights (required by the reference, projection.cpp:12-17) the
// unweighted blocks and divergence equal the weighted ones up to the weight
// factor, which cancels: Gamma = D M_w^-1 D^T W.
void gamma_apply(homfe_ctx* c, const double* s_in, double* out, cudaStream_t st) {
  launch_divergence(c->g, c->sp, s_in, true, c->d_r, st);
  precond_apply(c, c->d_r, c->d_z, nullptr, nullptr, st);
  QuadArgs a{c->d_z, c->d_hhi, nullptr, c->d_phase, c->d_cmat, out, nullptr};
  launch_quad(c->g, c->sp, kQuadGrad, a, st);
  c->launches += 5;
}

double qdot(homfe_ctx* c, const double* a, const double* b, int64_t n) {
  launch_dot_partials(a, b, n, c->d_partials, c->stream);
  double v = 0.0;
  reduce_to_host(c, 1, &v);
  return v;
}

// sb_newton_solve (projection.cpp:93-185) with strain_cg (:54-91). The
// unknown (fluctuating strain, compatible by construction) lives in d_strain.
bool sb_newton(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, const double* cref, double* avg_out,
               homfe_report* rep) {
  const auto t_total = Clock::now();
  validate_cfg(cfg);
  require_material(c);
  if (c->dist) throw ValidationError("sb_newton_solve: single-GPU contexts only");
  const int m = c->g.m;
  for (int k = 0; k < m; ++k)
    if (!std::isfinite(e[k])) throw ValidationError("load vector has non-finite entries");
  std::memset(rep, 0, sizeof(*rep));
  c->launches = 0;
  ensure_nl_buffers(c);
  ensure_sb_buffers(c);
  if ((int)c->models.size() != c->n_phases) {
    c->models.assign(c->n_phases, NLModel{0, 0.0, 0.0, 0.0, 0.0});
    HB_CUDA(cudaMemcpy(c->d_models, c->models.data(), c->models.size() * sizeof(NLModel), cudaMemcpyHostToDevice));
  }
  HB_CUDA(cudaMemcpyAsync(c->d_e, e, m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  // assemble_projection_blocks
  auto t0 = Clock::now();
  if (!c->have_ref || std::vector<double>(cref, cref + m * m) != c->c_ref) set_reference(c, cref);
  rep->assemblies = 1;
  rep->seconds_assembly += since(t0);
  const int64_t nq = c->g.np * c->sp.nq, ns = nq * m;
  const double wq = c->g.cell_volume / (double)nq;  // equal Gauss weights
  NLArgs na = nl_args(c, nullptr);
  na.qeps = c->d_strain;
  double bnorm0 = 0.0, inc_rel = INFINITY;
  bool have_inc = false, converged_state = false;
  auto sweep = [&]() {
    HB_CUDA(cudaMemsetAsync(c->d_status, 0, sizeof(int), c->stream));
    launch_sweep(c->g, c->sp, na, c->stream);
    int bad = 0;
    HB_CUDA(cudaMemcpyAsync(&bad, c->d_status, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (bad) throw NumericalError("evaluate: non-finite strain input");
    c->sig_valid = true;
  };
  for (int step = 0;; ++step) {
    t0 = Clock::now();
    sweep();
    rep->seconds_constitutive += since(t0);
    // b = -Gamma sigma
    gamma_apply(c, c->d_sig, c->d_sr, c->stream);
    launch_scale(c->d_sr, -1.0, ns, c->stream);
    const double bnorm = std::sqrt(std::max(0.0, qdot(c, c->d_sr, c->d_sr, ns)));
    if (step == 0) bnorm0 = bnorm;
    launch_qshift_norm2(c->d_strain, c->d_e, nq, m, c->d_partials, c->stream);
    double et2 = 0.0;
    reduce_to_host(c, 1, &et2);
    const bool b_is_zero = bnorm == 0.0 || bnorm <= 1e-12 * std::sqrt(et2);
    const bool residual_ok = bnorm <= cfg->eta_newton * bnorm0;
    const bool increment_ok = have_inc && inc_rel <= cfg->eta_newton;
    if (step > 0 && (increment_ok || residual_ok)) {
      rep->cause = 0;
      rep->converged = 1;
      converged_state = true;
      break;
    }
    if (step == cfg->max_newton) {
      rep->cause = 2;
      rep->converged = 0;
      break;
    }
    // strain_cg: r = b (d_sr), x = 0, p = r
    t0 = Clock::now();
    HB_CUDA(cudaMemsetAsync(c->d_sx, 0, ns * sizeof(double), c->stream));
    int iters = 0;
    double last = bnorm;
    bool cg_ok = false;
    if (b_is_zero) {
      cg_ok = true;
    } else {
      double rr = std::max(qdot(c, c->d_sr, c->d_sr, ns), 0.0);
      const double norm0 = std::sqrt(rr);
      last = norm0;
      if (norm0 == 0.0) {
        cg_ok = true;
      } else {
        HB_CUDA(cudaMemcpyAsync(c->d_sp, c->d_sr, ns * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
        for (int k = 1; k <= cfg->max_cg; ++k) {
          launch_tan_mult(c->g, c->sp, na, c->d_sp, c->d_scp, c->stream);
          gamma_apply(c, c->d_scp, c->d_sap, c->stream);
          const double pap = qdot(c, c->d_sp, c->d_sap, ns);
          if (pap <= 0.0)
            throw NumericalError("strain cg: non-positive curvature, operator is not positive definite");
          const double alpha = rr / pap;
          launch_axpy(c->d_sx, alpha, c->d_sp, ns, c->stream);
          launch_axpy(c->d_sr, -alpha, c->d_sap, ns, c->stream);
          const double rrn = std::max(qdot(c, c->d_sr, c->d_sr, ns), 0.0);
          iters = k;
          last = std::sqrt(rrn);
          c->launches += 4;
          if (std::sqrt(rrn) <= cfg->eta_cg * norm0) {
            cg_ok = true;
            break;
          }
          // p = r + (rrn / rr) p
          launch_scale(c->d_sp, rrn / rr, ns, c->stream);
          launch_axpy(c->d_sp, 1.0, c->d_sr, ns, c->stream);
          rr = rrn;
        }
      }
    }
    rep->seconds_cg += since(t0);
    launch_axpy(c->d_strain, 1.0, c->d_sx, ns, c->stream);
    const double num = std::sqrt(wq * qdot(c, c->d_sx, c->d_sx, ns));
    const double den = std::sqrt(wq * qdot(c, c->d_strain, c->d_strain, ns));
    inc_rel = den > 0.0 ? num / den : (num > 0.0 ? 1.0 : 0.0);
    have_inc = true;
    if (rep->n_steps < 32) {
      homfe_newton_step& sr = rep->steps[rep->n_steps];
      sr.cg_iterations = iters;
      sr.residual_initial = bnorm;
      sr.residual_final = last;
      sr.increment_rel = inc_rel;
      sr.precond_reassembled = step == 0 ? 1 : 0;
    }
    rep->n_steps += 1;
    rep->total_cg += iters;
    if (!cg_ok) {
      rep->cause = 1;
      rep->converged = 0;
      sweep();
      break;
    }
  }
  launch_quad_wsum(c->g, c->sp, c->d_sig, c->d_partials, c->stream);
  double avg[6];
  reduce_to_host(c, m, avg);
  for (int k = 0; k < m; ++k) avg_out[k] = avg[k] / c->g.cell_volume;
  rep->seconds_total = since(t_total);
  rep->kernel_launches = c->launches;
  return converged_state;
}

}  // namespace

// ===================================================================== C ABI
namespace {

bool is_multi(const homfe_ctx* c) { return c && !c->ranks.empty(); }

int multi_unsupported(const char* what) {
  g_err = std::string(what) + ": not available on a multi-GPU context (use one slab context per rank)";
  return HOMFE_VALIDATION;
}

// f(rank_ctx, rank) on every rank, each in its own host thread (the rank
// contexts' collectives need all ranks inside a call at once); the first
// failing rank's status and message are returned. HOMFE_NONCONVERGED is a
// result, not a failure: it is returned once every rank finished.
template <class F>
int multi_run(homfe_ctx* c, F&& f) {
  const int W = (int)c->ranks.size();
  std::vector<int> codes(W, HOMFE_OK);
  std::vector<std::string> errs(W);
  std::vector<std::thread> th;
  th.reserve(W);
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      codes[r] = f(c->ranks[r], r);
      if (codes[r] != HOMFE_OK) errs[r] = g_err;
    });
  for (auto& t : th) t.join();
  int soft = HOMFE_OK;
  for (int r = 0; r < W; ++r) {
    if (codes[r] == HOMFE_OK) continue;
    if (codes[r] == HOMFE_NONCONVERGED) {
      soft = HOMFE_NONCONVERGED;
      g_err = errs[r];
      continue;
    }
    g_err = errs[r];
    return codes[r];
  }
  return soft;
}

// component-planar global <-> rank slab (contiguous per component)
struct MultiSplit {
  int c;
  int64_t n_glob, n_loc;
  void scatter(const double* g, std::vector<double>& l, int r) const {
    l.resize((size_t)c * n_loc);
    for (int k = 0; k < c; ++k)
      std::memcpy(l.data() + (size_t)k * n_loc, g + (size_t)k * n_glob + (size_t)r * n_loc, n_loc * sizeof(double));
  }
  void gather(const std::vector<double>& l, double* g, int r) const {
    for (int k = 0; k < c; ++k)
      std::memcpy(g + (size_t)k * n_glob + (size_t)r * n_loc, l.data() + (size_t)k * n_loc, n_loc * sizeof(double));
  }
};

MultiSplit split_of(const homfe_ctx* c) {
  const homfe_ctx* r0 = c->ranks[0];
  return MultiSplit{r0->g.c, r0->g.np * (int64_t)c->ranks.size(), r0->g.np};
}

// vector op y = op(x) on the slabs
template <class F>
int multi_map(homfe_ctx* c, const double* x, double* y, F&& op) {
  const MultiSplit sp = split_of(c);
  std::vector<std::vector<double>> yl(c->ranks.size());
  const int code = multi_run(c, [&](homfe_ctx* rc, int r) {
    std::vector<double> xl;
    sp.scatter(x, xl, r);
    yl[r].assign(xl.size(), 0.0);
    return op(rc, xl.data(), yl[r].data());
  });
  if (code == HOMFE_OK || code == HOMFE_NONCONVERGED)
    for (size_t r = 0; r < yl.size(); ++r) sp.gather(yl[r], y, (int)r);
  return code;
}

std::atomic<uint64_t> g_multi_sim_group{7700000};

}  // namespace

extern "C" {

const char* homfe_gpu_last_error(void) { return g_err.c_str(); }

int homfe_isotropic_stiffness(double bulk, double shear, int32_t dim, double* out) {
  return guarded([&] { isotropic_stiffness(bulk, shear, dim, out); });
}

// Seeded inputs with the reference RNG convention (proj/tests/support/
// oracles.hpp:154-160, proj/src/microstructure.cpp:75-90):
// std::mt19937_64(seed), u = lo + (hi - lo) (gen() >> 11) 2^-53.
int homfe_random_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out) {
  return guarded([&] {
    std::mt19937_64 gen(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * ((double)(gen() >> 11) * 0x1.0p-53);
  });
}

// Standard normals by Box-Muller on consecutive uniform pairs of the same stream.
int homfe_random_normal(uint64_t seed, int64_t n, double* out) {
  return guarded([&] {
    std::mt19937_64 gen(seed);
    for (int64_t i = 0; i < n; i += 2) {
      const double u1 = (double)(gen() >> 11) * 0x1.0p-53;
      const double u2 = (double)(gen() >> 11) * 0x1.0p-53;
      const double r = std::sqrt(-2.0 * std::log1p(-u1));
      out[i] = r * std::cos(2.0 * M_PI * u2);
      if (i + 1 < n) out[i + 1] = r * std::sin(2.0 * M_PI * u2);
    }
  });
}

}  // extern "C"

namespace {

// Shared constructor. world == 0: single device (periodic grid on one GPU);
// world >= 1: slab `rank` of `world` along axis 0 with NCCL exchanges.
bool p2p_wanted(int world) {
  const char* penv = std::getenv("HOMFE_P2P");
  return world > 1 && world <= FusedFft::kMaxPeers && !(penv && penv[0] == '0');
}

// Peer access setup (slab mode, 2..8 ranks): every rank's two spectrum
// buffers (fused: T, T2; slab spectra: W, S) and p, through CUDA IPC handles
// gathered over NCCL (or the in-process transport's pointer exchange). On
// any IPC failure on any rank the context keeps the all-to-all transport.
void setup_peers(homfe_ctx* c, void* buf_a, void* buf_b) {
  const int G = c->g.world, me = c->g.rank;
  void* mine[3] = {buf_a, buf_b, c->d_p};
  void* ptrs[3][FusedFft::kMaxPeers] = {};
  if (c->sim) {
    for (int k = 0; k < 3; ++k)
      sim_exchange(c, mine[k], [&](SimGroup* S) {
        for (int q = 0; q < G; ++q) ptrs[k][q] = const_cast<void*>(S->ptr[q]);
      });
  } else {
    std::vector<cudaIpcMemHandle_t> h((size_t)G * 3);
    bool ok = true;
    for (int k = 0; k < 3; ++k) ok = ok && cudaIpcGetMemHandle(&h[(size_t)me * 3 + k], mine[k]) == cudaSuccess;
    // every rank takes part in the gather (a failed rank contributes zeros)
    char* d_h = dalloc<char>(h.size() * sizeof(cudaIpcMemHandle_t));
    const size_t per = 3 * sizeof(cudaIpcMemHandle_t);
    if (!ok) std::memset(&h[(size_t)me * 3], 0, per);
    HB_CUDA(cudaMemcpy(d_h + me * per, &h[(size_t)me * 3], per, cudaMemcpyHostToDevice));
    HB_NCCL(ncclAllGather(d_h + me * per, d_h, per, ncclChar, c->comm, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
    HB_CUDA(cudaMemcpy(h.data(), d_h, h.size() * sizeof(cudaIpcMemHandle_t), cudaMemcpyDeviceToHost));
    cudaFree(d_h);
    // agree on the outcome: all ranks pull, or none
    int flag = ok ? 1 : 0;
    for (int q = 0; q < G && flag; ++q) {
      if (q == me) {
        for (int k = 0; k < 3; ++k) ptrs[k][q] = mine[k];
        continue;
      }
      for (int k = 0; k < 3 && flag; ++k) {
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, h[(size_t)q * 3 + k], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          cudaGetLastError();
          flag = 0;
          break;
        }
        c->ipc_open.push_back(p);
        ptrs[k][q] = p;
      }
    }
    int* d_flag = dalloc<int>(1);
    HB_CUDA(cudaMemcpy(d_flag, &flag, sizeof(int), cudaMemcpyHostToDevice));
    HB_NCCL(ncclAllReduce(d_flag, d_flag, 1, ncclInt, ncclMin, c->comm, c->stream));
    HB_CUDA(cudaStreamSynchronize(c->stream));
    HB_CUDA(cudaMemcpy(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(d_flag);
    if (!flag) {
      for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
      c->ipc_open.clear();
      return;
    }
  }
  for (int q = 0; q < FusedFft::kMaxPeers; ++q) {
    const int qq = q < G ? q : 0;
    c->peer_a[q] = ptrs[0][qq];
    c->peer_b[q] = ptrs[1][qq];
    c->peer_p[q] = static_cast<double*>(ptrs[2][qq]);
  }
  c->d_bar = dalloc<double>(1);
  HB_CUDA(cudaMemset(c->d_bar, 0, sizeof(double)));
  c->peer = true;
}

homfe_ctx* create_impl(const homfe_grid_desc* desc, int rank, int world, const void* nccl_id) {
  if (!desc) throw ValidationError("create: null argument");
  const int d = desc->dim;
  if (d != 2 && d != 3) throw ValidationError("cell: dimension must be 2 or 3, got " + std::to_string(d));
  for (int a = 0; a < d; ++a) {
    if (desc->dims[a] < 2)
      throw ValidationError("cell.dims[" + std::to_string(a) + "]: must be >= 2, got " + std::to_string(desc->dims[a]));
    if (!(desc->lengths[a] > 0.0)) throw ValidationError("cell.lengths[" + std::to_string(a) + "]: must be > 0");
    if (desc->dims[a] > (1 << 24)) throw ValidationError("cell: dimension too large");
  }
  const int c = desc->components;
  if (c != 1 && c != d) throw ValidationError("nodal field shape does not match layout");
  const bool dist = world >= 1;
  const int G = dist ? world : 1;
  if (dist) {
    if (rank < 0 || rank >= world) throw ValidationError("slab: rank out of range");
    if (desc->stencil == HOMFE_FOUR_TRIANGLES_TWO_NODE)
      throw ValidationError("slab mode: one-node stencils only");
    if (desc->dims[0] % world != 0 || (d == 3 && desc->dims[1] % world != 0))
      throw ValidationError(d == 3 ? "slab mode: dims[0] and dims[1] must be divisible by the number of ranks"
                                   : "slab mode: dims[0] must be divisible by the number of ranks");
    if (!nccl_id) throw ValidationError("slab mode: missing NCCL unique id");
  }
  auto* ctx = new homfe_ctx();
  try {
    ctx->device = desc->device;
    HB_CUDA(cudaSetDevice(ctx->device));
    Grid& g = ctx->g;
    g.d = d;
    g.c = c;
    g.m = c == 1 ? d : mandel_dim(d);
    g.kind = desc->stencil;
    g.n0g = (int)desc->dims[0];
    g.n0 = g.n0g / G;
    g.n1 = (int)desc->dims[1];
    g.n2 = d == 3 ? (int)desc->dims[2] : 1;
    g.np = (int64_t)g.n0 * g.n1 * g.n2;
    g.npg = (int64_t)g.n0g * g.n1 * g.n2;
    g.dist = dist ? 1 : 0;
    g.rank = dist ? rank : 0;
    g.world = G;
    g.z0 = g.rank * g.n0;
    g.cell_volume = 1.0;
    for (int a = 0; a < 3; ++a) g.h[a] = a < d ? desc->lengths[a] / (double)desc->dims[a] : 1.0;
    for (int a = 0; a < d; ++a) g.cell_volume *= desc->lengths[a];
    if ((int64_t)c * g.np >= (int64_t)1 << 31) throw ValidationError("cell: grid too large for one device");
    ctx->dist = dist;
    ctx->sp = make_stencil(g.kind, d, g.h);
    g.nn = ctx->sp.nn;
    if (g.nn > 1 && dist) throw ValidationError("slab mode: one-node stencils only");
    ctx->nl = ctx->sp.noff;
    ctx->ne = ctx->nl * c;
    const int nh = (d == 3 ? g.n2 : g.n1) / 2 + 1;
    ctx->nf = (d == 3 ? (int64_t)g.n0g * g.n1 : (int64_t)g.n0g) * nh;  // global spectrum
    HB_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    HB_CUDA(cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking));
    HB_CUDA(cudaEventCreate(&ctx->ev0));
    HB_CUDA(cudaEventCreate(&ctx->ev1));
    if (dist) {
      if (std::memcmp(nccl_id, "HBSIMGRP", 8) == 0) {
        uint64_t gid = 0;
        std::memcpy(&gid, static_cast<const char*>(nccl_id) + 8, 8);
        std::lock_guard<std::mutex> lk(g_sim_mu);
        auto& grp = g_sim[gid];
        if (!grp) {
          grp = std::make_shared<SimGroup>();
          grp->world = world;
          grp->ptr.assign(world, nullptr);
          grp->red.assign((size_t)world * 256, 0.0);
          grp->ured.assign((size_t)world * 256, 0);
        }
        if (grp->world != world) throw ValidationError("slab sim: world mismatch");
        ctx->sim = grp.get();
        ctx->body_eager = true;  // host barriers cannot be captured
      } else {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        HB_NCCL(ncclCommInitRank(&ctx->comm, world, id, rank));
      }
      const size_t plane = (size_t)g.n1 * g.n2;
      ctx->d_hlo = dalloc<double>(c * plane);
      ctx->d_hhi = dalloc<double>(c * plane);
      ctx->d_ph_lo = dalloc<uint8_t>(plane);
      ctx->use_while = false;  // host-driven iterations around the collectives
    }
    const int64_t nv = ctx->nvec();
    ctx->d_x = dalloc<double>(nv);
    ctx->d_r = dalloc<double>(nv);
    ctx->d_p = dalloc<double>(nv);
    ctx->d_ap = dalloc<double>(nv);
    ctx->d_z = dalloc<double>(nv);
    ctx->d_u = dalloc<double>(nv);
    // spectrum scratch: cuFFT layout, or the tile-major layout of the fused
    // passes (16-column blocks, fftfused.cu) when that is larger
    const int64_t pitch = ((int64_t)(g.n2 / 2 + 1) + 15) / 16 * 16;
    const bool fz = d == 3 && (!dist || (fused_fft_eligible(g) && g.n1 % G == 0));  // slab spectra: own buffers
    const int64_t fused_sz = fz ? (int64_t)c * g.n0 * g.n1 * pitch : 0;
    ctx->d_spec = dalloc<double2>(std::max<int64_t>(dist ? 0 : (int64_t)c * g.nn * ctx->nf, fused_sz));
    ctx->d_phase = dalloc<uint8_t>(g.np);
    ctx->d_partials = dalloc<double>((size_t)kRedBlocks * 8);
    ctx->d_scal = dalloc<double>(64);
    ctx->d_red = dalloc<double>(256);
    ctx->d_e = dalloc<double>(8);
    ctx->d_st = dalloc<PcgState>(1);
    HB_CUDA(cudaMallocHost(&ctx->h_st, sizeof(PcgState)));
    HB_CUDA(cudaMallocHost(&ctx->h_scal, 256 * sizeof(double)));
    HB_CUDA(cudaMemset(ctx->d_u, 0, nv * sizeof(double)));
    if (!dist) {
      // cuFFT plans: batched over the c components (component-planar fields)
      int nn[3] = {g.n0, g.n1, g.n2};
      HB_CUFFT(cufftPlanMany(&ctx->fwd, d, nn, nullptr, 1, (int)g.np, nullptr, 1, (int)ctx->nf, CUFFT_D2Z,
                             c * g.nn));
      HB_CUFFT(cufftPlanMany(&ctx->inv, d, nn, nullptr, 1, (int)ctx->nf, nullptr, 1, (int)g.np, CUFFT_Z2D,
                             c * g.nn));
    }
    // per-axis phase tables for the analytic symbol (global grid)
    SpecParams& p = ctx->spp;
    std::memset(&p, 0, sizeof(p));
    p.kind = g.kind;
    p.d = d;
    p.c = c;
    p.n0 = g.n0g;
    p.n1 = g.n1;
    p.n1r = g.n1;
    p.k1off = 0;
    p.n2 = g.n2;
    p.nh = nh;
    p.nhv = nh;
    p.nf = ctx->nf;
    p.w = ctx->sp.w[0];
    p.inv_np = 1.0 / (double)g.npg;
    for (int a = 0; a < 3; ++a) p.h[a] = g.h[a];
    set_gram_factors(p);
    for (int a = 0; a < d; ++a) {
      const int nfull = a == 0 ? g.n0g : (a == 1 ? g.n1 : g.n2);
      const int len = a == d - 1 ? nh : nfull;
      std::vector<double4> tab(len);
      for (int k = 0; k < len; ++k) {
        const double t = 2.0 * M_PI * (double)k / (double)nfull;
        tab[k] = make_double4(std::sin(t), std::cos(t), std::sin(0.5 * t), std::cos(0.5 * t));
      }
      ctx->d_tab[a] = dalloc<double4>(len);
      HB_CUDA(cudaMemcpy(ctx->d_tab[a], tab.data(), len * sizeof(double4), cudaMemcpyHostToDevice));
      p.tab[a] = ctx->d_tab[a];
    }
    if (const char* env = std::getenv("HOMFE_NO_WHILE_GRAPH")) ctx->use_while = ctx->use_while && env[0] == '0';
    if (const char* env = std::getenv("HOMFE_FAST2D")) ctx->no_fast2d = env[0] == '0';
    const char* fenv = std::getenv("HOMFE_FUSED_FFT");
    const bool fused_ok = fused_fft_eligible(g) && g.n1 % G == 0;
    if (dist && d == 2) {
      // 2-D row slabs (c5): 1-D r2c along axis 1 of the local rows, the
      // half-spectrum columns split over the ranks (nhl = ceil(nh / G) each,
      // the last chunk zero-padded), 1-D c2c along axis 0 on the rank's
      // columns. The 3-D slab layouts with a unit last axis: S
      // [c][i0l][k1 < G nhl][1], W [c][i0][k1l][1] (slabfft.cu, unchanged).
      SlabDims& sd = ctx->sd;
      const int nhl = (nh + G - 1) / G;
      sd = SlabDims{c, g.n0g, g.n0, G * nhl, nhl, 1, g.rank, G};
      int nr[1] = {g.n1}, nsp[1] = {G * nhl};
      HB_CUFFT(cufftPlanMany(&ctx->p2f, 1, nr, nr, 1, g.n1, nsp, 1, G * nhl, CUFFT_D2Z, c * g.n0));
      HB_CUFFT(cufftPlanMany(&ctx->p2i, 1, nr, nsp, 1, G * nhl, nr, 1, g.n1, CUFFT_Z2D, c * g.n0));
      int n1d[1] = {g.n0g};
      const int rs = nhl;  // axis-0 stride of W
      HB_CUFFT(cufftPlanMany(&ctx->p1, 1, n1d, n1d, rs, 1, n1d, rs, 1, CUFFT_Z2Z, rs));
      const int64_t tot = sd.chunk() * G;
      ctx->d_S = dalloc<double2>(tot);
      ctx->d_W = dalloc<double2>(tot);
      HB_CUDA(cudaMemset(ctx->d_S, 0, tot * sizeof(double2)));  // padding columns stay zero
      HB_CUDA(cudaMemset(ctx->d_W, 0, tot * sizeof(double2)));
      if (p2p_wanted(G)) setup_peers(ctx, ctx->d_W, ctx->d_S);
      if (G == 1) {
        ctx->peer_a[0] = ctx->d_W;
        ctx->peer_b[0] = ctx->d_S;
      }
      if (!ctx->peer && G > 1) {
        ctx->d_send = dalloc<double2>(tot);
        ctx->d_recv = dalloc<double2>(tot);
      }
      ctx->slab_fft = true;
    } else if (dist && !fused_ok) {
      // slab spectra for any plane size: cuFFT per rank + transposes (slabfft.cu)
      SlabDims& sd = ctx->sd;
      sd = SlabDims{c, g.n0g, g.n0, g.n1, g.n1 / G, g.n2 / 2 + 1, g.rank, G};
      const int nh2 = sd.nh;
      int n2d[2] = {g.n1, g.n2};
      HB_CUFFT(cufftPlanMany(&ctx->p2f, 2, n2d, nullptr, 1, g.n1 * g.n2, nullptr, 1, g.n1 * nh2, CUFFT_D2Z,
                             c * g.n0));
      HB_CUFFT(cufftPlanMany(&ctx->p2i, 2, n2d, nullptr, 1, g.n1 * nh2, nullptr, 1, g.n1 * g.n2, CUFFT_Z2D,
                             c * g.n0));
      int n1d[1] = {g.n0g};
      const int rs = sd.n1l * nh2;  // axis-0 stride of W
      HB_CUFFT(cufftPlanMany(&ctx->p1, 1, n1d, n1d, rs, 1, n1d, rs, 1, CUFFT_Z2Z, rs));
      const int64_t tot = sd.chunk() * G;
      ctx->d_S = dalloc<double2>(tot);
      ctx->d_W = dalloc<double2>(tot);
      if (p2p_wanted(G)) setup_peers(ctx, ctx->d_W, ctx->d_S);
      if (G == 1) {
        ctx->peer_a[0] = ctx->d_W;
        ctx->peer_b[0] = ctx->d_S;
      }
      if (!ctx->peer && G > 1) {
        ctx->d_send = dalloc<double2>(tot);
        ctx->d_recv = dalloc<double2>(tot);
      }
      ctx->slab_fft = true;
    }
    if (!dist && g.d == 2 && g.c == 1 && g.kind == 1 && g.nn == 1 && g.n0 == 256 && g.n1 == 256) {
      const char* e2 = std::getenv("HOMFE_SMALL2D");
      if (!(e2 && e2[0] == '0')) {
        std::vector<double2> tw;  // four-step layout tw[k2 * 16 + n1] = W_256^{n1 k2} (fft.cuh)
        for (int k2 = 0; k2 < 16; ++k2)
          for (int n1 = 0; n1 < 16; ++n1) {
            const double t = -2.0 * M_PI * (double)(n1 * k2) / 256.0;
            tw.push_back(make_double2(std::cos(t), std::sin(t)));
          }
        ctx->d_tw256 = dalloc<double2>(tw.size());
        HB_CUDA(cudaMemcpy(ctx->d_tw256, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
        ctx->small2d = true;
      }
    }
    if (fused_ok && (dist || !(fenv && fenv[0] == '0'))) {
      const int n1 = g.n1, n0 = g.n0g;
      // twiddles: N <= 256 in the four-step layout tw[k2 * (N/16) + n1] =
      // W_N^{n1 k2}; N = 512 as the plain table W_N^k (fft.cuh)
      auto table = [](int n, std::vector<double2>& out) {
        if (n <= 256) {
          const int A = n / 16;
          for (int k2 = 0; k2 < 16; ++k2)
            for (int n1 = 0; n1 < A; ++n1) {
              const double t = -2.0 * M_PI * (double)(n1 * k2) / (double)n;
              out.push_back(make_double2(std::cos(t), std::sin(t)));
            }
        } else {
          for (int k = 0; k < n; ++k) {
            const double t = -2.0 * M_PI * (double)k / (double)n;
            out.push_back(make_double2(std::cos(t), std::sin(t)));
          }
        }
      };
      std::vector<double2> tw;
      table(n1, tw);
      table(n0, tw);
      ctx->d_tw = dalloc<double2>(tw.size());
      HB_CUDA(cudaMemcpy(ctx->d_tw, tw.data(), tw.size() * sizeof(double2), cudaMemcpyHostToDevice));
      FusedFft& f = ctx->ff;
      f.n0 = g.n0;
      f.np_plane = n1;
      f.c = c;
      f.np = g.np;
      f.n0g = g.n0g;
      f.rank = g.rank;
      f.world = G;
      f.n1l = n1 / G;
      f.T = ctx->d_spec;
      ctx->d_spec2 = dalloc<double2>(fused_sz);
      f.T2 = ctx->d_spec2;
      if (p2p_wanted(G)) setup_peers(ctx, f.T, f.T2);
      if (ctx->peer) {
        // pass 2 / 3 read source q's chunk for this rank in place:
        // base[q] + t(q, ...) == T_q + t(me, ...), i.e. base[q] = T_q + (me - q) chunk
        const int me = g.rank;
        for (int q = 0; q < FusedFft::kMaxPeers; ++q) {
          const int qq = q < G ? q : 0;
          const auto tq = reinterpret_cast<uintptr_t>(ctx->peer_a[q]);
          const auto t2q = reinterpret_cast<uintptr_t>(ctx->peer_b[q]);
          f.tpull[q] = reinterpret_cast<const double2*>(tq + (intptr_t)(me - qq) * f.chunk_t() * (intptr_t)sizeof(double2));
          f.t2pull[q] =
              reinterpret_cast<const double2*>(t2q + (intptr_t)(me - qq) * f.chunk_t2() * (intptr_t)sizeof(double2));
        }
      }
      if (G > 1 && !ctx->peer) {
        ctx->d_spec_r = dalloc<double2>(fused_sz);
        ctx->d_spec2_r = dalloc<double2>(fused_sz);
        f.Trecv = ctx->d_spec_r;
        f.T2recv = ctx->d_spec2_r;
      } else {
        f.Trecv = f.T;
        f.T2recv = f.T2;
      }
      if (!ctx->peer)
        for (int q = 0; q < FusedFft::kMaxPeers; ++q) {
          f.tpull[q] = f.Trecv;
          f.t2pull[q] = f.T2recv;
        }
      f.tw_plane = ctx->d_tw;
      f.tw0 = ctx->d_tw + n1;
      fused_make_maps(f);
      ctx->fused = true;
      if (const char* dbg = std::getenv("HOMFE_FFT_DBG")) f.dbg = std::atoi(dbg);
    }
  } catch (...) {
    homfe_gpu_destroy(ctx);
    throw;
  }
  return ctx;
}

}  // namespace

extern "C" {

int homfe_gpu_create(const homfe_grid_desc* desc, homfe_ctx** out) {
  return guarded([&] {
    if (!out) throw ValidationError("create: null argument");
    *out = create_impl(desc, 0, 0, nullptr);
  });
}

int homfe_gpu_create_multi(const homfe_grid_desc* desc, int32_t n_gpus, homfe_ctx** out) {
  return guarded([&] {
    if (!desc || !out) throw ValidationError("create: null argument");
    if (n_gpus < 1) throw ValidationError("create_multi: n_gpus must be >= 1");
    if (n_gpus == 1) {
      *out = create_impl(desc, 0, 0, nullptr);
      return;
    }
    // HOMFE_MULTI_SIM=1: every rank on desc->device with the in-process
    // transport (host barriers; tests on one GPU), else ranks on devices
    // desc->device ... desc->device + n_gpus - 1 over NCCL
    const char* sim_env = std::getenv("HOMFE_MULTI_SIM");
    const bool sim = sim_env && sim_env[0] == '1';
    if (!sim) {
      int ndev = 0;
      HB_CUDA(cudaGetDeviceCount(&ndev));
      if (desc->device < 0 || desc->device + n_gpus > ndev)
        throw ValidationError("create_multi: " + std::to_string(n_gpus) + " devices requested from device " +
                              std::to_string(desc->device) + ", " + std::to_string(ndev) + " visible");
    }
    unsigned char id[128] = {};
    if (sim) {
      std::memcpy(id, "HBSIMGRP", 8);
      const uint64_t gid = g_multi_sim_group.fetch_add(1);
      std::memcpy(id + 8, &gid, 8);
    } else {
      ncclUniqueId uid;
      HB_NCCL(ncclGetUniqueId(&uid));
      std::memcpy(id, &uid, sizeof(uid));
    }
    auto* m = new homfe_ctx();
    m->device = desc->device;
    m->ranks.assign(n_gpus, nullptr);
    std::vector<std::string> errs(n_gpus);
    std::vector<std::thread> th;
    for (int r = 0; r < n_gpus; ++r)
      th.emplace_back([&, r] {
        homfe_grid_desc d = *desc;
        d.device = sim ? desc->device : desc->device + r;
        try {
          m->ranks[r] = create_impl(&d, r, n_gpus, id);
        } catch (const std::exception& e) {
          errs[r] = e.what();
        }
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < n_gpus; ++r)
      if (!errs[r].empty()) {
        for (homfe_ctx* rc : m->ranks)
          if (rc) homfe_gpu_destroy(rc);
        m->ranks.clear();
        delete m;
        throw ValidationError(errs[r]);
      }
    const homfe_ctx* r0 = m->ranks[0];
    m->mp_np = r0->g.np * n_gpus;
    m->mp_nq = m->mp_np * r0->sp.nq;
    m->mp_nf = r0->nf;
    m->mp_c = r0->g.c;
    m->mp_m = r0->g.m;
    *out = m;
  });
}

int homfe_nccl_unique_id(void* out) {
  return guarded([&] {
    ncclUniqueId id;
    HB_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int homfe_gpu_create_dist(const homfe_grid_desc* desc, int32_t rank, int32_t world, const void* nccl_id,
                          homfe_ctx** out) {
  return guarded([&] {
    if (!out) throw ValidationError("create: null argument");
    if (world < 1) throw ValidationError("slab mode: world must be >= 1");
    *out = create_impl(desc, rank, world, nccl_id);
  });
}

int homfe_gpu_slab_transport(const homfe_ctx* c, int32_t* kind) {
  if (is_multi(c)) return homfe_gpu_slab_transport(c->ranks[0], kind);
  return guarded([&] {
    if (!c || !kind) throw ValidationError("slab_transport: null argument");
    *kind = c->peer ? 2 : (c->dist && c->g.world > 1 ? 1 : 0);
  });
}

int homfe_gpu_destroy(homfe_ctx* c) {
  if (!c) return HOMFE_OK;
  if (is_multi(c)) {
    for (homfe_ctx* rc : c->ranks) homfe_gpu_destroy(rc);
    delete c;
    return HOMFE_OK;
  }
  cudaSetDevice(c->device);
  destroy_graphs(c);
  if (c->fwd) cufftDestroy(c->fwd);
  if (c->inv) cufftDestroy(c->inv);
  double* bufs[] = {c->d_x, c->d_r, c->d_p, c->d_ap, c->d_z, c->d_u, c->d_ke, c->d_fe, c->d_cmat, c->d_hexmat, c->d_tri,
                    c->d_strain, c->d_sx, c->d_sr, c->d_sp, c->d_sap, c->d_scp, c->d_g0, c->d_gtr, c->d_tanc,
                    c->d_sig, c->d_qs, c->d_tpart,
                    c->d_quad, c->d_partials, c->d_scal, c->d_hist, c->d_e};
  for (double* b : bufs)
    if (b) cudaFree(b);
  if (c->d_models) cudaFree(c->d_models);
  if (c->d_qtab) cudaFree(c->d_qtab);
  if (c->d_blocks) cudaFree(c->d_blocks);
  if (c->d_blocks_raw) cudaFree(c->d_blocks_raw);
  if (c->d_phase0) cudaFree(c->d_phase0);
  if (c->d_model0) cudaFree(c->d_model0);
  if (c->d_cref) cudaFree(c->d_cref);
  if (c->d_status) cudaFree(c->d_status);
  for (auto* t : c->d_tab)
    if (t) cudaFree(t);
  if (c->d_spec) cudaFree(c->d_spec);
  if (c->d_tw) cudaFree(c->d_tw);
  if (c->d_tw256) cudaFree(c->d_tw256);
  if (c->d_spec2) cudaFree(c->d_spec2);
  if (c->d_spec_r) cudaFree(c->d_spec_r);
  if (c->d_spec2_r) cudaFree(c->d_spec2_r);
  for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
  if (c->d_bar) cudaFree(c->d_bar);
  if (c->p2f) cufftDestroy(c->p2f);
  if (c->p2i) cufftDestroy(c->p2i);
  if (c->p1) cufftDestroy(c->p1);
  for (double2* b : {c->d_S, c->d_W, c->d_send, c->d_recv})
    if (b) cudaFree(b);
  if (c->d_hlo) cudaFree(c->d_hlo);
  if (c->d_hhi) cudaFree(c->d_hhi);
  if (c->d_ph_lo) cudaFree(c->d_ph_lo);
  if (c->d_red) cudaFree(c->d_red);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->d_phase) cudaFree(c->d_phase);
  if (c->d_st) cudaFree(c->d_st);
  if (c->h_st) cudaFreeHost(c->h_st);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  delete c;
  return HOMFE_OK;
}

int homfe_gpu_sizes(const homfe_ctx* c, int64_t* np, int64_t* nq, int32_t* m, int64_t* nf) {
  if (is_multi(c)) {
    if (np) *np = c->mp_np;
    if (nq) *nq = c->mp_nq;
    if (m) *m = c->mp_m;
    if (nf) *nf = c->mp_nf;
    return HOMFE_OK;
  }
  return guarded([&] {
    if (np) *np = c->g.np;
    if (nq) *nq = c->g.np * c->sp.nq;
    if (m) *m = c->g.m;
    if (nf) *nf = c->nf;
  });
}

int homfe_gpu_set_material(homfe_ctx* c, int32_t n_phases, const double* t, const uint8_t* phase) {
  if (is_multi(c)) {
    const int64_t nl = c->ranks[0]->g.np;
    return multi_run(c, [&](homfe_ctx* rc, int r) {
      return homfe_gpu_set_material(rc, n_phases, t, phase ? phase + (size_t)r * nl : nullptr);
    });
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    c->nonlinear = false;
    c->qt_ok = false;
    set_material(c, n_phases, t, phase, false);
  });
}

int homfe_gpu_set_material_device(homfe_ctx* c, int32_t n_phases, const double* t, const uint8_t* d_phase) {
  if (is_multi(c)) return multi_unsupported("gpu_set_material_device");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    set_material(c, n_phases, t, d_phase, true);
  });
}

int homfe_gpu_precond_reset(homfe_ctx* c) {
  if (is_multi(c)) return multi_run(c, [&](homfe_ctx* rc, int) { return homfe_gpu_precond_reset(rc); });
  return guarded([&] {
    if (!c) throw ValidationError("precond_reset: null context");
    c->pm_valid = false;
    c->pm_mean.clear();
    c->pm_cref.clear();
  });
}

int homfe_gpu_solve(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, const double* warm_u,
                    double* u_out, double* avg_out, homfe_report* rep) {
  if (is_multi(c)) {
    const MultiSplit sp = split_of(c);
    std::vector<std::vector<double>> ul(c->ranks.size());
    std::vector<homfe_report> reps(c->ranks.size());
    std::vector<std::vector<double>> avgs(c->ranks.size(), std::vector<double>(6, 0.0));
    const int code = multi_run(c, [&](homfe_ctx* rc, int r) {
      std::vector<double> wl;
      if (warm_u) sp.scatter(warm_u, wl, r);
      ul[r].assign((size_t)sp.c * sp.n_loc, 0.0);
      return homfe_gpu_solve(rc, e, cfg, warm_u ? wl.data() : nullptr, ul[r].data(), avgs[r].data(), &reps[r]);
    });
    if (code == HOMFE_OK || code == HOMFE_NONCONVERGED) {
      if (u_out)
        for (size_t r = 0; r < ul.size(); ++r) sp.gather(ul[r], u_out, (int)r);
      if (avg_out) std::copy(avgs[0].begin(), avgs[0].begin() + c->mp_m, avg_out);
      if (rep) *rep = reps[0];
    }
    return code;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->nvec();
    if (warm_u) HB_CUDA(cudaMemcpyAsync(c->d_u, warm_u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    else HB_CUDA(cudaMemsetAsync(c->d_u, 0, n * sizeof(double), c->stream));
    homfe_report local;
    homfe_report* r = rep ? rep : &local;
    solve_dispatch(c, e, cfg, avg_out, r);
    if (u_out) HB_CUDA(cudaMemcpyAsync(u_out, c->d_u, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (!r->converged) throw NonConverged(r->cause == 1 ? "cg-stall" : "newton-cap");
  });
}

int homfe_gpu_set_material_models(homfe_ctx* c, int32_t n_phases, const homfe_material* models,
                                  const uint8_t* phase) {
  if (is_multi(c)) return multi_unsupported("gpu_set_material_models");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    if (!models) throw ValidationError("materials: null catalog");
    if (n_phases < 1) throw ValidationError("materials: catalog is empty");
    if (n_phases > kMaxPhases) throw ValidationError("materials: at most 256 phases");
    const int m = c->g.m, d = c->g.d;
    bool nonlinear = false;
    std::vector<double> eff((size_t)n_phases * m * m);
    std::vector<NLModel> nm(n_phases);
    for (int ph = 0; ph < n_phases; ++ph) {
      const homfe_material& md = models[ph];
      if (md.kind == HOMFE_MATERIAL_LINEAR) {
        std::copy(md.tangent, md.tangent + m * m, eff.begin() + (size_t)ph * m * m);
        nm[ph] = NLModel{0, 0.0, 0.0, 0.0, 0.0};
      } else if (md.kind == HOMFE_MATERIAL_J2) {
        if (!(md.bulk > 0.0) || !(md.shear > 0.0) || !(md.yield_stress > 0.0))
          throw ValidationError("j2_plastic: K, G and tau_y0 must be > 0");
        if (md.hardening < 0.0) throw ValidationError("j2_plastic: H must be >= 0");
        if (c->g.c == 1) throw ValidationError("materials: mixed thermal and mechanical models");
        if (c->dist) throw ValidationError("j2_plastic: the nonlinear path runs on one GPU");
        isotropic_stiffness(md.bulk, md.shear, d, &eff[(size_t)ph * m * m]);  // elastic tables
        nm[ph] = NLModel{1, md.bulk, md.shear, md.yield_stress, md.hardening};
        nonlinear = true;
      } else {
        throw ValidationError("materials: unknown model kind");
      }
    }
    c->nonlinear = false;
    set_material(c, n_phases, eff.data(), phase, false);
    ensure_nl_buffers(c);
    c->models = nm;
    HB_CUDA(cudaMemcpy(c->d_models, nm.data(), nm.size() * sizeof(NLModel), cudaMemcpyHostToDevice));
    c->nonlinear = nonlinear;
    // modal-kernel table for the J2 operator: isotropic linear phases as
    // (1, lambda + 2 mu / 3, mu), J2 phases as (0, k, G)
    bool qt_ok = nonlinear && c->g.c == 3 && c->g.d == 3;
    std::vector<double> qtab((size_t)n_phases * 3, 0.0);
    for (int ph = 0; ph < n_phases && qt_ok; ++ph) {
      if (nm[ph].kind == 1) {
        qtab[ph * 3 + 0] = 0.0;
        qtab[ph * 3 + 1] = nm[ph].k;
        qtab[ph * 3 + 2] = nm[ph].g;
        continue;
      }
      const double* cm = &eff[(size_t)ph * m * m];
      auto C = [&](int i, int j) { return cm[j * m + i]; };
      const double lam = C(0, 1), twomu = C(3, 3);
      const double tol = 8e-16 * (std::fabs(lam) + std::fabs(twomu));
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
          const double want = (i < 3 && j < 3) ? (i == j ? lam + twomu : lam) : (i == j ? twomu : 0.0);
          if (std::fabs(C(i, j) - want) > tol) qt_ok = false;
        }
      qtab[ph * 3 + 0] = 1.0;
      qtab[ph * 3 + 1] = lam + twomu / 3.0;
      qtab[ph * 3 + 2] = 0.5 * twomu;
    }
    if (const char* env = std::getenv("HOMFE_J2_FAST")) qt_ok = qt_ok && env[0] != '0';
    if (qt_ok) {
      if (!c->d_qtab) c->d_qtab = dalloc<double>((size_t)kMaxPhases * 3);
      HB_CUDA(cudaMemcpy(c->d_qtab, qtab.data(), qtab.size() * sizeof(double), cudaMemcpyHostToDevice));
    }
    if (qt_ok != c->qt_ok) destroy_graphs(c);
    c->qt_ok = qt_ok;
  });
}

int homfe_gpu_internal_width(homfe_ctx* c, int32_t* width, int64_t* num_quads) {
  if (is_multi(c)) return multi_unsupported("gpu_internal_width");
  return guarded([&] {
    if (width) *width = c->nonlinear ? 7 : 0;
    if (num_quads) *num_quads = c->g.np * c->sp.nq;
  });
}

int homfe_gpu_solve_state(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, const double* warm_u,
                          const double* g0, double* u_out, double* g_out, double* avg_out, homfe_report* rep) {
  if (is_multi(c)) return multi_unsupported("gpu_solve_state");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->nvec();
    const size_t gq = (size_t)c->g.np * c->sp.nq * 7;
    if (warm_u) HB_CUDA(cudaMemcpyAsync(c->d_u, warm_u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    else HB_CUDA(cudaMemsetAsync(c->d_u, 0, n * sizeof(double), c->stream));
    homfe_report local;
    homfe_report* r = rep ? rep : &local;
    if (c->nonlinear || c->g.nn > 1) {
      if (g0) HB_CUDA(cudaMemcpyAsync(c->d_g0, g0, gq * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      else HB_CUDA(cudaMemsetAsync(c->d_g0, 0, gq * sizeof(double), c->stream));
      const bool ok = newton_nl(c, e, cfg, avg_out, r);
      if (g_out)
        HB_CUDA(cudaMemcpyAsync(g_out, ok ? c->d_gtr : c->d_g0, gq * sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream));
    } else {
      newton(c, e, cfg, avg_out, r);
    }
    if (u_out) HB_CUDA(cudaMemcpyAsync(u_out, c->d_u, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (!r->converged) throw NonConverged(r->cause == 1 ? "cg-stall" : "newton-cap");
  });
}

int homfe_gpu_gamma_apply(homfe_ctx* c, const double* s_in, double* s_out) {
  if (is_multi(c)) return multi_unsupported("gpu_gamma_apply");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_reference(c);
    if (c->dist) throw ValidationError("gamma_apply: single-GPU contexts only");
    ensure_sb_buffers(c);
    const size_t n = (size_t)c->g.np * c->sp.nq * c->g.m;
    HB_CUDA(cudaMemcpyAsync(c->d_sp, s_in, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    gamma_apply(c, c->d_sp, c->d_sap, c->stream);
    HB_CUDA(cudaMemcpyAsync(s_out, c->d_sap, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_sb_solve(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, const double* c_ref,
                       const double* warm_strain, const double* g0, double* strain_out, double* g_out,
                       double* avg_out, homfe_report* rep) {
  if (is_multi(c)) return multi_unsupported("gpu_sb_solve");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    if (!c_ref) throw ValidationError("sb_newton_solve: reference tangent required");
    require_material(c);
    ensure_nl_buffers(c);
    ensure_sb_buffers(c);
    const int64_t nq = c->g.np * c->sp.nq;
    const size_t ns = (size_t)nq * c->g.m, gq = (size_t)nq * 7;
    if (warm_strain) HB_CUDA(cudaMemcpyAsync(c->d_strain, warm_strain, ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    else HB_CUDA(cudaMemsetAsync(c->d_strain, 0, ns * sizeof(double), c->stream));
    if (c->nonlinear) {
      if (g0) HB_CUDA(cudaMemcpyAsync(c->d_g0, g0, gq * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      else HB_CUDA(cudaMemsetAsync(c->d_g0, 0, gq * sizeof(double), c->stream));
    }
    homfe_report local;
    homfe_report* r = rep ? rep : &local;
    const bool ok = sb_newton(c, e, cfg, c_ref, avg_out, r);
    if (strain_out)
      HB_CUDA(cudaMemcpyAsync(strain_out, c->d_strain, ns * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (g_out && c->nonlinear)
      HB_CUDA(cudaMemcpyAsync(g_out, ok ? c->d_gtr : c->d_g0, gq * sizeof(double), cudaMemcpyDeviceToHost,
                              c->stream));
    sync(c);
    if (!r->converged) throw NonConverged(r->cause == 1 ? "cg-stall" : "newton-cap");
  });
}

int homfe_gpu_eigenvalue_bounds(homfe_ctx* c, const double* tangent, int32_t pixel_constant, const double* c_ref,
                                double* lower, double* upper, double* cond) {
  if (is_multi(c)) return multi_unsupported("gpu_eigenvalue_bounds");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    if (c->dist) throw ValidationError("eigenvalue_bounds: single-GPU contexts only");
    const int m = c->g.m;
    // C_ref = L L^T (spectral.cpp:41-53)
    std::vector<double> L(m * m, 0.0), Li(m * m, 0.0);
    for (int j = 0; j < m; ++j) {
      double sum = c_ref[j * m + j];
      for (int k = 0; k < j; ++k) sum -= L[j * m + k] * L[j * m + k];
      if (!(sum > 0.0)) throw ValidationError("eigenvalue_bounds: reference must be positive definite");
      L[j * m + j] = std::sqrt(sum);
      for (int i = j + 1; i < m; ++i) {
        double t = c_ref[j * m + i];
        for (int k = 0; k < j; ++k) t -= L[i * m + k] * L[j * m + k];
        L[i * m + j] = t / L[j * m + j];
      }
    }
    for (int col = 0; col < m; ++col)
      for (int i = 0; i < m; ++i) {
        double t = i == col ? 1.0 : 0.0;
        for (int k = 0; k < i; ++k) t -= L[i * m + k] * Li[k * m + col];
        Li[i * m + col] = t / L[i * m + i];
      }
    const int64_t nq = c->g.np * c->sp.nq, nn = c->nodes();
    const int cc = c->g.c;
    Scratch scratch;
    double* d_t = scratch.alloc<double>((size_t)nq * m * m);
    double* d_lo = scratch.alloc<double>((size_t)nn * cc);
    double* d_hi = scratch.alloc<double>((size_t)nn * cc);
    double* d_lo2 = scratch.alloc<double>((size_t)nn * cc);
    double* d_hi2 = scratch.alloc<double>((size_t)nn * cc);
    HB_CUDA(cudaMemcpyAsync(d_t, tangent, (size_t)nq * m * m * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const int st = bounds_device(c->g, c->sp, d_t, pixel_constant, Li.data(), cc, d_lo, d_hi, c->stream);
    if (st == 2) throw ValidationError("eigenvalue_bounds: tangent must be positive definite per point");
    // sorted sequences (spectral.cpp:115-116): device radix sort
    size_t tmp_bytes = 0;
    const int nk = (int)(nn * cc);
    HB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_lo, d_lo2, nk, 0, 64, c->stream));
    void* d_tmp = scratch.alloc<unsigned char>(tmp_bytes);
    HB_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_bytes, d_lo, d_lo2, nk, 0, 64, c->stream));
    HB_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, tmp_bytes, d_hi, d_hi2, nk, 0, 64, c->stream));
    HB_CUDA(cudaMemcpyAsync(lower, d_lo2, (size_t)nk * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    HB_CUDA(cudaMemcpyAsync(upper, d_hi2, (size_t)nk * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (!(lower[0] > 0.0)) throw ValidationError("condition_estimate: bounds must be positive");
    if (cond) *cond = upper[nk - 1] / lower[0];
  });
}

int homfe_gpu_stress_field(homfe_ctx* c, double* out) {
  if (is_multi(c)) return multi_unsupported("gpu_stress_field");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_material(c);
    if (c->dist) throw ValidationError("stress_field: single-GPU contexts only");
    if (!c->sig_valid) {
      // linear solve: sigma = C (e + D u) at the last solution (solver.cpp:321-324)
      ensure_nl_buffers(c);
      if ((int)c->models.size() != c->n_phases) {
        c->models.assign(c->n_phases, NLModel{0, 0.0, 0.0, 0.0, 0.0});
        HB_CUDA(cudaMemcpy(c->d_models, c->models.data(), c->models.size() * sizeof(NLModel),
                           cudaMemcpyHostToDevice));
      }
      nl_sweep(c);
    }
    const size_t nq = (size_t)c->g.np * c->sp.nq * c->g.m;
    HB_CUDA(cudaMemcpyAsync(out, c->d_sig, nq * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_solve_device(homfe_ctx* c, const double* e, const homfe_solve_cfg* cfg, const double* d_warm,
                           double* d_u_out, double* avg_out, homfe_report* rep) {
  if (is_multi(c)) return multi_unsupported("gpu_solve_device");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->nvec();
    if (d_warm) HB_CUDA(cudaMemcpyAsync(c->d_u, d_warm, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    else HB_CUDA(cudaMemsetAsync(c->d_u, 0, n * sizeof(double), c->stream));
    homfe_report local;
    homfe_report* r = rep ? rep : &local;
    solve_dispatch(c, e, cfg, avg_out, r);
    if (d_u_out) HB_CUDA(cudaMemcpyAsync(d_u_out, c->d_u, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    sync(c);
    if (!r->converged) throw NonConverged(r->cause == 1 ? "cg-stall" : "newton-cap");
  });
}

int homfe_gpu_apply_K(homfe_ctx* c, const double* u, double* ku) {
  if (is_multi(c))
    return multi_map(c, u, ku, [](homfe_ctx* rc, const double* x, double* y) { return homfe_gpu_apply_K(rc, x, y); });
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_material(c);
    const int64_t n = c->nvec();
    if (c->peer) peer_barrier(c, c->stream);  // no peer still reads the previous d_p
    HB_CUDA(cudaMemcpyAsync(c->d_p, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    apply_K(c, c->d_p, c->d_ap, nullptr, 1.0, nullptr, nullptr, c->stream);
    HB_CUDA(cudaMemcpyAsync(ku, c->d_ap, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_set_reference(homfe_ctx* c, const double* c_ref) {
  if (is_multi(c)) return multi_run(c, [&](homfe_ctx* rc, int) { return homfe_gpu_set_reference(rc, c_ref); });
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    set_reference(c, c_ref);
  });
}

int homfe_gpu_apply_minv(homfe_ctx* c, const double* r, double* z) {
  if (is_multi(c))
    return multi_map(c, r, z, [](homfe_ctx* rc, const double* x, double* y) { return homfe_gpu_apply_minv(rc, x, y); });
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_reference(c);
    const int64_t n = c->nvec();
    HB_CUDA(cudaMemcpyAsync(c->d_r, r, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    precond_apply(c, c->d_r, c->d_z, nullptr, nullptr, c->stream);
    HB_CUDA(cudaMemcpyAsync(z, c->d_z, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_reference_blocks(homfe_ctx* c, double* blocks) {
  if (is_multi(c)) return multi_unsupported("gpu_reference_blocks");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_reference(c);
    if (c->g.nn > 1) {
      const size_t cntb = (size_t)c->nf * c->g.c * c->g.nn * c->g.c * c->g.nn;
      HB_CUDA(cudaMemcpyAsync(blocks, c->d_blocks_raw, cntb * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      return;
    }
    const size_t cnt = (size_t)c->nf * c->g.c * c->g.c;
    Scratch scratch;
    double2* d = scratch.alloc<double2>(cnt);
    launch_symbol_dump(c->spp, d, c->stream);
    HB_CUDA(cudaMemcpyAsync(blocks, d, cnt * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

static double* quad_buffer(homfe_ctx* c) {
  if (!c->d_quad) c->d_quad = dalloc<double>((size_t)c->g.np * c->sp.nq * c->g.m);
  return c->d_quad;
}

int homfe_gpu_gradient(homfe_ctx* c, const double* u, double* grad) {
  if (is_multi(c)) return multi_unsupported("gpu_gradient");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->nvec();
    double* q = quad_buffer(c);
    HB_CUDA(cudaMemcpyAsync(c->d_p, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    QuadArgs a{c->d_p, nullptr, nullptr, c->d_phase, c->d_cmat, q, nullptr};
    launch_quad(c->g, c->sp, kQuadGrad, a, c->stream);
    HB_CUDA(cudaMemcpyAsync(grad, q, (size_t)c->g.np * c->sp.nq * c->g.m * sizeof(double), cudaMemcpyDeviceToHost,
                            c->stream));
    sync(c);
  });
}

int homfe_gpu_divergence(homfe_ctx* c, const double* s, int32_t weighted, double* out) {
  if (is_multi(c)) return multi_unsupported("gpu_divergence");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const int64_t n = c->nvec();
    double* q = quad_buffer(c);
    HB_CUDA(cudaMemcpyAsync(q, s, (size_t)c->g.np * c->sp.nq * c->g.m * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
    launch_divergence(c->g, c->sp, q, weighted != 0, c->d_ap, c->stream);
    HB_CUDA(cudaMemcpyAsync(out, c->d_ap, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_apply_tangent_field(homfe_ctx* c, const double* tangent, const double* u, double* ku) {
  if (is_multi(c)) return multi_unsupported("gpu_apply_tangent_field");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    if (!tangent || !u || !ku) throw ValidationError("apply_tangent_field: null argument");
    const int64_t n = c->nvec();
    const size_t nq = (size_t)c->g.np * c->sp.nq, mm = (size_t)c->g.m * c->g.m;
    Scratch scr;
    double* d_t = scr.alloc<double>(nq * mm);
    double* q = quad_buffer(c);
    HB_CUDA(cudaMemcpyAsync(d_t, tangent, nq * mm * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    HB_CUDA(cudaMemcpyAsync(c->d_p, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    QuadArgs a{c->d_p, nullptr, nullptr, c->d_phase, c->d_cmat, q, nullptr};
    launch_quad(c->g, c->sp, kQuadGrad, a, c->stream);          // eps_q = D u
    launch_tangent_field(c->g, c->sp, d_t, q, c->stream);        // sigma_q = C_q eps_q
    launch_divergence(c->g, c->sp, q, true, c->d_ap, c->stream);  // D^T W sigma
    HB_CUDA(cudaMemcpyAsync(ku, c->d_ap, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
  });
}

int homfe_gpu_weighted_dot(homfe_ctx* c, const double* a, const double* b, double* out) {
  if (is_multi(c)) return multi_unsupported("gpu_weighted_dot");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    if (!a || !b || !out) throw ValidationError("weighted_dot: null argument");
    HB_CUDA(cudaSetDevice(c->device));
    const size_t n = (size_t)c->g.np * c->sp.nq * c->g.m;
    Scratch scratch;
    double* da = scratch.alloc<double>(n);
    double* db = a == b ? da : scratch.alloc<double>(n);
    HB_CUDA(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    if (db != da) HB_CUDA(cudaMemcpyAsync(db, b, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    launch_quad_wdot(c->g, c->sp, da, db, c->d_partials, c->stream);
    reduce_to_host(c, 1, out);
  });
}

int homfe_gpu_volume_average(homfe_ctx* c, const double* s, double* out) {
  if (is_multi(c)) return multi_unsupported("gpu_volume_average");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    double* q = quad_buffer(c);
    HB_CUDA(cudaMemcpyAsync(q, s, (size_t)c->g.np * c->sp.nq * c->g.m * sizeof(double), cudaMemcpyHostToDevice,
                            c->stream));
    launch_quad_wsum(c->g, c->sp, q, c->d_partials, c->stream);
    double v[6];
    reduce_to_host(c, c->g.m, v);
    for (int k = 0; k < c->g.m; ++k) out[k] = v[k] / c->g.cell_volume;
  });
}

int homfe_gpu_pcg(homfe_ctx* c, const double* b, double eta, int32_t it_max, double* x, int32_t* iterations,
                  double* history, int32_t* converged) {
  if (is_multi(c)) {
    std::vector<int32_t> its(c->ranks.size()), conv(c->ranks.size());
    std::vector<double> hist0;
    if (history) hist0.assign((size_t)std::max(it_max, 0) + 1, 0.0);
    const int code = multi_map(c, b, x, [&](homfe_ctx* rc, const double* bl, double* xl) {
      int r = 0;
      while (c->ranks[r] != rc) ++r;
      return homfe_gpu_pcg(rc, bl, eta, it_max, xl, &its[r], r == 0 && history ? hist0.data() : nullptr, &conv[r]);
    });
    if (code == HOMFE_OK) {
      if (iterations) *iterations = its[0];
      if (converged) *converged = conv[0];
      if (history) std::copy(hist0.begin(), hist0.begin() + its[0] + 1, history);
    }
    return code;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_material(c);
    require_reference(c);
    if (it_max < 0) throw ValidationError("pcg: it_max must be >= 0");
    const int64_t n = c->nvec();
    HB_CUDA(cudaMemcpyAsync(c->d_r, b, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const PcgResult r = run_pcg(c, eta, it_max, history);
    HB_CUDA(cudaMemcpyAsync(x, c->d_x, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

int homfe_gpu_pcg_observed(homfe_ctx* c, const double* b, double eta, int32_t it_max, double* x,
                           int32_t* iterations, double* history, int32_t* converged, homfe_iterate_observer obs,
                           void* user) {
  if (is_multi(c)) return multi_unsupported("gpu_pcg_observed");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_material(c);
    require_reference(c);
    if (it_max < 0) throw ValidationError("pcg: it_max must be >= 0");
    if (c->dist) throw ValidationError("pcg_observed: single-GPU contexts only");
    const int64_t n = c->nvec();
    HB_CUDA(cudaMemcpyAsync(c->d_r, b, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const PcgResult r = run_pcg(c, eta, it_max, history, obs, user);
    HB_CUDA(cudaMemcpyAsync(x, c->d_x, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    sync(c);
    if (iterations) *iterations = r.iterations;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

// Per-stage CUDA-event timing of one PCG iteration on the context's current
// buffers (after a solve): 0 K apply, 1 x/r update, 2 forward FFT,
// 3 spectral solve, 4 inverse FFT, 5 p update, 6 the two tiny scalar kernels,
// 7 their sum. Averages over `reps` launches.
int homfe_gpu_kernel_times(homfe_ctx* c, int32_t reps, double* ms) {
  if (is_multi(c)) return multi_unsupported("gpu_kernel_times");
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    require_material(c);
    require_reference(c);
    if (reps < 1) throw ValidationError("kernel_times: reps must be >= 1");
    if (c->hist_cap < 2) {
      destroy_graphs(c);
      c->hist_cap = 2;
      c->d_hist = dalloc<double>(2);
    }
    const int64_t n = c->nvec();
    cudaStream_t s = c->stream;
    // live, never-finishing state with alpha = beta = 0: full memory traffic,
    // unchanged values
    write_state(c, 0.0, 1 << 30, 1);
    sync(c);
    cudaEvent_t a, b;
    HB_CUDA(cudaEventCreate(&a));
    HB_CUDA(cudaEventCreate(&b));
    auto timeit = [&](auto&& fn) {
      fn();  // warm
      HB_CUDA(cudaEventRecord(a, s));
      for (int i = 0; i < reps; ++i) fn();
      HB_CUDA(cudaEventRecord(b, s));
      HB_CUDA(cudaEventSynchronize(b));
      float t = 0.f;
      HB_CUDA(cudaEventElapsedTime(&t, a, b));
      return (double)t / reps;
    };
    ms[0] = timeit([&] { apply_K(c, c->d_p, c->d_ap, nullptr, 1.0, c->d_partials, c->d_st, s); });
    if (c->fused) {
      // pass 1 (r update + forward plane FFTs), pass 2 (pencils + solve)
      ms[1] = timeit([&] { fused_forward(c->ff, c->spp, c->d_r, c->d_ap, c->d_st, nullptr, s, 1); });
      ms[2] = -1.0;
      ms[3] = timeit([&] { fused_forward(c->ff, c->spp, c->d_r, c->d_ap, c->d_st, c->d_partials, s, 2); });
      ms[4] = -1.0;
      ms[5] = timeit([&] { fused_inverse(c->ff, c->d_p, c->d_x, nullptr, c->d_st, 0, s); });
      ms[6] = timeit([&] {
        launch_pcg_alpha(c->d_st, c->d_partials, s);
        launch_pcg_beta(c->d_st, c->d_partials, c->d_hist, s);
      });
      ms[7] = ms[0] + ms[1] + ms[3] + ms[5] + ms[6];
      cudaEventDestroy(a);
      cudaEventDestroy(b);
      return;
    }
    ms[1] = timeit([&] { launch_update_r(c->d_r, c->d_ap, n, c->d_st, s); });
    if (c->slab_fft) {  // with the transposes (exchange included)
      ms[2] = timeit([&] { slab_forward(c, c->d_r, s); });
      ms[3] = timeit([&] { slab_solve(c, c->d_st, c->d_partials, s); });
      ms[4] = timeit([&] { slab_inverse(c, c->d_z, s); });
    } else {
      ms[2] = timeit([&] { fft_forward(c, c->d_r, s); });
      ms[3] = timeit([&] { launch_spectral(c->spp, c->d_spec, c->d_st, c->d_partials, s); });
      ms[4] = timeit([&] { fft_inverse(c, c->d_z, s); });
    }
    ms[5] = timeit([&] { launch_update_xp(c->d_x, c->d_p, c->d_z, n, c->d_st, s); });
    ms[6] = timeit([&] {
      launch_pcg_alpha(c->d_st, c->d_partials, s);
      launch_pcg_beta(c->d_st, c->d_partials, c->d_hist, s);
    });
    ms[7] = ms[0] + ms[1] + ms[2] + ms[3] + ms[4] + ms[5] + ms[6];
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

int homfe_gpu_path_info(const homfe_ctx* c, int32_t* flags) {
  if (is_multi(c)) {
    const int code = homfe_gpu_path_info(c->ranks[0], flags);
    if (code == HOMFE_OK && flags) *flags |= HOMFE_PATH_MULTI;
    return code;
  }
  return guarded([&] {
    if (!c || !flags) throw ValidationError("path_info: null argument");
    *flags = (c->fused ? HOMFE_PATH_FUSED_FFT : 0) | (c->hex_fast ? HOMFE_PATH_HEX_MODAL : 0) |
             (c->use_while ? HOMFE_PATH_WHILE_GRAPH : 0) | (c->slab_fft ? HOMFE_PATH_SLAB_SPECTRA : 0) |
             (c->dist ? HOMFE_PATH_SLAB : 0) | (c->peer ? HOMFE_PATH_PEER_PULL : 0) |
             (elem2d_eligible(c->g) && !c->no_fast2d ? HOMFE_PATH_ELEM2D : 0) |
             (c->small2d && small2d_eligible(c->g, c->n_phases) ? HOMFE_PATH_SMALL2D : 0);
  });
}

int homfe_gpu_index_maps(homfe_ctx* c, int64_t* strides3, int64_t* nbr, int32_t* n_off) {
  if (is_multi(c)) return multi_unsupported("gpu_index_maps");
  if (c && c->dist) {
    g_err = "not available in slab mode (use a single-device context)";
    return HOMFE_VALIDATION;
  }
  return guarded([&] {
    HB_CUDA(cudaSetDevice(c->device));
    const Grid& g = c->g;
    if (strides3) {
      strides3[0] = g.d == 3 ? (int64_t)g.n1 * g.n2 : g.n1;
      strides3[1] = g.d == 3 ? g.n2 : 1;
      strides3[2] = g.d == 3 ? 1 : 0;
    }
    if (n_off) *n_off = c->sp.noff;
    if (nbr) {
      const size_t cnt = (size_t)g.np * c->sp.noff;
      int64_t* d = dalloc<int64_t>(cnt);
      launch_index_maps(g, c->sp, d, c->stream);
      HB_CUDA(cudaMemcpyAsync(nbr, d, cnt * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      sync(c);
      cudaFree(d);
    }
  });
}

}  // extern "C"
