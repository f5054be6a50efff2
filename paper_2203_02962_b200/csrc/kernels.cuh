// kernels.cuh -- launchers of the homfe B200 device kernels.
#pragma once

#include <cuComplex.h>

#include <vector>

#include "common.cuh"

namespace hb {

constexpr int kBlock = 256;
constexpr int kRedBlocks = 1184;  // 8 x 148 SMs: fixed grid => deterministic sums

struct ElemArgs {
  const double* u;
  const double* halo_lo;  // dist: plane z0-1 of u ([c][plane]); nullable otherwise
  const double* halo_hi;  // dist: plane z0+nz of u
  const uint8_t* ph_lo;   // dist: phase plane z0-1
  double* out;
  const uint8_t* phase;
  const double* ke;       // n_phases x NE x NE, row-major
  int n_phases;
  const double* fe;       // nullable: n_phases x NE load vectors
  double scale;           // out = scale * (K u + f)
  double* partials;       // nullable: per-block sum of u . out
  const PcgState* st;     // nullable: skip when st->done
  int64_t halo_cs;        // component stride of the halo planes (0: one plane, i.e.
                          // exchanged buffers; np when they point into a peer's field)
};

// Node-centric K u (+ f) from per-phase element matrices; any grid size.
void launch_apply_elem(const Grid& g, const ElemArgs& a, cudaStream_t s);
// Element-centric modal fast path for trilinear hex on cubic voxels
// (hexfast.cu). Tables: per-phase material data in the modal basis.
bool hex_fast_eligible(const Grid& g);
bool hex_fast_tables(const Grid& g, int n_phases, const double* cmats, std::vector<double>& iso,
                     std::vector<double>& gen);
void launch_hex_fast(const Grid& g, const ElemArgs& a, const double* d_mat, bool iso, cudaStream_t s);
// 2-D one-node pixel stencils: warp-strip element-matrix K u (quad2d.cu)
bool elem2d_eligible(const Grid& g);
void elem2d_tri_tables(const Grid& g, int n_phases, const double* cmats, std::vector<double>& tab);
void launch_elem2d(const Grid& g, const ElemArgs& a, const double* d_tri, cudaStream_t s);
// Nonlinear (J2) path, j2.cu. Per phase: kind 0 linear (catalog matrix in
// cmat), 1 J2 (bulk k, shear g, yield stress tau0, hardening).
struct NLModel {
  int kind;
  double k, g, tau0, hard;
};
struct NLArgs {
  const double* u;        // nodal field (c x N)
  const double* e;        // macro strain (m), sweep only
  const uint8_t* phase;
  const NLModel* models;
  const double* cmat;     // n_phases x m x m column-major
  const double* g0;       // committed internal state (7 per quad)
  double* g_trial;        // trial internal state (7 per quad)
  double* tanc;           // compact tangent (a, b, n[6]) per quad
  double* sig;            // stress quad field (m per quad)
  double* partials;       // sweep: per block m x m of sum_q w C_q
  int* status;            // sweep: set to 1 on a non-finite strain
  int width;              // internal width (7 when any J2 phase)
  const double* qeps;     // sweep: quad strain field (strain-based scheme) instead of D u
};
void launch_sweep(const Grid& g, const StencilParams& sp, const NLArgs& a, cudaStream_t s);
// y_q = C_q x_q over the quad field (tangent_multiply, strain-based scheme)
void launch_tan_mult(const Grid& g, const StencilParams& sp, const NLArgs& a, const double* x, double* y,
                     cudaStream_t s);
// per-block partials of sum_q |x_q + E|^2 (E nullable)
void launch_qshift_norm2(const double* x, const double* e, int64_t nq, int m, double* partials, cudaStream_t s);
// eigenvalue_bounds (spectral.cpp:33-118) on the device: per-point pencil
// extremes, node min/max over supports, sorted; returns 0 or a status
// (1: reference not SPD handled by the host; 2: tangent not PD at a point)
int bounds_device(const Grid& g, const StencilParams& sp, const double* d_tangent, int pixel_constant,
                  const double* linv_rowmajor, int c, double* d_lower, double* d_upper, cudaStream_t s);
void launch_tan_stress(const Grid& g, const StencilParams& sp, const NLArgs& a, const PcgState* st, cudaStream_t s);
// impulse-probed block preconditioner (probe.cu), Nn = 2 stencils
void launch_probe_store(const double2* spec, int b, int64_t nf, int col, double2* blocks, cudaStream_t s);
void launch_probe_invert(double2* blocks, int64_t nf, int b, int nn, int* status, cudaStream_t s);
void launch_probe_apply(double2* spec, const double2* blocks, int64_t nf, int b, double scale, cudaStream_t s);
void launch_phase_counts(const uint8_t* ph, int64_t n, unsigned long long* counts, cudaStream_t s);
// J2 path: K u with per-Gauss-point compact tangents (false if not eligible)
bool launch_hex_fast_qt(const Grid& g, const ElemArgs& a, const double* d_qtab, const double* d_tanc,
                        cudaStream_t s);
// mode 0: sum_q w |D u + e|^2 / h^3 (1 partial per block); 1: sum_q w C (D u + e) / h^3 (m per block)
bool launch_hex_quad(const Grid& g, int mode, const double* u, const double* halo_hi, const double* e,
                     const uint8_t* phase, const double* cmat, double* partials, cudaStream_t s);

enum QuadMode { kQuadGrad = 0, kQuadNorm2 = 1, kQuadStress = 2 };
struct QuadArgs {
  const double* u;        // nullable => zero field
  const double* halo_hi;  // dist: plane z0+nz of u ([c][plane])
  const double* e;        // nullable => no macroscopic term (device, m doubles)
  const uint8_t* phase;
  const double* cmat;     // n_phases x m x m column-major (stress mode)
  double* gout;           // grad mode: num_quads x m
  double* partials;       // norm2: 1 per block; stress: m per block
};
void launch_quad(const Grid& g, const StencilParams& sp, int mode, const QuadArgs& a, cudaStream_t s);
void launch_divergence(const Grid& g, const StencilParams& sp, const double* sfield, bool weighted,
                       double* out, cudaStream_t s);
void launch_tangent_field(const Grid& g, const StencilParams& sp, const double* tangent, double* q, cudaStream_t s);
void launch_quad_wdot(const Grid& g, const StencilParams& sp, const double* a, const double* b, double* partials,
                      cudaStream_t s);
void launch_quad_wsum(const Grid& g, const StencilParams& sp, const double* sfield, double* partials,
                      cudaStream_t s);
void launch_index_maps(const Grid& g, const StencilParams& sp, int64_t* nbr, cudaStream_t s);

// Vectors / reductions (deterministic: fixed grids, fixed-order finals).
void launch_dot_partials(const double* a, const double* b, int64_t n, double* partials, cudaStream_t s);
void launch_comp_sums(const double* a, int c, int64_t np, double* partials, cudaStream_t s);
void launch_sub_means(double* a, int c, int64_t np, const double* sums, cudaStream_t s, double count = 0.0);
void launch_final_sum(const double* partials, int nblocks, int nvals, double* out, cudaStream_t s);
void launch_scale(double* a, double sc, int64_t n, cudaStream_t s);
void launch_axpy(double* y, double a, const double* x, int64_t n, cudaStream_t s);

// PCG steps (solver.cpp:62-94) with device-resident scalars.
void launch_pcg_init(PcgState* st, const double* partials, double* hist, cudaStream_t s, int nblocks = kRedBlocks);
void launch_pcg_alpha(PcgState* st, const double* partials, cudaStream_t s, int nblocks = kRedBlocks);
void launch_update_r(double* r, const double* ap, int64_t n, const PcgState* st, cudaStream_t s);
void launch_pcg_beta(PcgState* st, const double* partials, double* hist, cudaStream_t s, int nblocks = kRedBlocks);
void launch_update_xp(double* x, double* p, const double* z, int64_t n, const PcgState* st, cudaStream_t s);
void launch_set_while(cudaGraphConditionalHandle h, const PcgState* st, cudaStream_t s);
void launch_update_xp_cond(double* x, double* p, const double* z, int64_t n, const PcgState* st,
                           cudaGraphConditionalHandle h, cudaStream_t s);

// Spectral solve z_hat = K_ref_hat(xi)^+ r_hat / N_p (precond.cpp:126-162),
// with the analytic symbol of the Nn = 1 stencils.
struct SpecParams {
  int kind, d, c;
  int n0, n1, n2;       // real dims (n2 = 1 in 2-D)
  int nh;               // last-axis spectrum length N_last/2 + 1
  int64_t nf;
  double w, inv_np;
  double h[3];
  double A[81];         // c = d: tensor A_ijkl; c = 1: C_ref (d x d) in A[0..d*d)
  int iso;              // C_ref isotropic: K_hat = (lam + mu) M + mu tr(M) I (c = d) / kappa tr(M)
  double lam, mu;       // isotropic reference moduli (mu = kappa for c = 1)
  const double4* tab[3];  // per axis: (sin, cos, sin(t/2), cos(t/2))
  int n1r, k1off;         // 3-D: axis-1 rows held (n1, or a slab rank's n1/W) and the first one's k1;
                          // 2-D slab: k1off = first half-spectrum column held (nh = columns held)
  int nhv;                // valid last-axis spectrum length N_last/2 + 1 (2-D slab chunks are padded)
  // division-free Gram factors (set_gram_factors): cd[a] = 8 w / h_a^2,
  // co[a][b] = 4 w / (h_a h_b)
  double cd[3], co[3][3];
};
inline void set_gram_factors(SpecParams& p) {
  for (int a = 0; a < 3; ++a) {
    p.cd[a] = 8.0 * p.w / (p.h[a] * p.h[a]);
    for (int b = 0; b < 3; ++b) p.co[a][b] = 4.0 * p.w / (p.h[a] * p.h[b]);
  }
}
void launch_spectral(const SpecParams& p, double2* spec, const PcgState* st, double* partials,
                     cudaStream_t s);
// whole PCG solve of a 256^2 scalar TwoTriangles problem in one persistent
// 16-CTA cluster (small2d.cu); false = not launched (cluster unschedulable)
bool small2d_eligible(const Grid& g, int n_phases);
bool launch_pcg_small2d(const SpecParams& sp, double* x, double* r, double* p, const uint8_t* phase,
                        const double* tri_tab, int n_phases, const double2* tw, PcgState* st, double* hist,
                        cudaStream_t s);


// Slab-decomposed spectra for any plane size (slabfft.cu): planes S
// [c][n0l][n1][nh] (2-D cuFFT of the local planes) <-> k1 rows W
// [c][n0][n1l][nh] (1-D cuFFT along axis 0). `dst[q]` is either a send chunk
// (all-to-all layout [q][c][i0l][k1l][k2], `push` = 0) or peer q's own W / S
// (`push` = 1: the transpose is stored straight into the peer over NVLink).
struct SlabDims {
  int c, n0, n0l, n1, n1l, nh, me, world;
  __host__ __device__ int64_t chunk() const { return (int64_t)c * n0l * n1l * nh; }
};
void launch_slab_pack_fwd(const SlabDims& d, const double2* S, double2* const* dst, int push, cudaStream_t s);
void launch_slab_unpack_fwd(const SlabDims& d, const double2* recv, double2* W, cudaStream_t s);
void launch_slab_pack_inv(const SlabDims& d, const double2* W, double2* const* dst, int push, cudaStream_t s);
void launch_slab_unpack_inv(const SlabDims& d, const double2* recv, double2* S, cudaStream_t s);

// Fused three-pass preconditioner (fftfused.cu): 3-D grids with square
// 128^2 / 256^2 planes. T has the cuFFT D2Z layout [c][n0][n1][n2/2+1].
struct FusedFft {
  int n0, np_plane, c;        // n0: LOCAL planes (slab), np_plane = n1 = n2
  int64_t np;                 // LOCAL pixels per component
  int n0g, rank, world, n1l;  // global planes, slab rank, ranks, k1 rows per rank
  double2* T;                 // pass-1 output (send side)
  double2* Trecv;             // pass-2 input (== T when world == 1)
  double2* T2;                // pass-2 output (send side)
  double2* T2recv;            // pass-3 input (== T2 when world == 1)
  const double2* tw_plane;    // W_{n1} table
  const double2* tw0;         // W_{n0g} table
  int dbg;                    // profiling: skipped phases (HOMFE_FFT_DBG)
  alignas(64) unsigned char t2map[128];  // CUtensorMap of T2 (pass-2 TMA stores), fused_make_maps
  // where pass 2 / pass 3 read the chunk of source peer q: base pointers such
  // that base[q] + TLayout::t(q, ...) (resp. t2) addresses it. Exchanged
  // receive buffers: base[q] = Trecv. Peer pull (NVLink, no all-to-all):
  // base[q] = T of rank q + (rank - q) * chunk, i.e. q's send-side chunk for me.
  static constexpr int kMaxPeers = 8;
  const double2* tpull[kMaxPeers];
  const double2* t2pull[kMaxPeers];
  int64_t chunk_t() const { return (int64_t)c * n1l * ((np_plane / 2 + 4) / 4) * n0 * 4; }
  int64_t chunk_t2() const { return (int64_t)c * n0 * n1l * (((np_plane / 2 + 16) / 16) * 16); }
};
bool fused_fft_eligible(const Grid& g);
void fused_make_maps(FusedFft& f);  // after T2 is allocated
void fused_forward(const FusedFft& f, const SpecParams& sp, double* r, const double* ap, const PcgState* st,
                   double* partials, cudaStream_t s, int which = 3);
void fused_inverse(const FusedFft& f, double* p, double* x, double* z, const PcgState* st, int init,
                   cudaStream_t s);
void launch_pcg_beta_cond(PcgState* st, const double* partials, double* hist, cudaGraphConditionalHandle h,
                          cudaStream_t s);
void launch_symbol_check(const SpecParams& p, double* partials, cudaStream_t s);
void launch_symbol_dump(const SpecParams& p, double2* blocks, cudaStream_t s);

}  // namespace hb
