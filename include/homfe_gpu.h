/*
 * homfe_gpu.h -- C ABI of the B200-native PCG hot path of the displacement-
 * based, FFT-preconditioned, matrix-free FE homogenization scheme
 * (arXiv 2203.02962; reference library `homfe`).
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, never
 * throws, and returns a status code that mirrors the reference CLI exit codes
 * (proj/tools/homog.cpp:23-26) and exception classes
 * (proj/include/homfe/common.hpp:15-25):
 *   HOMFE_OK 0, HOMFE_VALIDATION 2 (ValidationError), HOMFE_NONCONVERGED 3
 *   (cg-stall / newton-cap), HOMFE_NUMERICAL 4 (NumericalError).
 * homfe_gpu_last_error() returns the thread-local message of the last failure.
 *
 * Layouts are the reference's:
 *   nodal fields   component-planar  data[c * num_nodes + node]     (fields.hpp:16-36)
 *   quad fields    point-interleaved data[q * m + k], q = p * nq + lq (fields.hpp:40-61)
 *   materials      n_phases blocks of m x m, column-major Mandel      (fields.hpp:64-82)
 *   phase map      uint8 per pixel, row-major, last axis fastest      (io.cpp:65-86)
 * Host-buffer entry points copy in and out inside the call; the *_device
 * variants take device pointers on the context's device.
 *
 * One context per host thread (mirrors proj/include/homfe/fft.hpp:18-20);
 * every call is synchronous with respect to the host.
 */
#ifndef HOMFE_GPU_H
#define HOMFE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HOMFE_OK 0
#define HOMFE_VALIDATION 2
#define HOMFE_NONCONVERGED 3
#define HOMFE_NUMERICAL 4
#define HOMFE_DEVICE 5 /* CUDA / cuFFT failure (no reference equivalent) */

/* StencilKind, in the order of proj/include/homfe/grid.hpp:30-35. */
#define HOMFE_BILINEAR_QUAD 0
#define HOMFE_TWO_TRIANGLES 1
#define HOMFE_FOUR_TRIANGLES_TWO_NODE 2 /* probed complex blocks (probe.cu) */
#define HOMFE_TRILINEAR_HEX 3

/* ReferencePolicy::Kind (proj/include/homfe/solver.hpp:82-101). */
#define HOMFE_REF_IDENTITY_SCALED 0
#define HOMFE_REF_VOLUME_MEAN 1
#define HOMFE_REF_EXPLICIT 2

typedef struct homfe_ctx homfe_ctx;

/* CellSpec + StencilKind + physics (grid.hpp:14-28, material.hpp:100-118). */
typedef struct {
  int32_t dim;          /* 2 or 3 */
  int32_t stencil;      /* HOMFE_* stencil kind */
  int64_t dims[3];      /* pixel counts N_1..N_d, each >= 2 */
  double lengths[3];    /* cell edge lengths, each > 0 */
  int32_t components;   /* nodal components c: 1 (thermal) or dim (elasticity) */
  int32_t device;       /* CUDA device ordinal */
} homfe_grid_desc;

/* SolveConfig + ReferencePolicy (solver.hpp:16-31, 82-101). */
typedef struct {
  double eta_newton;            /* default 1e-5 */
  double eta_cg;                /* default 1e-5 */
  int32_t max_newton;           /* default 25 */
  int32_t max_cg;               /* default 20000 */
  double reassembly_threshold;  /* default 0.1 (no effect for linear tangents) */
  int32_t criterion;            /* 0 strain increment (default), 1 displacement */
  int32_t reference_policy;     /* HOMFE_REF_*, default volume mean */
  double reference_scale;       /* identity-scaled policy */
  const double* reference_matrix; /* explicit policy: m x m column-major */
} homfe_solve_cfg;

/* NewtonStep / SolveReport (solver.hpp:35-55). */
typedef struct {
  int32_t cg_iterations;
  double residual_initial;
  double residual_final;
  double increment_rel;
  int32_t precond_reassembled;
} homfe_newton_step;

typedef struct {
  int32_t n_steps;
  homfe_newton_step steps[32];
  int32_t cause;            /* 0 converged, 1 cg-stall, 2 newton-cap */
  int32_t converged;
  int32_t assemblies;       /* PrecondManager::assemblies() */
  int32_t total_cg;
  double seconds_constitutive, seconds_cg, seconds_assembly, seconds_total;
  double cg_device_ms;      /* CUDA-event time of all PCG iterations */
  int64_t kernel_launches;  /* kernels launched by this solve */
} homfe_report;

const char* homfe_gpu_last_error(void);

/* Context: grid, device buffers, cuFFT plans. Replaces GridLayout + FftGrid +
   the buffers owned by NodalField/FrequencyBlockDiag (grid.hpp:75-129,
   fft.hpp:22-57, precond.hpp:28-79). */
int homfe_gpu_create(const homfe_grid_desc* desc, homfe_ctx** out);
/* One context over n_gpus devices of this process (the
   reference's callers are single-process, proj/tools/homog.cpp:41-43): the
   slab decomposition of homfe_gpu_create_dist with rank r on device
   desc->device + r and one host thread per rank inside every call. Host
   buffers are GLOBAL (component-planar over the whole grid); supported:
   set_material, set_reference, precond_reset, solve, apply_K, apply_minv,
   pcg, sizes, path_info, slab_transport, destroy (the rest return
   HOMFE_VALIDATION). n_gpus = 1 is homfe_gpu_create. */
int homfe_gpu_create_multi(const homfe_grid_desc* desc, int32_t n_gpus, homfe_ctx** out);
int homfe_gpu_destroy(homfe_ctx* ctx);

/* Slab decomposition along axis 0 (the reference is
   single-process, SPEC.md:204 sketches only a partition contract). `desc` is
   the GLOBAL grid; rank r of `world` owns planes [r n0/world, (r+1) n0/world).
   One process per GPU; `nccl_id` (128 bytes from homfe_nccl_unique_id on
   rank 0, broadcast by the caller) initialises the NCCL communicator used for
   halo planes, the FFT transposes and scalar all-reductions. Afterwards every
   host-buffer entry point (set_material, solve, apply_K, apply_minv, pcg)
   takes and returns this rank's slab; scalars (<sigma>, iteration counts) are
   global. 3-d trilinear-hex grids (fused passes on 128^2 / 256^2 planes,
   slab spectra through cuFFT on any other plane) and 2-d one-node pixel
   stencils (row slabs along axis 0). */
int homfe_nccl_unique_id(void* out128);
int homfe_gpu_create_dist(const homfe_grid_desc* desc, int32_t rank, int32_t world, const void* nccl_id,
                          homfe_ctx** out);
/* Slab transport in use: 0 single device (or world 1), 1 all-to-all + halo
   sends (NCCL, HOMFE_P2P=0), 2 peer pull (passes 2/3 and the K halo read
   the peers' fields over NVLink; stream barriers only). No reference
   counterpart (the reference is single-process). */
int homfe_gpu_slab_transport(const homfe_ctx* ctx, int32_t* kind);

/* MaterialMap for linear models (material.hpp:100-118): per-phase m x m
   column-major tangents (conductivity d x d, or Mandel stiffness) and the
   uint8 phase of every pixel. Validates like MaterialMap::validate
   (material.cpp:252-277) and check_spd (material.cpp:13-29). */
int homfe_gpu_set_material(homfe_ctx* ctx, int32_t n_phases, const double* tangents,
                           const uint8_t* phase);
int homfe_gpu_set_material_device(homfe_ctx* ctx, int32_t n_phases, const double* tangents,
                                  const uint8_t* d_phase);

/* The context plays the caller's PrecondManager (solver.hpp:105-129): the
   assembled reference, the volume-averaged tangent at the last assembly and
   the drift rule persist across solves (load steps share one manager,
   solver.cpp:306-318). homfe_gpu_precond_reset starts a new manager. */
int homfe_gpu_precond_reset(homfe_ctx* ctx);

/* newton_solve (solver.hpp:163-166) for linear materials (J2 catalogs and
   two-node stencils run the general branch from a zero state): macroscopic load
   e (m), config, optional warm start u (c * num_nodes); outputs the periodic
   fluctuation u, the homogenized stress <sigma> (m) and the report. */
int homfe_gpu_solve(homfe_ctx* ctx, const double* e, const homfe_solve_cfg* cfg,
                    const double* warm_u, double* u_out, double* avg_stress_out,
                    homfe_report* report);
int homfe_gpu_solve_device(homfe_ctx* ctx, const double* e, const homfe_solve_cfg* cfg,
                           const double* d_warm_u, double* d_u_out, double* avg_stress_out,
                           homfe_report* report);

/* ---- nonlinear materials (J2 plasticity) --------------------- */
#define HOMFE_MATERIAL_LINEAR 0
#define HOMFE_MATERIAL_J2 1
/* Catalog entry, MaterialModel factories (material.cpp:37-101):
   LINEAR: tangent = m x m column-major Mandel (linear_elastic / conductivity);
   J2: j2_plastic(bulk, shear, yield_stress, hardening), mechanical only. */
typedef struct {
  int32_t kind;
  double tangent[36];
  double bulk, shear, yield_stress, hardening;
} homfe_material;
/* MaterialMap (material.hpp:100-118) with a general catalog. Linear-only
   catalogs behave exactly as homfe_gpu_set_material. */
int homfe_gpu_set_material_models(homfe_ctx* ctx, int32_t n_phases, const homfe_material* models,
                                  const uint8_t* phase);
/* InternalState shape (material.hpp:83-97): width 7 (J2) or 0, num_quads. */
int homfe_gpu_internal_width(homfe_ctx* ctx, int32_t* width, int64_t* num_quads);
/* newton_solve (solver.hpp:163-166) with the committed internal state g0
   (width x num_quads, quad-major; NULL = zeros) and the outgoing state g_out
   (trial state on convergence, g0 otherwise; NULL = not returned). */
int homfe_gpu_solve_state(homfe_ctx* ctx, const double* e, const homfe_solve_cfg* cfg,
                          const double* warm_u, const double* g0, double* u_out, double* g_out,
                          double* avg_stress_out, homfe_report* report);
/* NewtonOutcome::stress of the last solve (num_quads x m, quad-interleaved
   QuadField layout, fields.hpp:40-62): stress (elasticity) or flux (thermal). */
int homfe_gpu_stress_field(homfe_ctx* ctx, double* out);

/* ---- strain-based scheme and spectral bounds --------------- */
/* gamma_apply (projection.cpp:29-41) with the reference set by
   homfe_gpu_set_reference: s_in / s_out num_quads x m QuadFields. */
int homfe_gpu_gamma_apply(homfe_ctx* ctx, const double* s_in, double* s_out);
/* sb_newton_solve (projection.cpp:93-185): Newton on the fluctuating strain
   with Gamma-projected CG, fixed reference c_ref (m x m col-major). strain in
   (warm, nullable) / out: num_quads x m; g0 / g_out as homfe_gpu_solve_state. */
int homfe_gpu_sb_solve(homfe_ctx* ctx, const double* e, const homfe_solve_cfg* cfg, const double* c_ref,
                       const double* warm_strain, const double* g0, double* strain_out, double* g_out,
                       double* avg_stress_out, homfe_report* report);
/* eigenvalue_bounds + condition_estimate (spectral.cpp:33-127): tangent =
   num_quads blocks m x m col-major; lower / upper = components * num_nodes,
   sorted ascending. */
int homfe_gpu_eigenvalue_bounds(homfe_ctx* ctx, const double* tangent, int32_t pixel_constant,
                                const double* c_ref, double* lower, double* upper, double* cond);

/* ---- parity hooks (host buffers) ---------------------------------------- */
/* apply_tangent_operator (operators.hpp:31-33) with the material set above. */
int homfe_gpu_apply_K(homfe_ctx* ctx, const double* u, double* ku);
/* Build M^-1 for c_ref (assemble_reference + invert_blocks, precond.hpp:90-102;
   NumericalError on singular blocks) and apply it (precond.hpp:104-106). */
int homfe_gpu_set_reference(homfe_ctx* ctx, const double* c_ref);
int homfe_gpu_apply_minv(homfe_ctx* ctx, const double* r, double* z);
/* Dense Fourier symbol K_ref(xi) of the stored reference, nf blocks of
   (c Nn) x (c Nn) complex, column-major within the block like
   FrequencyBlockDiag (precond.hpp:38-45), for comparison with assembled
   blocks. */
int homfe_gpu_reference_blocks(homfe_ctx* ctx, double* blocks_c);
/* gradient_apply / divergence_apply (operators.hpp:20-25). */
int homfe_gpu_gradient(homfe_ctx* ctx, const double* u, double* grad);
int homfe_gpu_divergence(homfe_ctx* ctx, const double* s, int32_t weighted, double* out);
/* apply_tangent_operator with a general per-quadrature TangentField
   (operators.hpp:31-33, operators.cpp:247-257): ku = D^T W C_q D u, tangent =
   num_quads column-major m x m blocks in the reference's TangentField::data
   layout (fields.hpp:64-82), any values (not pixel-constant, not symmetric).
   Needs no material; the field is staged in device memory for the call
   (m^2 doubles per quadrature point). */
int homfe_gpu_apply_tangent_field(homfe_ctx* ctx, const double* tangent, const double* u, double* ku);
/* volume_average (fields.hpp:94-95) of an m-component quad field. */
int homfe_gpu_volume_average(homfe_ctx* ctx, const double* s, double* out);
/* pcg_solve (solver.hpp:75-78) with A = K(material), M^-1 = reference set by
   homfe_gpu_set_reference; history holds it_max + 1 doubles. */
int homfe_gpu_pcg(homfe_ctx* ctx, const double* b, double eta, int32_t it_max, double* x,
                  int32_t* iterations, double* history, int32_t* converged);
/* pcg_solve with an IterateObserver (solver.hpp:57-78, solver.cpp:87):
   `observer(user, k, x_k)` receives a host copy of the iterate after every
   iteration k >= 1 (x before the final mean removal, as in the reference).
   Runs the iterations one graph launch at a time (inspection, not speed). */
typedef void (*homfe_iterate_observer)(void* user, int32_t iteration, const double* x);
int homfe_gpu_pcg_observed(homfe_ctx* ctx, const double* b, double eta, int32_t it_max, double* x,
                           int32_t* iterations, double* history, int32_t* converged,
                           homfe_iterate_observer observer, void* user);
/* weighted_dot (fields.hpp:86-88): sum_q w_q a(q).b(q) of two m-component
   quad fields (m of the context). */
int homfe_gpu_weighted_dot(homfe_ctx* ctx, const double* a, const double* b, double* out);
/* Index maps for bit-exact comparison: strides (3) and the periodic neighbour
   table nbr[p * n_offsets + o] (grid.cpp:267-288, operators.cpp:65-84),
   computed on the device. */
int homfe_gpu_index_maps(homfe_ctx* ctx, int64_t* strides3, int64_t* nbr, int32_t* n_offsets);

/* Which kernels the context runs (no reference counterpart; lets parity
   tests assert that they exercise the path the benchmark times). Bits:
   fused three-pass FFT preconditioner (fftfused.cu), modal hex K (hexfast.cu),
   conditional-WHILE PCG graph, slab spectra (slabfft.cu), slab context,
   peer-pull transport, 2-D warp-strip K (quad2d.cu). */
#define HOMFE_PATH_FUSED_FFT 1
#define HOMFE_PATH_HEX_MODAL 2
#define HOMFE_PATH_WHILE_GRAPH 4
#define HOMFE_PATH_SLAB_SPECTRA 8
#define HOMFE_PATH_SLAB 16
#define HOMFE_PATH_PEER_PULL 32
#define HOMFE_PATH_ELEM2D 64
#define HOMFE_PATH_MULTI 128
#define HOMFE_PATH_SMALL2D 256 /* whole PCG loop in one persistent 16-CTA cluster (256^2 scalar) */
int homfe_gpu_path_info(const homfe_ctx* ctx, int32_t* flags);

/* Per-stage CUDA-event timing of one PCG iteration on the current buffers
   (call after a solve): ms[0..7] = K apply, x/r update, forward FFT, spectral
   solve, inverse FFT, p update, scalar kernels, their sum. */
int homfe_gpu_kernel_times(homfe_ctx* ctx, int32_t reps, double* ms);

/* isotropic_stiffness (proj/include/homfe/mandel.hpp:61-62): 3K P_vol +
   2G P_dev in Mandel notation, plane strain in 2-D; column-major output. */
int homfe_isotropic_stiffness(double bulk, double shear, int32_t dim, double* out);

/* Seeded synthetic inputs, reference RNG convention (std::mt19937_64(seed),
   (gen() >> 11) * 2^-53; proj/tests/support/oracles.hpp:154-160). */
int homfe_random_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out);
int homfe_random_normal(uint64_t seed, int64_t n, double* out);

/* Sizes of the context. */
int homfe_gpu_sizes(const homfe_ctx* ctx, int64_t* num_pixels, int64_t* num_quads,
                    int32_t* m, int64_t* num_frequencies);

#ifdef __cplusplus
}
#endif

#endif
