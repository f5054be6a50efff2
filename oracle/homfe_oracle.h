/*
 * homfe_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * C ABI of the CPU restatement of the reference (`homfe`, arXiv 2203.02962)
 * PCG hot path. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * (paper_2203_02962_b200/) never does.
 *
 * Status codes mirror the reference CLI (proj/tools/homog.cpp:23-26):
 *   0 ok, 2 ValidationError, 3 non-convergence, 4 NumericalError.
 */
#ifndef HOMFE_ORACLE_H
#define HOMFE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* StencilKind order of proj/include/homfe/grid.hpp:30-35. */
enum {
  OR_BILINEAR_QUAD = 0,
  OR_TWO_TRIANGLES = 1,
  OR_FOUR_TRIANGLES_TWO_NODE = 2,
  OR_TRILINEAR_HEX = 3
};

typedef struct {
  int32_t dim;          /* 2 or 3 */
  int32_t stencil;      /* OR_* */
  int64_t dims[3];      /* pixel counts, row-major, last axis fastest */
  double lengths[3];    /* cell edge lengths */
} or_grid;

typedef struct {
  double eta_newton, eta_cg;
  int32_t max_newton, max_cg;
  double reassembly_threshold;
  int32_t criterion;    /* 0 strain increment, 1 displacement increment */
  int32_t policy;       /* 0 identity-scaled, 1 volume-mean, 2 explicit */
  double policy_scale;
  const double* policy_matrix; /* m*m col-major, for explicit */
} or_solve_cfg;

typedef struct {
  int32_t cg_iterations;
  double residual_initial, residual_final, increment_rel;
  int32_t precond_reassembled;
} or_newton_step;

typedef struct {
  int32_t n_steps;
  or_newton_step steps[32];
  int32_t cause;        /* 0 converged, 1 cg-stall, 2 newton-cap */
  int32_t converged;
  int32_t assemblies;
  double seconds_cg, seconds_total, seconds_assembly;
} or_report;

const char* or_last_error(void);

/* Grid / layout (grid.cpp). */
int or_layout_info(const or_grid* g, int64_t* num_pixels, int32_t* nodes_per_pixel,
                   int32_t* quads_per_pixel, int64_t* strides3, double* quad_weights);
/* Periodic neighbour table: nbr[p*n_offsets + o] = flat pixel index reached from
   pixel p by stencil offset o (operators.cpp PixelWalker semantics). */
int or_neighbor_table(const or_grid* g, int64_t* nbr, int32_t* n_offsets);
/* Stencil table: per quad, per entry (offset, node, dphi[3]). */
int or_stencil_table(const or_grid* g, int32_t* n_entries_per_quad, int32_t* offsets,
                     int32_t* nodes, double* dphi);

/* Mandel / materials (mandel.cpp, material.cpp). */
int or_isotropic_stiffness(double bulk, double shear, int32_t d, double* out);

/* Operators (operators.cpp). Fields use the reference layouts:
   nodal component-planar [c][Nn*Np], quad fields interleaved [q][m],
   tangents column-major m*m per quadrature point. */
int or_gradient(const or_grid* g, int32_t c, const double* u, double* grad);
int or_divergence(const or_grid* g, int32_t c, const double* s, int32_t weighted,
                  double* out);
int or_apply_tangent(const or_grid* g, int32_t c, const double* tangent,
                     const double* u, int32_t weighted, double* out);
/* Same operator, tangent given per phase (n_phases m*m blocks) plus phase map;
   bitwise identical to or_apply_tangent on the expanded TangentField. */
int or_apply_phase(const or_grid* g, int32_t c, int32_t n_phases, const double* cmat,
                   const uint8_t* phase, const double* u, int32_t weighted, double* out);
int or_apply_reference(const or_grid* g, int32_t c, const double* c_ref,
                       const double* u, int32_t weighted, double* out);

/* FFT with FFTW conventions (fft.cpp): unnormalised r2c / c2r, half spectrum. */
int or_fft_forward(int32_t rank, const int64_t* dims, const double* in, double* out_c);
int or_fft_inverse(int32_t rank, const int64_t* dims, const double* in_c, double* out);

/* Preconditioner (precond.cpp). Opaque handle. */
typedef struct or_precond or_precond;
int or_precond_assemble(const or_grid* g, const double* c_ref, int32_t c,
                        int32_t weighted, int32_t invert, or_precond** out);
/* Same blocks from the exact symbol of the reference operator, evaluated in
   long double (one-node stencils): no impulse-probing rounding. Test
   infrastructure for the noise-floor protocol of SURVEY 8(c) item 5. */
int or_precond_exact(const or_grid* g, const double* c_ref, int32_t c, int32_t weighted, int32_t invert,
                     or_precond** out);
/* Preconditioner from a given symbol (nf x bdim x bdim complex, row-major per
   block), inverted like invert_blocks: used to separate the reference's own
   impulse-probing rounding from implementation differences in parity tests. */
int or_precond_from_symbol(const or_grid* g, int32_t c, const double* blocks_rm, int32_t weighted,
                           or_precond** out);
int or_precond_blocks(const or_precond* p, int64_t* num_freq, int32_t* bdim,
                      double* blocks_c /* nullable: nf*bdim*bdim complex */);
int or_precond_apply(const or_grid* g, const or_precond* p, const double* r, double* z);
void or_precond_destroy(or_precond* p);

/* PCG (solver.cpp:50-97) with A = phase-indexed K and M^-1 = p.
   history must hold it_max+1 doubles. */
int or_pcg(const or_grid* g, int32_t c, int32_t n_phases, const double* cmat,
           const uint8_t* phase, const or_precond* p, const double* b, double eta,
           int32_t it_max, double* x, int32_t* iterations, double* history,
           int32_t* converged);

/* Timing variant (bench.py CPU arms): fixed it_max iterations (eta = 0),
   iter_seconds[k-1] = steady_clock duration of iteration k (K apply, update,
   M^-1, dot, direction update). */
int or_pcg_timed(const or_grid* g, int32_t c, int32_t n_phases, const double* cmat,
                 const uint8_t* phase, const or_precond* p, const double* b, int32_t it_max,
                 double* x, double* iter_seconds);

/* Linear Newton solve (solver.cpp:171-296) for a phase-indexed linear catalog.
   thermal=1: c=1, m=d; else c=d, m=mandel_dim(d). */
int or_newton_solve(const or_grid* g, int32_t thermal, int32_t n_phases,
                    const double* cmat, const uint8_t* phase, const double* e,
                    const or_solve_cfg* cfg, const double* warm_u, double* u_out,
                    double* avg_stress_out, or_report* report);

/* Material catalog entry (material.cpp:37-101): kind 0 linear (tangent m*m
   col-major), kind 1 J2 plasticity (bulk, shear, yield stress, hardening). */
typedef struct {
  int32_t kind;
  double tangent[36];
  double bulk, shear, yield_stress, hardening;
} or_material;

/* J2 radial return (material.cpp:122-226, j2_return + plane-strain embedding):
   eps m Mandel, g_in 7 (plastic strain Mandel 6 + accumulated); outputs sigma
   (m), tangent (m*m col-major, nullable), g_new (7, nullable). */
int or_j2_evaluate(int32_t d, double bulk, double shear, double yield_stress, double hardening,
                   const double* eps, const double* g_in, double* sigma, double* tangent, double* g_new);

/* Newton solve (solver.cpp:171-296) for a general catalog (linear and J2),
   with PrecondManager::ensure (solver.cpp:120-142: volume-mean tangent drift,
   reassembly when the resolved C_ref changes). g0 / g_out: internal state
   (width 7 per quad, quad-major) or NULL (zeros / not returned). g_out is the
   trial state on convergence, g0 otherwise (solver.cpp:228-290). */
int or_newton_solve_models(const or_grid* g, int32_t thermal, int32_t n_phases, const or_material* models,
                           const uint8_t* phase, const double* g0, const double* e, const or_solve_cfg* cfg,
                           const double* warm_u, double* u_out, double* g_out, double* avg_stress_out,
                           or_report* report);

/* PrecondManager (solver.hpp:105-129) shared across load steps: the same
   Newton solve with the caller's manager (assembly, C_ref and the tangent
   mean at the last assembly persist, solver.cpp:306-318). */
typedef struct or_manager or_manager;
or_manager* or_manager_create(void);
void or_manager_destroy(or_manager* m);
int or_manager_assemblies(const or_manager* m);
int or_newton_solve_managed(const or_grid* g, int32_t thermal, int32_t n_phases, const or_material* models,
                            const uint8_t* phase, const double* g0, const double* e, const or_solve_cfg* cfg,
                            const double* warm_u, double* u_out, double* g_out, double* avg_stress_out,
                            or_report* report, or_manager* manager);

/* Strain-based scheme (projection.cpp): gamma_apply with the
   unweighted reference blocks (projection.cpp:22-41), and the SB Newton
   solve with Gamma-projected strain CG (projection.cpp:43-185). strain in /
   out: QuadField num_quads x m (warm may be NULL). */
int or_gamma_apply(const or_grid* g, const double* c_ref, int32_t c, const double* s, double* out);
int or_sb_newton_solve(const or_grid* g, int32_t thermal, int32_t n_phases, const or_material* models,
                       const uint8_t* phase, const double* g0, const double* e, const or_solve_cfg* cfg,
                       const double* c_ref, const double* warm_strain, double* strain_out, double* g_out,
                       double* avg_stress_out, or_report* report);
/* eigenvalue_bounds (spectral.cpp:33-118): tangent = num_quads m x m blocks
   (col-major), pixel_constant shortcut flag; lower / upper = c * num_nodes
   sorted; cond = condition_estimate (spectral.cpp:121-127). */
int or_eigenvalue_bounds(const or_grid* g, const double* tangent, int32_t pixel_constant, const double* c_ref,
                         int32_t c, double* lower, double* upper, double* cond);

/* Field reductions (fields.cpp). */
int or_volume_average(const or_grid* g, int32_t m, const double* s, double* out);
int or_weighted_dot(const or_grid* g, int32_t m, const double* a, const double* b,
                    double* out);

/* Deterministic RNG convention (tests/support/oracles.hpp:154-160):
   std::mt19937_64(seed), u = lo + (hi-lo)*(gen()>>11)*2^-53. */
// Worker threads of the timing variant (1 = the reference's serial loop order).
int or_set_threads(int32_t n);
int or_uniform(uint64_t seed, int64_t n, double lo, double hi, double* out);

#ifdef __cplusplus
}
#endif

#endif
