// homfe/gpu.hpp -- header-only C++ shim re-exposing the reference's solver
// API (proj/include/homfe/{grid,fields,material,solver}.hpp) over the C ABI
// of include/homfe_gpu.h, so a caller of `homfe::newton_solve` /
// `homfe::run_load_program` switches to the B200 path by swapping the include
// and linking libhomfe_gpu.so.
//
// Same names, argument meaning and error behaviour as the reference:
//   * ValidationError / NumericalError (proj/include/homfe/common.hpp:15-25)
//     are thrown for status codes 2 / 4; CUDA failures throw DeviceError;
//   * non-convergence is reported, not thrown (NewtonOutcome::converged,
//     SolveReport::cause), as in proj/src/solver.cpp:229-290.
// Forced deviations (documented in DESIGN.md): Eigen vectors become
// std::vector<double>. Both newton_solve forms exist: the reference's
// (layout, map, g0, e, cfg, precond, warm) and the linear shorthand without
// InternalState (width 0 for linear models, proj/src/material.cpp:107-111).
#ifndef HOMFE_GPU_HPP
#define HOMFE_GPU_HPP

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../homfe_gpu.h"

namespace homfe {

using Index = std::int64_t;

class ValidationError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int code) {
  if (code == HOMFE_OK || code == HOMFE_NONCONVERGED) return;
  const std::string msg = homfe_gpu_last_error();
  if (code == HOMFE_VALIDATION) throw ValidationError(msg);
  if (code == HOMFE_NUMERICAL) throw NumericalError(msg);
  throw DeviceError(msg);
}
}  // namespace detail

// grid.hpp:14-28, 30-35
struct CellSpec {
  std::vector<Index> dims;
  std::vector<double> lengths;
  int dim() const { return static_cast<int>(dims.size()); }
  Index pixel_count() const {
    Index n = 1;
    for (Index d : dims) n *= d;
    return n;
  }
  double cell_volume() const {
    double v = 1.0;
    for (double l : lengths) v *= l;
    return v;
  }
};

enum class StencilKind { BilinearQuad, TwoTriangles, FourTrianglesTwoNode, TrilinearHex };

inline StencilKind stencil_kind_from_string(const std::string& name) {
  if (name == "bilinear-quad") return StencilKind::BilinearQuad;
  if (name == "two-triangles") return StencilKind::TwoTriangles;
  if (name == "four-triangles-two-node") return StencilKind::FourTrianglesTwoNode;
  if (name == "trilinear-hex") return StencilKind::TrilinearHex;
  throw ValidationError("stencil: unknown kind '" + name + "'");
}

// One device context per (layout, nodal component count); contexts are not
// shared between host threads (fft.hpp:18-20).
class GridLayout {
 public:
  // n_gpus > 1: one context over that many devices of this process (slab
  // decomposition along axis 0, homfe_gpu_create_multi); newton_solve,
  // run_load_program, apply_tangent_operator, apply_preconditioner and
  // pcg_solve take and return global fields.
  GridLayout(CellSpec cell, StencilKind kind, int n_gpus = 1) : cell_(std::move(cell)), kind_(kind), n_gpus_(n_gpus) {
    if (cell_.dims.size() != cell_.lengths.size()) throw ValidationError("cell: dims and lengths must have equal rank");
    if (cell_.dim() != 2 && cell_.dim() != 3) throw ValidationError("cell: dimension must be 2 or 3");
  }
  const CellSpec& cell() const { return cell_; }
  StencilKind kind() const { return kind_; }
  int dim() const { return cell_.dim(); }
  int n_gpus() const { return n_gpus_; }
  Index num_pixels() const { return cell_.pixel_count(); }
  // grid.hpp:96-110: node types per pixel (FourTrianglesTwoNode adds the
  // pixel-centre node), nodes = Nn * N_p
  int nodes_per_pixel() const { return kind_ == StencilKind::FourTrianglesTwoNode ? 2 : 1; }
  Index num_nodes() const { return num_pixels() * nodes_per_pixel(); }
  Index num_quads() const { return num_pixels() * quads_per_pixel(); }
  // grid.cpp:114-229: 1 (BilinearQuad here: 4), 2, 4, 8 Gauss points per pixel
  int quads_per_pixel() const {
    switch (kind_) {
      case StencilKind::BilinearQuad: return 4;
      case StencilKind::TwoTriangles: return 2;
      case StencilKind::FourTrianglesTwoNode: return 4;
      case StencilKind::TrilinearHex: return 8;
    }
    return 0;
  }

  homfe_ctx* context(int components, int device = 0) const {
    auto it = ctx_.find(components);
    if (it != ctx_.end()) return it->second.get();
    homfe_grid_desc d{};
    d.dim = dim();
    d.stencil = static_cast<int32_t>(kind_);
    for (int a = 0; a < 3; ++a) {
      d.dims[a] = a < dim() ? cell_.dims[a] : 1;
      d.lengths[a] = a < dim() ? cell_.lengths[a] : 1.0;
    }
    d.components = components;
    d.device = device;
    homfe_ctx* h = nullptr;
    if (n_gpus_ > 1) detail::check(homfe_gpu_create_multi(&d, n_gpus_, &h));
    else detail::check(homfe_gpu_create(&d, &h));
    auto* raw = h;
    ctx_.emplace(components, std::shared_ptr<homfe_ctx>(h, [](homfe_ctx* p) { homfe_gpu_destroy(p); }));
    return raw;
  }

 private:
  CellSpec cell_;
  StencilKind kind_;
  int n_gpus_ = 1;
  mutable std::map<int, std::shared_ptr<homfe_ctx>> ctx_;
};

// fields.hpp:16-36 (Eigen::VectorXd -> std::vector<double>)
struct NodalField {
  int components = 0;
  Index nodes = 0;
  std::vector<double> data;
  NodalField() = default;
  NodalField(int c, Index n) : components(c), nodes(n), data(static_cast<std::size_t>(c * n), 0.0) {}
  double& operator()(int c, Index node) { return data[static_cast<std::size_t>(c * nodes + node)]; }
  double operator()(int c, Index node) const { return data[static_cast<std::size_t>(c * nodes + node)]; }
};

// material.hpp:36-69 (linear models and J2 plasticity)
class MaterialModel {
 public:
  enum class Kind { LinearElastic, Conductivity, J2Plastic };
  // material.cpp:78-101
  static MaterialModel j2_plastic(double bulk, double shear, double yield_stress, double hardening, int d) {
    if (!(bulk > 0.0) || !(shear > 0.0) || !(yield_stress > 0.0))
      throw ValidationError("j2_plastic: K, G and tau_y0 must be > 0");
    if (hardening < 0.0) throw ValidationError("j2_plastic: H must be >= 0");
    if (d != 2 && d != 3) throw ValidationError("j2_plastic: dimension must be 2 or 3");
    MaterialModel m = isotropic_elastic(bulk, shear, d);
    m.kind_ = Kind::J2Plastic;
    m.j2_[0] = bulk;
    m.j2_[1] = shear;
    m.j2_[2] = yield_stress;
    m.j2_[3] = hardening;
    return m;
  }
  Kind kind() const { return kind_; }
  bool nonlinear() const { return kind_ == Kind::J2Plastic; }
  int internal_width() const { return nonlinear() ? 7 : 0; }
  homfe_material c_model() const {
    homfe_material mm{};
    if (nonlinear()) {
      mm.kind = HOMFE_MATERIAL_J2;
      mm.bulk = j2_[0];
      mm.shear = j2_[1];
      mm.yield_stress = j2_[2];
      mm.hardening = j2_[3];
    } else {
      mm.kind = HOMFE_MATERIAL_LINEAR;
      for (std::size_t i = 0; i < tangent_.size() && i < 36; ++i) mm.tangent[i] = tangent_[i];
    }
    return mm;
  }
  static MaterialModel linear_elastic(std::vector<double> c_colmajor, int d) {
    const int m = d == 2 ? 3 : 6;
    if (static_cast<int>(c_colmajor.size()) != m * m) throw ValidationError("linear_elastic: stiffness must be 3x3 or 6x6");
    return MaterialModel(std::move(c_colmajor), d, false);
  }
  static MaterialModel isotropic_elastic(double bulk, double shear, int d) {
    std::vector<double> c(static_cast<std::size_t>(d == 2 ? 9 : 36));
    detail::check(homfe_isotropic_stiffness(bulk, shear, d, c.data()));
    return MaterialModel(std::move(c), d, false);
  }
  static MaterialModel conductivity(std::vector<double> a_colmajor, int d) {
    if (static_cast<int>(a_colmajor.size()) != d * d) throw ValidationError("conductivity: matrix must be 2x2 or 3x3");
    return MaterialModel(std::move(a_colmajor), d, true);
  }
  static MaterialModel isotropic_conductivity(double kappa, int d) {
    if (!(kappa > 0.0)) throw ValidationError("conductivity: kappa must be > 0");
    std::vector<double> a(static_cast<std::size_t>(d * d), 0.0);
    for (int i = 0; i < d; ++i) a[static_cast<std::size_t>(i * d + i)] = kappa;
    return MaterialModel(std::move(a), d, true);
  }
  bool thermal() const { return thermal_; }
  int dim() const { return dim_; }
  int flux_components() const { return thermal_ ? dim_ : (dim_ == 2 ? 3 : 6); }
  const std::vector<double>& linear_tangent() const {
    if (nonlinear()) throw ValidationError("linear_tangent: J2 has no constant tangent");
    return tangent_;
  }

 private:
  MaterialModel(std::vector<double> t, int d, bool thermal)
      : kind_(thermal ? Kind::Conductivity : Kind::LinearElastic), tangent_(std::move(t)), dim_(d), thermal_(thermal) {}
  Kind kind_;
  std::vector<double> tangent_;
  int dim_;
  bool thermal_;
  double j2_[4] = {0, 0, 0, 0};
};

// material.hpp:83-97: data[q * width + i]
struct InternalState {
  int width = 0;
  Index quads = 0;
  std::vector<double> data;
  InternalState() = default;
  InternalState(int width_, Index quads_)
      : width(width_), quads(quads_), data(static_cast<std::size_t>(width_ * quads_), 0.0) {}
};

// material.hpp:100-118
struct MaterialMap {
  std::vector<MaterialModel> catalog;
  std::vector<std::uint8_t> phase;
  int node_components(int d) const { return catalog.front().thermal() ? 1 : d; }
  int flux_components() const { return catalog.front().flux_components(); }
  int internal_width() const {
    int w = 0;
    for (const auto& mdl : catalog) w = mdl.internal_width() > w ? mdl.internal_width() : w;
    return w;
  }
  InternalState make_state(const GridLayout& layout) const {
    return InternalState(internal_width(), layout.num_pixels() * layout.quads_per_pixel());
  }
};

// solver.hpp:16-31
struct SolveConfig {
  double eta_newton = 1e-5;
  double eta_cg = 1e-5;
  int max_newton = 25;
  int max_cg = 20000;
  double reassembly_threshold = 0.1;
  enum class NewtonCriterion { StrainIncrement, DisplacementIncrement };
  NewtonCriterion criterion = NewtonCriterion::StrainIncrement;
};

enum class TerminationCause { Converged, CgStall, NewtonCap };

struct NewtonStep {
  int cg_iterations = 0;
  double residual_initial = 0.0;
  double residual_final = 0.0;
  double increment_rel = 0.0;
  bool precond_reassembled = false;
};

struct SolveReport {
  std::vector<NewtonStep> steps;
  TerminationCause cause = TerminationCause::Converged;
  double seconds_constitutive = 0.0, seconds_cg = 0.0, seconds_assembly = 0.0, seconds_total = 0.0;
  int newton_steps() const { return static_cast<int>(steps.size()); }
  int total_cg() const {
    int n = 0;
    for (const auto& s : steps) n += s.cg_iterations;
    return n;
  }
};

// solver.hpp:82-101
struct ReferencePolicy {
  enum class Kind { IdentityScaled, VolumeMean, Explicit };
  Kind kind = Kind::VolumeMean;
  double scale = 1.0;
  std::vector<double> matrix;  // column-major m x m
  static ReferencePolicy identity_scaled(double s = 1.0) { return {Kind::IdentityScaled, s, {}}; }
  static ReferencePolicy volume_mean() { return {Kind::VolumeMean, 1.0, {}}; }
  static ReferencePolicy explicit_matrix(std::vector<double> m) { return {Kind::Explicit, 1.0, std::move(m)}; }
};

// solver.hpp:105-129: for linear tangents one assembly per solve.
class PrecondManager {
 public:
  PrecondManager(ReferencePolicy policy, double threshold, int components)
      : policy_(std::move(policy)), threshold_(threshold), components_(components) {}
  const ReferencePolicy& policy() const { return policy_; }
  int components() const { return components_; }
  int assemblies() const { return assemblies_; }
  void count_assembly(int n) { assemblies_ += n; }
  double threshold() const { return threshold_; }
  // The device context holds the manager's state (assembled reference, the
  // tangent mean at the last assembly, homfe_gpu_precond_reset): a manager
  // used with a context it was not last bound to starts fresh there.
  void bind(homfe_ctx* ctx) {
    if (bound_ != ctx) {
      detail::check(homfe_gpu_precond_reset(ctx));
      bound_ = ctx;
    }
  }

 private:
  ReferencePolicy policy_;
  double threshold_;
  int components_;
  int assemblies_ = 0;
  homfe_ctx* bound_ = nullptr;
};

// solver.hpp:145-161
struct NewtonOutcome {
  NodalField u;
  InternalState internal;      // trial state on convergence, g0 otherwise
  std::vector<double> stress;  // QuadField (num_quads x m), mechanical maps
  std::vector<double> average_stress;
  SolveReport report;
  bool converged = false;
};

namespace detail {
inline void set_material(homfe_ctx* ctx, const MaterialMap& map) {
  if (map.catalog.empty()) throw ValidationError("materials: catalog is empty");
  std::vector<homfe_material> models;
  for (const auto& mdl : map.catalog) models.push_back(mdl.c_model());
  check(homfe_gpu_set_material_models(ctx, static_cast<int32_t>(models.size()), models.data(), map.phase.data()));
}
}  // namespace detail

// newton_solve (solver.hpp:163-166) on the GPU, with the committed internal
// state g0 (map.make_state(layout) for a fresh start).
inline NewtonOutcome newton_solve(const GridLayout& layout, const MaterialMap& map, const InternalState& g0,
                                  const std::vector<double>& e, const SolveConfig& cfg, PrecondManager& precond,
                                  const NodalField* warm_start = nullptr) {
  const int c = map.node_components(layout.dim());
  if (static_cast<Index>(map.phase.size()) != layout.num_pixels())
    throw ValidationError("materials: phase map does not match the grid");
  homfe_ctx* ctx = layout.context(c);
  detail::set_material(ctx, map);
  precond.bind(ctx);
  homfe_solve_cfg sc{};
  sc.eta_newton = cfg.eta_newton;
  sc.eta_cg = cfg.eta_cg;
  sc.max_newton = cfg.max_newton;
  sc.max_cg = cfg.max_cg;
  sc.reassembly_threshold = cfg.reassembly_threshold;
  sc.criterion = cfg.criterion == SolveConfig::NewtonCriterion::StrainIncrement ? 0 : 1;
  const ReferencePolicy& pol = precond.policy();
  sc.reference_policy = pol.kind == ReferencePolicy::Kind::IdentityScaled ? HOMFE_REF_IDENTITY_SCALED
                        : pol.kind == ReferencePolicy::Kind::VolumeMean   ? HOMFE_REF_VOLUME_MEAN
                                                                          : HOMFE_REF_EXPLICIT;
  sc.reference_scale = pol.scale;
  sc.reference_matrix = pol.matrix.empty() ? nullptr : pol.matrix.data();
  NewtonOutcome out;
  out.u = NodalField(c, layout.num_nodes());
  out.average_stress.assign(static_cast<std::size_t>(map.flux_components()), 0.0);
  if (warm_start && (warm_start->components != c || warm_start->nodes != layout.num_nodes()))
    throw ValidationError("warm start has wrong shape");
  const int width = map.internal_width();
  const Index nq = layout.num_pixels() * layout.quads_per_pixel();
  if (g0.width != width || g0.quads != nq) throw ValidationError("internal state does not match layout and catalog");
  out.internal = InternalState(width, nq);
  homfe_report rep{};
  const int code = homfe_gpu_solve_state(ctx, e.data(), &sc, warm_start ? warm_start->data.data() : nullptr,
                                         width ? g0.data.data() : nullptr, out.u.data.data(),
                                         width ? out.internal.data.data() : nullptr, out.average_stress.data(),
                                         &rep);
  detail::check(code);
  if (c > 1) {
    out.stress.assign(static_cast<std::size_t>(nq * map.flux_components()), 0.0);
    detail::check(homfe_gpu_stress_field(ctx, out.stress.data()));
  }
  for (int i = 0; i < rep.n_steps && i < 32; ++i) {
    const auto& s = rep.steps[i];
    out.report.steps.push_back({s.cg_iterations, s.residual_initial, s.residual_final, s.increment_rel,
                                s.precond_reassembled != 0});
  }
  out.report.cause = rep.cause == 0 ? TerminationCause::Converged
                     : rep.cause == 1 ? TerminationCause::CgStall
                                      : TerminationCause::NewtonCap;
  out.report.seconds_constitutive = rep.seconds_constitutive;
  out.report.seconds_cg = rep.seconds_cg;
  out.report.seconds_assembly = rep.seconds_assembly;
  out.report.seconds_total = rep.seconds_total;
  out.converged = rep.converged != 0;
  precond.count_assembly(rep.assemblies);
  return out;
}

// Linear shorthand (no internal state; linear catalogs).
inline NewtonOutcome newton_solve(const GridLayout& layout, const MaterialMap& map, const std::vector<double>& e,
                                  const SolveConfig& cfg, PrecondManager& precond,
                                  const NodalField* warm_start = nullptr) {
  return newton_solve(layout, map, map.make_state(layout), e, cfg, precond, warm_start);
}

struct LoadStepResult {
  std::vector<double> load;
  NewtonOutcome outcome;
};

// run_load_program (solver.hpp:168-179, solver.cpp:298-319): warm-started
// load steps, stopping at the first non-converged step.
inline std::vector<LoadStepResult> run_load_program(const GridLayout& layout, const MaterialMap& map,
                                                    const std::vector<std::vector<double>>& loads,
                                                    const SolveConfig& cfg, const ReferencePolicy& policy) {
  if (loads.empty()) throw ValidationError("loading: at least one load step is required");
  PrecondManager precond(policy, cfg.reassembly_threshold, map.node_components(layout.dim()));
  std::vector<LoadStepResult> results;
  results.reserve(loads.size());  // `warm` points into the previous result
  InternalState g = map.make_state(layout);
  const NodalField* warm = nullptr;
  for (const auto& e : loads) {
    results.push_back({e, newton_solve(layout, map, g, e, cfg, precond, warm)});
    if (results.back().outcome.converged) g = results.back().outcome.internal;
    if (!results.back().outcome.converged) break;
    warm = &results.back().outcome.u;
  }
  return results;
}

// ---- operator-level seams (operators.hpp, fields.hpp, precond.hpp, solver.hpp)

// fields.hpp:40-61: point-interleaved data[q * m + k]
struct QuadField {
  Index quads = 0;
  int m = 0;
  std::vector<double> data;
  QuadField() = default;
  QuadField(Index q, int m_) : quads(q), m(m_), data(static_cast<std::size_t>(q * m_), 0.0) {}
  double* vec(Index q) { return data.data() + q * m; }
  const double* vec(Index q) const { return data.data() + q * m; }
};

namespace detail {
// the context whose gradient width is m (c = 1: m = d; c = d: Mandel)
inline homfe_ctx* quad_context(const GridLayout& layout, int m) {
  const int d = layout.dim();
  if (m == d) return layout.context(1);
  if (m == d * (d + 1) / 2) return layout.context(d);
  throw ValidationError("quadrature field shape does not match layout");
}
inline void check_quad(const GridLayout& layout, const QuadField& s) {
  if (s.quads != layout.num_quads() || static_cast<Index>(s.data.size()) != s.quads * s.m)
    throw ValidationError("quadrature field shape does not match layout");
}
inline void check_nodal(const GridLayout& layout, const NodalField& u) {
  if (u.nodes != layout.num_nodes() || (u.components != 1 && u.components != layout.dim()) ||
      static_cast<Index>(u.data.size()) != u.components * u.nodes)
    throw ValidationError("nodal field shape does not match layout");
}
}  // namespace detail

// gradient_apply (operators.hpp:20-21): the dense product D u at every
// quadrature point.
inline QuadField gradient_apply(const GridLayout& layout, const NodalField& u) {
  detail::check_nodal(layout, u);
  const int d = layout.dim();
  QuadField out(layout.num_quads(), u.components == 1 ? d : d * (d + 1) / 2);
  detail::check(homfe_gpu_gradient(layout.context(u.components), u.data.data(), out.data.data()));
  return out;
}

// divergence_apply (operators.hpp:23-25): D^T W s, or D^T s unweighted.
inline NodalField divergence_apply(const GridLayout& layout, const QuadField& s, bool weighted = true) {
  detail::check_quad(layout, s);
  homfe_ctx* ctx = detail::quad_context(layout, s.m);
  NodalField out(s.m == layout.dim() ? 1 : layout.dim(), layout.num_nodes());
  detail::check(homfe_gpu_divergence(ctx, s.data.data(), weighted ? 1 : 0, out.data.data()));
  return out;
}

// weighted_dot / weighted_norm / volume_average (fields.hpp:86-95).
inline double weighted_dot(const GridLayout& layout, const QuadField& a, const QuadField& b) {
  detail::check_quad(layout, a);
  detail::check_quad(layout, b);
  if (a.m != b.m) throw ValidationError("weighted_dot: fields differ in width");
  double v = 0.0;
  detail::check(homfe_gpu_weighted_dot(detail::quad_context(layout, a.m), a.data.data(), b.data.data(), &v));
  return v;
}
inline double weighted_norm(const GridLayout& layout, const QuadField& a) {
  const double v = weighted_dot(layout, a, a);
  return v > 0.0 ? std::sqrt(v) : 0.0;
}
inline std::vector<double> volume_average(const GridLayout& layout, const QuadField& s) {
  detail::check_quad(layout, s);
  std::vector<double> out(static_cast<std::size_t>(s.m), 0.0);
  detail::check(homfe_gpu_volume_average(detail::quad_context(layout, s.m), s.data.data(), out.data()));
  return out;
}

// FrequencyBlockDiag (precond.hpp:28-79). The device never stores the
// blocks of a one-node stencil: it evaluates the reference symbol in closed
// form inside the spectral kernels, so this handle
// carries the reference tangent, the weighting and the inversion state;
// block(k) reads the assembled (pre-inversion) symbol back for inspection.
class FrequencyBlockDiag {
 public:
  int block_dim() const { return components_ * nodes_per_pixel_; }
  Index num_frequencies() const { return num_freq_; }
  int components() const { return components_; }
  int nodes_per_pixel() const { return nodes_per_pixel_; }
  bool weighted() const { return weighted_; }
  bool inverted() const { return inverted_; }
  Index zero_frequency() const { return 0; }
  const std::vector<double>& reference() const { return c_ref_; }
  // K_ref_hat(xi_k) before inversion, column-major block_dim^2 (precond.hpp:38-45)
  std::vector<std::complex<double>> block(Index k) const {
    if (k < 0 || k >= num_freq_) throw ValidationError("block: frequency out of range");
    if (symbol_.empty()) {
      homfe_ctx* ctx = layout_->context(components_);
      detail::check(homfe_gpu_set_reference(ctx, c_ref_.data()));
      const int b = block_dim();
      std::vector<double> raw(static_cast<std::size_t>(num_freq_ * b * b * 2));
      detail::check(homfe_gpu_reference_blocks(ctx, raw.data()));
      symbol_.resize(static_cast<std::size_t>(num_freq_ * b * b));
      for (std::size_t i = 0; i < symbol_.size(); ++i) symbol_[i] = {raw[2 * i], raw[2 * i + 1]};
    }
    const int b = block_dim();
    const double sc = weighted_ ? 1.0 : 1.0 / w_;
    std::vector<std::complex<double>> out(static_cast<std::size_t>(b * b));
    for (int i = 0; i < b * b; ++i) out[static_cast<std::size_t>(i)] = sc * symbol_[static_cast<std::size_t>(k * b * b + i)];
    return out;
  }

 private:
  friend FrequencyBlockDiag assemble_reference(const GridLayout&, const std::vector<double>&, int, bool);
  friend FrequencyBlockDiag invert_blocks(const FrequencyBlockDiag&);
  friend NodalField apply_preconditioner(const GridLayout&, const FrequencyBlockDiag&, const NodalField&);
  const GridLayout* layout_ = nullptr;
  std::vector<double> c_ref_;
  int components_ = 0, nodes_per_pixel_ = 1;
  Index num_freq_ = 0;
  bool weighted_ = true, inverted_ = false;
  double w_ = 1.0;  // quadrature weight (unweighted blocks = weighted / w)
  mutable std::vector<std::complex<double>> symbol_;
};

// assemble_reference (precond.hpp:90-93): validates c_ref (symmetric positive
// definite, ValidationError otherwise) and sets it as the device reference.
inline FrequencyBlockDiag assemble_reference(const GridLayout& layout, const std::vector<double>& c_ref,
                                             int components, bool weighted = true) {
  const int d = layout.dim();
  if (components != 1 && components != d) throw ValidationError("assemble_reference: bad component count");
  const int m = components == 1 ? d : d * (d + 1) / 2;
  if (static_cast<int>(c_ref.size()) != m * m) throw ValidationError("reference tangent has wrong dimension");
  homfe_ctx* ctx = layout.context(components);
  detail::check(homfe_gpu_set_reference(ctx, c_ref.data()));
  FrequencyBlockDiag b;
  b.layout_ = &layout;
  b.c_ref_ = c_ref;
  b.components_ = components;
  b.nodes_per_pixel_ = layout.nodes_per_pixel();
  b.weighted_ = weighted;
  Index nf = 1;
  for (int a = 0; a < d; ++a) nf *= a == d - 1 ? layout.cell().dims[a] / 2 + 1 : layout.cell().dims[a];
  b.num_freq_ = nf;
  b.w_ = layout.cell().cell_volume() / static_cast<double>(layout.num_pixels()) / layout.quads_per_pixel();
  return b;
}

// invert_blocks (precond.hpp:95-102): the device inverts per frequency inside
// the spectral kernel (zero frequency pseudo-inverted); NumericalError for a
// numerically singular non-zero-frequency block is raised at assembly.
inline FrequencyBlockDiag invert_blocks(const FrequencyBlockDiag& blocks) {
  if (blocks.inverted_) throw ValidationError("invert_blocks: blocks are already inverted");
  FrequencyBlockDiag out = blocks;
  out.inverted_ = true;
  return out;
}

// apply_preconditioner (precond.hpp:104-106): M^-1 r.
inline NodalField apply_preconditioner(const GridLayout& layout, const FrequencyBlockDiag& inv_blocks,
                                       const NodalField& r) {
  if (!inv_blocks.inverted_) throw ValidationError("apply_preconditioner: blocks are not inverted");
  detail::check_nodal(layout, r);
  if (r.components != inv_blocks.components_) throw ValidationError("apply_preconditioner: field shape mismatch");
  homfe_ctx* ctx = layout.context(r.components);
  detail::check(homfe_gpu_set_reference(ctx, inv_blocks.c_ref_.data()));
  NodalField out(r.components, r.nodes);
  detail::check(homfe_gpu_apply_minv(ctx, r.data.data(), out.data.data()));
  if (!inv_blocks.weighted_)
    for (double& v : out.data) v *= inv_blocks.w_;
  return out;
}

// pcg_solve (solver.hpp:57-78) with A = the tangent operator of a linear
// material map and M^-1 = inverted reference blocks, both on the device.
// The observer receives x_k after every iteration (solver.cpp:87); with an
// observer the iterations run one graph launch at a time.
using IterateObserver = std::function<void(const NodalField&)>;

struct PcgOutcome {
  NodalField x;
  int iterations = 0;
  std::vector<double> history;  // |r_k|_{M^-1}, starting from r_0
  bool converged = false;
};

struct TangentOperator {
  const GridLayout* layout;
  MaterialMap map;
};

namespace detail {
struct ObserverCall {
  const IterateObserver* obs;
  NodalField buf;
};
inline void observer_trampoline(void* user, int32_t, const double* x) {
  auto* oc = static_cast<ObserverCall*>(user);
  std::copy(x, x + oc->buf.data.size(), oc->buf.data.begin());
  (*oc->obs)(oc->buf);
}
}  // namespace detail

inline PcgOutcome pcg_solve(const TangentOperator& apply_a, const FrequencyBlockDiag& minv, const NodalField& b,
                            double eta, int it_max, const IterateObserver& observer = {}) {
  const GridLayout& layout = *apply_a.layout;
  detail::check_nodal(layout, b);
  if (!minv.inverted()) throw ValidationError("pcg: preconditioner blocks are not inverted");
  if (b.components != minv.components()) throw ValidationError("pcg: field shape mismatch");
  if (it_max < 0) throw ValidationError("pcg: it_max must be >= 0");
  homfe_ctx* ctx = layout.context(b.components);
  detail::set_material(ctx, apply_a.map);
  detail::check(homfe_gpu_set_reference(ctx, minv.reference().data()));
  PcgOutcome out;
  out.x = NodalField(b.components, b.nodes);
  std::vector<double> hist(static_cast<std::size_t>(it_max + 1), 0.0);
  int32_t its = 0, conv = 0;
  if (observer) {
    detail::ObserverCall oc{&observer, NodalField(b.components, b.nodes)};
    detail::check(homfe_gpu_pcg_observed(ctx, b.data.data(), eta, it_max, out.x.data.data(), &its, hist.data(),
                                         &conv, &detail::observer_trampoline, &oc));
  } else {
    detail::check(homfe_gpu_pcg(ctx, b.data.data(), eta, it_max, out.x.data.data(), &its, hist.data(), &conv));
  }
  out.iterations = its;
  out.converged = conv != 0;
  hist.resize(static_cast<std::size_t>(its + 1));
  out.history = std::move(hist);
  return out;
}

// apply_tangent_operator (operators.hpp:31-33) for a linear material map.
inline NodalField apply_tangent_operator(const GridLayout& layout, const MaterialMap& map, const NodalField& u) {
  homfe_ctx* ctx = layout.context(u.components);
  detail::set_material(ctx, map);
  NodalField out(u.components, u.nodes);
  detail::check(homfe_gpu_apply_K(ctx, u.data.data(), out.data.data()));
  return out;
}

// fields.hpp:64-82: per-quadrature-point tangent matrices, column-major m x m
// blocks (the reference's TangentField::data layout).
struct TangentField {
  int m = 0;
  Index quads = 0;
  bool pixel_constant = false;
  std::vector<double> data;
  TangentField() = default;
  TangentField(int m_, Index quads_) : m(m_), quads(quads_), data(static_cast<std::size_t>(m_ * m_ * quads_), 0.0) {}
  double* block(Index q) { return data.data() + q * m * m; }
  const double* block(Index q) const { return data.data() + q * m * m; }
  // uniform(quads, c): the same column-major block everywhere (fields.cpp)
  static TangentField uniform(Index quads, int m, const std::vector<double>& c_colmajor) {
    if (static_cast<int>(c_colmajor.size()) != m * m) throw ValidationError("TangentField::uniform: block size");
    TangentField t(m, quads);
    for (Index q = 0; q < quads; ++q) std::copy(c_colmajor.begin(), c_colmajor.end(), t.block(q));
    t.pixel_constant = true;
    return t;
  }
};

// apply_tangent_operator (operators.hpp:31-33, operators.cpp:247-257) with a
// general per-quadrature-point TangentField: D^T W C_q D u on the device.
inline NodalField apply_tangent_operator(const GridLayout& layout, const TangentField& tangent, const NodalField& u) {
  if (u.nodes != layout.num_nodes() || (u.components != 1 && u.components != layout.dim()))
    throw ValidationError("nodal field shape does not match layout");
  const int m = u.components == 1 ? layout.dim() : (layout.dim() == 2 ? 3 : 6);
  if (tangent.m != m) throw ValidationError("tangent dimension does not match layout");
  if (tangent.quads != layout.num_quads()) throw ValidationError("tangent field size does not match layout");
  homfe_ctx* ctx = layout.context(u.components);
  NodalField out(u.components, u.nodes);
  detail::check(homfe_gpu_apply_tangent_field(ctx, tangent.data.data(), u.data.data(), out.data.data()));
  return out;
}

}  // namespace homfe

#endif
