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

#include <cstdint>
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
  GridLayout(CellSpec cell, StencilKind kind) : cell_(std::move(cell)), kind_(kind) {
    if (cell_.dims.size() != cell_.lengths.size()) throw ValidationError("cell: dims and lengths must have equal rank");
    if (cell_.dim() != 2 && cell_.dim() != 3) throw ValidationError("cell: dimension must be 2 or 3");
  }
  const CellSpec& cell() const { return cell_; }
  StencilKind kind() const { return kind_; }
  int dim() const { return cell_.dim(); }
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
    detail::check(homfe_gpu_create(&d, &h));
    auto* raw = h;
    ctx_.emplace(components, std::shared_ptr<homfe_ctx>(h, [](homfe_ctx* p) { homfe_gpu_destroy(p); }));
    return raw;
  }

 private:
  CellSpec cell_;
  StencilKind kind_;
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

 private:
  ReferencePolicy policy_;
  double threshold_;
  int components_;
  int assemblies_ = 0;
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

// apply_tangent_operator (operators.hpp:31-33) for a linear material map.
inline NodalField apply_tangent_operator(const GridLayout& layout, const MaterialMap& map, const NodalField& u) {
  homfe_ctx* ctx = layout.context(u.components);
  detail::set_material(ctx, map);
  NodalField out(u.components, u.nodes);
  detail::check(homfe_gpu_apply_K(ctx, u.data.data(), out.data.data()));
  return out;
}

}  // namespace homfe

#endif
