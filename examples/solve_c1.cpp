// Drop-in example: the reference's C++ solver API (homfe::newton_solve,
// run_load_program) served by the B200 library through include/homfe/gpu.hpp.
// Build: g++ -std=c++17 -I include examples/solve_c1.cpp
//          -L paper_2203_02962_b200/_lib -lhomfe_gpu -Wl,-rpath,<that dir>
#include <cmath>
#include <cstdio>

#include "homfe/gpu.hpp"

int main() {
  using namespace homfe;
  const Index n = 64;
  GridLayout layout({{n, n}, {1.0, 1.0}}, StencilKind::TwoTriangles);
  MaterialMap map;
  map.catalog = {MaterialModel::isotropic_conductivity(1.0, 2), MaterialModel::isotropic_conductivity(10.0, 2)};
  map.phase.assign(static_cast<std::size_t>(n * n), 0);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      const double x = (i + 0.5) / n - 0.5, y = (j + 0.5) / n - 0.5;
      if (x * x + y * y < 0.09) map.phase[static_cast<std::size_t>(i * n + j)] = 1;
    }
  SolveConfig cfg;
  cfg.eta_cg = 1e-8;
  try {
    const auto results = run_load_program(layout, map, {{1.0, 0.0}, {0.0, 1.0}}, cfg,
                                          ReferencePolicy::explicit_matrix({1.0, 0.0, 0.0, 1.0}));
    for (const auto& r : results) {
      std::printf("load (%g, %g): converged %d, newton %d, cg %d, <q> = (%.12f, %.12f)\n", r.load[0], r.load[1],
                  int(r.outcome.converged), r.outcome.report.newton_steps(), r.outcome.report.total_cg(),
                  r.outcome.average_stress[0], r.outcome.average_stress[1]);
    }
    // error path mirrors the reference: bad tolerance -> ValidationError
    cfg.eta_cg = 2.0;
    PrecondManager pm(ReferencePolicy::volume_mean(), 0.1, 1);
    try {
      newton_solve(layout, map, {1.0, 0.0}, cfg, pm);
      std::printf("expected ValidationError\n");
      return 1;
    } catch (const ValidationError& e) {
      std::printf("ValidationError: %s\n", e.what());
    }
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
  return 0;
}
