// Drop-in example with a nonlinear catalog: J2 inclusions in an elastic
// matrix under a two-step load program (homfe::run_load_program with the
// committed internal state), then one explicit newton_solve from the
// returned state (the reference's 7-argument signature).
// Build: g++ -std=c++17 -I include examples/solve_j2.cpp
//          -L paper_2203_02962_b200/_lib -lhomfe_gpu -Wl,-rpath,<that dir>
#include <cstdio>

#include "homfe/gpu.hpp"

int main() {
  using namespace homfe;
  const Index n = 32;
  GridLayout layout({{n, n}, {1.0, 1.0}}, StencilKind::TwoTriangles);
  MaterialMap map;
  map.catalog = {MaterialModel::isotropic_elastic(1.0, 0.5, 2), MaterialModel::j2_plastic(2.0, 1.0, 2e-3, 0.05, 2)};
  map.phase.assign(static_cast<std::size_t>(n * n), 0);
  for (Index i = 0; i < n; ++i)
    for (Index j = 0; j < n; ++j) {
      const double x = (i + 0.5) / n - 0.5, y = (j + 0.5) / n - 0.5;
      if (x * x + y * y < 0.1) map.phase[static_cast<std::size_t>(i * n + j)] = 1;
    }
  SolveConfig cfg;
  cfg.eta_cg = 1e-8;
  cfg.eta_newton = 1e-7;
  try {
    const auto results = run_load_program(layout, map, {{2e-3, -1e-3, 2e-3}, {4e-3, -2e-3, 4e-3}}, cfg,
                                          ReferencePolicy::volume_mean());
    double peak = 0.0;
    for (const auto& r : results) {
      peak = 0.0;
      for (Index q = 0; q < r.outcome.internal.quads; ++q) {
        const double a = r.outcome.internal.data[static_cast<std::size_t>(q * 7 + 6)];
        peak = a > peak ? a : peak;
      }
      std::printf("load (%g, %g, %g): converged %d, newton %d, cg %d, <s12> = %.12e, max ep_acc = %.6e\n",
                  r.load[0], r.load[1], r.load[2], int(r.outcome.converged), r.outcome.report.newton_steps(),
                  r.outcome.report.total_cg(), r.outcome.average_stress[2], peak);
    }
    if (results.size() != 2 || !(peak > 0.0)) return 1;
    PrecondManager pm(ReferencePolicy::volume_mean(), cfg.reassembly_threshold, 2);
    const NewtonOutcome again =
        newton_solve(layout, map, results[1].outcome.internal, {4e-3, -2e-3, 4e-3}, cfg, pm, &results[1].outcome.u);
    std::printf("restart from the committed state: converged %d, newton %d, stress quads %zu\n",
                int(again.converged), again.report.newton_steps(), again.stress.size() / 3);
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
  return 0;
}
