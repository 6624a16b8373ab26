// Drop-in check: the reference's own Plant closed loop (plant.cpp:133-181)
// driven by smpc::gpu::make_gpu_controller vs the reference make_controller,
// from the same scenario JSON (argv[1]). Prints one JSON line per
// controller: the first solve's rho / eta / U*[0] and the closed-loop log.
// Built by tests/test_drop_in.py against /root/reference headers + oracle/_ref
// (the unmodified reference library) + libsmpc_b200.so.
#include <cstdio>
#include <memory>
#include <string>

#include "smpc/controllers.hpp"
#include "smpc/plant.hpp"
#include "smpc/scenario.hpp"
#include "../../paper_2409_07563_b200/cpp/smpc_gpu_controller.hpp"

using namespace smpc;

static void run(const char* label, std::shared_ptr<Controller> ctl, const ScenarioConfig& sc, double seconds) {
  const StateVector x0 = ctl->dynamics().state_from_named_values(sc.initial_state);
  const ControllerSolution first = ctl->compute_control(x0);
  std::printf("{\"impl\": \"%s\", \"rho\": %.17g, \"eta\": %.17g, \"u0\": [", label, first.weights.baseline,
              first.weights.normalizer);
  for (int c = 0; c < first.controls.control_dim(); ++c) std::printf("%s%.9g", c ? ", " : "", first.controls.at(0)[c]);
  ctl->reset_mean();
  PlantConfig pc;
  pc.replan_rate = sc.plant.replan_rate;
  pc.dt_min = sc.plant.dt_min;
  Plant plant(pc, ctl);
  std::shared_ptr<const DynamicsModel> dyn = make_dynamics(sc.dynamics);
  SimulatedSystem sim(dyn, x0, sc.plant.disturbance_std, 1);
  const LoopResult res = plant.run_control_loop(sim, seconds);
  std::printf("], \"solves\": %d, \"accumulated_cost\": %.17g, \"mean_solve_ms\": %.6f, \"x\": [", res.solve_count,
              res.accumulated_cost, res.mean_solve_ms);
  for (size_t r = 0; r < res.rows.size(); ++r) {
    std::printf("%s[", r ? ", " : "");
    for (int i = 0; i < res.rows[r].x.dim(); ++i) std::printf("%s%.9g", i ? ", " : "", res.rows[r].x[i]);
    std::printf("]");
  }
  std::printf("]}\n");
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  try {
    const ScenarioConfig sc = load_scenario(argv[1]);
    const double seconds = std::stod(argv[2]);
    EngineConfig ec;
    ec.num_workers = 4;
    run("reference", make_controller(sc, ec), sc, seconds);
    run("b200", gpu::make_gpu_controller(sc), sc, seconds);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
  return 0;
}
