// Drop-in check for USER models: a damped spring-mass written as the
// reference's own DynamicsModel / CostFunction subclasses (dynamics.hpp:17-74,
// costs.hpp:16-37) drives (a) the unmodified reference MppiController and
// (b) smpc::gpu::GpuMppiController, whose solve runs the same model's device
// twin compiled out of tree against include/smpc_b200_plugin.cuh
// (tests/native/user_model.cu, loaded with dlopen). Both then run the
// reference Plant closed loop. Prints one JSON line per controller.
// Built by tests/test_drop_in.py; test infrastructure only.
#include <dlfcn.h>

#include <cstdio>
#include <memory>
#include <string>

#include "smpc/controllers.hpp"
#include "smpc/plant.hpp"
#include "smpc/scenario.hpp"
#include "../../paper_2409_07563_b200/cpp/smpc_gpu_controller.hpp"

using namespace smpc;

// p' = v, v' = (f - k p - c v) * 0.5, |f| <= f_max  (user_model.cu SpringMass)
class SpringMassModel : public DynamicsModel {
 public:
  SpringMassModel(float k, float c, float f_max)
      : DynamicsModel(ModelDims{2, 1, 2}, "spring_mass", {"P", "V"}), k_(k), c_(c) {
    set_control_bounds({-f_max}, {f_max});
  }
  using DynamicsModel::state_derivative;
  void state_derivative(const float* x, const float* u, float* dx) const override {
    dx[0] = x[1];
    dx[1] = ((u[0] - k_ * x[0]) - c_ * x[1]) * 0.5f;
  }

 private:
  float k_, c_;
};

// (p - 1)^2 + 0.1 v^2 + 0.01 u^2, terminal 10 (p - 1)^2  (user_model.cu SpringCost)
class SpringCostFn : public CostFunction {
 public:
  SpringCostFn() : CostFunction("spring_cost", 2, 1) {}
  double running_cost_raw(const float* y, const float* u, int) const override {
    const double dp = static_cast<double>(y[0]) - 1.0;
    const double v = y[1], f = u[0];
    return (dp * dp + 0.1 * (v * v)) + 0.01 * (f * f);
  }
  double terminal_cost_raw(const float* y) const override {
    const double dp = static_cast<double>(y[0]) - 1.0;
    return 10.0 * (dp * dp);
  }
};

static void run(const char* label, std::shared_ptr<Controller> ctl, std::shared_ptr<const DynamicsModel> dyn,
                const ScenarioConfig& sc, double seconds) {
  const StateVector x0 = dyn->state_from_named_values(sc.initial_state);
  const ControllerSolution first = ctl->compute_control(x0);
  int argmax = 0;
  for (size_t m = 1; m < first.weights.weights.size(); ++m)
    if (first.weights.weights[m] > first.weights.weights[argmax]) argmax = (int)m;
  std::printf("{\"impl\": \"%s\", \"rho\": %.17g, \"eta\": %.17g, \"argmax_w\": %d, \"u\": [", label,
              first.weights.baseline, first.weights.normalizer, argmax);
  for (int t = 0; t < first.controls.horizon(); ++t) std::printf("%s%.9g", t ? ", " : "", first.controls.at(t)[0]);
  ctl->reset_mean();
  PlantConfig pc;
  pc.replan_rate = sc.plant.replan_rate;
  pc.dt_min = sc.plant.dt_min;
  Plant plant(pc, ctl);
  SimulatedSystem sim(dyn, x0, 0.0, 1);
  const LoopResult res = plant.run_control_loop(sim, seconds);
  std::printf("], \"solves\": %d, \"accumulated_cost\": %.17g, \"x\": [", res.solve_count, res.accumulated_cost);
  for (size_t r = 0; r < res.rows.size(); ++r)
    std::printf("%s[%.9g, %.9g]", r ? ", " : "", res.rows[r].x[0], res.rows[r].x[1]);
  std::printf("]}\n");
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  try {
    void* h = dlopen(argv[1], RTLD_NOW);
    if (!h) {
      std::fprintf(stderr, "dlopen: %s\n", dlerror());
      return 2;
    }
    using OpsFn = smpc_model_ops (*)(float, float, float);
    const OpsFn spring_ops = reinterpret_cast<OpsFn>(dlsym(h, "spring_ops"));
    const smpc_model_ops ops = spring_ops(2.0f, 0.5f, 3.0f);
    ScenarioConfig sc;
    sc.num_samples = 2048;
    sc.horizon = 50;
    sc.dt = 0.02;
    sc.lambda = 1.0;
    sc.control_std = {1.0};
    sc.rng_seed = 5;
    sc.initial_state = {{"P", -0.5}};
    const double seconds = std::stod(argv[2]);
    auto dyn = std::make_shared<const SpringMassModel>(2.0f, 0.5f, 3.0f);
    auto cost = std::make_shared<const SpringCostFn>();
    EngineConfig ec;
    ec.num_workers = 4;
    auto ref = std::make_shared<MppiController>(dyn, cost, make_sampler_config(sc, 1), MppiSettings{
        sc.num_samples, sc.iterations, sc.lambda, sc.dt, sc.horizon, {}}, ec);
    run("reference", ref, dyn, sc, seconds);
    run("b200", std::make_shared<gpu::GpuMppiController>(dyn, cost, sc, ops), dyn, sc, seconds);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
  return 0;
}
