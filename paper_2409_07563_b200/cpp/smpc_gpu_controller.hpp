// smpc_gpu_controller.hpp — drop-in B200 controllers for the reference
// `smpc` C++ library (/root/reference/proj/core).
//
// Header-only adapter a maintainer adds next to controllers.hpp. It derives
// from the reference's own abstract smpc::Controller (controllers.hpp:42-84),
// so every caller of that interface — Plant (plant.hpp:63-66, takes
// std::shared_ptr<Controller>), bench_timing-style loops, user code — drives
// the GPU iteration unchanged:
//
//   auto ctl = smpc::gpu::make_gpu_controller(scenario);   // mppi | dmd | tube
//   smpc::Plant plant(plant_config, ctl);                    // reference Plant
//
// The hot path (sample -> rollout -> weights -> update -> nominal rollout)
// runs through the C ABI in include/smpc_b200.h; nothing here does per-sample
// work. Controller::mean_ stays the source of truth for the warm start (the
// base class's shift_control_sequence / set_mean / reset_mean keep working):
// it is uploaded before and read back after every solve.
#pragma once

#include <cmath>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "smpc/controllers.hpp"
#include "smpc/costmap.hpp"
#include "smpc/costs.hpp"
#include "smpc/dynamics.hpp"
#include "smpc/feedback.hpp"
#include "smpc/scenario.hpp"
#include "smpc_b200.h"

namespace smpc::gpu {

/// smpc_status -> the reference's exception types (types.hpp:24-33).
inline void check(smpc_status st, const smpc_ctx* ctx) {
  if (st == SMPC_OK) return;
  const std::string msg = smpc_last_error(ctx);
  if (st == SMPC_ERR_CONFIG) throw ConfigError(msg);
  throw Error(msg);
}

/// Owns the flattened problem plus the arrays its pointers refer to.
struct Problem {
  smpc_problem p{};
  std::vector<float> std_per_step, step_sizes;
  std::vector<uint8_t> costmap;
};

/// ScenarioConfig (scenario.hpp:118-140) -> smpc_problem, with the same
/// kind strings as make_dynamics / make_cost / make_controller.
inline Problem make_problem(const ScenarioConfig& sc, int device = 0, bool plugin = false) {
  Problem out;
  smpc_problem& p = out.p;
  p.abi_version = SMPC_B200_ABI_VERSION;
  p.num_samples = sc.num_samples;
  p.horizon = sc.horizon;
  p.iterations = sc.iterations;
  p.dt = sc.dt;
  p.lambda = sc.lambda;
  p.seed = sc.rng_seed;
  p.n_control_std = static_cast<int32_t>(sc.control_std.size());
  for (size_t i = 0; i < sc.control_std.size() && i < SMPC_MAX_DIM; ++i)
    p.control_std[i] = static_cast<float>(sc.control_std[i]);
  for (const auto& row : sc.sampler.std_per_step)
    for (double v : row) out.std_per_step.push_back(static_cast<float>(v));
  p.zero_mean_fraction = sc.sampler.zero_mean_fraction;
  p.include_mean_sample = sc.sampler.include_mean_sample ? 1 : 0;
  p.importance_sampling = sc.sampler.importance_sampling ? 1 : 0;
  const std::string& ck = sc.controller.kind;
  p.controller_kind = ck == "dmd"    ? SMPC_CTRL_DMD
                      : ck == "tube" ? SMPC_CTRL_TUBE
                      : ck == "cem"  ? SMPC_CTRL_CEM
                                     : SMPC_CTRL_MPPI;
  if (ck != "mppi" && ck != "dmd" && ck != "tube" && ck != "cem")
    throw ConfigError("controller.kind '" + ck + "' is not recognized");
  if (ck == "dmd") {  // controllers.cpp:315-321
    if (!sc.controller.step_size_per_step.empty()) {
      for (double g : sc.controller.step_size_per_step) out.step_sizes.push_back(static_cast<float>(g));
    } else {
      out.step_sizes.push_back(static_cast<float>(sc.controller.step_size));
    }
  }
  p.nominal_reset_bound = sc.controller.nominal_reset_bound;
  p.elite_fraction = sc.controller.elite_fraction;
  const DynamicsSection& d = sc.dynamics;
  if (plugin) {  // a user model: its device functors carry the model and cost (smpc_create_with_ops)
    p.dynamics_kind = SMPC_DYN_PLUGIN;
  } else if (d.kind == "unicycle") {
    p.dynamics_kind = SMPC_DYN_UNICYCLE;
  } else if (d.kind == "cartpole") {
    p.dynamics_kind = SMPC_DYN_CARTPOLE;
    const double v[] = {d.cart_mass, d.pole_mass, d.pole_length, d.gravity};
    p.n_dyn_params = 4;
    for (int i = 0; i < 4; ++i) p.dyn_params[i] = v[i];
  } else if (d.kind == "diff_drive") {
    p.dynamics_kind = SMPC_DYN_DIFF_DRIVE;
    const double v[] = {d.wheel_radius, d.wheel_length, d.v_min, d.v_max, d.w_min, d.w_max};
    p.n_dyn_params = 6;
    for (int i = 0; i < 6; ++i) p.dyn_params[i] = v[i];
  } else if (d.kind == "double_integrator") {
    p.dynamics_kind = SMPC_DYN_DOUBLE_INTEGRATOR;
  } else {
    throw ConfigError("dynamics.kind '" + d.kind + "' is not recognized");
  }
  const CostSection& c = sc.cost;
  if (plugin) {
  } else if (c.kind == "road") {
    p.cost_kind = SMPC_COST_ROAD;
    const double v[] = {c.road_half_width, c.road_linear_coeff, c.road_quadratic_coeff};
    p.n_cost_params = 3;
    for (int i = 0; i < 3; ++i) p.cost_params[i] = v[i];
  } else if (c.kind == "circle_track") {
    p.cost_kind = SMPC_COST_CIRCLE_TRACK;
    const double v[] = {c.inner_radius, c.outer_radius, c.crash_cost, c.speed_target, c.speed_coeff,
                        c.angular_momentum_target, c.angular_momentum_coeff};
    p.n_cost_params = 7;
    for (int i = 0; i < 7; ++i) p.cost_params[i] = v[i];
  } else if (c.kind == "diff_drive_nav") {
    p.cost_kind = SMPC_COST_DIFF_DRIVE_NAV;
    const double v[] = {c.goal_x, c.goal_y, c.goal_yaw, c.dist_coeff, c.yaw_coeff, c.obstacle_cost};
    p.n_cost_params = 6;
    for (int i = 0; i < 6; ++i) p.cost_params[i] = v[i];
    // make_cost (costs.cpp:136-141): the file, or an all-free map of the configured size
    const Costmap2D map = !c.costmap_path.empty()
                              ? Costmap2D::load(c.costmap_path)
                              : Costmap2D(c.map_width, c.map_height, c.map_resolution, c.map_origin_x,
                                          c.map_origin_y);
    out.costmap.resize(static_cast<size_t>(map.cells_x()) * map.cells_y());
    for (int iy = 0; iy < map.cells_y(); ++iy)
      for (int ix = 0; ix < map.cells_x(); ++ix)
        out.costmap[static_cast<size_t>(iy) * map.cells_x() + ix] = map.cell(ix, iy) ? 1 : 0;
    p.costmap_cells_x = map.cells_x();
    p.costmap_cells_y = map.cells_y();
    p.costmap_resolution = map.resolution();
    p.costmap_origin_x = map.origin_x();
    p.costmap_origin_y = map.origin_y();
  } else if (c.kind == "quadratic") {
    p.cost_kind = SMPC_COST_QUADRATIC;
    p.n_quad = static_cast<int32_t>(c.weights.size());
    for (size_t i = 0; i < c.weights.size() && i < SMPC_MAX_DIM; ++i) {
      p.quad_weights[i] = static_cast<float>(c.weights[i]);
      p.quad_target[i] = c.target.empty() ? 0.0f : static_cast<float>(c.target[i]);
    }
  } else {
    throw ConfigError("cost.kind '" + c.kind + "' is not recognized");
  }
  p.device = device;
  p.update_skip_mass = 0.0;  // exact reference semantics by default
  if (!out.std_per_step.empty()) p.std_per_step = out.std_per_step.data();
  if (!out.step_sizes.empty()) {
    p.step_sizes = out.step_sizes.data();
    p.n_step_sizes = static_cast<int32_t>(out.step_sizes.size());
  }
  if (!out.costmap.empty()) p.costmap = out.costmap.data();
  return out;
}

/// MppiController / DMD / CemController on the B200: drop-in for
/// smpc::MppiController (controllers.hpp:89-97) and smpc::CemController
/// (controllers.hpp:103-116).
class GpuMppiController : public Controller {
 public:
  GpuMppiController(const ScenarioConfig& scenario, int device = 0, double update_skip_mass = 0.0)
      : GpuMppiController(scenario, make_problem(scenario, device), update_skip_mass) {}

  /// A user model: the user's own reference-side DynamicsModel / CostFunction
  /// subclasses (dynamics.hpp:17-74, costs.hpp:16-37 — Plant and
  /// SimulatedSystem keep using them) plus their device twins compiled
  /// against include/smpc_b200_plugin.cuh (ops, from smpc_ops_for). The
  /// scenario supplies the sampler / controller / plant sections.
  GpuMppiController(std::shared_ptr<const DynamicsModel> dynamics, std::shared_ptr<const CostFunction> cost,
                    const ScenarioConfig& scenario, const smpc_model_ops& ops, int device = 0,
                    double update_skip_mass = 0.0)
      : Controller(scenario.controller.kind, dynamics, std::move(cost),
                   make_sampler_config(scenario, dynamics->dims().n_u), settings_from(scenario), single_worker()),
        problem_(make_problem(scenario, device, true)) {
    problem_.p.update_skip_mass = update_skip_mass;
    check(smpc_create_with_ops(&problem_.p, &ops, &ctx_), nullptr);
  }

  ~GpuMppiController() override { smpc_destroy(ctx_); }
  GpuMppiController(const GpuMppiController&) = delete;
  GpuMppiController& operator=(const GpuMppiController&) = delete;

  ControllerSolution compute_control(const StateVector& x0) override {
    upload_mean(0, mean_);
    const int T = horizon(), n_u = dynamics().dims().n_u, n_x = dynamics().dims().n_x,
              n_y = dynamics().dims().n_y;
    std::vector<float> controls(static_cast<size_t>(T) * n_u), states(static_cast<size_t>(T + 1) * n_x),
        outputs(static_cast<size_t>(T) * n_y);
    std::vector<double> weights(static_cast<size_t>(settings_.num_samples));
    smpc_solution sol{};
    sol.controls = controls.data();
    sol.states = states.data();
    sol.outputs = outputs.data();
    sol.weights = weights.data();
    check(smpc_compute_control(ctx_, x0.data(), &sol), ctx_);
    mean_ = to_trajectory(controls, T, n_u);
    return to_solution(sol, controls, states, outputs, std::move(weights), T, n_x, n_y);
  }

 protected:
  GpuMppiController(const ScenarioConfig& scenario, Problem prob, double skip, std::string name = "")
      : Controller(name.empty() ? scenario.controller.kind : name, make_dynamics(scenario.dynamics),
                   cost_of(scenario), make_sampler_config(scenario, n_u_of(scenario)),
                   settings_from(scenario), single_worker()),
        problem_(std::move(prob)) {
    problem_.p.update_skip_mass = skip;
    check(smpc_create(&problem_.p, &ctx_), nullptr);
  }

  // The reference's own model / cost objects back dynamics() / cost() (used by
  // Plant for logging); the solve itself never calls them.
  static std::shared_ptr<const CostFunction> cost_of(const ScenarioConfig& sc) {
    const std::unique_ptr<DynamicsModel> dyn = make_dynamics(sc.dynamics);
    return make_cost(sc.cost, *dyn);
  }
  static int n_u_of(const ScenarioConfig& sc) { return make_dynamics(sc.dynamics)->dims().n_u; }

  static MppiSettings settings_from(const ScenarioConfig& sc) {
    MppiSettings s;
    s.num_samples = sc.num_samples;
    s.iterations = sc.iterations;
    s.lambda = sc.lambda;
    s.dt = sc.dt;
    s.horizon = sc.horizon;
    return s;
  }
  // The base class owns a (never used) CPU RolloutEngine: keep it thread-free.
  static EngineConfig single_worker() {
    EngineConfig e;
    e.num_workers = 1;
    e.strategy = StrategyChoice::Kind::kFused;
    return e;
  }

  void upload_mean(int system, const ControlTrajectory& m) {
    const int T = m.horizon(), n_u = m.control_dim();
    std::vector<float> flat(static_cast<size_t>(T) * n_u);
    for (int t = 0; t < T; ++t)
      for (int c = 0; c < n_u; ++c) flat[static_cast<size_t>(t) * n_u + c] = m.at(t)[c];
    check(smpc_set_mean(ctx_, system, flat.data()), ctx_);
  }

  ControlTrajectory to_trajectory(const std::vector<float>& flat, int T, int n_u) const {
    std::vector<ControlVector> cs;
    cs.reserve(static_cast<size_t>(T));
    for (int t = 0; t < T; ++t) {
      Vec v(n_u);
      for (int c = 0; c < n_u; ++c) v[c] = flat[static_cast<size_t>(t) * n_u + c];
      cs.emplace_back(std::move(v));
    }
    return ControlTrajectory(settings_.dt, std::move(cs));
  }

  ControllerSolution to_solution(const smpc_solution& sol, const std::vector<float>& controls,
                                 const std::vector<float>& states, const std::vector<float>& outputs,
                                 std::vector<double> weights, int T, int n_x, int n_y) const {
    ControllerSolution out;
    out.controls = to_trajectory(controls, T, static_cast<int>(controls.size() / T));
    for (int t = 0; t <= T; ++t) {
      Vec v(n_x);
      for (int i = 0; i < n_x; ++i) v[i] = states[static_cast<size_t>(t) * n_x + i];
      out.states.emplace_back(std::move(v));
    }
    for (int t = 0; t < T; ++t) {
      Vec v(n_y);
      for (int i = 0; i < n_y; ++i) v[i] = outputs[static_cast<size_t>(t) * n_y + i];
      out.outputs.outputs.emplace_back(std::move(v));
    }
    out.weights.baseline = sol.summary.baseline;
    out.weights.normalizer = sol.summary.normalizer;
    out.weights.weights = std::move(weights);
    out.solve_time_ms = sol.solve_time_ms;
    return out;
  }

  Problem problem_;
  smpc_ctx* ctx_ = nullptr;
};

/// TubeMppiController on the B200 (controllers.hpp:134-160): nominal and real
/// systems share one noise batch per iteration, rolled out by the same
/// threads. The PID correction is the reference's own PidController.
class GpuTubeMppiController : public GpuMppiController {
 public:
  GpuTubeMppiController(const ScenarioConfig& scenario, int device = 0, double update_skip_mass = 0.0)
      : GpuMppiController(scenario, make_problem(scenario, device), update_skip_mass, "tube"),
        pid_(make_pid_gains(scenario.feedback, dynamics().dims().n_u, dynamics().dims().n_x,
                            static_cast<float>(scenario.dt))),
        real_mean_(mean_) {
    pid_state_ = pid_.make_state();
  }

  TubeSolution tube_compute_control(const StateVector& x_real) {
    upload_mean(0, mean_);
    upload_mean(1, real_mean_);
    const int T = horizon(), n_u = dynamics().dims().n_u, n_x = dynamics().dims().n_x,
              n_y = dynamics().dims().n_y;
    std::vector<float> nc(static_cast<size_t>(T) * n_u), rc(nc.size());
    std::vector<float> ns(static_cast<size_t>(T + 1) * n_x), rs(ns.size());
    std::vector<float> no(static_cast<size_t>(T) * n_y), ro(no.size());
    std::vector<float> nominal(static_cast<size_t>(n_x));
    smpc_tube_solution sol{};
    sol.nominal.controls = nc.data();
    sol.nominal.states = ns.data();
    sol.nominal.outputs = no.data();
    sol.real.controls = rc.data();
    sol.real.states = rs.data();
    sol.real.outputs = ro.data();
    sol.nominal_state = nominal.data();
    check(smpc_tube_compute_control(ctx_, x_real.data(), &sol), ctx_);
    mean_ = to_trajectory(nc, T, n_u);
    real_mean_ = to_trajectory(rc, T, n_u);
    TubeSolution out;
    out.nominal = to_solution(sol.nominal, nc, ns, no, {}, T, n_x, n_y);
    out.real = to_solution(sol.real, rc, rs, ro, {}, T, n_x, n_y);
    Vec nv(n_x);
    for (int i = 0; i < n_x; ++i) nv[i] = nominal[static_cast<size_t>(i)];
    out.nominal_state = StateVector(std::move(nv));
    // applied = u0 + PID(x_real -> nominal) (controllers.cpp:269-273)
    const ControlVector corr = pid_.feedback(x_real, out.nominal_state, pid_state_);
    Vec applied(corr.dim());
    for (Eigen::Index c = 0; c < applied.size(); ++c) applied[c] = mean_.at(0)[c] + corr[c];
    out.applied = ControlVector(std::move(applied));
    return out;
  }

  ControllerSolution compute_control(const StateVector& x0) override { return tube_compute_control(x0).nominal; }

  void shift_control_sequence(double elapsed_s, double dt_min) override {
    Controller::shift_control_sequence(elapsed_s, dt_min);
    ControlTrajectory nominal = mean_;
    mean_ = real_mean_;
    Controller::shift_control_sequence(elapsed_s, dt_min);
    real_mean_ = mean_;
    mean_ = std::move(nominal);
  }

 private:
  PidController pid_;
  PidState pid_state_;
  ControlTrajectory real_mean_;
};

/// make_controller (controllers.cpp:294-344) for the B200 path.
inline std::shared_ptr<Controller> make_gpu_controller(const ScenarioConfig& scenario, int device = 0,
                                                       double update_skip_mass = 0.0) {
  const std::vector<std::string> errors = validate(scenario);
  if (!errors.empty()) {
    std::string message = "scenario invalid:";
    for (const auto& e : errors) message += "\n  " + e;
    throw ConfigError(message);
  }
  if (scenario.controller.kind == "tube")
    return std::make_shared<GpuTubeMppiController>(scenario, device, update_skip_mass);
  // mppi / dmd / cem share the single-system context; CEM's elite selection
  // replaces the softmin weights on the device (controllers.cpp:149-203).
  if (scenario.controller.kind == "mppi" || scenario.controller.kind == "dmd" || scenario.controller.kind == "cem")
    return std::make_shared<GpuMppiController>(scenario, device, update_skip_mass);
  throw ConfigError("controller.kind '" + scenario.controller.kind + "' is not recognized");
}

}  // namespace smpc::gpu
