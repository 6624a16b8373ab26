// ref_capi.cpp — thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled by oracle/Makefile into
// oracle/_ref/libsmpc_ref.so). TEST / BASELINE INFRASTRUCTURE ONLY: used to
// pin the oracle restatement (tests/golden via oracle/gen_golden.py) and as
// bench.py's `--impl reference` / cpu_baseline arm. Nothing here is shipped
// or called by the product path.
//
// Every function constructs the reference's own public types (DynamicsModel
// and CostFunction subclasses, GaussianSampler, RolloutEngine,
// MppiController, TubeMppiController) and calls their public methods.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "../include/smpc_b200.h"
#include "smpc/controllers.hpp"
#include "smpc/costmap.hpp"
#include "smpc/costs.hpp"
#include "smpc/dynamics.hpp"
#include "smpc/engine.hpp"
#include "smpc/plant.hpp"
#include "smpc/rng.hpp"
#include "smpc/sampling.hpp"

using namespace smpc;

namespace {

void set_err(char* err, size_t n, const std::string& msg) {
  if (err && n) {
    std::strncpy(err, msg.c_str(), n - 1);
    err[n - 1] = 0;
  }
}

double dp(const smpc_problem* p, int i, double d) { return i < p->n_dyn_params ? p->dyn_params[i] : d; }
double cp(const smpc_problem* p, int i, double d) { return i < p->n_cost_params ? p->cost_params[i] : d; }

std::shared_ptr<const DynamicsModel> make_dyn(const smpc_problem* p) {
  switch (p->dynamics_kind) {
    case SMPC_DYN_UNICYCLE:
      return std::make_shared<UnicycleModel>();
    case SMPC_DYN_CARTPOLE: {
      CartpoleParams c;
      c.cart_mass = (float)dp(p, 0, 1.0);
      c.pole_mass = (float)dp(p, 1, 1.0);
      c.pole_length = (float)dp(p, 2, 1.0);
      c.gravity = (float)dp(p, 3, 9.81);
      return std::make_shared<CartpoleModel>(c);
    }
    case SMPC_DYN_DIFF_DRIVE: {
      DiffDriveParams d;
      d.wheel_radius = (float)dp(p, 0, 1.0);
      d.wheel_length = (float)dp(p, 1, 1.0);
      d.v_min = (float)dp(p, 2, -0.35);
      d.v_max = (float)dp(p, 3, 0.5);
      d.w_min = (float)dp(p, 4, -0.5);
      d.w_max = (float)dp(p, 5, 0.5);
      return std::make_shared<DiffDriveModel>(d);
    }
    case SMPC_DYN_DOUBLE_INTEGRATOR:
      return std::make_shared<DoubleIntegrator2DModel>();
  }
  throw ConfigError("dynamics.kind is not recognized");
}

std::shared_ptr<const CostFunction> make_cst(const smpc_problem* p, const DynamicsModel& dyn) {
  const ModelDims& dims = dyn.dims();
  switch (p->cost_kind) {
    case SMPC_COST_ROAD: {
      RoadCostParams r;
      r.half_width = (float)cp(p, 0, 1.0);
      r.linear_coeff = (float)cp(p, 1, 1.0);
      r.quadratic_coeff = (float)cp(p, 2, 10.0);
      return std::make_shared<RoadCost>(r, dims.n_y, dims.n_u);
    }
    case SMPC_COST_CIRCLE_TRACK: {
      CircleTrackCostParams c;
      c.inner_radius = (float)cp(p, 0, 1.875);
      c.outer_radius = (float)cp(p, 1, 2.125);
      c.crash_cost = (float)cp(p, 2, 1000.0);
      c.speed_target = (float)cp(p, 3, 2.0);
      c.speed_coeff = (float)cp(p, 4, 2.0);
      c.angular_momentum_target = (float)cp(p, 5, 4.0);
      c.angular_momentum_coeff = (float)cp(p, 6, 2.0);
      return std::make_shared<CircleTrackCost>(c);
    }
    case SMPC_COST_DIFF_DRIVE_NAV: {
      DiffDriveNavCostParams n;
      n.goal_x = (float)cp(p, 0, 2.0);
      n.goal_y = (float)cp(p, 1, 2.0);
      n.goal_yaw = (float)cp(p, 2, 0.0);
      n.dist_coeff = (float)cp(p, 3, 5.0);
      n.yaw_coeff = (float)cp(p, 4, 5.0);
      n.obstacle_cost = (float)cp(p, 5, 20.0);
      const double res = p->costmap_resolution;
      auto map = std::make_shared<Costmap2D>(p->costmap_cells_x * res, p->costmap_cells_y * res,
                                             res, p->costmap_origin_x, p->costmap_origin_y);
      if (map->cells_x() != p->costmap_cells_x || map->cells_y() != p->costmap_cells_y) {
        throw Error("ref_capi: costmap geometry does not round-trip");
      }
      if (p->costmap) {
        for (int iy = 0; iy < p->costmap_cells_y; ++iy)
          for (int ix = 0; ix < p->costmap_cells_x; ++ix)
            map->set_cell(ix, iy, p->costmap[(size_t)iy * p->costmap_cells_x + ix] != 0);
      }
      return std::make_shared<DiffDriveNavCost>(n, map);
    }
    case SMPC_COST_QUADRATIC: {
      std::vector<float> t(p->quad_target, p->quad_target + p->n_quad);
      std::vector<float> w(p->quad_weights, p->quad_weights + p->n_quad);
      return std::make_shared<QuadraticCost>(t, w, dims.n_u);
    }
  }
  throw ConfigError("cost.kind is not recognized");
}

GaussianSamplerConfig sampler_cfg(const smpc_problem* p, int n_u) {
  GaussianSamplerConfig c;
  c.std_dev.assign(p->control_std, p->control_std + p->n_control_std);
  if (c.std_dev.size() == 1 && n_u > 1) c.std_dev.assign((size_t)n_u, c.std_dev[0]);
  if (p->std_per_step) {
    for (int t = 0; t < p->horizon; ++t)
      c.std_per_step.emplace_back(p->std_per_step + (size_t)t * n_u,
                                  p->std_per_step + (size_t)(t + 1) * n_u);
  }
  c.zero_mean_fraction = p->zero_mean_fraction;
  c.include_mean_sample = p->include_mean_sample != 0;
  c.importance_sampling = p->importance_sampling != 0;
  c.seed = p->seed;
  return c;
}

ControlTrajectory traj(const float* mean, int T, int n_u, double dt) {
  std::vector<ControlVector> cs;
  for (int t = 0; t < T; ++t) {
    Vec v(n_u);
    for (int c = 0; c < n_u; ++c) v[c] = mean[(size_t)t * n_u + c];
    cs.emplace_back(v);
  }
  return ControlTrajectory(dt, std::move(cs));
}

void untraj(const ControlTrajectory& tr, float* out) {
  const int n_u = tr.control_dim();
  for (int t = 0; t < tr.horizon(); ++t)
    for (int c = 0; c < n_u; ++c) out[(size_t)t * n_u + c] = tr.at(t)[c];
}

StateVector state(const float* x, int n) {
  Vec v(n);
  for (int i = 0; i < n; ++i) v[i] = x[i];
  return StateVector(v);
}

EngineConfig engine_cfg(int workers, int strategy) {
  EngineConfig e;
  e.num_workers = workers;
  e.strategy = strategy == 0   ? StrategyChoice::Kind::kSplit
               : strategy == 1 ? StrategyChoice::Kind::kFused
                               : StrategyChoice::Kind::kAuto;
  return e;
}

MppiSettings settings(const smpc_problem* p) {
  MppiSettings s;
  s.num_samples = p->num_samples;
  s.iterations = p->iterations;
  s.lambda = p->lambda;
  s.dt = p->dt;
  s.horizon = p->horizon;
  if (p->step_sizes && p->n_step_sizes > 0)
    s.step_sizes.assign(p->step_sizes, p->step_sizes + p->n_step_sizes);
  return s;
}

void fill_solution(const ControllerSolution& sol, float* controls, float* states, float* outputs,
                   double* weights, double* summary4) {
  if (controls) untraj(sol.controls, controls);
  if (states) {
    size_t k = 0;
    for (const auto& x : sol.states)
      for (int i = 0; i < x.dim(); ++i) states[k++] = x[i];
  }
  if (outputs) {
    size_t k = 0;
    for (const auto& y : sol.outputs.outputs)
      for (int i = 0; i < y.dim(); ++i) outputs[k++] = y[i];
  }
  const auto& w = sol.weights.weights;
  if (weights) std::copy(w.begin(), w.end(), weights);
  if (summary4) {
    summary4[0] = sol.weights.baseline;
    summary4[1] = sol.weights.normalizer;
    // argmin cost == first maximum weight (weights are monotone in cost).
    summary4[2] = (double)(std::max_element(w.begin(), w.end()) - w.begin());
    summary4[3] = sol.solve_time_ms;
  }
}

struct RefController {
  std::unique_ptr<Controller> ctl;
  bool tube = false;
  int n_x = 0, n_u = 0, n_y = 0;
};

}  // namespace

extern "C" {

void ref_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const auto w = philox::block({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = w[i];
}

void ref_quad(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, float out[4]) {
  const auto z = NormalStream(seed).quad(a, b, c);
  for (int i = 0; i < 4; ++i) out[i] = z[i];
}

int ref_generate_samples(const smpc_problem* p, const float* mean, uint32_t stream, int workers,
                         float* eps, uint8_t* flags, char* err, size_t errn) {
  try {
    auto dyn = make_dyn(p);
    const int n_u = dyn->dims().n_u;
    GaussianSampler sampler(sampler_cfg(p, n_u), n_u);
    WorkerPool pool(workers);
    const NoiseBatch b = sampler.generate_samples(traj(mean, p->horizon, n_u, p->dt),
                                                  p->num_samples, stream, &pool);
    std::copy(b.eps.begin(), b.eps.end(), eps);
    if (flags)
      for (int m = 0; m < p->num_samples; ++m)
        flags[m] = (uint8_t)((b.is_mean_sample[m] ? 1 : 0) | (b.is_zero_mean[m] ? 2 : 0));
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

// Rollout of an injected batch through RolloutEngine (split=0 / fused=1),
// with the importance adjustment computed by the reference sampler about
// means[s] when p->importance_sampling is set.
int ref_rollout(const smpc_problem* p, int S, const float* x0s, const float* means,
                const float* eps, int strategy, int workers, double* costs, float* outputs,
                char* err, size_t errn) {
  try {
    auto dyn = make_dyn(p);
    auto cost = make_cst(p, *dyn);
    const ModelDims d = dyn->dims();
    const int T = p->horizon, M = p->num_samples;
    GaussianSampler sampler(sampler_cfg(p, d.n_u), d.n_u);
    NoiseBatch batch;
    batch.num_samples = M;
    batch.horizon = T;
    batch.control_dim = d.n_u;
    batch.mean = traj(means, T, d.n_u, p->dt);
    batch.eps.assign(eps, eps + (size_t)M * T * d.n_u);
    batch.is_mean_sample.assign((size_t)M, 0);
    batch.is_zero_mean.assign((size_t)M, 0);
    batch.importance_enabled.assign((size_t)M, p->importance_sampling ? 1 : 0);
    RolloutRequest req;
    req.dynamics = dyn.get();
    req.cost = cost.get();
    req.noise = &batch;
    for (int s = 0; s < S; ++s) {
      req.initial_states.push_back(state(x0s + (size_t)s * d.n_x, d.n_x));
      req.means.push_back(traj(means + (size_t)s * T * d.n_u, T, d.n_u, p->dt));
      if (p->importance_sampling)
        req.cost_adjustments.push_back(
            sampler.importance_weight_adjustment(batch, req.means.back(), p->lambda));
    }
    RolloutEngine engine(engine_cfg(workers, strategy));
    const RolloutResult r = strategy == 0 ? engine.rollout_split(req) : engine.rollout_fused(req);
    for (int s = 0; s < S; ++s) std::copy(r.costs[s].begin(), r.costs[s].end(), costs + (size_t)s * M);
    if (outputs) {
      if (!r.outputs) throw Error("ref_rollout: outputs need the split strategy");
      std::copy(r.outputs->data.begin(), r.outputs->data.end(), outputs);
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

int ref_compute_weights(const double* costs, int64_t n, double lambda, double* weights,
                        double* baseline, double* normalizer, char* err, size_t errn) {
  try {
    const WeightResult w = RolloutEngine::compute_weights(std::span<const double>(costs, (size_t)n), lambda);
    std::copy(w.weights.begin(), w.weights.end(), weights);
    *baseline = w.baseline;
    *normalizer = w.normalizer;
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

void* ref_controller_create(const smpc_problem* p, int workers, int strategy, char* err, size_t errn) {
  try {
    auto dyn = make_dyn(p);
    auto cost = make_cst(p, *dyn);
    auto rc = new RefController();
    rc->n_x = dyn->dims().n_x;
    rc->n_u = dyn->dims().n_u;
    rc->n_y = dyn->dims().n_y;
    const GaussianSamplerConfig sc = sampler_cfg(p, rc->n_u);
    if (p->controller_kind == SMPC_CTRL_TUBE) {
      PidGains g;
      g.kp = GainMatrix::Zero(rc->n_u, rc->n_x);
      g.ki = GainMatrix::Zero(rc->n_u, rc->n_x);
      g.kd = GainMatrix::Zero(rc->n_u, rc->n_x);
      g.dt = (float)p->dt;
      rc->ctl = std::make_unique<TubeMppiController>(dyn, cost, sc, settings(p), g,
                                                     p->nominal_reset_bound,
                                                     engine_cfg(workers, strategy));
      rc->tube = true;
    } else if (p->controller_kind == SMPC_CTRL_CEM) {
      CemSettings cem;
      cem.elite_fraction = p->elite_fraction;
      rc->ctl = std::make_unique<CemController>(dyn, cost, sc, settings(p), cem, engine_cfg(workers, strategy));
    } else {
      rc->ctl = std::make_unique<MppiController>(dyn, cost, sc, settings(p),
                                                 engine_cfg(workers, strategy),
                                                 p->controller_kind == SMPC_CTRL_DMD ? "dmd" : "mppi");
    }
    return rc;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return nullptr;
  }
}

void ref_controller_destroy(void* h) { delete static_cast<RefController*>(h); }

// Plant::run_control_loop (plant.cpp:133-181) on a fresh single-system
// controller with the reference's own Plant and SimulatedSystem (seeded as
// make_simulated_system does, plant.cpp:224-230). rows: steps x (2+n_x+n_u).
int ref_run_control_loop(const smpc_problem* p, double replan_rate, double dt_min, double disturbance_std,
                         const float* x0, double duration_s, int workers, double* accumulated, double* rows,
                         int64_t* n_rows, char* err, size_t errn) {
  try {
    void* h = ref_controller_create(p, workers, 1, err, errn);
    if (!h) return 3;
    std::unique_ptr<RefController> rc(static_cast<RefController*>(h));
    std::shared_ptr<Controller> ctl(std::move(rc->ctl));
    PlantConfig pc;
    pc.replan_rate = replan_rate;
    pc.dt_min = dt_min;
    Plant plant(pc, ctl);
    auto dyn = make_dyn(p);
    SimulatedSystem sim(dyn, state(x0, dyn->dims().n_x), disturbance_std, p->seed ^ 0x9E3779B97F4A7C15ull);
    const LoopResult r = plant.run_control_loop(sim, duration_s);
    *accumulated = r.accumulated_cost;
    *n_rows = (int64_t)r.rows.size();
    if (rows) {
      size_t k = 0;
      for (const auto& row : r.rows) {
        rows[k++] = row.t;
        for (int i = 0; i < row.x.dim(); ++i) rows[k++] = row.x[i];
        for (int i = 0; i < row.u.dim(); ++i) rows[k++] = row.u[i];
        rows[k++] = row.running_cost;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

int ref_set_mean(void* h, const float* mean) {
  auto* rc = static_cast<RefController*>(h);
  rc->ctl->set_mean(traj(mean, rc->ctl->horizon(), rc->n_u, rc->ctl->dt()));
  return 0;
}

int ref_get_mean(void* h, float* mean) {
  untraj(static_cast<RefController*>(h)->ctl->mean(), mean);
  return 0;
}

int ref_shift_control_sequence(void* h, double elapsed_s, double dt_min, char* err, size_t errn) {
  try {
    static_cast<RefController*>(h)->ctl->shift_control_sequence(elapsed_s, dt_min);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

// summary4 = {baseline, normalizer, argmin, solve_time_ms}
int ref_compute_control(void* h, const float* x0, float* controls, float* states, float* outputs,
                        double* weights, double* summary4, char* err, size_t errn) {
  try {
    auto* rc = static_cast<RefController*>(h);
    const ControllerSolution sol = rc->ctl->compute_control(state(x0, rc->n_x));
    fill_solution(sol, controls, states, outputs, weights, summary4);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

int ref_tube_compute_control(void* h, const float* x_real, float* nominal_controls,
                             float* nominal_states, double* nominal_summary4, float* real_controls,
                             float* real_states, double* real_summary4, float* nominal_state,
                             char* err, size_t errn) {
  try {
    auto* rc = static_cast<RefController*>(h);
    auto* tube = dynamic_cast<TubeMppiController*>(rc->ctl.get());
    if (!tube) throw Error("ref_tube_compute_control: not a tube controller");
    const TubeSolution sol = tube->tube_compute_control(state(x_real, rc->n_x));
    fill_solution(sol.nominal, nominal_controls, nominal_states, nullptr, nullptr, nominal_summary4);
    fill_solution(sol.real, real_controls, real_states, nullptr, nullptr, real_summary4);
    if (nominal_state)
      for (int i = 0; i < rc->n_x; ++i) nominal_state[i] = sol.nominal_state[i];
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errn, e.what());
    return 3;
  }
}

}  // extern "C"
