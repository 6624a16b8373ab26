// Builds device functors from the POD params and dispatches the cost kind for
// one dynamics model. Included once per dynamics TU (inst_*.cu) so the
// (dynamics x cost x systems x noise-mode) kernel instantiations compile in
// parallel translation units.
#pragma once

#include "kernels.cuh"

namespace smpc_dev {

template <class D>
struct is_bicycle : std::false_type {};
template <bool F>
struct is_bicycle<BicycleDyn<F>> : std::true_type {};

inline RoadCostDev make_road(const CostParams& c) {
  RoadCostDev r;
  r.half_width = c.p[0];
  r.lin_d = (double)c.p[1];
  r.quad_d = (double)c.p[2];
  r.lin_hw_d = r.lin_d * (double)c.p[0];  // static_cast<double>(linear) * half_width (costs.cpp:40)
  return r;
}

// CircleTrackCost ctor precomputes the squared radii in float (costs.cpp:50-51).
inline CircleTrackCostDev make_circle(const CostParams& c) {
  volatile float inner = c.p[0], outer = c.p[1];
  CircleTrackCostDev k;
  k.inner_sq = inner * inner;
  k.outer_sq = outer * outer;
  k.speed_target = c.p[3];
  k.am_target = c.p[5];
  volatile double zero = 0.0;
  k.crash0_d = zero + (double)c.p[2];  // cost = 0.0; cost += crash (costs.cpp:57-58)
  k.speed_coeff_d = (double)c.p[4];
  k.am_coeff_d = (double)c.p[6];
  return k;
}

inline NavCostDev make_nav(const CostParams& c) {
  NavCostDev n;
  n.goal_x = c.p[0], n.goal_y = c.p[1], n.goal_yaw = c.p[2];
  n.dist_d = (double)c.p[3], n.yaw_d = (double)c.p[4];
  volatile double one = 1.0, zero = 0.0;  // occupancy() returns 1.0f / 0.0f
  n.obst_occ_d = (double)c.p[5] * one;
  n.obst_free_d = (double)c.p[5] * zero;
  n.origin_x = c.origin_x, n.origin_y = c.origin_y, n.inv_resolution = c.inv_resolution;
  n.cells_x = c.cells_x, n.cells_y = c.cells_y;
  n.grid = c.grid;
  return n;
}

template <int NY>
inline QuadraticCostDev<NY> make_quad(const CostParams& c) {
  QuadraticCostDev<NY> q;
  for (int i = 0; i < NY; ++i) q.target_d[i] = (double)c.target[i], q.weights_d[i] = (double)c.weights[i];
  return q;
}

template <class Dyn>
cudaError_t rollout_dispatch(const Dyn& dyn, const IterArgs& a, int cost_kind, cudaStream_t st) {
  switch (cost_kind) {
    case 0:  // road: needs n_y >= 2 (costs.cpp:30); not offered for the builder-defined bicycle
      if constexpr (Dyn::NY >= 2 && !is_bicycle<Dyn>::value) return launch_rollout_t(a, dyn, make_road(a.cost), st);
      break;
    case 1:  // circle_track: (n_y, n_u) = (4, 2)
      if constexpr (Dyn::NY == 4 && Dyn::NU == 2) return launch_rollout_t(a, dyn, make_circle(a.cost), st);
      break;
    case 2:  // diff_drive_nav: (n_y, n_u) = (3, 2)
      if constexpr (Dyn::NY == 3 && Dyn::NU == 2) return launch_rollout_t(a, dyn, make_nav(a.cost), st);
      break;
    case 3:  // quadratic: n_quad == n_y (checked on the host)
      return launch_rollout_t(a, dyn, make_quad<Dyn::NY>(a.cost), st);
  }
  return cudaErrorInvalidValue;
}

template <class Dyn>
cudaError_t rmppi_dispatch(const Dyn& dyn, const IterArgs& a, int cost_kind, cudaStream_t st) {
  switch (cost_kind) {
    case 0:
      if constexpr (Dyn::NY >= 2 && !is_bicycle<Dyn>::value) return launch_rmppi_select_t(a, dyn, make_road(a.cost), st);
      break;
    case 1:
      if constexpr (Dyn::NY == 4 && Dyn::NU == 2) return launch_rmppi_select_t(a, dyn, make_circle(a.cost), st);
      break;
    case 2:
      if constexpr (Dyn::NY == 3 && Dyn::NU == 2) return launch_rmppi_select_t(a, dyn, make_nav(a.cost), st);
      break;
    case 3:
      return launch_rmppi_select_t(a, dyn, make_quad<Dyn::NY>(a.cost), st);
  }
  return cudaErrorInvalidValue;
}

template <class Dyn>
cudaError_t plant_dispatch(const Dyn& dyn, const IterArgs& a, int cost_kind, const PlantStepArgs& p,
                           cudaStream_t st) {
  switch (cost_kind) {
    case 0:
      if constexpr (Dyn::NY >= 2 && !is_bicycle<Dyn>::value) return launch_plant_step_t(a, dyn, make_road(a.cost), p, st);
      break;
    case 1:
      if constexpr (Dyn::NY == 4 && Dyn::NU == 2) return launch_plant_step_t(a, dyn, make_circle(a.cost), p, st);
      break;
    case 2:
      if constexpr (Dyn::NY == 3 && Dyn::NU == 2) return launch_plant_step_t(a, dyn, make_nav(a.cost), p, st);
      break;
    case 3:
      return launch_plant_step_t(a, dyn, make_quad<Dyn::NY>(a.cost), p, st);
  }
  return cudaErrorInvalidValue;
}

#define SMPC_DEFINE_OPS(NAME, DYN_T, ...)                                                       \
  namespace {                                                                                   \
  DYN_T NAME##_make(const DynParams& p) { __VA_ARGS__ }                                         \
  cudaError_t NAME##_rollout(const IterArgs& a, int ck, cudaStream_t st) {                       \
    return rollout_dispatch(NAME##_make(a.dyn), a, ck, st);                                      \
  }                                                                                             \
  cudaError_t NAME##_rmppi(const IterArgs& a, int ck, cudaStream_t st) {                          \
    return rmppi_dispatch(NAME##_make(a.dyn), a, ck, st);                                        \
  }                                                                                             \
  cudaError_t NAME##_plant(const IterArgs& a, int ck, const PlantStepArgs& p, cudaStream_t st) {   \
    return plant_dispatch(NAME##_make(a.dyn), a, ck, p, st);                                     \
  }                                                                                             \
  cudaError_t NAME##_update(const IterArgs& a, cudaStream_t st) {                                \
    return launch_update_t(a, NAME##_make(a.dyn), st);                                           \
  }                                                                                             \
  cudaError_t NAME##_combine(const IterArgs& a, cudaStream_t st) {                               \
    return launch_combine_t(a, NAME##_make(a.dyn), st);                                          \
  }                                                                                             \
  cudaError_t NAME##_generate(const IterArgs& a, float* e, uint8_t* f, cudaStream_t st) {        \
    return launch_generate_t<DYN_T::NU>(a, e, f, st);                                            \
  }                                                                                             \
  ModelOps NAME##_ops() {                                                                       \
    return ModelOps{NAME##_rollout, NAME##_rmppi, NAME##_plant, launch_weights, NAME##_update, NAME##_combine, \
                    NAME##_generate, DYN_T::NX, DYN_T::NU, DYN_T::NY};                           \
  }                                                                                             \
  }

}  // namespace smpc_dev
