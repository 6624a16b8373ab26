// User models for the B200 MPPI library without editing or rebuilding it —
// the device counterpart of subclassing the reference's DynamicsModel /
// CostFunction (dynamics.hpp:17-74, costs.hpp:16-37).
//
// A user writes two trivially copyable functors in their own .cu file:
//
//   struct MyModel {                       // DynamicsModel: dims + raw step
//     static constexpr int NX, NU, NY;     //   ModelDims (types.hpp:44-61)
//     static constexpr int ANGULAR;        //   wrapped state channel or -1
//     static constexpr bool BOUNDED;       //   clamp_control is applied
//     static constexpr bool POST_STEP;     //   post_step(x) after each Euler step
//     __device__ void state_derivative(const float* x, const float* u, float* dx) const;
//     __device__ void clamp_control(const float* u, float* out) const;
//     // optional: HEAVY_STEP, state_derivative_fast / post_step_fast (branch-free,
//     //           NaN where inexact -> the sample is replayed with the exact path)
//   };
//   struct MyCost {                        // CostFunction: running + terminal
//     static constexpr bool USES_MAP;      //   reads the problem's costmap (grid)
//     static constexpr bool USES_CONTROL;  //   optional; default true
//     __device__ double running_cost(const float* y, const float* u, int t) const;
//     __device__ double terminal_cost(const float* y) const;
//     // optional: running_cost_fast (same contract as state_derivative_fast)
//   };
//
// then, in that same translation unit:
//
//   #include "smpc_b200_plugin.cuh"
//   auto model = smpc_ops_for(MyModel{...}, MyCost{...});
//   smpc_model_ops ops = model.ops("my_model");
//   smpc_create_with_ops(&problem, &ops, &ctx);   // then every smpc_* call as usual
//
// smpc_ops_for instantiates this library's kernel templates (csrc/kernels.cuh:
// fused rollout + Philox sampler + importance term + block argmin, weighted
// update + nominal rollout, multi-GPU combine, closed-loop plant step, noise
// materialisation, RMPPI candidate scoring) for the user's functors inside the
// user's own shared object; the library calls them through the table. Build:
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false \
//        -Xcompiler -fPIC -shared -I include -I paper_2409_07563_b200/csrc my_model.cu -o libmy_model.so
// (-fmad=false keeps the IEEE-op semantics the reference's CPU build has.)
#pragma once

#include "smpc_b200.h"
#include "kernels.cuh"

template <class Dyn, class Cost>
struct smpc_plugin_model {
  struct Pair {
    Dyn dyn;
    Cost cost;
  } pair;
  static_assert(std::is_trivially_copyable<Pair>::value, "plugin functors must be trivially copyable");

  static const Pair& of(const void* u) { return *static_cast<const Pair*>(u); }
  static const smpc_dev::IterArgs& args(const void* a) { return *static_cast<const smpc_dev::IterArgs*>(a); }
  static int32_t rollout(const void* a, const void* u, void* st) {
    return (int32_t)smpc_dev::launch_rollout_t(args(a), of(u).dyn, of(u).cost, (cudaStream_t)st);
  }
  static int32_t update(const void* a, const void* u, void* st) {
    return (int32_t)smpc_dev::launch_update_t(args(a), of(u).dyn, (cudaStream_t)st);
  }
  static int32_t combine(const void* a, const void* u, void* st) {
    return (int32_t)smpc_dev::launch_combine_t(args(a), of(u).dyn, (cudaStream_t)st);
  }
  static int32_t generate(const void* a, const void*, float* e, uint8_t* f, void* st) {
    return (int32_t)smpc_dev::launch_generate_t<Dyn::NU>(args(a), e, f, (cudaStream_t)st);
  }
  static int32_t plant_step(const void* a, const void* u, const void* p, void* st) {
    return (int32_t)smpc_dev::launch_plant_step_t(args(a), of(u).dyn, of(u).cost,
                                                  *static_cast<const smpc_dev::PlantStepArgs*>(p), (cudaStream_t)st);
  }
  static int32_t rmppi_select(const void* a, const void* u, void* st) {
    if constexpr (smpc_dev::is_warp_coop<Dyn>::value)
      return (int32_t)smpc_dev::launch_rmppi_select_coop_t(args(a), of(u).dyn, of(u).cost, (cudaStream_t)st);
    else
      return (int32_t)smpc_dev::launch_rmppi_select_t(args(a), of(u).dyn, of(u).cost, (cudaStream_t)st);
  }

  // The table for smpc_create_with_ops; this object must outlive that call
  // (the library copies the functor pair).
  smpc_model_ops ops(const char* name) const {
    smpc_model_ops o{};
    o.abi_version = SMPC_B200_ABI_VERSION;
    o.args_bytes = (int32_t)sizeof(smpc_dev::IterArgs);
    o.n_x = Dyn::NX;
    o.n_u = Dyn::NU;
    o.n_y = Dyn::NY;
    o.name = name;
    o.user = &pair;
    o.user_bytes = (int64_t)sizeof(pair);
    o.rollout = &rollout;
    o.update = &update;
    o.combine = &combine;
    o.generate = &generate;
    o.plant_step = &plant_step;
    o.rmppi_select = &rmppi_select;
    return o;
  }
};

template <class Dyn, class Cost>
smpc_plugin_model<Dyn, Cost> smpc_ops_for(const Dyn& dyn, const Cost& cost) {
  return smpc_plugin_model<Dyn, Cost>{{dyn, cost}};
}
