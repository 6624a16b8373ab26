// An OUT-OF-TREE user model + cost compiled against the public plugin header
// (include/smpc_b200_plugin.cuh) into its own shared object — nothing in the
// library is edited or rebuilt (the reference's DynamicsModel / CostFunction
// subclassing, dynamics.hpp:17-74, costs.hpp:16-37). Test infrastructure
// (tests/test_plugin.py, tests/test_gpu_plugin.py).
//
//   user_di_ops:     a double integrator + quadratic cost written here from
//                    the reference's equations (dynamics.cpp:173-181,
//                    costs.cpp:86-109): must reproduce the built-in pair bit
//                    for bit.
//   spring_ops:      a new model (damped spring-mass, 2 states, 1 control)
//                    with a control-dependent cost: checked against a numpy
//                    float32/float64 restatement.
#include "smpc_b200_plugin.cuh"

namespace user {

struct UserDoubleIntegrator {
  static constexpr int NX = 4, NU = 2, NY = 4, ANGULAR = -1;
  static constexpr bool BOUNDED = false;
  static constexpr bool POST_STEP = false;
  __device__ __forceinline__ void state_derivative(const float* x, const float* u, float* dx) const {
    dx[0] = x[2];
    dx[1] = x[3];
    dx[2] = u[0];
    dx[3] = u[1];
  }
  __device__ __forceinline__ void clamp_control(const float*, float*) const {}
};

struct UserQuadratic {
  static constexpr bool USES_MAP = false;
  static constexpr bool USES_CONTROL = false;
  double target[4], weight[4];
  __device__ __forceinline__ double running_cost(const float* y, const float*, int) const {
    double c = 0.0;
    for (int i = 0; i < 4; ++i) {
      const double d = __dsub_rn((double)y[i], target[i]);
      c = __dadd_rn(c, __dmul_rn(__dmul_rn(weight[i], d), d));
    }
    return c;
  }
  __device__ __forceinline__ double terminal_cost(const float* y) const { return running_cost(y, nullptr, 0); }
};

// p' = v, v' = (f - k p - c v) / m  with m = 2 (so / m is an exact * 0.5)
struct SpringMass {
  static constexpr int NX = 2, NU = 1, NY = 2, ANGULAR = -1;
  static constexpr bool BOUNDED = true;
  static constexpr bool POST_STEP = false;
  float k, c, f_max;
  __device__ __forceinline__ void clamp_control(const float* u, float* out) const {
    const float a = u[0] < -f_max ? -f_max : u[0];
    out[0] = f_max < a ? f_max : a;
  }
  __device__ __forceinline__ void state_derivative(const float* x, const float* u, float* dx) const {
    dx[0] = x[1];
    dx[1] = __fmul_rn(__fsub_rn(__fsub_rn(u[0], __fmul_rn(k, x[0])), __fmul_rn(c, x[1])), 0.5f);
  }
};

// (p - 1)^2 + 0.1 v^2 + 0.01 u^2 (u: the clamped sampled control, engine.cpp:40-48), terminal 10 (p - 1)^2
struct SpringCost {
  static constexpr bool USES_MAP = false;
  static constexpr bool USES_CONTROL = true;
  __device__ __forceinline__ double running_cost(const float* y, const float* u, int) const {
    const double dp = __dsub_rn((double)y[0], 1.0);
    const double v = (double)y[1], f = (double)u[0];
    return __dadd_rn(__dadd_rn(__dmul_rn(dp, dp), __dmul_rn(0.1, __dmul_rn(v, v))), __dmul_rn(0.01, __dmul_rn(f, f)));
  }
  __device__ __forceinline__ double terminal_cost(const float* y) const {
    const double dp = __dsub_rn((double)y[0], 1.0);
    return __dmul_rn(10.0, __dmul_rn(dp, dp));
  }
};

smpc_plugin_model<UserDoubleIntegrator, UserQuadratic> g_di;
smpc_plugin_model<SpringMass, SpringCost> g_spring;

}  // namespace user

extern "C" smpc_model_ops user_di_ops(const double* target, const double* weight) {
  user::UserQuadratic q;
  for (int i = 0; i < 4; ++i) q.target[i] = target[i], q.weight[i] = weight[i];
  user::g_di = smpc_ops_for(user::UserDoubleIntegrator{}, q);
  return user::g_di.ops("user_double_integrator");
}

extern "C" smpc_model_ops spring_ops(float k, float c, float f_max) {
  user::g_spring = smpc_ops_for(user::SpringMass{k, c, f_max}, user::SpringCost{});
  return user::g_spring.ops("spring_mass");
}
