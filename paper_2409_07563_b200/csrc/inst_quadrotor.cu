// Kernel instantiations: the builder-defined 13-state quadrotor (models.cuh).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(quad, QuadrotorDyn, {
  // p = {mass, gravity, tau, thrust_max, rate_max}; derived in float exactly
  // as oracle/smpc_oracle.c:quadrotor_params does
  QuadrotorDyn q;
  const float mass = p.p[0], g = p.p[1], tau = p.p[2], tmax = p.p[3], rmax = p.p[4];
  volatile float one = 1.0f;
  q.inv_mass = one / mass;
  q.inv_tau = one / tau;
  q.gravity = g;
  q.hover = mass * g;
  for (int i = 0; i < 3; ++i) q.lo[i] = -rmax, q.hi[i] = rmax;
  q.lo[3] = -q.hover;
  q.hi[3] = tmax - q.hover;
  return q;
})
ModelOps ops_quadrotor() { return quad_ops(); }
}  // namespace smpc_dev
