// Kernel instantiations: the builder-defined kinematic bicycle (models.cuh),
// both glibc sinf/cosf ifunc variants.
#include "inst_common.cuh"

namespace smpc_dev {
#define SMPC_BICYCLE_MAKE(F)                                  \
  BicycleDyn<F> b;                                            \
  b.wheelbase = p.p[0];                                       \
  b.lo[0] = p.p[1], b.hi[0] = p.p[2];                         \
  b.lo[1] = p.p[3], b.hi[1] = p.p[4];                         \
  return b;
SMPC_DEFINE_OPS(bc_fma, BicycleDyn<true>, SMPC_BICYCLE_MAKE(true))
SMPC_DEFINE_OPS(bc_gen, BicycleDyn<false>, SMPC_BICYCLE_MAKE(false))
ModelOps ops_bicycle(bool fma_libm) { return fma_libm ? bc_fma_ops() : bc_gen_ops(); }
}  // namespace smpc_dev
