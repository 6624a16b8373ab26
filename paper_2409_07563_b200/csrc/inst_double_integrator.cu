// Kernel instantiations: DoubleIntegrator2DModel (dynamics.cpp:173-181).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(di, DoubleIntegratorDyn, (void)p; return DoubleIntegratorDyn{};)
ModelOps ops_double_integrator() { return di_ops(); }
}  // namespace smpc_dev
