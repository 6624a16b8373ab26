// Kernel instantiations: UnicycleModel (dynamics.cpp:122-131).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(uni_fma, UnicycleDyn<true>, (void)p; return UnicycleDyn<true>{};)
SMPC_DEFINE_OPS(uni_gen, UnicycleDyn<false>, (void)p; return UnicycleDyn<false>{};)
ModelOps ops_unicycle(bool fma_libm) { return fma_libm ? uni_fma_ops() : uni_gen_ops(); }
}  // namespace smpc_dev
