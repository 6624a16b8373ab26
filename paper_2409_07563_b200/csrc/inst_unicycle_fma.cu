// Kernel instantiations: UnicycleModel (dynamics.cpp:122-131), glibc sinf/cosf FMA ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(uni_fma, UnicycleDyn<true>, (void)p; return UnicycleDyn<true>{};)
ModelOps uni_fma_ops_ext() { return uni_fma_ops(); }
}  // namespace smpc_dev
