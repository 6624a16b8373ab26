// Kernel instantiations: UnicycleModel (dynamics.cpp:122-131), glibc sinf/cosf generic ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(uni_gen, UnicycleDyn<false>, (void)p; return UnicycleDyn<false>{};)
ModelOps uni_fma_ops_ext();
ModelOps ops_unicycle(bool fma_libm) { return fma_libm ? uni_fma_ops_ext() : uni_gen_ops(); }
}  // namespace smpc_dev
