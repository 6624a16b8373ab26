// Kernel instantiations: DiffDriveModel (dynamics.cpp:158-171), glibc sinf/cosf FMA ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(dd_fma, DiffDriveDyn<true>, return DiffDriveDyn<true>{{p.p[2], p.p[4]}, {p.p[3], p.p[5]}};)
ModelOps dd_fma_ops_ext() { return dd_fma_ops(); }
}  // namespace smpc_dev
