// Kernel instantiations: DiffDriveModel (dynamics.cpp:158-171), glibc sinf/cosf generic ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(dd_gen, DiffDriveDyn<false>, return DiffDriveDyn<false>{{p.p[2], p.p[4]}, {p.p[3], p.p[5]}};)
ModelOps dd_fma_ops_ext();
ModelOps ops_diff_drive(bool fma_libm) { return fma_libm ? dd_fma_ops_ext() : dd_gen_ops(); }
}  // namespace smpc_dev
