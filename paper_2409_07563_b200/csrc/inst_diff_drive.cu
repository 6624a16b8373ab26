// Kernel instantiations: DiffDriveModel (dynamics.cpp:158-171), control
// bounds {v_min, w_min} / {v_max, w_max} from params [2..5].
#include "inst_common.cuh"

namespace smpc_dev {
#define SMPC_DD(F) return DiffDriveDyn<F>{{p.p[2], p.p[4]}, {p.p[3], p.p[5]}};
SMPC_DEFINE_OPS(dd_fma, DiffDriveDyn<true>, SMPC_DD(true))
SMPC_DEFINE_OPS(dd_gen, DiffDriveDyn<false>, SMPC_DD(false))
ModelOps ops_diff_drive(bool fma_libm) { return fma_libm ? dd_fma_ops() : dd_gen_ops(); }
}  // namespace smpc_dev
