// Kernel instantiations: the builder-defined kinematic bicycle (models.cuh), glibc sinf/cosf generic ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(bc_gen, BicycleDyn<false>, BicycleDyn<false> b; b.wheelbase = p.p[0]; b.inv_wheelbase = exact_inverse_pow2f(p.p[0]); b.lo[0] = p.p[1], b.hi[0] = p.p[2]; b.lo[1] = p.p[3], b.hi[1] = p.p[4]; return b;)
ModelOps bc_fma_ops_ext();
ModelOps ops_bicycle(bool fma_libm) { return fma_libm ? bc_fma_ops_ext() : bc_gen_ops(); }
}  // namespace smpc_dev
