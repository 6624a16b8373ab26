// Kernel instantiations: CartpoleModel (dynamics.cpp:133-156), glibc sinf/cosf FMA ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(cp_fma, CartpoleDyn<true>, return CartpoleDyn<true>{p.p[0], p.p[1], p.p[2], p.p[3], exact_inverse_pow2f(p.p[2])};)
ModelOps cp_fma_ops_ext() { return cp_fma_ops(); }
}  // namespace smpc_dev
