// Kernel instantiations: CartpoleModel (dynamics.cpp:133-156), glibc sinf/cosf generic ifunc
// variant (one variant per translation unit so the two compile in parallel).
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(cp_gen, CartpoleDyn<false>, return CartpoleDyn<false>{p.p[0], p.p[1], p.p[2], p.p[3], exact_inverse_pow2f(p.p[2])};)
ModelOps cp_fma_ops_ext();
ModelOps ops_cartpole(bool fma_libm) { return fma_libm ? cp_fma_ops_ext() : cp_gen_ops(); }
}  // namespace smpc_dev
