// Kernel instantiations: CartpoleModel (dynamics.cpp:133-156), both glibc
// sinf/cosf ifunc variants.
#include "inst_common.cuh"

namespace smpc_dev {
SMPC_DEFINE_OPS(cp_fma, CartpoleDyn<true>, return CartpoleDyn<true>{p.p[0], p.p[1], p.p[2], p.p[3]};)
SMPC_DEFINE_OPS(cp_gen, CartpoleDyn<false>, return CartpoleDyn<false>{p.p[0], p.p[1], p.p[2], p.p[3]};)
ModelOps ops_cartpole(bool fma_libm) { return fma_libm ? cp_fma_ops() : cp_gen_ops(); }
}  // namespace smpc_dev
