// Host-side probe: which glibc sinf/cosf ifunc variant (FMA or generic) does
// this process dispatch to? The reference's dynamics call the host libm, so
// the device ports (glibc_math.cuh) must follow the same variant. The probe
// inputs are the first bit patterns where the two variants differ (found by
// tests/native/check_glibc_math.cpp over all 2^32 floats).
// Compiled by g++ with -ffp-contract=off -fno-builtin (no constant folding of
// sinf through MPFR, no contraction in the generic port).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "glibc_math.cuh"

extern "C" int32_t smpc_host_libm_uses_fma(void) {
  static const uint32_t kProbes[] = {0x42a35c07u, 0x418a3addu, 0x41bc76d9u, 0x4255b0a9u, 0x42687a55u};
  int fma_votes = 0, gen_votes = 0;
  for (uint32_t bits : kProbes) {
    float x;
    memcpy(&x, &bits, 4);
    volatile float vx = x;
    const float hs = sinf(vx), hc = cosf(vx);
    if (hs == smpc_glibc::sinf_glibc<true>(x) && hc == smpc_glibc::cosf_glibc<true>(x)) ++fma_votes;
    if (hs == smpc_glibc::sinf_glibc<false>(x) && hc == smpc_glibc::cosf_glibc<false>(x)) ++gen_votes;
  }
  return fma_votes >= gen_votes ? 1 : 0;
}
