// Bit-exact device ports of the glibc 2.39 single-precision transcendentals
// that sit on the MPPI hot path of the reference:
//   * logf  — normal_icdf tail branch        (proj/core/include/smpc/rng.hpp:80)
//   * sinf / cosf — unicycle / cartpole / diff-drive state_derivative
//                                            (proj/core/src/dynamics.cpp:128-129,
//                                             :144-145, :168-169)
// The reference calls the host's glibc libm (un-vendored, glibc 2.39 in this
// image). CUDA's logf/sinf/cosf differ from glibc by 1-2 ulp on ~1% of inputs,
// which would make sampled trajectories differ from the reference after the
// first step. These ports restate glibc's algorithms (ARM optimized-routines
// logf / sinf / cosf: double-precision evaluation, one final rounding to
// float) with the constant tables read out of this image's libm.so.6
// (__logf_data @ +0xb7d40, __sincosf_table @ +0xb8120, __inv_pio4 @ +0xb80c0),
// so every double operation is the same IEEE operation the host performs.
//
// Device arithmetic uses explicit _rn intrinsics (no FMA contraction whatever
// -fmad says); the host build (used only by the exhaustive CPU check) must be
// compiled with -ffp-contract=off. Exhaustive equality against the host libm
// over all 2^32 float inputs: tests/test_glibc_math.py.
//
// Third-party notice. The algorithms and constant tables restated here come
// from glibc 2.39 (sysdeps/ieee754/flt-32: e_logf.c, s_sinf.c, s_cosf.c,
// sincosf.h, e_logf_data.c, s_sincosf_data.c), which takes them from ARM's
// optimized-routines. glibc is licensed LGPL-2.1-or-later; optimized-routines
// is MIT OR Apache-2.0 WITH LLVM-exception. This file is a restatement of
// those routines and carries their licences; see THIRD_PARTY_NOTICES.md.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define GM_HD __host__ __device__ __forceinline__
#else
#define GM_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define GM_DMUL(a, b) __dmul_rn((a), (b))
#define GM_DADD(a, b) __dadd_rn((a), (b))
#define GM_DSUB(a, b) __dsub_rn((a), (b))
#define GM_DFMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define GM_DMUL(a, b) ((a) * (b))
#define GM_DADD(a, b) ((a) + (b))
#define GM_DSUB(a, b) ((a) - (b))
#define GM_DFMA(a, b, c) fma((a), (b), (c))
#endif

namespace smpc_glibc {

struct LogfEntry {
  double invc, logc;
};

struct SincosfTable {
  double sign[4];
  double hpi_inv;  // 2/pi * 2^24 (x86-64 build: no TOINT_INTRINSICS)
  double hpi;
  double c0, c1, s1, c2, s2, c3, s3, c4;
};

#define SMPC_LOGF_ROWS                                                                          \
  {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2}, \
      {0x1.49539f0f010bp+0, -0x1.01eae7f513a67p-2},                                             \
      {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},                                            \
      {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3},                                            \
      {0x1.25e227b0b8eap+0, -0x1.1aa2bc79c81p-3},                                               \
      {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4},                                            \
      {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},                                            \
      {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1p+0, 0x0p+0},                          \
      {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5}, {0x1.ca4b31f026aap-1, 0x1.c5e53aa362eb4p-4}, \
      {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3}, {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d22477p-3}, \
      {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2}, {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2}

#define SMPC_SINCOSF_ROWS                                                                       \
  {{1.0, -1.0, -1.0, 1.0}, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, 0x1p+0,                  \
   -0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, 0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7,     \
   -0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, 0x1.99343027bf8c3p-16},                       \
      {{1.0, -1.0, -1.0, 1.0}, 0x1.45f306dc9c883p+23, 0x1.921fb54442d18p+0, -0x1p+0,             \
       0x1.ffffffd0c621cp-2, -0x1.555545995a603p-3, -0x1.55553e1068f19p-5, 0x1.1107605230bc4p-7, \
       0x1.6c087e89a359dp-10, -0x1.994eb3774cf24p-13, -0x1.99343027bf8c3p-16}

#define SMPC_INV_PIO4_ROWS                                                          \
  0xa2u, 0xa2f9u, 0xa2f983u, 0xa2f9836eu, 0xf9836e4eu, 0x836e4e44u, 0x6e4e4415u,    \
      0x4e441529u, 0x441529fcu, 0x1529fc27u, 0x29fc2757u, 0xfc2757d1u, 0x2757d1f5u, \
      0x57d1f534u, 0xd1f534ddu, 0xf534ddc0u, 0x34ddc0dbu, 0xddc0db62u, 0xc0db6295u, \
      0xdb629599u, 0x6295993cu, 0x95993c43u, 0x993c4390u, 0x3c439041u

// Namespace-scope tables: a __constant__-bank copy for device code and a plain
// const copy for host code (the same literals).
#if defined(__CUDACC__)
static __constant__ LogfEntry kLogfTabDev[16] = {SMPC_LOGF_ROWS};
static __constant__ SincosfTable kSincosfTabDev[2] = {SMPC_SINCOSF_ROWS};
static __constant__ uint32_t kInvPio4Dev[24] = {SMPC_INV_PIO4_ROWS};
#endif
static const LogfEntry kLogfTabHost[16] = {SMPC_LOGF_ROWS};
static const SincosfTable kSincosfTabHost[2] = {SMPC_SINCOSF_ROWS};
static const uint32_t kInvPio4Host[24] = {SMPC_INV_PIO4_ROWS};

#if defined(__CUDA_ARCH__)
#define GM_LOGF_TAB kLogfTabDev
#define GM_SINCOSF_TAB kSincosfTabDev
#define GM_INV_PIO4 kInvPio4Dev
GM_HD uint32_t f2u(float x) { return __float_as_uint(x); }
GM_HD float u2f(uint32_t x) { return __uint_as_float(x); }
#else
#define GM_LOGF_TAB kLogfTabHost
#define GM_SINCOSF_TAB kSincosfTabHost
#define GM_INV_PIO4 kInvPio4Host
GM_HD uint32_t f2u(float x) {
  union {
    float f;
    uint32_t u;
  } v;
  v.f = x;
  return v.u;
}
GM_HD float u2f(uint32_t x) {
  union {
    float f;
    uint32_t u;
  } v;
  v.u = x;
  return v.f;
}
#endif

// ---------------------------------------------------------------------------
// logf: glibc 2.39 sysdeps/ieee754/flt-32/e_logf.c
// ---------------------------------------------------------------------------
GM_HD float logf_glibc(float x) {
  const double kLn2 = 0x1.62e42fefa39efp-1;
  const double A0 = -0x1.00ea348b88334p-2, A1 = 0x1.5575b0be00b6ap-2, A2 = -0x1.ffffef20a4123p-2;
  uint32_t ix = f2u(x);
  if (ix == 0x3f800000u) return 0.0f;
  if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
    if (ix * 2 == 0) return -u2f(0x7f800000u);  // -inf (divide by zero)
    if (ix == 0x7f800000u) return x;             // log(inf) = inf
    if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return u2f(0x7fc00000u);  // NaN
    ix = f2u(x * 0x1p23f);  // subnormal: exact scaling
    ix -= 23u << 23;
  }
  const uint32_t tmp = ix - 0x3f330000u;
  const int i = (int)((tmp >> (23 - 4)) % 16u);
  const int k = (int32_t)tmp >> 23;
  const uint32_t iz = ix - (tmp & 0xff800000u);
  const double invc = GM_LOGF_TAB[i].invc;
  const double logc = GM_LOGF_TAB[i].logc;
  const double z = (double)u2f(iz);
  const double r = GM_DSUB(GM_DMUL(z, invc), 1.0);
  const double y0 = GM_DADD(logc, GM_DMUL((double)k, kLn2));
  const double r2 = GM_DMUL(r, r);
  double y = GM_DADD(GM_DMUL(A1, r), A2);
  y = GM_DADD(GM_DMUL(A0, r2), y);
  y = GM_DADD(GM_DMUL(y, r2), GM_DADD(y0, r));
  return (float)y;
}

// ---------------------------------------------------------------------------
// sinf / cosf: glibc 2.39 sysdeps/ieee754/flt-32/s_sinf.c, s_cosf.c, sincosf.h
// ---------------------------------------------------------------------------
GM_HD uint32_t abstop12(float x) { return (f2u(x) >> 20) & 0x7ffu; }

// glibc builds two ifunc variants of sinf/cosf: generic C (no contraction) and
// an -mfma -mavx2 build in which GCC contracts every `a + b*c` below into one
// fused multiply-add. They differ on 34 of 2^32 inputs (all with 17 < |x| < 120,
// where reduce_fast cancels), so the port is templated on the variant and the
// engine selects the one the host libm dispatches to (smpc_host_libm_uses_fma).
#define GM_MADD(FMA, a, b, c) ((FMA) ? GM_DFMA((b), (c), (a)) : GM_DADD((a), GM_DMUL((b), (c))))

template <bool FMA>
GM_HD float sinf_poly(double x, double x2, const SincosfTable* p, int n) {
  if ((n & 1) == 0) {
    const double x3 = GM_DMUL(x, x2);
    const double s1 = GM_MADD(FMA, p->s2, x2, p->s3);
    const double x7 = GM_DMUL(x3, x2);
    const double s = GM_MADD(FMA, x, x3, p->s1);
    return (float)GM_MADD(FMA, s, x7, s1);
  }
  const double x4 = GM_DMUL(x2, x2);
  const double c2 = GM_MADD(FMA, p->c3, x2, p->c4);
  const double c1 = GM_MADD(FMA, p->c0, x2, p->c1);
  const double x6 = GM_DMUL(x4, x2);
  const double c = GM_MADD(FMA, c1, x4, p->c2);
  return (float)GM_MADD(FMA, c, x6, c2);
}

// |x| < 120: single multiply-subtract reduction with the 2^24-prescaled 2/pi.
template <bool FMA>
GM_HD double reduce_fast(double x, const SincosfTable* p, int* np) {
  const double r = GM_DMUL(x, p->hpi_inv);
  const int n = ((int32_t)r + 0x800000) >> 24;
  *np = n;
  return FMA ? GM_DFMA(-(double)n, p->hpi, x) : GM_DSUB(x, GM_DMUL((double)n, p->hpi));
}

// |x| >= 120: reduction against 4/pi bits.
GM_HD double reduce_large(uint32_t xi, int* np) {
  const uint32_t* arr = &GM_INV_PIO4[(xi >> 26) & 15];
  const int shift = (xi >> 23) & 7;
  xi = (xi & 0xffffffu) | 0x800000u;
  xi <<= shift;
  uint64_t res0 = (uint64_t)(uint32_t)(xi * arr[0]);
  const uint64_t res1 = (uint64_t)xi * arr[4];
  const uint64_t res2 = (uint64_t)xi * arr[8];
  res0 = (res2 >> 32) | (res0 << 32);
  res0 += res1;
  const uint64_t n = (res0 + (1ULL << 61)) >> 62;
  res0 -= n << 62;
  const double x = (double)(int64_t)res0;
  *np = (int)n;
  return GM_DMUL(x, 0x1.921fb54442d18p-62);
}

template <bool FMA>
GM_HD float sinf_glibc(float y) {
  double x = y;
  const SincosfTable* p = &GM_SINCOSF_TAB[0];
  int n;
  if (abstop12(y) < abstop12(0x1.921fb6p-1f)) {
    const double s = GM_DMUL(x, x);
    if (abstop12(y) < abstop12(0x1p-12f)) return y;
    return sinf_poly<FMA>(x, s, p, 0);
  } else if (abstop12(y) < abstop12(120.0f)) {
    x = reduce_fast<FMA>(x, p, &n);
    const double s = p->sign[n & 3];
    if (n & 2) p = &GM_SINCOSF_TAB[1];
    return sinf_poly<FMA>(GM_DMUL(x, s), GM_DMUL(x, x), p, n);
  } else if (abstop12(y) < 0x7f8u) {
    const uint32_t xi = f2u(y);
    const int sign = xi >> 31;
    x = reduce_large(xi, &n);
    const double s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &GM_SINCOSF_TAB[1];
    return sinf_poly<FMA>(GM_DMUL(x, s), GM_DMUL(x, x), p, n);
  }
  return u2f(0x7fc00000u);  // inf or NaN -> NaN
}

template <bool FMA>
GM_HD float cosf_glibc(float y) {
  double x = y;
  const SincosfTable* p = &GM_SINCOSF_TAB[0];
  int n;
  if (abstop12(y) < abstop12(0x1.921fb6p-1f)) {
    const double x2 = GM_DMUL(x, x);
    if (abstop12(y) < abstop12(0x1p-12f)) return 1.0f;
    return sinf_poly<FMA>(x, x2, p, 1);
  } else if (abstop12(y) < abstop12(120.0f)) {
    x = reduce_fast<FMA>(x, p, &n);
    const double s = p->sign[n & 3];
    if (n & 2) p = &GM_SINCOSF_TAB[1];
    return sinf_poly<FMA>(GM_DMUL(x, s), GM_DMUL(x, x), p, n ^ 1);
  } else if (abstop12(y) < 0x7f8u) {
    const uint32_t xi = f2u(y);
    const int sign = xi >> 31;
    x = reduce_large(xi, &n);
    const double s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &GM_SINCOSF_TAB[1];
    return sinf_poly<FMA>(GM_DMUL(x, s), GM_DMUL(x, x), p, n ^ 1);
  }
  return u2f(0x7fc00000u);
}

// sinf and cosf of the same argument with ONE range reduction (the
// state_derivatives call both, dynamics.cpp:128-129, :144-145, :168-169).
// Same branches, same reduction, then the two polynomial evaluations of
// sinf_glibc / cosf_glibc: equal to the separate ports by construction and
// checked exhaustively (smpc_libm_hash rows 3-4 against the host libm).
template <bool FMA>
GM_HD void sincosf_glibc(float y, float* sp, float* cp) {
  double x = y;
  const SincosfTable* p = &GM_SINCOSF_TAB[0];
  int n;
  if (abstop12(y) < abstop12(0x1.921fb6p-1f)) {
    const double x2 = GM_DMUL(x, x);
    if (abstop12(y) < abstop12(0x1p-12f)) {
      *sp = y;
      *cp = 1.0f;
      return;
    }
    *sp = sinf_poly<FMA>(x, x2, p, 0);
    *cp = sinf_poly<FMA>(x, x2, p, 1);
    return;
  }
  if (abstop12(y) < abstop12(120.0f)) {
    x = reduce_fast<FMA>(x, p, &n);
    const double s = p->sign[n & 3];
    if (n & 2) p = &GM_SINCOSF_TAB[1];
    const double xs = GM_DMUL(x, s), xx = GM_DMUL(x, x);
    *sp = sinf_poly<FMA>(xs, xx, p, n);
    *cp = sinf_poly<FMA>(xs, xx, p, n ^ 1);
    return;
  }
  if (abstop12(y) < 0x7f8u) {
    const uint32_t xi = f2u(y);
    const int sign = xi >> 31;
    x = reduce_large(xi, &n);
    const double s = p->sign[(n + sign) & 3];
    if ((n + sign) & 2) p = &GM_SINCOSF_TAB[1];
    const double xs = GM_DMUL(x, s), xx = GM_DMUL(x, x);
    *sp = sinf_poly<FMA>(xs, xx, p, n);
    *cp = sinf_poly<FMA>(xs, xx, p, n ^ 1);
    return;
  }
  *sp = *cp = u2f(0x7fc00000u);
}

// sincosf_glibc without a branch for |x| < 120 (the rollout's unchecked
// loop): the |x| < pi/4 path is the reduce_fast path with n = 0 (x - 0*hpi ==
// x, sign[0] == 1, table 0: the same operations), the |x| < 2^-12 early
// returns are selects, and |x| >= 120, inf and NaN give NaN (the sample is
// then replayed with the exact sincosf_glibc). No constant-bank table reads:
// __sincosf_table[1] is table 0 with every cosine coefficient negated and the
// same sine coefficients, so its cosine polynomial is the exact negation of
// table 0's (round-to-nearest is symmetric; the cosine polynomial is >= 0.7,
// never an exact zero), and sign[n & 3] = {1,-1,-1,1} is a conditional
// negation. Equal to sincosf_glibc on every |x| < 120 (exhaustive:
// smpc_fast_math_check).
template <bool FMA>
GM_HD void sincosf_glibc_fast(float y, float* sp, float* cp) {
  constexpr double hpi_inv = 0x1.45f306dc9c883p+23, hpi = 0x1.921fb54442d18p+0;
  constexpr double c0 = 0x1p+0, c1 = -0x1.ffffffd0c621cp-2, c2 = 0x1.55553e1068f19p-5, c3 = -0x1.6c087e89a359dp-10,
                   c4 = 0x1.99343027bf8c3p-16;
  constexpr double s1 = -0x1.555545995a603p-3, s2 = 0x1.1107605230bc4p-7, s3 = -0x1.994eb3774cf24p-13;
  const double xd = (double)y;
  const double r = GM_DMUL(xd, hpi_inv);
  const int n = ((int32_t)r + 0x800000) >> 24;
  const double x = FMA ? GM_DFMA(-(double)n, hpi, xd) : GM_DSUB(xd, GM_DMUL((double)n, hpi));
  const double xs = ((n + 1) & 2) ? -x : x;  // x * sign[n & 3]
  const double x2 = GM_DMUL(x, x);
  // sine polynomial (sinf_poly, n even): table-independent
  const double x3 = GM_DMUL(xs, x2);
  const double sa = GM_MADD(FMA, s2, x2, s3);
  const double x7 = GM_DMUL(x3, x2);
  const double sb = GM_MADD(FMA, xs, x3, s1);
  const float S = (float)GM_MADD(FMA, sb, x7, sa);
  // cosine polynomial (sinf_poly, n odd) with table 0, negated for table 1
  const double x4 = GM_DMUL(x2, x2);
  const double ca = GM_MADD(FMA, c3, x2, c4);
  const double cb = GM_MADD(FMA, c0, x2, c1);
  const double x6 = GM_DMUL(x4, x2);
  const double cc = GM_MADD(FMA, cb, x4, c2);
  const float C0 = (float)GM_MADD(FMA, cc, x6, ca);
  const float C = (n & 2) ? -C0 : C0;
  float sv = (n & 1) ? C : S;
  float cv = (n & 1) ? S : C;
  const uint32_t top = abstop12(y);
  const bool tiny = top < abstop12(0x1p-12f);
  sv = tiny ? y : sv;
  cv = tiny ? 1.0f : cv;
  const bool ok = top < abstop12(120.0f);
  *sp = ok ? sv : u2f(0x7fc00000u);
  *cp = ok ? cv : u2f(0x7fc00000u);
}

// Order-independent fingerprint of a function over all 2^32 float inputs
// (test infrastructure: the device result is compared with the same sum over
// the host libm, tests/golden/libm_hash.json). NaN outputs hash as the
// canonical quiet NaN; the sum is bucketed by the input's top 8 bits so a
// mismatch names a 2^24-wide input range.
GM_HD uint64_t libm_hash_term(uint32_t in, float out) {
  const uint32_t bits = out != out ? 0x7fc00000u : f2u(out);
  uint64_t z = (((uint64_t)in << 32) | bits) + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

}  // namespace smpc_glibc
