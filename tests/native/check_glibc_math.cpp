// Exhaustive CPU check: the glibc 2.39 ports in glibc_math.cuh (host build,
// -ffp-contract=off) against this host's libm logf/sinf/cosf, over a strided
// subset or all 2^32 float bit patterns. Test infrastructure only.
// Usage: check_glibc_math <stride> <threads> <fma:0|1>
// <fma> selects the port variant; run with GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA
// to compare the generic variant against the generic libm dispatch.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>

#include "../../paper_2409_07563_b200/csrc/glibc_math.cuh"

static inline bool same(float a, float b) {
  if (std::isnan(a) && std::isnan(b)) return true;
  uint32_t ua, ub;
  std::memcpy(&ua, &a, 4);
  std::memcpy(&ub, &b, 4);
  return ua == ub;
}

int main(int argc, char** argv) {
  const uint64_t stride = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1;
  const int threads = argc > 2 ? std::atoi(argv[2]) : (int)std::thread::hardware_concurrency();
  const bool fma_variant = argc > 3 ? std::atoi(argv[3]) != 0 : true;
  std::atomic<uint64_t> bad_log{0}, bad_sin{0}, bad_cos{0}, bad_fast{0}, checked{0};
  // fingerprint of the HOST libm over the visited inputs ([fn][top byte of x]),
  // the value the device-side exhaustive check (smpc_libm_hash) must reproduce
  std::vector<std::atomic<uint64_t>> hash(3 * 256);
  for (auto& h : hash) h = 0;
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    pool.emplace_back([&, w] {
      uint64_t bl = 0, bs = 0, bc = 0, bf = 0, n = 0;
      std::vector<uint64_t> hl(3 * 256, 0);
      for (uint64_t i = (uint64_t)w * stride; i < (1ULL << 32); i += stride * threads) {
        uint32_t u = (uint32_t)i;
        float x;
        std::memcpy(&x, &u, 4);
        const float lg = logf(x), sn = sinf(x), cs = cosf(x);
        hl[0 * 256 + (u >> 24)] += smpc_glibc::libm_hash_term(u, lg);
        hl[1 * 256 + (u >> 24)] += smpc_glibc::libm_hash_term(u, sn);
        hl[2 * 256 + (u >> 24)] += smpc_glibc::libm_hash_term(u, cs);
        if (!same(smpc_glibc::logf_glibc(x), lg)) {
          if (bl < 3) std::fprintf(stderr, "logf mismatch %08x\n", u);
          ++bl;
        }
        if (!same((fma_variant ? smpc_glibc::sinf_glibc<true>(x) : smpc_glibc::sinf_glibc<false>(x)), sn)) {
          if (bs < 3) std::fprintf(stderr, "sinf mismatch %08x\n", u);
          ++bs;
        }
        if (!same((fma_variant ? smpc_glibc::cosf_glibc<true>(x) : smpc_glibc::cosf_glibc<false>(x)), cs)) {
          if (bc < 3) std::fprintf(stderr, "cosf mismatch %08x\n", u);
          ++bc;
        }
        {  // the branch-free rollout variant: equal to the port for |x| < 120, NaN beyond
          float s0, c0, s1, c1;
          if (fma_variant) {
            smpc_glibc::sincosf_glibc<true>(x, &s0, &c0);
            smpc_glibc::sincosf_glibc_fast<true>(x, &s1, &c1);
          } else {
            smpc_glibc::sincosf_glibc<false>(x, &s0, &c0);
            smpc_glibc::sincosf_glibc_fast<false>(x, &s1, &c1);
          }
          const bool ok = std::fabs(x) < 120.0f ? (same(s0, s1) && same(c0, c1)) : (std::isnan(s1) && std::isnan(c1));
          if (!ok) {
            if (bf < 3) std::fprintf(stderr, "sincosf_fast mismatch %08x\n", u);
            ++bf;
          }
        }
        ++n;
      }
      for (int k = 0; k < 3 * 256; ++k) hash[k] += hl[k];
      bad_log += bl;
      bad_fast += bf;
      bad_sin += bs;
      bad_cos += bc;
      checked += n;
    });
  }
  for (auto& t : pool) t.join();
  if (const char* hp = std::getenv("SMPC_LIBM_HASH_OUT")) {
    if (FILE* f = std::fopen(hp, "w")) {
      for (int k = 0; k < 3 * 256; ++k) std::fprintf(f, "%llu\n", (unsigned long long)hash[k].load());
      std::fclose(f);
    }
  }
  std::printf("{\"checked\": %llu, \"logf_mismatch\": %llu, \"sinf_mismatch\": %llu, \"cosf_mismatch\": %llu, "
              "\"sincosf_fast_mismatch\": %llu}\n",
              (unsigned long long)checked.load(), (unsigned long long)bad_log.load(),
              (unsigned long long)bad_sin.load(), (unsigned long long)bad_cos.load(),
              (unsigned long long)bad_fast.load());
  return (bad_log | bad_sin | bad_cos | bad_fast) ? 1 : 0;
}
