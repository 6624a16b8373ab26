// Neural-network (AutoRally-style MLP) dynamics rollout on the 5th-generation
// tensor cores (BASELINE.json configs[3]; builder-defined model, see
// models.cuh:MlpDyn — no reference counterpart, tolerance parity against the
// restated oracle oracle/smpc_oracle.c:mlp_derivative).
//
// One CTA = 128 samples of one system (one tcgen05 M=128 tile; grid.y =
// system, so Tube's nominal and real rollouts are separate CTAs that
// regenerate the same Philox draw — cheaper than doubling the per-thread
// state). Per timestep:
//
//   SIMT   u = clamp(mean + eps); h1 = tanh(W1 [roll,vx,vy,r,u] + b1)    (6x32)
//          h1 -> shared memory as TF32 hi/lo pairs in the UMMA K-major
//          no-swizzle core-matrix layout (row = sample)
//   tcgen05 D[s] (TMEM, 128 lanes x 32 fp32 columns) = H1 W2^T in 3xTF32:
//          hi*hi + hi*lo + lo*hi, 4 K-steps of 8 -> 12 MMAs per system,
//          issued by one thread, completion via tcgen05.commit -> mbarrier
//   SIMT   tcgen05.ld (32x32b.x32: thread = TMEM lane = sample row) ->
//          h2 = tanh(D + b2) -> (roll,vx,vy,r)' = W3 h2 + b3 (32x4) ->
//          kinematics -> explicit Euler -> wrap yaw -> running cost
//
// Layer 2 (32x32, 76% of the MACs) is the dense batched contraction the
// tensor cores take; layers 1 and 3 stay in registers (K = 6 and N = 4 are
// below a tcgen05 tile and need no round trip). The costs, argmin reduction,
// weights, update and nominal rollout are the shared MPPI kernels
// (kernels.cuh), so MPPI, DMD, CEM and Tube all run on this rollout.
#include <cuda_runtime.h>

#include "inst_common.cuh"

namespace smpc_dev {
namespace mlpk {

using namespace mlp_layout;

// Instruction descriptor, kind::tf32: D fp32 (bits 4-5 = 1), A/B TF32
// (bits 7-9 = 2, 10-12 = 2), both K-major, N = 32 (bits 17-22 = N>>3),
// M = 128 (bits 24-28 = M>>4).
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
constexpr int kTile = 128;                      // samples per CTA (= M)
constexpr int kHBytes = kTile * HID * 4;        // one TF32 operand tile [128 x 32]
constexpr int kWBytes = HID * HID * 4;          // W2 operand tile [32 x 32]
constexpr uint32_t kLBO = 128;                  // next 4-element K chunk
constexpr uint32_t kSBO = HID * 32;             // next 8-row group (K = 32: 8 chunks x 128 B)

// Byte offset of element (r, k) in a K-major SWIZZLE_NONE tile with HID columns:
// core matrices of 8 rows x 16 B, K chunks LBO apart, row groups SBO apart.
__device__ __forceinline__ uint32_t core_off(int r, int k) {
  return (uint32_t)((r >> 3) * kSBO + (k >> 2) * kLBO + (r & 7) * 16 + (k & 3) * 4);
}

// UMMA shared-memory matrix descriptor (sm_100): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout 0 =
// SWIZZLE_NONE [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(kLBO >> 4) << 16) | ((uint64_t)(kSBO >> 4) << 32) |
         (1ull << 46);
}

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---- packed f32x2 helpers (the MLP path has no bit-exactness contract, so
// FFMA2 contraction is used freely here) ----------------------------------
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) { return f2pack(lo, hi); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return f2fma(a, b, c); }
__device__ __forceinline__ float ex2f(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcpf(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// Two tanh at once: sign(x) (1 - 2 / (2^{2|x| log2 e} + 1)); abs error ~1e-7.
__device__ __forceinline__ f2 tanh2(f2 x) {
  float a, b;
  f2unpack(x, a, b);
  const f2 ax = pk(fabsf(a), fabsf(b));
  const f2 t = fma2(ax, f2splat_bits(0x4038AA3Bu) /* 2 log2 e */, 0ull);
  float t0, t1;
  f2unpack(t, t0, t1);
  const f2 den = fma2(pk(ex2f(t0), ex2f(t1)), f2splat_bits(0x3F800000u), f2splat_bits(0x3F800000u));  // e + 1
  float d0, d1;
  f2unpack(den, d0, d1);
  const f2 r = fma2(pk(rcpf(d0), rcpf(d1)), f2splat_bits(0xC0000000u) /* -2 */, f2splat_bits(0x3F800000u));
  float r0, r1;
  f2unpack(r, r0, r1);
  return pk(copysignf(r0, a), copysignf(r1, b));
}

// Two tanh on the FMA pipe only (no MUFU): the clamped odd rational
// x P(x^2) / Q(x^2) (degree 13 / 6, the minimax form Eigen uses for float
// tanh; abs error ~1e-7 on the clamp range, where tanh saturates to 1 in
// float), the division by Q in [4.9e-3, 1] as an integer-seeded reciprocal
// with three Newton steps. The layer-2 epilogue mixes it with tanh2 so the
// XU (ex2 + rcp) and FMA pipes share the 64 tanh per sample-step.
__device__ __forceinline__ f2 tanh2_fma(f2 x) {
#define SPL(c) f2splat_bits(__float_as_uint(c))
  float a, b;
  f2unpack(x, a, b);
  const float lim = 7.90531110763549805f;
  a = fminf(fmaxf(a, -lim), lim);
  b = fminf(fmaxf(b, -lim), lim);
  const f2 xc = pk(a, b);
  const f2 x2 = fma2(xc, xc, 0ull);
  f2 p = fma2(x2, SPL(-2.76076847742355e-16f), SPL(2.00018790482477e-13f));
  p = fma2(x2, p, SPL(-8.60467152213735e-11f));
  p = fma2(x2, p, SPL(5.12229709037114e-08f));
  p = fma2(x2, p, SPL(1.48572235717979e-05f));
  p = fma2(x2, p, SPL(6.37261928875436e-04f));
  p = fma2(x2, p, SPL(4.89352455891786e-03f));
  p = fma2(xc, p, 0ull);
  f2 q = fma2(x2, SPL(1.19825839466702e-06f), SPL(1.18534705686654e-04f));
  q = fma2(x2, q, SPL(2.26843463243900e-03f));
  q = fma2(x2, q, SPL(4.89352518554385e-03f));
  float q0, q1;
  f2unpack(q, q0, q1);
  f2 r = pk(__uint_as_float(0x7EF311C3u - __float_as_uint(q0)), __uint_as_float(0x7EF311C3u - __float_as_uint(q1)));
  const f2 nq = q ^ 0x8000000080000000ull;  // -q
#pragma unroll
  for (int it = 0; it < 3; ++it) r = fma2(r, fma2(nq, r, SPL(1.0f)), r);  // r += r (1 - q r)
#undef SPL
  return fma2(p, r, 0ull);
}

#ifndef SMPC_MLP_FMA_TANH
#define SMPC_MLP_FMA_TANH 1  // layer-2 epilogue: every other tanh pair on the FMA pipe (A/B: 0 = all MUFU)
#endif

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity));
}

// 32 consecutive fp32 TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Shared-memory carve-up (bytes); host and device agree through this struct.
struct Smem {
  int w2hi, w2lo, h0, xs, params, sig2, sigma, mean, bar, total;
  // RM: both RMPPI systems in one CTA: an A-operand pair per system and the
  // nominal states exchanged for the real system's feedback
  __host__ __device__ Smem(int S, int TU, bool RM = false) {
    w2hi = 0;
    w2lo = w2hi + kWBytes;
    h0 = w2lo + kWBytes;                        // [sys][hi|lo][128 x 32]
    xs = h0 + (RM ? 2 : 1) * 2 * kHBytes;       // RM: nominal x_t of each sample [128][8]
    params = xs + (RM ? kTile * 8 * 4 : 0);     // W1 b1 b2 W3 b3 (fp32)
    sig2 = (params + (TOTAL - HID * HID) * 4 + 15) / 16 * 16;
    sigma = sig2 + TU * 8;
    mean = sigma + TU * 4;
    bar = (mean + S * TU * 4 + 15) / 16 * 16;   // mbarrier (8 B) + TMEM base (4 B); mean = all S systems
    total = bar + 16;
  }
};

// RM = RMPPI (a.rmppi, S = 2): one CTA of 256 threads holds both systems of
// the same 128 samples (threads 0-127 nominal, 128-255 real), two M = 128
// MMAs per K-step into TMEM columns [0,32) and [32,64), so the real system's
// sampled control gets u + K (x_real,t - x_nominal,t) of its own sample
// (states exchanged through shared memory, one extra CTA barrier per step).
template <class Dyn, class Cost, bool INJ, bool IMP, bool RM>
__global__ void __launch_bounds__(RM ? 2 * kTile : kTile, RM ? 2 : 4)
    mlp_rollout_kernel(const IterArgs a, const Dyn dyn, Cost cost) {
  constexpr int NU = 2, NX = 7, NY = 7;
  constexpr int NTH = RM ? 2 * kTile : kTile;
  const int S = a.S;
  const int sys = RM ? (int)(threadIdx.x >> 7) : (int)blockIdx.y;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (aborted(a)) return;
  const int T = a.T, TU = T * NU;
  const Smem L(S, TU, RM);
  float* prm = reinterpret_cast<float*>(smem + L.params);  // W1T [0,192) b1 [192,224) b2 [224,256) W3T [256,384) b3 [384,388)
  const float* sW1 = prm;
  const float* sB1 = prm + HID * IN;
  const float* sB2 = sB1 + HID;
  const float* sW3 = sB2 + HID;
  const float* sB3 = sW3 + OUT * HID;
  double* sig2_s = reinterpret_cast<double*>(smem + L.sig2);
  float* sigma_s = reinterpret_cast<float*>(smem + L.sigma);
  float* mean_s = reinterpret_cast<float*>(smem + L.mean);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.bar + 8);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int row = tid & (kTile - 1);  // sample row of this thread's system tile (= its TMEM lane)
  float* xs_s = reinterpret_cast<float*>(smem + L.xs);

  // ---- one-time staging: W2 as TF32 hi/lo operand tiles, the SIMT layers, sampler tables
  const float* w = dyn.w;
  for (int e = tid; e < HID * HID; e += NTH) {
    const int n = e / HID, k = e % HID;  // W2[n][k]: B operand row n (output unit), K-major
    const float v = __ldg(w + W2 + e);
    const float hi = to_tf32(v);
    *reinterpret_cast<float*>(smem + L.w2hi + core_off(n, k)) = hi;
    *reinterpret_cast<float*>(smem + L.w2lo + core_off(n, k)) = to_tf32(v - hi);
  }
  // SIMT layers, transposed for packed broadcast reads: W1T[k][j], b1, b2, W3T[j][q], b3
  for (int e = tid; e < HID * IN; e += NTH) prm[(e % IN) * HID + e / IN] = __ldg(w + W1 + e);
  for (int e = tid; e < HID; e += NTH) prm[HID * IN + e] = __ldg(w + B1 + e), prm[HID * IN + HID + e] = __ldg(w + B2 + e);
  for (int e = tid; e < OUT * HID; e += NTH) prm[HID * IN + 2 * HID + (e % HID) * OUT + e / HID] = __ldg(w + W3 + e);
  for (int e = tid; e < OUT; e += NTH) prm[HID * IN + 2 * HID + OUT * HID + e] = __ldg(w + B3 + e);
  for (int k = tid; k < TU; k += NTH) {
    sigma_s[k] = a.sigma[k];
    if (IMP) sig2_s[k] = a.sig2_pow2 ? 1.0 / a.sig2[k] : a.sig2[k];  // exact inverse of a power of two
  }
  for (int k = tid; k < S * TU; k += NTH) mean_s[k] = a.mean_in[k];
  constexpr int kCols = RM ? 64 : 32;  // fp32 accumulator columns: 32 per system
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) mbar_init(bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int i = blockIdx.x * kTile + row;
  const bool active = i < a.M_local;
  const long long m = (a.sample_idx && active) ? a.sample_idx[i] : a.m_begin + i;
  const bool is_mean = a.with_mean && m == 0;
  const bool zero_mean = m >= a.zero_begin;
  const uint32_t stream = noise_stream(a);

  float x[NX], y[NY];
  double total = 0.0, imp = 0.0;
#pragma unroll
  for (int c = 0; c < NX; ++c) x[c] = a.x0[sys * NX + c];
  unsigned long long err = kNoError;
  float4 zq = make_float4(0.f, 0.f, 0.f, 0.f);
  // small-N mode: pre-generated quads, prefetched one quad ahead
  const size_t zi = (size_t)(active ? i : 0);
  float4 zn = a.zq ? __ldg(a.zq + zi) : make_float4(0.f, 0.f, 0.f, 0.f);
  uint32_t phase = 0;
  unsigned char* hhi = smem + L.h0 + (RM ? sys * 2 * kHBytes : 0);
  unsigned char* hlo = hhi + kHBytes;
  const float* mean_sys = mean_s + sys * TU;  // u = mean_s + eps; eps drawn about system 0's mean

  for (int t = 0; t < T; ++t) {
    // ---- RMPPI ancillary feedback on the real system from the nominal state
    // of the same sample at time t: fb_c = sum_j K[c][j] (x_real,j - x_nom,j)
    float fb[NU] = {0.0f, 0.0f};
    if constexpr (RM) {
      if (sys == 0) {
#pragma unroll
        for (int c = 0; c < NX; ++c) xs_s[row * 8 + c] = x[c];
      }
      __syncthreads();
      if (sys == 1) {
#pragma unroll
        for (int c = 0; c < NU; ++c) {
          float acc = 0.0f;
#pragma unroll
          for (int j = 0; j < NX; ++j) acc = F_ADD(acc, F_MUL(a.fb_gain[c * NX + j], F_SUB(x[j], xs_s[row * 8 + j])));
          fb[c] = acc;
        }
      }
    }
    // ---- noise (sampling.cpp:64-88) and the sampled, clamped control
    float u[NU], uc[NU];
#pragma unroll
    for (int c = 0; c < NU; ++c) {
      const int k = t * NU + c;
      float e;
      if constexpr (INJ) {
        e = active ? a.eps_in[(size_t)(m - a.m_begin) * TU + k] : 0.0f;
      } else {
        if ((k & 3) == 0) {
          if (a.zq) {
            zq = zn;
            if ((k >> 2) + 1 < (TU + 3) / 4) zn = __ldg(a.zq + (size_t)((k >> 2) + 1) * a.M_local + zi);
          } else {
            zq = normal_quad_fast(a, stream, (uint32_t)m, (uint32_t)(k >> 2));
          }
        }
        float ev = F_MUL(sigma_s[k], quad_lane(zq, k & 3));
        if (zero_mean) ev = F_SUB(ev, mean_s[k]);
        e = is_mean ? 0.0f : ev;
      }
      const float mu = mean_sys[k];
      u[c] = F_ADD(mu, e);
      if constexpr (IMP) {
        const double me = D_MUL((double)mu, (double)e);
        imp = D_ADD(imp, a.sig2_pow2 ? D_MUL(me, sig2_s[k]) : __ddiv_rn(me, sig2_s[k]));
      }
      if constexpr (RM) {
        if (sys == 1) u[c] = F_ADD(u[c], fb[c]);
      }
    }
    dyn.clamp_control(u, uc);
    // ---- layer 1 (SIMT) -> this sample's row of the hi/lo A operand
    const float in[IN] = {x[3], x[4], x[5], x[6], uc[0], uc[1]};
    f2 inb[IN];
#pragma unroll
    for (int k = 0; k < IN; ++k) inb[k] = pk(in[k], in[k]);
#pragma unroll
    for (int j0 = 0; j0 < HID; j0 += 4) {
      // units j0..j0+3 as two packed pairs, 6 FFMA2 each
      const ulonglong2 bb = *reinterpret_cast<const ulonglong2*>(sB1 + j0);
      f2 acc0 = bb.x, acc1 = bb.y;
#pragma unroll
      for (int k = 0; k < IN; ++k) {
        const ulonglong2 wk = *reinterpret_cast<const ulonglong2*>(sW1 + k * HID + j0);
        acc0 = fma2(wk.x, inb[k], acc0);
        acc1 = fma2(wk.y, inb[k], acc1);
      }
      float h[4];
      f2unpack(tanh2(acc0), h[0], h[1]);
      f2unpack(tanh2(acc1), h[2], h[3]);
      float hv[4], lv[4];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        hv[jj] = to_tf32(h[jj]);
        lv[jj] = to_tf32(h[jj] - hv[jj]);
      }
      *reinterpret_cast<float4*>(hhi + core_off(row, j0)) = make_float4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<float4*>(hlo + core_off(row, j0)) = make_float4(lv[0], lv[1], lv[2], lv[3]);
    }
    // ---- layer 2 on the tensor cores: D = H1 W2^T (3xTF32), one issuing thread
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0) {
      const uint32_t bhi = smem_u32(smem + L.w2hi), blo = smem_u32(smem + L.w2lo);
#pragma unroll
      for (int ss = 0; ss < (RM ? 2 : 1); ++ss) {
        const uint32_t ahi = smem_u32(smem + L.h0 + ss * 2 * kHBytes), alo = ahi + kHBytes;
        const uint32_t d = tmem + (uint32_t)(ss * 32);  // system ss: accumulator columns [32 ss, 32 ss + 32)
#pragma unroll
        for (int kk = 0; kk < HID / 8; ++kk) {  // K-step of 8 TF32 = 2 core-matrix chunks = 256 B
          const uint32_t off = (uint32_t)kk * 2u * kLBO;
          mma_tf32(d, smem_desc(ahi + off), smem_desc(bhi + off), kk > 0 ? 1u : 0u);
          mma_tf32(d, smem_desc(ahi + off), smem_desc(blo + off), 1u);
          mma_tf32(d, smem_desc(alo + off), smem_desc(bhi + off), 1u);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                   : "memory");
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    // ---- epilogue: layer 3 + kinematics + Euler + running cost
    float d2[HID];
    tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(RM ? sys * 32 : 0), d2);
    const ulonglong2 b3v = *reinterpret_cast<const ulonglong2*>(sB3);
    f2 o01 = b3v.x, o23 = b3v.y;
#pragma unroll
    for (int j = 0; j < HID; j += 2) {
      const f2 hb = fma2(pk(d2[j], d2[j + 1]), f2splat_bits(0x3F800000u), *reinterpret_cast<const f2*>(sB2 + j));
      float h0, h1;
      f2unpack((SMPC_MLP_FMA_TANH && ((j >> 1) & 1)) ? tanh2_fma(hb) : tanh2(hb), h0, h1);
      const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(sW3 + j * OUT);        // W3T[j][0..3]
      const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(sW3 + (j + 1) * OUT);  // W3T[j+1][0..3]
      const f2 hh0 = pk(h0, h0), hh1 = pk(h1, h1);
      o01 = fma2(w0.x, hh0, o01);
      o23 = fma2(w0.y, hh0, o23);
      o01 = fma2(w1.x, hh1, o01);
      o23 = fma2(w1.y, hh1, o23);
    }
    float o[OUT];
    f2unpack(o01, o[0], o[1]);
    f2unpack(o23, o[2], o[3]);
    float dx[NX];
    dyn.kinematics(x, dx);
#pragma unroll
    for (int q = 0; q < OUT; ++q) dx[3 + q] = o[q];
    float xn[NX];
#pragma unroll
    for (int c = 0; c < NX; ++c) xn[c] = F_ADD(x[c], F_MUL(a.dt, dx[c]));
    xn[2] = wrap_angle(xn[2]);
#pragma unroll
    for (int c = 0; c < NY; ++c) y[c] = xn[c];
    const double ct = cost.running_cost(y, uc, t);
    if (active && err == kNoError) {  // engine.cpp:51-65, first failure per sample
      int ch = -1;
#pragma unroll
      for (int c = NX - 1; c >= 0; --c)
        if (!isfinite(xn[c])) ch = c;
      if (ch >= 0) err = make_error_key(0, sys, m, t, 0, ch);
      else if (!(ct >= 0.0 && ct <= DBL_MAX)) err = make_error_key(0, sys, m, t, 1, 0);
    }
    total = D_ADD(total, ct);
    if (a.outputs && active) {
      float* op = a.outputs + (((size_t)sys * a.M_local + i) * T + t) * NY;
#pragma unroll
      for (int c = 0; c < NY; ++c) op[c] = y[c];
    }
#pragma unroll
    for (int c = 0; c < NX; ++c) x[c] = xn[c];
  }

  // ---- release TMEM (the allocating warp), then totals (engine.cpp:236-238, :263-265)
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
  }
  double J = INFINITY;
  if (active) {
    if (err == kNoError) {
      const double term = cost.terminal_cost(y);
      if (!(term >= 0.0 && term <= DBL_MAX)) err = make_error_key(0, sys, m, T - 1, 2, 0);
      J = D_ADD(total, term);
      if constexpr (IMP) J = D_ADD(J, D_MUL(a.lambda, imp));
      if (!isfinite(J) && err == kNoError) err = make_error_key(1, sys, m, 0, 0, 0);
    } else {
      J = NAN;
    }
    a.costs[(size_t)sys * a.M_local + i] = J;
  }
  if (err != kNoError) atomicMin(&a.header->err_key, err);

  // ---- block (min, argmin) of this system; the last CTA of the whole grid
  // reduces every system (same output as publish_block_min, 2-D grid).
  // (RM: one pass per system over the whole 256-thread CTA)
#pragma unroll
  for (int ss = 0; ss < (RM ? 2 : 1); ++ss) {
    const bool mine = !RM || sys == ss;
    double j = active && mine ? J : INFINITY;
    if (!(j == j)) j = INFINITY;
    long long mm = active && mine ? m : LLONG_MAX;
    block_argmin<NTH>(j, mm);
    if (tid == 0) {
      const int s_out = RM ? ss : sys;
      a.blk_min[s_out * a.n_roll_blocks + blockIdx.x] = j;
      a.blk_arg[s_out * a.n_roll_blocks + blockIdx.x] = mm;
    }
  }
  if (!last_block_done(&a.counters[0], gridDim.x * gridDim.y)) return;
  for (int s = 0; s < S; ++s) {
    double j = INFINITY;
    long long mm = LLONG_MAX;
    for (int b = tid; b < a.n_roll_blocks; b += NTH) {
      const double j2 = ((volatile double*)a.blk_min)[s * a.n_roll_blocks + b];
      const long long m2 = ((volatile long long*)a.blk_arg)[s * a.n_roll_blocks + b];
      if (better(j2, m2, j, mm)) j = j2, mm = m2;
    }
    block_argmin<NTH>(j, mm);
    if (tid == 0) {
      double* g = a.gather1 + (size_t)a.rank * a.g1s + s * 2;
      g[0] = j;
      g[1] = __longlong_as_double(mm);
    }
  }
}

template <class Dyn, class Cost, bool RM>
cudaError_t launch_rm(const IterArgs& a, const Dyn& dyn, const Cost& cost, cudaStream_t st) {
  const Smem L(a.S, a.T * 2, RM);
  const size_t smem = (size_t)L.total;
  const dim3 grid((unsigned)((a.M_local + kTile - 1) / kTile), RM ? 1u : (unsigned)a.S), block(RM ? 2 * kTile : kTile);
  auto k = mlp_rollout_kernel<Dyn, Cost, false, false, RM>;
  if (a.eps_in)
    k = a.importance ? mlp_rollout_kernel<Dyn, Cost, true, true, RM> : mlp_rollout_kernel<Dyn, Cost, true, false, RM>;
  else if (a.importance)
    k = mlp_rollout_kernel<Dyn, Cost, false, true, RM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<grid, block, smem, st>>>(a, dyn, cost);
  return cudaGetLastError();
}

template <class Dyn, class Cost>
cudaError_t launch(const IterArgs& a, const Dyn& dyn, const Cost& cost, cudaStream_t st) {
  if (a.rmppi && a.S == 2) return launch_rm<Dyn, Cost, true>(a, dyn, cost, st);
  return launch_rm<Dyn, Cost, false>(a, dyn, cost, st);
}

template <class Dyn>
cudaError_t rollout(const Dyn& dyn, const IterArgs& a, int cost_kind, cudaStream_t st) {
  switch (cost_kind) {
    case 0: return launch(a, dyn, make_road(a.cost), st);
    case 3: return launch(a, dyn, make_quad<7>(a.cost), st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace mlpk

namespace {
template <bool F>
MlpDyn<F> mlp_make(const DynParams& p) {
  MlpDyn<F> d;
  d.w = p.tensor;
  return d;
}
template <bool F>
cudaError_t mlp_rollout(const IterArgs& a, int ck, cudaStream_t st) {
  return mlpk::rollout(mlp_make<F>(a.dyn), a, ck, st);
}
template <bool F>
cudaError_t mlp_plant(const IterArgs& a, int ck, const PlantStepArgs& p, cudaStream_t st) {
  switch (ck) {
    case 0: return launch_plant_step_t(a, mlp_make<F>(a.dyn), make_road(a.cost), p, st);
    case 3: return launch_plant_step_t(a, mlp_make<F>(a.dyn), make_quad<7>(a.cost), p, st);
  }
  return cudaErrorInvalidValue;
}
template <bool F>
cudaError_t mlp_rmppi(const IterArgs& a, int ck, cudaStream_t st) {
  switch (ck) {
    case 0: return launch_rmppi_select_coop_t(a, mlp_make<F>(a.dyn), make_road(a.cost), st);
    case 3: return launch_rmppi_select_coop_t(a, mlp_make<F>(a.dyn), make_quad<7>(a.cost), st);
  }
  return cudaErrorInvalidValue;
}
template <bool F>
cudaError_t mlp_update(const IterArgs& a, cudaStream_t st) {
  return launch_update_t(a, mlp_make<F>(a.dyn), st);
}
template <bool F>
cudaError_t mlp_combine(const IterArgs& a, cudaStream_t st) {
  return launch_combine_t(a, mlp_make<F>(a.dyn), st);
}
cudaError_t mlp_generate(const IterArgs& a, float* e, uint8_t* f, cudaStream_t st) {
  return launch_generate_t<2>(a, e, f, st);
}
}  // namespace

ModelOps ops_mlp(bool fma_libm) {
  if (fma_libm)
    return ModelOps{mlp_rollout<true>, mlp_rmppi<true>, mlp_plant<true>, launch_weights, mlp_update<true>,
                    mlp_combine<true>, mlp_generate, 7, 2, 7};
  return ModelOps{mlp_rollout<false>, mlp_rmppi<false>, mlp_plant<false>, launch_weights, mlp_update<false>,
                  mlp_combine<false>, mlp_generate, 7, 2, 7};
}

}  // namespace smpc_dev
