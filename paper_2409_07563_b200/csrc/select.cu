// Device ordering of samples by (cost, index): the CEM elite selection
// (CemController::compute_control, controllers.cpp:161-198) and the
// partial_sort behind it, for any context's last rollout.
//
//   k smallest by (J_m, m)   <- std::partial_sort(order, order+k, ..., cmp)
//                               with cmp = (J_a != J_b) ? J_a < J_b : a < b
//                               (controllers.cpp:165-171)
//
// Selection is an MSB radix select over an order-preserving 64-bit image of
// the cost (8 passes of 8-bit digits, each an L2-resident scan of the costs
// with a shared-memory histogram; the last CTA of each pass picks the digit).
// It ends with the threshold key K* and the number `need` of samples with
// key == K* that are elites; those are the lowest-indexed ones (the
// comparator's tie-break), found with per-CTA counts and an exclusive prefix.
// The elites are then compacted in ascending m into the same candidate list
// the MPPI weighted-update kernel consumes, with e_m = 1 and eta = 1, so the
// update kernel accumulates exactly sum_elites eps (controllers.cpp:175-180)
// and commit_update applies mean + acc / k (:186).
//
// The explicit elite ORDER (only needed for reporting, smpc_sorted_samples)
// is a bitonic sort of the k compacted (key, m) pairs.
#include <algorithm>

#include "kernels.cuh"

namespace smpc_dev {

// Order-preserving image of a double (total order; -0 folded onto +0 so the
// comparator's J_a != J_b tie semantics hold).
__device__ __forceinline__ unsigned long long cost_key(double j) {
  if (j == 0.0) j = 0.0;
  const unsigned long long b = (unsigned long long)__double_as_longlong(j);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256) select_init_kernel(SelectState* st, long long k) {
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->k_rem = k;
    st->k = k;
  }
  st->hist[threadIdx.x] = 0u;
}

// One radix pass: digit (key >> shift) & 255 over the keys that share the
// already-selected higher digits.
__global__ void __launch_bounds__(256) select_pass_kernel(const double* costs, long long n, SelectState* st,
                                                          int pass, unsigned int* counter) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0u;
  __syncthreads();
  const int shift = 56 - 8 * pass;
  const unsigned long long prefix = st->prefix;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long key = cost_key(costs[i]);
    const bool match = pass == 0 || ((key ^ prefix) >> (shift + 8)) == 0ull;
    if (match) atomicAdd(&h[(key >> shift) & 255u], 1u);
  }
  __syncthreads();
  if (h[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], h[threadIdx.x]);
  if (!last_block_done(counter, gridDim.x)) return;
  // Last CTA: inclusive scan of the 256 global bins, pick the bin holding rank k_rem.
  __shared__ unsigned long long cum[256];
  const unsigned int mine = ((volatile unsigned int*)st->hist)[threadIdx.x];
  cum[threadIdx.x] = mine;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const unsigned long long v = threadIdx.x >= off ? cum[threadIdx.x - off] : 0ull;
    __syncthreads();
    cum[threadIdx.x] += v;
    __syncthreads();
  }
  const long long k_rem = st->k_rem;
  const unsigned long long before = cum[threadIdx.x] - mine;
  __syncthreads();
  if ((long long)before < k_rem && k_rem <= (long long)cum[threadIdx.x]) {
    st->prefix = prefix | ((unsigned long long)threadIdx.x << shift);
    st->k_rem = k_rem - (long long)before;
  }
  st->hist[threadIdx.x] = 0u;
}

// Per weights-CTA range: how many keys equal K* (for the lowest-index tie-break).
__global__ void __launch_bounds__(256) select_eq_count_kernel(const IterArgs a, const SelectState* st, int* eq_cnt,
                                                              long long* eq_off, unsigned int* counter) {
  const long long beg = (long long)blockIdx.x * a.M_local / gridDim.x;
  const long long end = (long long)(blockIdx.x + 1) * a.M_local / gridDim.x;
  const unsigned long long kstar = st->prefix;
  long long c = 0;
  for (long long i = beg + threadIdx.x; i < end; i += blockDim.x) c += cost_key(a.costs[i]) == kstar;
  c = block_sum<256>(c);
  if (threadIdx.x == 0) eq_cnt[blockIdx.x] = (int)c;
  if (!last_block_done(counter, gridDim.x)) return;
  if (threadIdx.x == 0) {  // n_w_blocks <= 592: a serial prefix is ~1 us
    long long run = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      eq_off[b] = run;
      run += ((volatile int*)eq_cnt)[b];
    }
  }
}

// Marks elites (e_m = 1, else 0) and compacts them per CTA range in ascending
// m into cand (the update kernel's work list, mean sample excluded: its eps is
// identically zero); the last CTA turns the counts into offsets and publishes
// eta = 1 / elite count for the update and commit.
__global__ void __launch_bounds__(256) select_mark_kernel(const IterArgs a, const SelectState* st, const long long* eq_off,
                                                          unsigned int* counter) {
  __shared__ int warp_cnt[8], warp_eq[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long beg = (long long)blockIdx.x * a.M_local / gridDim.x;
  const long long end = (long long)(blockIdx.x + 1) * a.M_local / gridDim.x;
  const unsigned long long kstar = st->prefix;
  const long long need = st->k_rem;
  long long eq_seen = eq_off[blockIdx.x];
  long long ncand = 0;
  for (long long c0 = beg; c0 < end; c0 += 256) {
    const long long i = c0 + threadIdx.x;
    bool elite = false, eq = false;
    unsigned long long key = ~0ull;
    if (i < end) {
      key = cost_key(a.costs[i]);
      eq = key == kstar;
    }
    const unsigned beq = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_eq[warp] = __popc(beq);
    __syncthreads();
    int eq_before = 0, eq_total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      eq_before += (w < warp) ? warp_eq[w] : 0;
      eq_total += warp_eq[w];
    }
    if (i < end) {
      const long long eq_rank = eq_seen + eq_before + __popc(beq & ((1u << lane) - 1u));
      elite = key < kstar || (eq && eq_rank < need);
      a.weights[i] = elite ? 1.0 : 0.0;
    }
    eq_seen += eq_total;
    const bool take = elite && !(a.with_mean && a.m_begin + i == 0);
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_cnt[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      before += (w < warp) ? warp_cnt[w] : 0;
      total += warp_cnt[w];
    }
    if (take) {
      const long long pos = beg + ncand + before + __popc(bal & ((1u << lane) - 1u));
      a.cand[pos] = (int)i;
      if (a.cand_e) a.cand_e[pos] = 1.0;  // elites: e_m = 1, eta = 1
    }
    ncand += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.cand_cnt[blockIdx.x] = (int)ncand;
  if (!last_block_done(counter, gridDim.x)) return;
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      a.cand_off[b] = run;
      run += ((volatile int*)a.cand_cnt)[b];
    }
    a.cand_off[gridDim.x] = run;
    double* g = a.gather2 + (size_t)a.rank * a.g2s;
    g[0] = 1.0;              // eta for the update: w_m = e_m / 1 = 1 exactly
    g[1] = (double)st->k;    // elites ("nonzero" weights)
  }
}

// ---- explicit order of the selected samples (bitonic over (key, m)) ---------

// (key, m) pairs padded to a power of two with +inf keys.
__global__ void pad_pairs_kernel(unsigned long long* keys, long long* idx, long long n_pad) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  keys[i] = ~0ull;
  idx[i] = LLONG_MAX;
}

// Every selected sample (e_m != 0 marks them, mean sample included — cand
// omits it); slots are taken in arbitrary order, the sort fixes the order.
__global__ void scatter_selected_kernel(const IterArgs a, unsigned long long* keys, long long* idx,
                                        unsigned long long* slot) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.M_local;
       i += (long long)gridDim.x * blockDim.x) {
    if (a.weights[i] != 0.0) {
      const unsigned long long p = atomicAdd(slot, 1ull);
      keys[p] = cost_key(a.costs[i]);
      idx[p] = a.m_begin + i;
    }
  }
}

__device__ __forceinline__ bool pair_less(unsigned long long ka, long long ia, unsigned long long kb, long long ib) {
  return ka < kb || (ka == kb && ia < ib);
}

__global__ void bitonic_step_kernel(unsigned long long* keys, long long* idx, long long n, long long j, long long k) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long l = i ^ j;
  if (l <= i) return;
  const bool up = (i & k) == 0;
  const unsigned long long ki = keys[i], kl = keys[l];
  const long long ii = idx[i], il = idx[l];
  const bool swap = up ? pair_less(kl, il, ki, ii) : pair_less(ki, ii, kl, il);
  if (swap) {
    keys[i] = kl, keys[l] = ki;
    idx[i] = il, idx[l] = ii;
  }
}

cudaError_t launch_select(const IterArgs& a, SelectState* st, long long k, unsigned int* counters, int* eq_cnt,
                          long long* eq_off, cudaStream_t s) {
  select_init_kernel<<<1, 256, 0, s>>>(st, k);
  const int nblk = std::max(1, std::min(a.n_w_blocks, (int)((a.M_local + 255) / 256)));
  for (int pass = 0; pass < 8; ++pass)
    select_pass_kernel<<<nblk, 256, 0, s>>>(a.costs, a.M_local, st, pass, counters + 0);
  select_eq_count_kernel<<<a.n_w_blocks, 256, 0, s>>>(a, st, eq_cnt, eq_off, counters + 1);
  select_mark_kernel<<<a.n_w_blocks, 256, 0, s>>>(a, st, eq_off, counters + 2);
  return cudaGetLastError();
}

cudaError_t launch_sort_selected(const IterArgs& a, long long k, unsigned long long* keys, long long* idx,
                                 unsigned long long* slot, cudaStream_t s) {
  long long n_pad = 1;
  while (n_pad < k) n_pad <<= 1;
  const int threads = 256;
  const unsigned blocks = (unsigned)((n_pad + threads - 1) / threads);
  pad_pairs_kernel<<<blocks, threads, 0, s>>>(keys, idx, n_pad);
  cudaMemsetAsync(slot, 0, sizeof(unsigned long long), s);
  scatter_selected_kernel<<<592, 256, 0, s>>>(a, keys, idx, slot);
  for (long long kk = 2; kk <= n_pad; kk <<= 1)
    for (long long j = kk >> 1; j > 0; j >>= 1) bitonic_step_kernel<<<blocks, threads, 0, s>>>(keys, idx, n_pad, j, kk);
  return cudaGetLastError();
}

}  // namespace smpc_dev
