// Host/device launch descriptors shared by the kernel instantiation units and
// the C-ABI host code. Plain PODs: the host fills them once per context and
// the kernels read them as by-value kernel parameters.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace smpc_dev {

constexpr int kMaxNX = 16;
constexpr int kMaxNU = 4;
constexpr int kMaxNY = 16;
constexpr int kRolloutThreads = 128;

// SMPC_DYN_MLP parameter blob (smpc_b200.h): W1[32][6] b1[32] W2[32][32]
// b2[32] W3[4][32] b3[4], fp32 row-major.
namespace mlp_layout {
constexpr int IN = 6, HID = 32, OUT = 4;
constexpr int W1 = 0, B1 = W1 + HID * IN, W2 = B1 + HID, B2 = W2 + HID * HID, W3 = B2 + HID, B3 = W3 + OUT * HID;
constexpr int TOTAL = B3 + OUT;  // 1412
}  // namespace mlp_layout

constexpr int kUpdateThreads = 256;
constexpr int kUpdateWarps = kUpdateThreads / 32;
#ifndef SMPC_UPDATE_MIN_BLOCKS2
#define SMPC_UPDATE_MIN_BLOCKS2 2
#endif
constexpr int kUpdateCtasPerSm = SMPC_UPDATE_MIN_BLOCKS2;  // resident update CTAs per SM
#ifndef SMPC_UPDATE_QUADS_PER_UNIT
#define SMPC_UPDATE_QUADS_PER_UNIT 2
#endif
constexpr int kUpdateQuadsPerUnit = SMPC_UPDATE_QUADS_PER_UNIT;  // quads per update work unit
constexpr size_t kFinishStageMaxBytes = 200 * 1024;
// Split small-N rollout: samples per cost CTA, so that its per-(sample, t)
// costs and importance terms stay within 96 KB of shared memory.
__host__ __device__ inline int split_samples_per_cta(int T, int NU, bool imp) {
  int sb = 32;
  const long long per = (long long)T * (1 + (imp ? NU : 0)) * 8;
  while (sb > 1 && per * sb > 96 * 1024) sb >>= 1;
  return sb;
}
constexpr int kUpdateSlot = kUpdateQuadsPerUnit * 4;  // per-warp partial: the group's QW*4 entry sums
// Shards up to this many samples pre-generate the iteration's noise in one
// parallel pass (gen_zq_kernel) instead of inside each sample's serial chain.
constexpr long long kZqMaxSamples = 16384;

// Error key (lowest key wins = what a single-worker reference would throw):
//   [63:62] stage  0 rollout, 1 compute_weights, 2 finish_solution
//   [61]    system
//   [60:30] sample (global index)
//   [29:6]  timestep
//   [5:4]   phase  0 non-finite state, 1 invalid running cost, 2 terminal
//   [3:0]   channel
constexpr unsigned long long kNoError = ~0ull;
__host__ __device__ inline unsigned long long make_error_key(unsigned stage, unsigned s, long long m,
                                                             int t, unsigned phase, unsigned ch) {
  return ((unsigned long long)stage << 62) | ((unsigned long long)(s & 1) << 61) |
         ((unsigned long long)(m & 0x7fffffffLL) << 30) | ((unsigned long long)(t & 0xffffff) << 6) |
         ((unsigned long long)(phase & 3) << 4) | (unsigned long long)(ch & 15);
}

// Philox round keys (see philox_normal.cuh) and the runtime {1,1} / {-0,-0}
// f32x2 operands that keep ptxas from contracting packed mul+add.
struct PhiloxKeys {
  uint32_t k0[10], k1[10];
};
struct PackConst {
  unsigned long long one;    // {1.0f, 1.0f}
  unsigned long long mzero;  // {-0.0f, -0.0f}
};

// Model / cost parameters as plain floats (device functors are built from these).
struct DynParams {
  float p[8];
  const float* tensor;  // device copy of smpc_problem::dyn_tensor (SMPC_DYN_MLP)
};
struct CostParams {
  float p[8];
  int n_quad;
  float target[kMaxNY], weights[kMaxNY];
  // costmap (diff_drive_nav)
  const uint8_t* grid;  // device pointer
  int cells_x, cells_y;
  float origin_x, origin_y, inv_resolution;
  int map_in_smem;
};

// Radix-select state (select.cu): the k-th smallest (cost, index) key.
struct SelectState {
  unsigned long long prefix;  // threshold key K* (complete after the 8 passes)
  long long k_rem;            // elites with key == K* (lowest indices first)
  long long k;                // elites in total
  unsigned int hist[256];
};

// Per-context iteration state on the device.
struct ResultHeader {
  unsigned long long err_key;
  unsigned long long abort_key;
  unsigned long long solve_count;
  double rho[2];
  double eta[2];
  long long argmin[2];
  long long nonzero[2];
  float next_nominal_state[kMaxNX];
  // RMPPI: the nominal state chosen for this solve and its candidate index
  float rmppi_nominal[kMaxNX];
  int rmppi_choice;
  // closed loop (smpc_run_control_loop): sticky first error of the loop and
  // the accumulated applied running cost (plant.cpp:175)
  unsigned long long loop_err;
  double loop_cost;
};

// One SimulatedSystem::step of the closed loop (plant.cpp:31-48, :160-178).
struct PlantStepArgs {
  float* x;               // simulated state [NX] (device)
  float* x0_out;          // the controller's x0 buffer: the next update_state snapshot
  const float* controls;  // last solution's controls [T][NU]
  int idx;                // control_for_time index (plant.cpp:106-115)
  uint32_t step;          // SimulatedSystem::step_count_ and the cost's t
  float dt;               // (float) controller dt
  float scale;            // (float)(disturbance_std * sqrt(dt)); 0 = no disturbance
  PhiloxKeys rk;          // round keys of NormalStream(rng_seed ^ 0x9E3779B97F4A7C15)
  double t;
  double* log;            // [steps][2 + NX + NU] rows {t, x, u, c} or nullptr
};

__host__ __device__ inline double exact_inverse_pow2(double x) {
  // 1/x if x is a power of two whose inverse is a normal double (then x*inv
  // equals x/lambda bit for bit for every operand), else 0
  if (!(x > 0.0) || x > 0x1p1000 || x < 0x1p-1000) return 0.0;
  int e;
  const double m = frexp(x, &e);
  return m == 0.5 ? ldexp(1.0, 1 - e) : 0.0;
}

struct IterArgs {
  // problem
  int T, S;
  int M_local;
  long long m_begin;
  long long M_global;
  float dt;
  double lambda;
  double inv_lambda_pow2;  // 1/lambda when lambda is a power of two (x/lambda == x*inv exactly), else 0
  int sig2_pow2;           // every sigma^2 is a power of two: the importance term multiplies by 1/sigma^2 (exact)
  uint32_t key0, key1;
  PhiloxKeys rk;         // round keys of (key0, key1)
  PackConst pk;
  // Phi^-1 tail lookup on the Philox word w (see philox_normal.cuh): with
  // u = w + tail_off (mod 2^32), the draw is a tail iff u < tail_lim, and its
  // value is tail[u >> 9] (upper tail first, then the lower tail).
  uint32_t tail_off, tail_lim;
  int with_mean;
  long long zero_begin;
  int importance;
  int world, rank;
  // noise stream: stream = solve_count*256 + iter (stream_for, controllers.cpp:63-66),
  // or the explicit value when solve_count == nullptr
  const unsigned long long* solve_count;
  int iter;
  uint32_t stream;
  // inputs
  const float* mean_in;  // [S][T][NU]
  float* mean_out;       // [S][T][NU]
  const float* x0;       // [S][NX]
  const float* sigma;    // [T][NU]
  const double* sig2;    // [T][NU]
  const double* gamma;   // [T]
  const float* eps_in;   // injected [M_local][T][NU] or nullptr
  const float* tail;     // Phi^-1 tail table
  unsigned long long tail_tex;  // the same table as a 1-D texture object (index-addressed fetch)
  // normal_icdf over the sampler's whole domain (2^23 floats, 32 MB, built
  // once per device with the same device arithmetic as the in-register
  // path): a texture object, or 0
  unsigned long long full_tex;
  // rollout outputs
  double* costs;   // [S][M_local]
  float* outputs;  // [S][M_local][T][NY] or nullptr
  // reduction scratch
  int n_roll_blocks;
  double* blk_min;       // [S][n_roll_blocks]
  long long* blk_arg;    // [S][n_roll_blocks]
  unsigned int* counters;  // [8] arrival counters (self-resetting)
  double* gather1;       // [world][S][2]  (rho_g, argmin_g as double bits)
  double* weights;       // [S][M_local] e_m (unnormalised) -> weights
  int n_w_blocks;
  double* blk_eta;       // [S][n_w_blocks]
  long long* blk_nz;     // [S][n_w_blocks]
  double* gather2;       // [world][S][2]  (eta_g, nonzero_g)
  int* cand;             // [S][M_local] update candidates, compacted per weights-CTA range
  double* cand_e;        // [S][M_local] e_m of each candidate (same positions as cand), or nullptr
  int* cand_cnt;         // [S][n_w_blocks]
  long long* cand_off;   // [S][n_w_blocks + 1] exclusive prefix of cand_cnt
  int n_u_blocks;
  double* blk_part;      // [S][QG][upd_slots][QW][4] per-warp quad sums, by rank among the group's warps
  int upd_slots;         // max warps covering one quad group
  unsigned int* upd_gcnt;  // [S][QG] warps done per quad group (self-resetting)
  double* upd_gsum;      // [S][QG][QW][4] reduced quad-group sums (written by each group's last warp)
  double* gather3;       // [world][S][T*NU]
  // per-rank strides (doubles) of gather1/2/3: separate buffers in the exact
  // three-collective mode; one packed record [g1 | g2 | g3] per rank in the
  // single-collective mode (one ncclAllGather per iteration)
  int g1s, g2s, g3s;
  int comm_single;        // single-collective mode: local baselines + rescaled combine
  int finish_staged;      // finish_solution's states fit the update kernel's shared staging (set at launch)
  // Split small-N rollout (the reference's split strategy, engine.cpp:130-209):
  // the rollout kernel runs only the dynamics chain and stores the outputs
  // (and controls) [S][T][NY|NU][M_local] (sample-minor); a parallel cost
  // kernel evaluates the running costs / importance terms over (sample, t)
  // and sums them in the reference's order. A sample whose fast chain flags
  // is replayed exactly by the rollout kernel (rflag[i] = 1, its J written).
  int split;
  // Injected noise staged by TMA (cp.async.bulk.tensor 2-D, 128 samples x 32
  // floats per box, SWIZZLE_128B) into double-buffered shared memory: the
  // host-side CUtensorMap (launch passes it by value) and whether it is valid
  // (eps rows 16-byte multiples).
  const void* eps_map;
  int eps_tma;
  int tu4;  // T * n_u % 4 == 0: float4 reads of injected eps rows
  float* ytraj;
  float* utraj;
  unsigned char* rflag;
  // results
  ResultHeader* header;
  float* controls;  // [S][T][NU]
  float* states;    // [S][T+1][NX]
  float* outs_nom;  // [S][T][NY]
  int do_finish;    // final iteration of a solve: nominal rollout + solve_count++
  int begin_keys;   // this kernel opens the solve: reset the error / abort keys (no begin_solve launch)
  int normalize_weights;  // write w = e/eta back (only when the caller wants weights)
  double skip_w;          // update skips samples with w_m < skip_w (0 = exact)
  double cem_k;           // CEM: elite count k (commit mean + acc / k); 0 = MPPI / Tube
  // RMPPI (S = 2): the real system's sampled control gets the ancillary
  // feedback u += K (x_real,t - x_nominal,t) of the same sample; candidate
  // nominal states z_i on the segment previous-nominal -> real (x0[0] ->
  // x0[1] on entry) are scored by their mean-trajectory cost.
  int rmppi;
  float fb_gain[kMaxNU * kMaxNX];  // K, row-major [NU][NX]
  int n_cand;
  double cost_threshold;
  double* rm_score;  // [32] candidate scores (warp-cooperative models' select)
  float* rm_z;       // [32][kMaxNX] candidate states
  // Indexed rollout (export_sample_trajectories re-roll): thread i rolls out
  // global sample sample_idx[i] (nullptr: m_begin + i)
  const long long* sample_idx;
  // user-model plugin (smpc_create_with_ops): the smpc_model_ops table and
  // the context's copy of its functor pair, read by the host trampolines
  const void* plugin_ops;
  const void* plugin_user;
  // Small-N mode: the iteration's standard-normal quads pre-generated by
  // gen_zq_kernel, [Q][M_local] float4 (nullptr: regenerate in the rollout)
  const float4* zq;
  DynParams dyn;
  CostParams cost;
};

// One set of launchers per (dynamics kind, libm variant); cost kind and S are
// dispatched inside. Defined in inst_*.cu.
struct ModelOps {
  cudaError_t (*rollout)(const IterArgs&, int cost_kind, cudaStream_t);
  cudaError_t (*rmppi_select)(const IterArgs&, int cost_kind, cudaStream_t);
  cudaError_t (*plant_step)(const IterArgs&, int cost_kind, const PlantStepArgs&, cudaStream_t);
  cudaError_t (*weights)(const IterArgs&, cudaStream_t);
  cudaError_t (*update)(const IterArgs&, cudaStream_t);
  cudaError_t (*combine)(const IterArgs&, cudaStream_t);
  cudaError_t (*generate)(const IterArgs&, float* eps_out, uint8_t* flags_out, cudaStream_t);
  int nx, nu, ny;
};

ModelOps ops_unicycle(bool fma_libm);
ModelOps ops_cartpole(bool fma_libm);
ModelOps ops_diff_drive(bool fma_libm);
ModelOps ops_double_integrator();
ModelOps ops_quadrotor();
ModelOps ops_mlp(bool fma_libm);
ModelOps ops_plugin();  // trampolines into IterArgs::plugin_ops (smpc_capi.cu)
ModelOps ops_bicycle(bool fma_libm);

cudaError_t launch_select(const IterArgs& a, SelectState* st, long long k, unsigned int* counters, int* eq_cnt,
                          long long* eq_off, cudaStream_t stream);
cudaError_t launch_sort_selected(const IterArgs& a, long long k, unsigned long long* keys, long long* idx,
                                 unsigned long long* slot, cudaStream_t stream);
cudaError_t build_tail_table(float* table, uint32_t j_lo, uint32_t j_hi, cudaStream_t stream);
cudaError_t launch_begin_solve(ResultHeader* h, cudaStream_t stream);
cudaError_t launch_shift_mean(float* mean, int S, int T, int NU, long long steps, cudaStream_t stream);
cudaError_t launch_gen_zq(const IterArgs& a, int nu, float4* zq, cudaStream_t stream);
cudaError_t launch_icdf_domain(const IterArgs& a, float* out, cudaStream_t stream);
cudaError_t launch_weights(const IterArgs& a, cudaStream_t stream);
cudaError_t launch_normalize_weights(const IterArgs& a, cudaStream_t stream);
cudaError_t launch_min_only(const double* costs, long long n, double* blk_min, long long* blk_arg,
                            int nblk, unsigned int* counter, double* out_rho, long long* out_arg,
                            cudaStream_t stream);

}  // namespace smpc_dev
