// C-ABI implementation (include/smpc_b200.h): context lifecycle, validation
// with the reference's error texts, device buffers, the captured per-solve
// CUDA graph, the engine/sampler boundary calls and NCCL multi-GPU plumbing.
// Host code only — all arithmetic on the hot path runs in the kernels.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/smpc_b200.h"
#include "launch.h"

using namespace smpc_dev;

extern "C" int32_t smpc_host_libm_uses_fma(void);  // libm_probe.cpp

namespace {

thread_local std::string g_create_error;

// ---- minimal NCCL surface, loaded with dlopen so single-GPU use never needs it
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclChar = 0, ncclUint8 = 1, ncclFloat64 = 8 };
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    for (const char* n : names) {
      api.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (api.handle) {
      api.GetUniqueId = (ncclResult_t(*)(ncclUniqueId*))dlsym(api.handle, "ncclGetUniqueId");
      api.CommInitRank = (ncclResult_t(*)(ncclComm_t*, int, ncclUniqueId, int))dlsym(api.handle, "ncclCommInitRank");
      api.AllGather = (ncclResult_t(*)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t))dlsym(
          api.handle, "ncclAllGather");
      api.CommDestroy = (ncclResult_t(*)(ncclComm_t))dlsym(api.handle, "ncclCommDestroy");
      api.GetErrorString = (const char* (*)(ncclResult_t))dlsym(api.handle, "ncclGetErrorString");
    }
  }
  return api.GetUniqueId ? &api : nullptr;
}

struct ConfigError {
  std::string msg;
};
struct RuntimeError {
  std::string msg;
};
struct CudaError {
  std::string msg;
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) throw CudaError{std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

// Zeroed device buffer. cudaMemset runs on the legacy default stream, which
// does NOT order with the contexts' non-blocking streams, so the fill is
// waited for here (allocation paths are cold): kernels rely on zeroed
// arrival counters and scratch.
template <typename T>
T* dalloc(size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  CK(cudaMalloc(&p, n * sizeof(T)));
  CK(cudaMemset(p, 0, n * sizeof(T)));
  CK(cudaStreamSynchronize(nullptr));
  return static_cast<T*>(p);
}

const char* controller_name(int kind) {
  return kind == SMPC_CTRL_DMD     ? "dmd"
         : kind == SMPC_CTRL_TUBE  ? "tube"
         : kind == SMPC_CTRL_CEM   ? "cem"
         : kind == SMPC_CTRL_RMPPI ? "rmppi"
                                   : "mppi";
}

}  // namespace

struct smpc_ctx {
  smpc_problem p{};
  std::vector<float> std_per_step, step_sizes, fb_gain;
  std::vector<uint8_t> costmap;
  ModelOps ops{};
  int nx = 0, nu = 0, ny = 0, S = 1, T = 0, I = 1;
  long long M = 0, M_local = 0, m_begin = 0;
  bool fma = true;
  cudaStream_t stream = nullptr;
  // device buffers
  float *d_mean = nullptr, *d_x0 = nullptr, *d_sigma = nullptr, *d_tail = nullptr;
  double *d_sig2 = nullptr, *d_gamma = nullptr, *d_costs = nullptr, *d_weights = nullptr;
  double *d_blk_min = nullptr, *d_blk_eta = nullptr, *d_blk_part = nullptr;
  double* d_upd_gsum = nullptr;
  unsigned int* d_upd_gcnt = nullptr;
  double *d_gather1 = nullptr, *d_gather2 = nullptr, *d_gather3 = nullptr;
  int *d_cand = nullptr, *d_cand_cnt = nullptr;
  double* d_cand_e = nullptr;
  unsigned long long tail_tex = 0;
  unsigned long long full_tex = 0;  // per-device full-domain normal_icdf table (shared, never freed)
  int upd_slots = 4;
  long long* d_cand_off = nullptr;
  long long *d_blk_arg = nullptr, *d_blk_nz = nullptr;
  unsigned int* d_counters = nullptr;
  uint8_t* d_costmap = nullptr;
  float* d_dyn_tensor = nullptr;
  float4* d_zq = nullptr;  // small-N mode noise buffer [Q][M_local]
  // split small-N rollout (dynamics chain + parallel exact costs): samples per
  // cost CTA (0 = off), trajectories [S][T][NY|NU][M_local], replay flags
  int split_sb = 0;
  long long blk_cap = 0;  // entries of d_blk_min / d_blk_arg
  float *d_ytraj = nullptr, *d_utraj = nullptr;
  unsigned char* d_rflag = nullptr;
  bool use_zq = false;     // noise strategy: split (d_zq pass) vs fused (in-register)
  smpc_noise_choice noise_choice = {SMPC_NOISE_AUTO, 0.0, 0.0, 0};
  bool noise_resolved = false;  // set by smpc_select_noise_strategy (default: split iff M_local <= 16384)
  // CEM elite selection / sample ordering (select.cu)
  SelectState* d_select = nullptr;
  int* d_eq_cnt = nullptr;
  long long* d_eq_off = nullptr;
  long long cem_k = 0;
  unsigned char* d_result = nullptr;
  unsigned char* h_result = nullptr;  // pinned
  size_t result_bytes = 0, off_controls = 0, off_states = 0, off_outs = 0;
  float* h_x0 = nullptr;  // pinned staging
  // scratch for the engine / sampler boundary
  float *d_ro_x0 = nullptr, *d_ro_mean = nullptr, *d_eps = nullptr, *d_outputs = nullptr;
  size_t eps_cap = 0, outputs_cap = 0;
  double* d_wscratch = nullptr;
  size_t wscratch_cap = 0;
  uint8_t* d_flags = nullptr;
  size_t flags_cap = 0;
  IterArgs base{};
  int n_roll_blocks = 1, n_w_blocks = 1, n_u_blocks = 1;
  // graph
  cudaGraphExec_t graph = nullptr;
  cudaEvent_t ev_stage = nullptr;
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  double rollout_ms_total = 0.0;
  long long rollout_launches = 0;
  // multi-GPU
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  int comm_mode = SMPC_COMM_SINGLE;  // one all-gather per iteration (smpc_comm_set_mode)
  double* d_gather_rec = nullptr;    // [8][rec] packed per-rank records of the single-collective mode
  // injected noise (device [M_local][T][n_u]) for every solve, and the TMA
  // descriptors of it and of the engine-boundary copy d_eps
  const float* d_inj = nullptr;
  smpc_model_ops plugin{};            // user model (smpc_create_with_ops), with its functor pair copied
  std::vector<unsigned char> plugin_user;
  alignas(64) CUtensorMap inj_map;
  alignas(64) CUtensorMap eps_map;
  bool inj_tma = false, eps_tma = false;
  double* d_rm_score = nullptr;      // RMPPI candidate scratch (warp-cooperative models)
  float* d_rm_z = nullptr;
  // host state
  uint64_t solve_count = 0;
  std::string err;
  long long err_sample = -1;
  int err_t = -1, err_ch = -1;
  std::vector<float> nominal_state;
  bool nominal_started = false;
  std::vector<float> host_mean[2];

  ResultHeader* header() { return reinterpret_cast<ResultHeader*>(d_result); }
  ResultHeader* h_header() { return reinterpret_cast<ResultHeader*>(h_result); }
};

namespace {

void set_error(smpc_ctx* c, const std::string& msg) {
  if (c) {
    c->err = msg;
    c->err_sample = -1;
    c->err_t = -1;
    c->err_ch = -1;
  } else {
    g_create_error = msg;
  }
}

template <class F>
smpc_status guarded(smpc_ctx* c, F&& f) {
  try {
    f();
    return SMPC_OK;
  } catch (const ConfigError& e) {
    set_error(c, e.msg);
    return SMPC_ERR_CONFIG;
  } catch (const RuntimeError& e) {
    set_error(c, e.msg);
    return SMPC_ERR_RUNTIME;
  } catch (const CudaError& e) {
    set_error(c, e.msg);
    return SMPC_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(c, e.what());
    return SMPC_ERR_RUNTIME;
  }
}

double pd(const smpc_problem& p, int i, double d) { return i < p.n_dyn_params ? p.dyn_params[i] : d; }
double pc(const smpc_problem& p, int i, double d) { return i < p.n_cost_params ? p.cost_params[i] : d; }

// Validation mirroring the reference constructors' checks and messages:
// Controller ctor (controllers.cpp:23-49), GaussianSampler ctor
// (sampling.cpp:7-30), model ctors (dynamics.cpp:133-171), cost ctors and
// make_cost (costs.cpp:27-162), RolloutEngine::validate (engine.cpp:81-127).
// ---- user-model plugin trampolines (smpc_create_with_ops) --------------------
const smpc_model_ops* plugin_of(const IterArgs& a) { return static_cast<const smpc_model_ops*>(a.plugin_ops); }
cudaError_t plugin_rollout(const IterArgs& a, int, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->rollout(&a, a.plugin_user, st);
}
cudaError_t plugin_rmppi(const IterArgs& a, int, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->rmppi_select(&a, a.plugin_user, st);
}
cudaError_t plugin_plant(const IterArgs& a, int, const PlantStepArgs& p, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->plant_step(&a, a.plugin_user, &p, st);
}
cudaError_t plugin_update(const IterArgs& a, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->update(&a, a.plugin_user, st);
}
cudaError_t plugin_combine(const IterArgs& a, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->combine(&a, a.plugin_user, st);
}
cudaError_t plugin_generate(const IterArgs& a, float* e, uint8_t* f, cudaStream_t st) {
  return (cudaError_t)plugin_of(a)->generate(&a, a.plugin_user, e, f, st);
}

void validate(smpc_ctx* c) {
  const smpc_problem& p = c->p;
  if (p.abi_version != SMPC_B200_ABI_VERSION) throw ConfigError{"smpc_problem: ABI version mismatch"};
  const std::string name = controller_name(p.controller_kind);
  switch (p.dynamics_kind) {
    case SMPC_DYN_UNICYCLE: c->ops = ops_unicycle(c->fma); break;
    case SMPC_DYN_CARTPOLE:
      if (!(pd(p, 0, 1) > 0) || !(pd(p, 1, 1) > 0) || !(pd(p, 2, 1) > 0) ||
          !((float)pd(p, 0, 1) > 0.0f) || !((float)pd(p, 1, 1) > 0.0f) || !((float)pd(p, 2, 1) > 0.0f))
        throw RuntimeError{"cartpole: masses and pole length must be > 0"};
      c->ops = ops_cartpole(c->fma);
      break;
    case SMPC_DYN_DIFF_DRIVE:
      if (!((float)pd(p, 0, 1) > 0.0f) || !((float)pd(p, 1, 1) > 0.0f))
        throw RuntimeError{"diff_drive: wheel geometry must be > 0"};
      if (!((float)pd(p, 2, -0.35) < (float)pd(p, 3, 0.5)))
        throw RuntimeError{"diff_drive: control bound lower must be < upper on channel 0"};
      if (!((float)pd(p, 4, -0.5) < (float)pd(p, 5, 0.5)))
        throw RuntimeError{"diff_drive: control bound lower must be < upper on channel 1"};
      c->ops = ops_diff_drive(c->fma);
      break;
    case SMPC_DYN_DOUBLE_INTEGRATOR: c->ops = ops_double_integrator(); break;
    case SMPC_DYN_QUADROTOR:  // builder-defined (models.cuh:QuadrotorDyn)
      if (!((float)pd(p, 0, 1.0) > 0.0f) || !((float)pd(p, 2, 0.05) > 0.0f))
        throw RuntimeError{"quadrotor: mass and rate time constant must be > 0"};
      if (!((float)pd(p, 3, 39.24) > (float)pd(p, 0, 1.0) * (float)pd(p, 1, 9.81)) || !((float)pd(p, 4, 5.0) > 0.0f))
        throw RuntimeError{"quadrotor: thrust_max must exceed hover thrust and rate_max must be > 0"};
      c->ops = ops_quadrotor();
      break;
    case SMPC_DYN_BICYCLE:  // builder-defined (models.cuh:BicycleDyn)
      if (!((float)pd(p, 0, 0.5) > 0.0f)) throw RuntimeError{"bicycle: wheelbase must be > 0"};
      if (!((float)pd(p, 1, -0.35) < (float)pd(p, 2, 0.5)))
        throw RuntimeError{"bicycle: control bound lower must be < upper on channel 0"};
      if (!((float)pd(p, 3, -0.6) < (float)pd(p, 4, 0.6)))
        throw RuntimeError{"bicycle: control bound lower must be < upper on channel 1"};
      c->ops = ops_bicycle(c->fma);
      break;
    case SMPC_DYN_PLUGIN: {  // user functors (smpc_create_with_ops): launchers from the plugin
      const smpc_model_ops& o = c->plugin;
      if (o.abi_version != SMPC_B200_ABI_VERSION || o.args_bytes != (int32_t)sizeof(IterArgs))
        throw ConfigError{"smpc_model_ops: built against a different library version"};
      if (!o.rollout || !o.update || !o.combine || !o.generate || !o.plant_step)
        throw ConfigError{"smpc_model_ops: missing launcher"};
      if (o.n_x < 1 || o.n_u < 1 || o.n_y < 1) throw ConfigError{"smpc_model_ops: invalid dimensions"};
      c->ops = ModelOps{plugin_rollout, o.rmppi_select ? plugin_rmppi : nullptr, plugin_plant, launch_weights,
                        plugin_update, plugin_combine, plugin_generate, o.n_x, o.n_u, o.n_y};
      break;
    }
    case SMPC_DYN_MLP:  // builder-defined (models.cuh:MlpDyn, tcgen05 rollout in mlp.cu)
      if (!p.dyn_tensor || p.dyn_tensor_len != mlp_layout::TOTAL)
        throw RuntimeError{"mlp: dyn_tensor must hold " + std::to_string(mlp_layout::TOTAL) +
                           " floats (W1 b1 W2 b2 W3 b3, smpc_b200.h)"};
      for (int64_t k = 0; k < p.dyn_tensor_len; ++k)
        if (!std::isfinite(p.dyn_tensor[k])) throw RuntimeError{"mlp: network parameters must be finite"};
      c->ops = ops_mlp(c->fma);
      break;
    default: throw ConfigError{"dynamics.kind is not recognized"};
  }
  c->nx = c->ops.nx, c->nu = c->ops.nu, c->ny = c->ops.ny;
  if (p.controller_kind != SMPC_CTRL_MPPI && p.controller_kind != SMPC_CTRL_DMD &&
      p.controller_kind != SMPC_CTRL_TUBE && p.controller_kind != SMPC_CTRL_CEM && p.controller_kind != SMPC_CTRL_RMPPI)
    throw ConfigError{"controller.kind is not recognized"};
  // cost (make_cost + ctor checks); a plugin's cost functor is its own
  int cost_ny = c->ny, cost_nu = c->nu;
  std::string cost_name;
  switch (p.dynamics_kind == SMPC_DYN_PLUGIN ? -1 : p.cost_kind) {
    case -1: cost_name = "plugin"; break;
    case SMPC_COST_ROAD:
      cost_name = "road";
      if (c->ny < 2) throw RuntimeError{"road cost needs at least 2 output channels"};
      if (p.dynamics_kind == SMPC_DYN_BICYCLE) throw ConfigError{"road cost is not offered for the bicycle model"};
      if (!((float)pc(p, 0, 1.0) > 0.0f)) throw RuntimeError{"road cost: half_width must be > 0"};
      break;
    case SMPC_COST_CIRCLE_TRACK: {
      cost_name = "circle_track";
      const float in = (float)pc(p, 0, 1.875), out = (float)pc(p, 1, 2.125);
      if (!(in > 0.0f) || !(in < out)) throw RuntimeError{"circle_track cost: need 0 < inner_radius < outer_radius"};
      cost_ny = 4, cost_nu = 2;
      break;
    }
    case SMPC_COST_DIFF_DRIVE_NAV:
      cost_name = "diff_drive_nav";
      cost_ny = 3, cost_nu = 2;
      if (!(p.costmap_resolution > 0.0)) throw RuntimeError{"costmap: resolution must be > 0"};
      if (p.costmap_cells_x < 1 || p.costmap_cells_y < 1) throw RuntimeError{"costmap: dimensions give an empty grid"};
      break;
    case SMPC_COST_QUADRATIC:
      cost_name = "quadratic";
      if (p.n_quad < 1 || p.n_quad > SMPC_MAX_DIM)
        throw RuntimeError{"quadratic cost: target and weights must be non-empty and equal length"};
      for (int i = 0; i < p.n_quad; ++i)
        if (!(p.quad_weights[i] >= 0.0f)) throw RuntimeError{"quadratic cost: weights must be >= 0"};
      cost_ny = p.n_quad;
      break;
    default: throw ConfigError{"cost.kind is not recognized"};
  }
  static const char* dyn_names[] = {"unicycle", "cartpole", "diff_drive", "double_integrator", "quadrotor", "mlp",
                                    "bicycle"};
  const char* dyn_name = p.dynamics_kind == SMPC_DYN_PLUGIN ? (c->plugin.name ? c->plugin.name : "plugin")
                                                             : dyn_names[p.dynamics_kind];
  if (cost_ny != c->ny)
    throw ConfigError{"cost '" + cost_name + "' expects " + std::to_string(cost_ny) +
                      " output channels but model '" + dyn_name + "' produces " +
                      std::to_string(c->ny)};
  if (cost_nu != c->nu) throw RuntimeError{"rollout request cost dimensions do not match the model"};
  // sampler
  if (p.n_control_std == 1 && c->nu > 1) {
  } else if (p.n_control_std != c->nu) {
    throw RuntimeError{"sampler: std_dev needs one entry per control channel"};
  }
  for (int i = 0; i < p.n_control_std; ++i)
    if (!(p.control_std[i] > 0.0f)) throw RuntimeError{"sampler: std_dev entries must be > 0"};
  if (p.std_per_step) {
    for (int i = 0; i < p.horizon * c->nu; ++i)
      if (!(p.std_per_step[i] > 0.0f)) throw RuntimeError{"sampler: std_per_step entries must be > 0"};
  }
  if (!(p.zero_mean_fraction >= 0.0 && p.zero_mean_fraction <= 1.0))
    throw RuntimeError{"sampler: zero_mean_fraction must be in [0, 1]"};
  // controller
  if (p.num_samples < 1) throw RuntimeError{name + ": num_samples must be >= 1"};
  if (p.iterations < 1 || p.iterations > 256) throw RuntimeError{name + ": iterations must be in [1, 256]"};
  if (!(p.lambda > 0.0)) throw RuntimeError{name + ": lambda must be > 0"};
  if (!(p.dt > 0.0)) throw RuntimeError{name + ": dt must be > 0"};
  if (p.horizon < 1) throw RuntimeError{name + ": horizon must be >= 1"};
  if (!(p.n_step_sizes == 0 || p.n_step_sizes == 1 || p.n_step_sizes == p.horizon))
    throw RuntimeError{name + ": step_sizes must be empty, scalar, or one per timestep"};
  for (int i = 0; i < p.n_step_sizes; ++i)
    if (!(p.step_sizes[i] > 0.0f && p.step_sizes[i] <= 1.0f))
      throw RuntimeError{name + ": step sizes must be in (0, 1]"};
  if (p.controller_kind == SMPC_CTRL_TUBE && !(p.nominal_reset_bound > 0.0))
    throw RuntimeError{"tube: nominal_reset_bound must be > 0"};
  if (p.controller_kind == SMPC_CTRL_RMPPI) {
    if (!c->ops.rmppi_select) throw ConfigError{"rmppi: not supported for this dynamics model"};
    if (p.num_candidates < 2 || p.num_candidates > 32) throw RuntimeError{"rmppi: num_candidates must be in [2, 32]"};
    if (p.cost_threshold != p.cost_threshold) throw RuntimeError{"rmppi: cost_threshold must not be NaN"};
    if (p.feedback_gain)
      for (int k = 0; k < c->nu * c->nx; ++k)
        if (!std::isfinite(p.feedback_gain[k])) throw RuntimeError{"rmppi: feedback gains must be finite"};
  }
  if (p.controller_kind == SMPC_CTRL_CEM && !(p.elite_fraction > 0.0 && p.elite_fraction <= 1.0))
    throw RuntimeError{"cem: elite_fraction must be in (0, 1]"};  // controllers.cpp:145-147
  if (!(p.update_skip_mass >= 0.0 && p.update_skip_mass < 1e-6))
    throw RuntimeError{name + ": update_skip_mass must be in [0, 1e-6)"};
  if (p.horizon > (1 << 22)) throw RuntimeError{name + ": horizon too large"};
  if (c->nx > kMaxNX || c->nu > kMaxNU || c->ny > kMaxNY) throw RuntimeError{"ModelDims: dimension exceeds capacity"};
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint32_t tail_table_size(uint32_t* j_lo_out, uint32_t* j_hi_out);

int gather_record(const smpc_ctx* c) { return 4 * c->S + c->S * c->T * c->nu; }



// TMA descriptor of an injected-noise tensor [rows][T*n_u] fp32 (reference
// layout, sampling.hpp:40-42): boxes of 32 floats x 128 rows, SWIZZLE_128B
// (the rollout kernel's tma_src). false when the rows are not 16-byte
// multiples or the driver entry point is unavailable (checked per-step path).
bool encode_eps_map(CUtensorMap* map, const float* d, long long rows, int tu) {
  if (tu % 4 != 0 || rows < 1) return false;
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      encode = (EncodeFn)fn;
  }
  if (!encode) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)tu, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)tu * sizeof(float)};
  const cuuint32_t box[2] = {32, (cuuint32_t)kRolloutThreads};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(d), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// normal_icdf over the sampler's whole 2^23-point domain, one 32 MB table per
// device shared by every context (it depends on nothing but the arithmetic),
// built by the same icdf_quad_words path the kernels evaluate in registers.
struct FullIcdfTable {
  float* d = nullptr;
  unsigned long long tex = 0;
};
std::mutex g_full_mu;
FullIcdfTable g_full[64];

unsigned long long full_icdf_table(const IterArgs& base, int device, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_full_mu);
  FullIcdfTable& t = g_full[device & 63];
  if (!t.tex) {
    float* d = nullptr;
    CK(cudaMalloc(&d, sizeof(float) << 23));
    CK(launch_icdf_domain(base, d, st));
    CK(cudaStreamSynchronize(st));
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = d;
    rd.res.linear.desc = cudaCreateChannelDesc<float>();
    rd.res.linear.sizeInBytes = sizeof(float) << 23;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
    t.d = d;
    t.tex = (unsigned long long)tex;
  }
  return t.tex;
}

void fill_args(smpc_ctx* c) {
  IterArgs& a = c->base;
  const smpc_problem& p = c->p;
  a.T = c->T;
  a.S = c->S;
  a.M_local = (int)c->M_local;
  a.m_begin = c->m_begin;
  a.M_global = c->M;
  a.dt = (float)p.dt;  // engine.cpp:136, :216
  a.lambda = p.lambda;
  a.inv_lambda_pow2 = exact_inverse_pow2(p.lambda);
  a.key0 = (uint32_t)p.seed;
  a.key1 = (uint32_t)(p.seed >> 32);
  for (int r = 0; r < 10; ++r) {  // Philox round keys (rng.hpp:24-25)
    a.rk.k0[r] = a.key0 + (uint32_t)r * 0x9E3779B9u;
    a.rk.k1[r] = a.key1 + (uint32_t)r * 0xBB67AE85u;
  }
  a.pk.one = 0x3f8000003f800000ull;    // {1.0f, 1.0f}
  a.pk.mzero = 0x8000000080000000ull;  // {-0.0f, -0.0f}
  {
    uint32_t j_lo, j_hi;
    tail_table_size(&j_lo, &j_hi);
    a.tail_off = ((1u << 23) - j_hi) << 9;           // rotates the upper tail to index 0
    a.tail_lim = (((1u << 23) - j_hi) + j_lo) << 9;  // upper + lower tail entries
  }
  a.with_mean = p.include_mean_sample != 0;
  // zero-mean quota filled from the tail (sampling.cpp:56-62)
  long long n_zero = (long long)ceil(p.zero_mean_fraction * (double)c->M);
  n_zero = std::min(n_zero, a.with_mean ? c->M - 1 : c->M);
  a.zero_begin = c->M - n_zero;
  // CEM ranks raw rollout costs: no importance adjustment (controllers.cpp:155-162).
  a.importance = p.importance_sampling != 0 && p.controller_kind != SMPC_CTRL_CEM;
  a.cem_k = p.controller_kind == SMPC_CTRL_CEM ? (double)c->cem_k : 0.0;
  a.rmppi = p.controller_kind == SMPC_CTRL_RMPPI;
  for (int k = 0; k < kMaxNU * kMaxNX; ++k) a.fb_gain[k] = 0.0f;
  for (size_t k = 0; k < c->fb_gain.size(); ++k) a.fb_gain[k] = c->fb_gain[k];
  a.n_cand = p.num_candidates;
  a.cost_threshold = p.cost_threshold;
  a.rm_score = c->d_rm_score;
  a.rm_z = c->d_rm_z;
  a.plugin_ops = p.dynamics_kind == SMPC_DYN_PLUGIN ? &c->plugin : nullptr;
  a.plugin_user = c->plugin_user.empty() ? nullptr : c->plugin_user.data();
  a.split = 0;  // enabled per launch with the split-noise buffer (enqueue_solve)
  a.eps_map = nullptr;
  a.eps_tma = 0;
  a.tu4 = (c->T * c->nu) % 4 == 0;
  a.ytraj = c->d_ytraj;
  a.utraj = c->d_utraj;
  a.rflag = c->d_rflag;
  a.world = c->world;
  a.rank = c->rank;
  a.solve_count = &c->header()->solve_count;
  a.iter = 0;
  a.stream = 0;
  a.mean_in = c->d_mean;
  a.mean_out = c->d_mean;
  a.x0 = c->d_x0;
  a.sigma = c->d_sigma;
  a.sig2 = c->d_sig2;
  a.gamma = c->d_gamma;
  a.eps_in = nullptr;
  a.sample_idx = nullptr;
  a.zq = nullptr;
  a.tail = c->d_tail;
  a.tail_tex = c->tail_tex;
  a.full_tex = c->full_tex;
  a.costs = c->d_costs;
  a.outputs = nullptr;
  a.n_roll_blocks = c->n_roll_blocks;
  a.blk_min = c->d_blk_min;
  a.blk_arg = c->d_blk_arg;
  a.counters = c->d_counters;
  a.gather1 = c->d_gather1;
  a.weights = c->d_weights;
  a.n_w_blocks = c->n_w_blocks;
  a.blk_eta = c->d_blk_eta;
  a.blk_nz = c->d_blk_nz;
  a.gather2 = c->d_gather2;
  a.cand = c->d_cand;
  a.cand_e = c->d_cand_e;
  a.upd_slots = c->upd_slots;
  a.cand_cnt = c->d_cand_cnt;
  a.cand_off = c->d_cand_off;
  a.n_u_blocks = c->n_u_blocks;
  a.blk_part = c->d_blk_part;
  a.upd_gsum = c->d_upd_gsum;
  a.upd_gcnt = c->d_upd_gcnt;
  a.gather3 = c->d_gather3;
  a.comm_single = c->comm_mode == SMPC_COMM_SINGLE;
  if (a.comm_single) {  // one record per rank: [S][2] (rho, argmin) | [S][2] (eta, nz) | [S][T*NU] sums
    const int rec = gather_record(c);
    a.gather1 = c->d_gather_rec;
    a.gather2 = c->d_gather_rec + 2 * c->S;
    a.gather3 = c->d_gather_rec + 4 * c->S;
    a.g1s = a.g2s = a.g3s = rec;
  } else {
    a.g1s = 2 * c->S;
    a.g2s = 2 * c->S;
    a.g3s = c->S * c->T * c->nu;
  }
  a.header = c->header();
  a.controls = reinterpret_cast<float*>(c->d_result + c->off_controls);
  a.states = reinterpret_cast<float*>(c->d_result + c->off_states);
  a.outs_nom = reinterpret_cast<float*>(c->d_result + c->off_outs);
  a.do_finish = 0;
  a.normalize_weights = 0;
  a.skip_w = p.update_skip_mass > 0.0 ? p.update_skip_mass / (double)c->M : 0.0;
  for (int i = 0; i < 8; ++i) a.dyn.p[i] = 0.f;
  switch (p.dynamics_kind) {
    case SMPC_DYN_CARTPOLE:
      a.dyn.p[0] = (float)pd(p, 0, 1.0), a.dyn.p[1] = (float)pd(p, 1, 1.0);
      a.dyn.p[2] = (float)pd(p, 2, 1.0), a.dyn.p[3] = (float)pd(p, 3, 9.81);
      break;
    case SMPC_DYN_DIFF_DRIVE: {
      const double d[6] = {1.0, 1.0, -0.35, 0.5, -0.5, 0.5};
      for (int i = 0; i < 6; ++i) a.dyn.p[i] = (float)pd(p, i, d[i]);
      break;
    }
    case SMPC_DYN_BICYCLE: {
      const double d[5] = {0.5, -0.35, 0.5, -0.6, 0.6};
      for (int i = 0; i < 5; ++i) a.dyn.p[i] = (float)pd(p, i, d[i]);
      break;
    }
    case SMPC_DYN_QUADROTOR: {
      const double d[5] = {1.0, 9.81, 0.05, 39.24, 5.0};
      for (int i = 0; i < 5; ++i) a.dyn.p[i] = (float)pd(p, i, d[i]);
      break;
    }
    default: break;
  }
  a.dyn.tensor = c->d_dyn_tensor;
  CostParams& cp = a.cost;
  memset(&cp, 0, sizeof(cp));
  switch (p.cost_kind) {
    case SMPC_COST_ROAD: {
      const double d[3] = {1.0, 1.0, 10.0};
      for (int i = 0; i < 3; ++i) cp.p[i] = (float)pc(p, i, d[i]);
      break;
    }
    case SMPC_COST_CIRCLE_TRACK: {
      const double d[7] = {1.875, 2.125, 1000.0, 2.0, 2.0, 4.0, 2.0};
      for (int i = 0; i < 7; ++i) cp.p[i] = (float)pc(p, i, d[i]);
      break;
    }
    case SMPC_COST_DIFF_DRIVE_NAV: {
      if (p.dynamics_kind == SMPC_DYN_PLUGIN) break;
      const double d[6] = {2.0, 2.0, 0.0, 5.0, 5.0, 20.0};
      for (int i = 0; i < 6; ++i) cp.p[i] = (float)pc(p, i, d[i]);
      cp.grid = c->d_costmap;
      cp.cells_x = p.costmap_cells_x;
      cp.cells_y = p.costmap_cells_y;
      cp.origin_x = (float)p.costmap_origin_x;
      cp.origin_y = (float)p.costmap_origin_y;
      cp.inv_resolution = (float)(1.0 / p.costmap_resolution);  // costmap.cpp:21
      cp.map_in_smem = (size_t)cp.cells_x * cp.cells_y <= 96 * 1024;
      break;
    }
    case SMPC_COST_QUADRATIC:
      cp.n_quad = p.n_quad;
      for (int i = 0; i < p.n_quad; ++i) cp.target[i] = p.quad_target[i], cp.weights[i] = p.quad_weights[i];
      break;
  }
  if (p.dynamics_kind == SMPC_DYN_PLUGIN && c->d_costmap) {  // a plugin cost with USES_MAP reads the problem's map
    cp.grid = c->d_costmap;
    cp.cells_x = p.costmap_cells_x;
    cp.cells_y = p.costmap_cells_y;
    cp.origin_x = (float)p.costmap_origin_x;
    cp.origin_y = (float)p.costmap_origin_y;
    cp.inv_resolution = (float)(1.0 / p.costmap_resolution);
    cp.map_in_smem = (size_t)cp.cells_x * cp.cells_y <= 96 * 1024;
  }
}

// Number of entries of the Phi^-1 tail table (see philox_normal.cuh), and the
// integer thresholds: j is a lower tail iff j < *j_lo_out, upper iff j >= *j_hi_out.
uint32_t tail_table_size(uint32_t* j_lo_out, uint32_t* j_hi_out) {
  static uint32_t cached_lo = 0, cached_hi = 0, cached_n = 0;
  if (cached_n) {
    if (j_lo_out) *j_lo_out = cached_lo;
    if (j_hi_out) *j_hi_out = cached_hi;
    return cached_n;
  }
  const float kLow = 0.02425f;
  const volatile float one = 1.0f;
  const float kHigh = one - kLow;
  uint32_t j_lo = 0, j_hi = 1u << 23;
  for (uint32_t j = 0; j < (1u << 23); ++j) {
    const float pj = (float)j * 0x1.0p-23f + 0x1.0p-24f;
    if (pj < kLow) j_lo = j + 1;
    if (pj > kHigh && j < j_hi) j_hi = j;
  }
  cached_lo = j_lo;
  cached_hi = j_hi;
  cached_n = std::max(j_lo, (1u << 23) - j_hi);
  if (j_lo_out) *j_lo_out = j_lo;
  if (j_hi_out) *j_hi_out = j_hi;
  return cached_n;
}

void decode_error(smpc_ctx* c, unsigned long long key) {
  const unsigned stage = (unsigned)(key >> 62);
  const long long m = (long long)((key >> 30) & 0x7fffffffULL);
  const int t = (int)((key >> 6) & 0xffffff);
  const unsigned phase = (unsigned)((key >> 4) & 3);
  const int ch = (int)(key & 15);
  char buf[256];
  if (stage == 0 && phase == 0) {
    snprintf(buf, sizeof buf, "rollout produced non-finite state channel %d at sample %lld timestep %d", ch, m, t);
  } else if (stage == 0) {
    snprintf(buf, sizeof buf, "rollout produced invalid running cost at sample %lld timestep %d", m, t);
  } else if (stage == 1) {
    snprintf(buf, sizeof buf, "compute_weights: non-finite cost at sample %lld", m);
  } else if (stage == 3) {  // closed-loop applied cost (CostFunction::running_cost, costs.cpp:12-14)
    static const char* cost_names[] = {"road", "circle_track", "diff_drive_nav", "quadratic"};
    const int ck = c->p.cost_kind;
    snprintf(buf, sizeof buf, "%s: running cost must be finite and >= 0", ck >= 0 && ck < 4 ? cost_names[ck] : "cost");
  } else if (phase == 1) {
    snprintf(buf, sizeof buf, "control vector has non-finite entry at channel %d", ch);
  } else {
    snprintf(buf, sizeof buf, "state vector has non-finite entry at channel %d", ch);
  }
  c->err = buf;
  c->err_sample = stage <= 1 ? m : -1;
  c->err_t = stage == 0 || stage == 3 ? t : -1;
  c->err_ch = (stage == 0 && phase == 0) || stage == 2 ? ch : -1;
}

// One solve's device work on c->stream (graph-captured or direct).
void enqueue_solve(smpc_ctx* c, bool timed) {
  // small-N mode: the first gen_zq resets the error keys itself
  const bool zq_opens = c->use_zq && !c->d_inj && c->p.controller_kind != SMPC_CTRL_RMPPI;
  if (!zq_opens) CK(launch_begin_solve(c->header(), c->stream));
  if (c->p.controller_kind == SMPC_CTRL_RMPPI) {  // nominal-state choice, once per solve
    IterArgs a = c->base;
    CK(c->ops.rmppi_select(a, c->p.cost_kind, c->stream));
  }
  for (int it = 0; it < c->I; ++it) {
    IterArgs a = c->base;
    a.iter = it;
    a.do_finish = it == c->I - 1;
    if (timed) CK(cudaEventRecord(c->ev[2 * it], c->stream));
    if (c->d_inj) {  // injected noise (smpc_set_injected_noise): rollout and update read it
      a.eps_in = c->d_inj;
      a.eps_tma = c->inj_tma;
      a.eps_map = &c->inj_map;
    } else if (c->use_zq) {  // split noise: one parallel pass, off the per-sample serial chain
      a.zq = c->d_zq;
      a.split = c->d_ytraj ? c->split_sb : 0;  // and the split dynamics / cost rollout
      IterArgs g = a;
      g.begin_keys = zq_opens && it == 0;
      CK(launch_gen_zq(g, c->nu, c->d_zq, c->stream));
    }
    CK(c->ops.rollout(a, c->p.cost_kind, c->stream));
    if (timed) CK(cudaEventRecord(c->ev[2 * it + 1], c->stream));
    if (c->p.controller_kind == SMPC_CTRL_CEM) {  // elite selection replaces compute_weights
      CK(launch_select(a, c->d_select, c->cem_k, c->d_counters + 8, c->d_eq_cnt, c->d_eq_off, c->stream));
      CK(c->ops.update(a, c->stream));
      continue;
    }
    const bool single = c->comm_mode == SMPC_COMM_SINGLE;
    if (c->world > 1 && !single) {
      const size_t n1 = (size_t)c->S * 2;
      if (nccl()->AllGather(c->d_gather1 + c->rank * n1, c->d_gather1, n1, ncclFloat64, c->comm, c->stream))
        throw CudaError{"ncclAllGather (rho) failed"};
    }
    CK(c->ops.weights(a, c->stream));
    if (c->world > 1 && !single) {
      const size_t n2 = (size_t)c->S * 2;
      if (nccl()->AllGather(c->d_gather2 + c->rank * n2, c->d_gather2, n2, ncclFloat64, c->comm, c->stream))
        throw CudaError{"ncclAllGather (eta) failed"};
    }
    CK(c->ops.update(a, c->stream));
    if (c->world > 1) {
      if (single) {  // (rho_g, argmin_g, eta_g, nz_g, S_g) of every rank in one collective
        const size_t n = (size_t)gather_record(c);
        if (nccl()->AllGather(c->d_gather_rec + c->rank * n, c->d_gather_rec, n, ncclFloat64, c->comm, c->stream))
          throw CudaError{"ncclAllGather (iteration record) failed"};
      } else {
        const size_t n3 = (size_t)c->S * c->T * c->nu;
        if (nccl()->AllGather(c->d_gather3 + c->rank * n3, c->d_gather3, n3, ncclFloat64, c->comm, c->stream))
          throw CudaError{"ncclAllGather (weighted sums) failed"};
      }
      CK(c->ops.combine(a, c->stream));
    }
  }
}

// ---- in-process shard group (one host thread, any devices) ------------------
// The same kernels and the same rank-indexed gather buffers as the NCCL path;
// each all-gather is done as device-to-device copies of every rank's slot into
// every rank's buffer, ordered with events. Used to run (and test) the
// world > 1 combine logic on a single GPU.
void group_allgather(smpc_ctx** cs, int n, int which) {
  for (int r = 0; r < n; ++r) CK(cudaEventRecord(cs[r]->ev_stage, cs[r]->stream));
  for (int d = 0; d < n; ++d) {
    smpc_ctx* dst = cs[d];
    for (int r = 0; r < n; ++r) {
      smpc_ctx* src = cs[r];
      if (r == d) continue;
      CK(cudaStreamWaitEvent(dst->stream, src->ev_stage, 0));
      size_t slot;
      double *from, *to;
      if (which == 0) {  // single-collective record
        slot = (size_t)gather_record(src);
        from = src->d_gather_rec, to = dst->d_gather_rec;
      } else if (which == 1) {
        slot = (size_t)src->S * 2;
        from = src->d_gather1, to = dst->d_gather1;
      } else if (which == 2) {
        slot = (size_t)src->S * 2;
        from = src->d_gather2, to = dst->d_gather2;
      } else {
        slot = (size_t)src->S * src->T * src->nu;
        from = src->d_gather3, to = dst->d_gather3;
      }
      CK(cudaMemcpyAsync(to + r * slot, from + r * slot, slot * sizeof(double), cudaMemcpyDefault, dst->stream));
    }
  }
}

void enqueue_group_solve(smpc_ctx** cs, int n) {
  for (int r = 0; r < n; ++r) CK(launch_begin_solve(cs[r]->header(), cs[r]->stream));
  const int I = cs[0]->I;
  for (int it = 0; it < I; ++it) {
    auto args = [&](smpc_ctx* c) {
      IterArgs a = c->base;
      a.iter = it;
      a.do_finish = it == I - 1;
      return a;
    };
    const bool single = cs[0]->comm_mode == SMPC_COMM_SINGLE;
    for (int r = 0; r < n; ++r) CK(cs[r]->ops.rollout(args(cs[r]), cs[r]->p.cost_kind, cs[r]->stream));
    if (!single) group_allgather(cs, n, 1);
    for (int r = 0; r < n; ++r) CK(cs[r]->ops.weights(args(cs[r]), cs[r]->stream));
    if (!single) group_allgather(cs, n, 2);
    for (int r = 0; r < n; ++r) CK(cs[r]->ops.update(args(cs[r]), cs[r]->stream));
    group_allgather(cs, n, single ? 0 : 3);
    for (int r = 0; r < n; ++r) CK(cs[r]->ops.combine(args(cs[r]), cs[r]->stream));
  }
}

void build_graph(smpc_ctx* c) {
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_solve(c, false);
  } catch (...) {
    cudaStreamEndCapture(c->stream, &g);
    throw;
  }
  CK(cudaStreamEndCapture(c->stream, &g));
  CK(cudaGraphInstantiate(&c->graph, g, 0));
  cudaGraphDestroy(g);
}

// Buffers of the split small-N rollout (when the model runs on the SIMT rollout).
void alloc_split(smpc_ctx* c, bool refill) {
  if (c->d_ytraj || c->p.dynamics_kind == SMPC_DYN_MLP) return;
  // A/B knob (default off: measured slower than the fused chain, whose cost
  // work the scheduler already overlaps with the dynamics chain)
  const char* e = getenv("SMPC_SPLIT");
  if (!e || atoi(e) == 0) return;
  c->d_ytraj = dalloc<float>((size_t)c->S * c->T * c->ny * c->M_local);
  c->d_utraj = dalloc<float>((size_t)c->S * c->T * c->nu * c->M_local);
  c->d_rflag = dalloc<unsigned char>((size_t)c->M_local);
  c->split_sb = split_samples_per_cta(c->T, c->nu, true);
  // the cost kernel publishes one block minimum per SB samples
  const long long need = (long long)c->S * ((c->M_local + c->split_sb - 1) / c->split_sb);
  if (need > c->blk_cap) {
    if (c->d_blk_min) cudaFree(c->d_blk_min);
    if (c->d_blk_arg) cudaFree(c->d_blk_arg);
    c->d_blk_min = dalloc<double>((size_t)need);
    c->d_blk_arg = dalloc<long long>((size_t)need);
    c->blk_cap = need;
  }
  if (refill) fill_args(c);
}

void set_noise(smpc_ctx* c, bool split) {
  if (split) alloc_split(c, true);
  if (split && !c->d_zq) c->d_zq = dalloc<float4>((size_t)((c->T * c->nu + 3) / 4) * c->M_local);
  if (c->use_zq != split) {
    c->use_zq = split;
    if (c->graph) {
      cudaGraphExecDestroy(c->graph);
      c->graph = nullptr;
    }
  }
}

// One iteration (noise, rollout, weights / elite selection, weighted
// update) of the current means from d_x0, with the update committed into a
// scratch mean: the controller state is untouched. Unlike the reference's
// CPU strategies, the device ones also differ in the update (split reads the
// materialised normals back), so the whole iteration is what is timed.
double time_iteration_median(smpc_ctx* c, bool split, int n) {
  IterArgs a = c->base;
  a.do_finish = 0;
  a.iter = 0;
  if (split) {
    a.zq = c->d_zq;
    a.split = c->d_ytraj ? c->split_sb : 0;
  }
  float* scratch = nullptr;
  CK(cudaMalloc(&scratch, sizeof(float) * (size_t)c->S * c->T * c->nu));
  a.mean_out = scratch;
  auto once = [&] {
    CK(launch_begin_solve(c->header(), c->stream));
    if (split) CK(launch_gen_zq(a, c->nu, c->d_zq, c->stream));
    CK(c->ops.rollout(a, c->p.cost_kind, c->stream));
    if (c->world > 1) return;  // the rest needs the collectives: rollout only
    if (c->p.controller_kind == SMPC_CTRL_CEM) {
      CK(launch_select(a, c->d_select, c->cem_k, c->d_counters + 8, c->d_eq_cnt, c->d_eq_off, c->stream));
    } else {
      CK(c->ops.weights(a, c->stream));
    }
    CK(c->ops.update(a, c->stream));
  };
  std::vector<double> t;
  try {
    for (int i = 0; i < 2; ++i) once();
    for (int i = 0; i < n; ++i) {
      CK(cudaEventRecord(c->ev[0], c->stream));
      once();
      CK(cudaEventRecord(c->ev[1], c->stream));
      CK(cudaEventSynchronize(c->ev[1]));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]));
      t.push_back(ms);
    }
  } catch (...) {
    cudaStreamSynchronize(c->stream);
    cudaFree(scratch);
    throw;
  }
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(scratch);
  std::sort(t.begin(), t.end());
  return t.size() % 2 ? t[t.size() / 2] : 0.5 * (t[t.size() / 2 - 1] + t[t.size() / 2]);
}

// The AUTO selection from the states already in d_x0.
smpc_noise_choice auto_select_noise(smpc_ctx* c, int32_t trials, double split_budget_bytes) {
  smpc_noise_choice ch = {SMPC_NOISE_AUTO, 0.0, 0.0, 0};
  const double split_bytes = 16.0 * (double)((c->T * c->nu + 3) / 4) * (double)c->M_local;
  if (split_bytes > split_budget_bytes) {
    ch.kind = SMPC_NOISE_FUSED;
  } else {
    const int n = std::max(3, trials > 0 ? trials : 5);
    set_noise(c, true);
    ch.split_median_ms = time_iteration_median(c, true, n);
    ch.fused_median_ms = time_iteration_median(c, false, n);
    ch.timed = 1;
    ch.kind = smpc_noise_strategy_rule(split_bytes, split_budget_bytes, ch.split_median_ms, ch.fused_median_ms);
  }
  set_noise(c, ch.kind == SMPC_NOISE_SPLIT);
  c->noise_choice = ch;
  c->noise_resolved = true;
  return ch;
}

void launch_solve(smpc_ctx* c) {
  if (c->timing) {
    enqueue_solve(c, true);
  } else {
    if (!c->graph) build_graph(c);
    CK(cudaGraphLaunch(c->graph, c->stream));
  }
}

void collect_timing(smpc_ctx* c) {
  if (!c->timing) return;
  for (int it = 0; it < c->I; ++it) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev[2 * it], c->ev[2 * it + 1]));
    c->rollout_ms_total += ms;
    c->rollout_launches += 1;
  }
}

// Copies the result region back and checks the error key.
void fetch_results(smpc_ctx* c) {
  CK(cudaMemcpyAsync(c->h_result, c->d_result, c->result_bytes, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  collect_timing(c);
  const ResultHeader* h = c->h_header();
  if (h->err_key != kNoError) {
    decode_error(c, h->err_key);
    throw RuntimeError{c->err};
  }
  c->solve_count = h->solve_count;
}

void upload_x0(smpc_ctx* c, const float* x0, int S) {
  memcpy(c->h_x0, x0, sizeof(float) * S * c->nx);
  CK(cudaMemcpyAsync(c->d_x0, c->h_x0, sizeof(float) * S * c->nx, cudaMemcpyHostToDevice, c->stream));
}

void copy_solution(smpc_ctx* c, int s, smpc_solution* out) {
  const ResultHeader* h = c->h_header();
  const float* controls = reinterpret_cast<const float*>(c->h_result + c->off_controls);
  const float* states = reinterpret_cast<const float*>(c->h_result + c->off_states);
  const float* outs = reinterpret_cast<const float*>(c->h_result + c->off_outs);
  const size_t TU = (size_t)c->T * c->nu;
  if (out->controls) memcpy(out->controls, controls + s * TU, sizeof(float) * TU);
  if (out->states) memcpy(out->states, states + (size_t)s * (c->T + 1) * c->nx, sizeof(float) * (c->T + 1) * c->nx);
  if (out->outputs) memcpy(out->outputs, outs + (size_t)s * c->T * c->ny, sizeof(float) * c->T * c->ny);
  out->summary.baseline = h->rho[s];
  out->summary.normalizer = h->eta[s];
  out->summary.argmin = h->argmin[s];
  out->summary.nonzero = h->nonzero[s];
}

void fetch_weights(smpc_ctx* c, int s, double* dst) {
  IterArgs a = c->base;
  CK(launch_normalize_weights(a, c->stream));
  CK(cudaMemcpyAsync(dst, c->d_weights + (size_t)s * c->M_local, sizeof(double) * c->M_local,
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

// ============================================================================
extern "C" {

const char* smpc_version(void) { return "paper_2409_07563_b200 0.1 (sm_100a)"; }

static smpc_status create_impl(const smpc_problem* problem, const smpc_model_ops* ops, smpc_ctx** out);

smpc_status smpc_create(const smpc_problem* problem, smpc_ctx** out) { return create_impl(problem, nullptr, out); }

smpc_status smpc_create_with_ops(const smpc_problem* problem, const smpc_model_ops* ops, smpc_ctx** out) {
  if (!ops) return SMPC_ERR_ARGUMENT;
  return create_impl(problem, ops, out);
}

static smpc_status create_impl(const smpc_problem* problem, const smpc_model_ops* ops, smpc_ctx** out) {
  if (!problem || !out) return SMPC_ERR_ARGUMENT;
  *out = nullptr;
  smpc_ctx* c = new smpc_ctx();
  c->p = *problem;
  if (ops) {
    c->plugin = *ops;
    if (ops->user && ops->user_bytes > 0)
      c->plugin_user.assign((const unsigned char*)ops->user, (const unsigned char*)ops->user + ops->user_bytes);
    c->plugin.user = c->plugin_user.empty() ? nullptr : c->plugin_user.data();
    c->p.dynamics_kind = SMPC_DYN_PLUGIN;
  } else if (problem->dynamics_kind == SMPC_DYN_PLUGIN) {
    g_create_error = "dynamics.kind plugin needs smpc_create_with_ops";
    delete c;
    return SMPC_ERR_CONFIG;
  }
  c->fma = smpc_host_libm_uses_fma() != 0;
  const smpc_status st = guarded(nullptr, [&] {
    validate(c);
    smpc_problem& p = c->p;
    c->T = p.horizon;
    c->I = p.iterations;
    c->M = p.num_samples;
    c->S = (p.controller_kind == SMPC_CTRL_TUBE || p.controller_kind == SMPC_CTRL_RMPPI) ? 2 : 1;
    if (p.feedback_gain) c->fb_gain.assign(p.feedback_gain, p.feedback_gain + (size_t)c->nu * c->nx);
    p.feedback_gain = nullptr;
    // k = max(1, (int)ceil(elite_fraction * M)) (controllers.cpp:164)
    c->cem_k = std::max(1, (int)std::ceil(p.elite_fraction * (double)p.num_samples));
    c->m_begin = 0;
    long long m_end = c->M;
    if (p.shard_end > 0) {
      if (p.shard_begin < 0 || p.shard_end > c->M || p.shard_begin >= p.shard_end)
        throw ConfigError{"smpc_problem: invalid shard range"};
      c->m_begin = p.shard_begin;
      m_end = p.shard_end;
    }
    c->M_local = m_end - c->m_begin;
    const int TU = c->T * c->nu;
    // own copies of borrowed arrays
    if (p.std_per_step) c->std_per_step.assign(p.std_per_step, p.std_per_step + TU);
    if (p.n_step_sizes > 0) c->step_sizes.assign(p.step_sizes, p.step_sizes + p.n_step_sizes);
    if (p.costmap) c->costmap.assign(p.costmap, p.costmap + (size_t)p.costmap_cells_x * p.costmap_cells_y);
    std::vector<float> dyn_tensor;
    if (p.dyn_tensor) dyn_tensor.assign(p.dyn_tensor, p.dyn_tensor + p.dyn_tensor_len);
    p.dyn_tensor = nullptr;
    p.std_per_step = nullptr;
    p.step_sizes = nullptr;
    p.costmap = nullptr;

    CK(cudaSetDevice(p.device));
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->n_roll_blocks = (int)((c->M_local + kRolloutThreads - 1) / kRolloutThreads);
    c->n_w_blocks = (int)std::min<long long>((c->M_local + 255) / 256, 148 * 4);
    // update grid: one wave of the update kernel's resident CTAs (kUpdateCtasPerSm per SM)
    {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device);
      int per_sm = kUpdateCtasPerSm;
      if (const char* e = getenv("SMPC_UPDATE_CTAS_PER_SM")) per_sm = std::max(1, atoi(e));  // A/B knob
      // enough warps for one work unit (quad group x 32 candidates) each when
      // every sample is a candidate, capped at one resident wave
      const long long QG = ((TU + 3) / 4 + kUpdateQuadsPerUnit - 1) / kUpdateQuadsPerUnit;
      const long long units = (c->M_local + 31) / 32 * QG;
      c->n_u_blocks = (int)std::max<long long>(1, std::min<long long>((units + kUpdateWarps - 1) / kUpdateWarps,
                                                                     (long long)sms * per_sm));
    }

    c->d_mean = dalloc<float>((size_t)c->S * TU);
    c->d_x0 = dalloc<float>((size_t)2 * kMaxNX);
    c->d_sigma = dalloc<float>((size_t)(TU + 3) / 4 * 4);  // float4-readable
    c->d_sig2 = dalloc<double>(TU);
    c->d_gamma = dalloc<double>(c->T);
    c->d_costs = dalloc<double>((size_t)c->S * c->M_local);
    c->d_weights = dalloc<double>((size_t)c->S * c->M_local);
    c->blk_cap = (long long)c->S * c->n_roll_blocks;
    c->d_blk_min = dalloc<double>((size_t)c->blk_cap);
    c->d_blk_arg = dalloc<long long>((size_t)c->blk_cap);
    c->d_blk_eta = dalloc<double>((size_t)c->S * c->n_w_blocks);
    c->d_blk_nz = dalloc<long long>((size_t)c->S * c->n_w_blocks);
    c->d_cand = dalloc<int>((size_t)c->S * c->M_local);
    c->d_cand_cnt = dalloc<int>((size_t)c->S * c->n_w_blocks);
    c->d_cand_off = dalloc<long long>((size_t)c->S * (c->n_w_blocks + 1));
    c->d_cand_e = dalloc<double>((size_t)c->S * c->M_local);
    {
      const long long warps = (long long)c->n_u_blocks * kUpdateWarps;
      const long long Q = (TU + 3) / 4, QG = (Q + kUpdateQuadsPerUnit - 1) / kUpdateQuadsPerUnit;
      // warps covering one quad group: <= 2 * warps / QG + 2 (each owns >= U / (2 W) units)
      c->upd_slots = (int)(2 * ((warps + QG - 1) / QG) + 3);
      c->d_blk_part = dalloc<double>((size_t)c->S * QG * c->upd_slots * kUpdateSlot);
      c->d_upd_gsum = dalloc<double>((size_t)c->S * QG * kUpdateSlot);
      c->d_upd_gcnt = dalloc<unsigned int>((size_t)c->S * QG);
    }
    c->d_counters = dalloc<unsigned int>(16);
    c->d_select = dalloc<SelectState>(1);
    {  // small-N mode below kZqMaxSamples samples per shard (latency-bound sizes)
      long long zq_max = kZqMaxSamples;
      if (const char* e = getenv("SMPC_ZQ_MAX_SAMPLES")) zq_max = atoll(e);  // A/B knob (0 = off)
      if (c->M_local <= zq_max) {
        c->d_zq = dalloc<float4>((size_t)((TU + 3) / 4) * c->M_local);
        c->use_zq = true;
        alloc_split(c, false);
      }
    }
    c->d_eq_cnt = dalloc<int>(c->n_w_blocks);
    c->d_eq_off = dalloc<long long>(c->n_w_blocks + 1);
    c->d_gather1 = dalloc<double>((size_t)c->S * 2 * 8);
    c->d_gather2 = dalloc<double>((size_t)c->S * 2 * 8);
    c->d_gather3 = dalloc<double>((size_t)c->S * TU * 8);
    c->d_gather_rec = dalloc<double>((size_t)gather_record(c) * 8);
    c->d_rm_score = dalloc<double>(32);
    c->d_rm_z = dalloc<float>(32 * kMaxNX);
    // result region: header | controls | states | outputs
    size_t off = align_up(sizeof(ResultHeader), 256);
    c->off_controls = off;
    off = align_up(off + sizeof(float) * c->S * TU, 256);
    c->off_states = off;
    off = align_up(off + sizeof(float) * c->S * (c->T + 1) * c->nx, 256);
    c->off_outs = off;
    off = align_up(off + sizeof(float) * c->S * c->T * c->ny, 256);
    c->result_bytes = off;
    c->d_result = dalloc<unsigned char>(off);
    CK(cudaMallocHost(&c->h_result, off));
    CK(cudaMallocHost(&c->h_x0, sizeof(float) * 2 * kMaxNX));
    {
      ResultHeader h;
      memset(&h, 0, sizeof h);
      h.err_key = kNoError;
      h.abort_key = kNoError;
      CK(cudaMemcpyAsync(c->d_result, &h, sizeof h, cudaMemcpyHostToDevice, c->stream));
    }
    // sigma / sigma^2 (sampling.hpp:56-60, sampling.cpp:123) and gamma (engine.cpp:397-401)
    std::vector<float> sig(TU);
    std::vector<double> sig2(TU), gam(c->T);
    for (int t = 0; t < c->T; ++t)
      for (int u = 0; u < c->nu; ++u) {
        const float s = !c->std_per_step.empty() ? c->std_per_step[t * c->nu + u]
                                                 : (p.n_control_std == 1 ? p.control_std[0] : p.control_std[u]);
        sig[t * c->nu + u] = s;
        const double sd = s;
        sig2[t * c->nu + u] = sd * sd;
      }
    for (int t = 0; t < c->T; ++t)
      gam[t] = c->step_sizes.empty() ? 1.0 : (double)c->step_sizes[c->step_sizes.size() == 1 ? 0 : t];
    CK(cudaMemcpyAsync(c->d_sigma, sig.data(), sizeof(float) * TU, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_sig2, sig2.data(), sizeof(double) * TU, cudaMemcpyHostToDevice, c->stream));
    {
      bool pow2 = true;
      for (double v : sig2) pow2 = pow2 && exact_inverse_pow2(v) != 0.0;
      c->base.sig2_pow2 = pow2 ? 1 : 0;  // fill_args leaves it alone
    }
    CK(cudaMemcpyAsync(c->d_gamma, gam.data(), sizeof(double) * c->T, cudaMemcpyHostToDevice, c->stream));
    if ((p.dynamics_kind != SMPC_DYN_PLUGIN && p.cost_kind == SMPC_COST_DIFF_DRIVE_NAV) ||
        (p.dynamics_kind == SMPC_DYN_PLUGIN && !c->costmap.empty())) {
      const size_t cells = (size_t)p.costmap_cells_x * p.costmap_cells_y;
      c->d_costmap = dalloc<uint8_t>(cells);
      if (!c->costmap.empty()) CK(cudaMemcpyAsync(c->d_costmap, c->costmap.data(), cells, cudaMemcpyHostToDevice, c->stream));
    }
    if (p.dynamics_kind == SMPC_DYN_MLP) {  // + W2 transposed for the warp-cooperative nominal rollout
      using namespace mlp_layout;
      for (int k = 0; k < HID; ++k)
        for (int j = 0; j < HID; ++j) dyn_tensor.push_back(dyn_tensor[W2 + j * HID + k]);
    }
    if (!dyn_tensor.empty()) {
      c->d_dyn_tensor = dalloc<float>(dyn_tensor.size());
      CK(cudaMemcpyAsync(c->d_dyn_tensor, dyn_tensor.data(), sizeof(float) * dyn_tensor.size(), cudaMemcpyHostToDevice, c->stream));
    }
    uint32_t j_lo, j_hi;
    tail_table_size(&j_lo, &j_hi);
    c->d_tail = dalloc<float>((size_t)((1u << 23) - j_hi) + j_lo);
    CK(build_tail_table(c->d_tail, j_lo, j_hi, c->stream));
    {
      cudaResourceDesc rd = {};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = c->d_tail;
      rd.res.linear.desc = cudaCreateChannelDesc<float>();
      rd.res.linear.sizeInBytes = sizeof(float) * ((size_t)((1u << 23) - j_hi) + j_lo);
      cudaTextureDesc td = {};
      td.readMode = cudaReadModeElementType;
      cudaTextureObject_t tex = 0;
      CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
      c->tail_tex = (unsigned long long)tex;
    }
    // Creation-time uploads are ordered on the context's (non-blocking) stream
    // and complete before the first solve: a pageable cudaMemcpy may return
    // before its DMA lands and is not ordered with a non-blocking stream (a
    // solve could read the zeroed result header, i.e. a spurious error key).
    CK(cudaStreamSynchronize(c->stream));
    c->host_mean[0].assign(TU, 0.f);
    c->host_mean[1].assign(TU, 0.f);
    c->nominal_state.assign(c->nx, 0.f);
    CK(cudaEventCreateWithFlags(&c->ev_stage, cudaEventDisableTiming));
    for (int i = 0; i < 2 * c->I; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->ev.push_back(e);
    }
    fill_args(c);
    c->full_tex = full_icdf_table(c->base, p.device, c->stream);
    c->base.full_tex = c->full_tex;
    CK(cudaStreamSynchronize(c->stream));
  });
  if (st != SMPC_OK) {
    smpc_destroy(c);
    return st;
  }
  *out = c;
  return SMPC_OK;
}

void smpc_destroy(smpc_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->tail_tex) cudaDestroyTextureObject((cudaTextureObject_t)c->tail_tex);
  for (auto e : c->ev) cudaEventDestroy(e);
  if (c->ev_stage) cudaEventDestroy(c->ev_stage);
  if (c->comm && nccl()) nccl()->CommDestroy(c->comm);
  void* ptrs[] = {c->d_mean, c->d_x0, c->d_sigma, c->d_tail, c->d_sig2, c->d_gamma, c->d_costs,
                  c->d_weights, c->d_blk_min, c->d_blk_eta, c->d_blk_part, c->d_gather1, c->d_gather2,
                  c->d_gather3, c->d_blk_arg, c->d_blk_nz, c->d_counters, c->d_costmap, c->d_result,
                  c->d_ro_x0, c->d_ro_mean, c->d_eps, c->d_outputs, c->d_wscratch, c->d_flags,
                  c->d_cand, c->d_cand_e, c->d_cand_cnt, c->d_cand_off, c->d_select, c->d_eq_cnt, c->d_eq_off,
                  c->d_dyn_tensor, c->d_zq, c->d_gather_rec, c->d_rm_score, c->d_rm_z,
                  c->d_ytraj, c->d_utraj, c->d_rflag, c->d_upd_gsum, c->d_upd_gcnt};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->h_result) cudaFreeHost(c->h_result);
  if (c->h_x0) cudaFreeHost(c->h_x0);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

const char* smpc_last_error(const smpc_ctx* c) { return c ? c->err.c_str() : g_create_error.c_str(); }

smpc_status smpc_error_location(const smpc_ctx* c, int64_t* sample, int32_t* timestep, int32_t* channel) {
  if (!c) return SMPC_ERR_ARGUMENT;
  if (sample) *sample = c->err_sample;
  if (timestep) *timestep = c->err_t;
  if (channel) *channel = c->err_ch;
  return SMPC_OK;
}

smpc_status smpc_get_dims(const smpc_ctx* c, int32_t* nx, int32_t* nu, int32_t* ny) {
  if (!c) return SMPC_ERR_ARGUMENT;
  if (nx) *nx = c->nx;
  if (nu) *nu = c->nu;
  if (ny) *ny = c->ny;
  return SMPC_OK;
}

smpc_status smpc_set_mean(smpc_ctx* c, int32_t system, const float* mean) {
  if (!c || !mean || system < 0 || system >= c->S) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const size_t TU = (size_t)c->T * c->nu;
    for (size_t k = 0; k < TU; ++k)
      if (!std::isfinite(mean[k])) throw RuntimeError{"control vector has non-finite entry at channel " + std::to_string(k % c->nu)};
    CK(cudaMemcpyAsync(c->d_mean + system * TU, mean, sizeof(float) * TU, cudaMemcpyHostToDevice, c->stream));
    if (c->p.controller_kind == SMPC_CTRL_RMPPI)  // one control sequence, mirrored into both systems
      CK(cudaMemcpyAsync(c->d_mean + (1 - system) * TU, mean, sizeof(float) * TU, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_get_mean(const smpc_ctx* cc, int32_t system, float* mean) {
  smpc_ctx* c = const_cast<smpc_ctx*>(cc);
  if (!c || !mean || system < 0 || system >= c->S) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const size_t TU = (size_t)c->T * c->nu;
    CK(cudaMemcpyAsync(mean, c->d_mean + system * TU, sizeof(float) * TU, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_get_solve_count(const smpc_ctx* c, uint64_t* n) {
  if (!c || !n) return SMPC_ERR_ARGUMENT;
  *n = c->solve_count;
  return SMPC_OK;
}

smpc_status smpc_set_solve_count(smpc_ctx* c, uint64_t n) {
  if (!c) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    CK(cudaMemcpyAsync(&c->header()->solve_count, &n, sizeof n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->solve_count = n;
  });
}

smpc_status smpc_compute_control(smpc_ctx* c, const float* x0, smpc_solution* out) {
  if (!c || !x0) return SMPC_ERR_ARGUMENT;
  if (c->S != 1) {
    // TubeMppiController::compute_control returns the nominal solution (controllers.cpp:281-283).
    smpc_tube_solution t{};
    if (out) t.nominal = *out;
    const smpc_status st = smpc_tube_compute_control(c, x0, &t);
    if (out) *out = t.nominal;
    return st;
  }
  return guarded(c, [&] {
    const double t0 = now_ms();
    for (int i = 0; i < c->nx; ++i)
      if (!std::isfinite(x0[i])) throw RuntimeError{"state vector has non-finite entry at channel " + std::to_string(i)};
    upload_x0(c, x0, 1);
    launch_solve(c);
    fetch_results(c);
    if (out) {
      copy_solution(c, 0, out);
      if (out->weights) fetch_weights(c, 0, out->weights);
      out->solve_time_ms = now_ms() - t0;
    }
  });
}

smpc_status smpc_tube_compute_control(smpc_ctx* c, const float* x_real, smpc_tube_solution* out) {
  if (!c || !x_real) return SMPC_ERR_ARGUMENT;
  if (c->S != 2) {
    set_error(c, "tube_compute_control: context is not a tube controller");
    return SMPC_ERR_RUNTIME;
  }
  const bool rmppi = c->p.controller_kind == SMPC_CTRL_RMPPI;
  return guarded(c, [&] {
    const double t0 = now_ms();
    for (int i = 0; i < c->nx; ++i)
      if (!std::isfinite(x_real[i])) throw RuntimeError{"state vector has non-finite entry at channel " + std::to_string(i)};
    // nominal-state bookkeeping (controllers.cpp:221-227); RMPPI chooses on the
    // device between the previous nominal state and x_real (rmppi_select_kernel)
    if (!c->nominal_started) {
      c->nominal_state.assign(x_real, x_real + c->nx);
      c->nominal_started = true;
    } else if (!rmppi && std::isfinite(c->p.nominal_reset_bound)) {
      float acc = 0.f;
      for (int i = 0; i < c->nx; ++i) {
        const float d = x_real[i] - c->nominal_state[i];
        acc += d * d;
      }
      if ((double)std::sqrt(acc) > c->p.nominal_reset_bound) c->nominal_state.assign(x_real, x_real + c->nx);
    }
    float x0s[2 * kMaxNX];
    memcpy(x0s, c->nominal_state.data(), sizeof(float) * c->nx);
    memcpy(x0s + c->nx, x_real, sizeof(float) * c->nx);
    upload_x0(c, x0s, 2);
    launch_solve(c);
    fetch_results(c);
    const double elapsed = now_ms() - t0;
    if (rmppi) {
      const float* z = c->h_header()->rmppi_nominal;
      c->nominal_state.assign(z, z + c->nx);
    }
    if (out) {
      if (out->nominal_state) memcpy(out->nominal_state, c->nominal_state.data(), sizeof(float) * c->nx);
      copy_solution(c, 0, &out->nominal);
      copy_solution(c, 1, &out->real);
      if (out->nominal.weights) fetch_weights(c, 0, out->nominal.weights);
      if (out->real.weights) fetch_weights(c, 1, out->real.weights);
      out->nominal.solve_time_ms = elapsed;
      out->real.solve_time_ms = elapsed;
    }
    // the nominal system advances only through the model (controllers.cpp:276-277)
    const float* nn = c->h_header()->next_nominal_state;
    c->nominal_state.assign(nn, nn + c->nx);
  });
}

smpc_status smpc_shift_control_sequence(smpc_ctx* c, double elapsed_s, double dt_min) {
  if (!c) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const std::string name = controller_name(c->p.controller_kind);
    if (!(dt_min > 0.0)) throw RuntimeError{name + ": dt_min must be > 0"};
    if (elapsed_s <= 0.0) return;
    // controllers.cpp:68-84 (Tube shifts both means, :285-292)
    const double quantized = (double)std::llrint(elapsed_s / dt_min) * dt_min;
    const long long steps = std::llrint(quantized / c->p.dt);
    if (steps <= 0) return;
    const int T = c->T, nu = c->nu;
    std::vector<float> m((size_t)T * nu), shifted((size_t)T * nu);
    for (int s = 0; s < c->S; ++s) {
      // on the context stream: ordered after a graph left running by smpc_launch_iteration
      CK(cudaMemcpyAsync(m.data(), c->d_mean + (size_t)s * T * nu, sizeof(float) * T * nu, cudaMemcpyDeviceToHost,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));
      if (steps >= T) {
        std::fill(shifted.begin(), shifted.end(), 0.f);
      } else {
        for (int t = 0; t < T; ++t) {
          const int src = std::min<long long>(t + steps, T - 1);
          for (int u = 0; u < nu; ++u) shifted[t * nu + u] = m[src * nu + u];
        }
      }
      CK(cudaMemcpyAsync(c->d_mean + (size_t)s * T * nu, shifted.data(), sizeof(float) * T * nu, cudaMemcpyHostToDevice,
                         c->stream));
      CK(cudaStreamSynchronize(c->stream));
    }
  });
}

smpc_status smpc_generate_samples(smpc_ctx* c, const float* mean, uint32_t stream, float* eps_out,
                                  uint8_t* flags_out) {
  if (!c || !mean || !eps_out) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const size_t TU = (size_t)c->T * c->nu;
    const size_t n = (size_t)c->M_local * TU;
    if (c->eps_cap < n) {
      if (c->d_eps) cudaFree(c->d_eps);
      c->d_eps = dalloc<float>(n);
      c->eps_cap = n;
    }
    if (c->flags_cap < (size_t)c->M_local) {
      if (c->d_flags) cudaFree(c->d_flags);
      c->d_flags = dalloc<uint8_t>(c->M_local);
      c->flags_cap = c->M_local;
    }
    if (!c->d_ro_mean) c->d_ro_mean = dalloc<float>(2 * TU);
    CK(cudaMemcpyAsync(c->d_ro_mean, mean, sizeof(float) * TU, cudaMemcpyHostToDevice, c->stream));
    IterArgs a = c->base;
    a.solve_count = nullptr;
    a.stream = stream;
    a.mean_in = c->d_ro_mean;
    CK(c->ops.generate(a, c->d_eps, c->d_flags, c->stream));
    CK(cudaMemcpyAsync(eps_out, c->d_eps, sizeof(float) * n, cudaMemcpyDeviceToHost, c->stream));
    if (flags_out) CK(cudaMemcpyAsync(flags_out, c->d_flags, c->M_local, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_rollout(smpc_ctx* c, int32_t S, const float* x0s, const float* means, const float* eps,
                         uint32_t stream, double* costs_out, float* outputs_out) {
  if (!c || !x0s || !means || !costs_out || (S != 1 && S != 2)) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const size_t TU = (size_t)c->T * c->nu;
    if (!c->d_ro_mean) c->d_ro_mean = dalloc<float>(2 * TU);
    if (!c->d_ro_x0) c->d_ro_x0 = dalloc<float>(2 * kMaxNX);
    CK(cudaMemcpyAsync(c->d_ro_mean, means, sizeof(float) * S * TU, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_ro_x0, x0s, sizeof(float) * S * c->nx, cudaMemcpyHostToDevice, c->stream));
    IterArgs a = c->base;
    a.S = S;
    a.solve_count = nullptr;
    a.stream = stream;
    a.iter = 0;
    a.mean_in = c->d_ro_mean;
    a.x0 = c->d_ro_x0;
    if (S > c->S) {  // scratch sized for the controller's S; grow for a 2-system request
      if (!c->d_wscratch || c->wscratch_cap < (size_t)2 * c->M_local) {
        if (c->d_wscratch) cudaFree(c->d_wscratch);
        c->wscratch_cap = (size_t)2 * c->M_local + 2 * (size_t)c->n_roll_blocks;
        c->d_wscratch = dalloc<double>(c->wscratch_cap);
      }
    }
    double* costs = S > c->S ? c->d_wscratch : c->d_costs;
    a.costs = costs;
    // blk_min/arg and gather1 must hold S systems
    double* blk_min = c->d_blk_min;
    long long* blk_arg = c->d_blk_arg;
    if (S > c->S) {
      blk_min = dalloc<double>((size_t)2 * c->n_roll_blocks);
      blk_arg = dalloc<long long>((size_t)2 * c->n_roll_blocks);
    }
    a.blk_min = blk_min;
    a.blk_arg = blk_arg;
    a.rank = 0;
    a.world = 1;
    // RolloutEngine::rollout takes its cost adjustments from the sampler
    // config whatever controller owns the engine (only CemController's own
    // compute_control drops them, controllers.cpp:155-162)
    a.importance = c->p.importance_sampling != 0;
    if (eps) {
      const size_t n = (size_t)c->M_local * TU;
      if (c->eps_cap < n) {
        if (c->d_eps) cudaFree(c->d_eps);
        c->d_eps = dalloc<float>(n);
        c->eps_cap = n;
        c->eps_tma = false;  // re-encode for the new buffer
      }
      CK(cudaMemcpyAsync(c->d_eps, eps, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
      if (!c->eps_tma) c->eps_tma = encode_eps_map(&c->eps_map, c->d_eps, c->M_local, (int)TU);
      a.eps_in = c->d_eps;
      a.eps_tma = c->eps_tma;
      a.eps_map = &c->eps_map;
    }
    if (outputs_out) {
      const size_t n = (size_t)S * c->M_local * c->T * c->ny;
      if (c->outputs_cap < n) {
        if (c->d_outputs) cudaFree(c->d_outputs);
        c->d_outputs = dalloc<float>(n);
        c->outputs_cap = n;
      }
      a.outputs = c->d_outputs;
    }
    // the kernel's abort gate reads the header: clear a previous failure first
    CK(launch_begin_solve(c->header(), c->stream));
    CK(c->ops.rollout(a, c->p.cost_kind, c->stream));
    ResultHeader h;
    CK(cudaMemcpyAsync(costs_out, costs, sizeof(double) * S * c->M_local, cudaMemcpyDeviceToHost, c->stream));
    if (outputs_out)
      CK(cudaMemcpyAsync(outputs_out, c->d_outputs, sizeof(float) * S * c->M_local * c->T * c->ny,
                         cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&h, c->header(), sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (S > c->S) {
      cudaFree(blk_min);
      cudaFree(blk_arg);
    }
    if (h.err_key != kNoError && (h.err_key >> 62) == 0) {
      decode_error(c, h.err_key);
      throw RuntimeError{c->err};
    }
  });
}

smpc_status smpc_compute_weights(smpc_ctx* c, const double* costs, int64_t count, double lambda,
                                 double* weights_out, smpc_weight_summary* summary) {
  if (!c || !costs || count < 0) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    if (!(lambda > 0.0)) throw RuntimeError{"compute_weights: lambda must be > 0"};
    if (count == 0) throw RuntimeError{"compute_weights: cost list is empty"};
    for (int64_t m = 0; m < count; ++m)
      if (!std::isfinite(costs[m])) throw RuntimeError{"compute_weights: non-finite cost at sample " + std::to_string(m)};
    const int nblk = (int)std::min<long long>((count + 255) / 256, 148 * 4);
    const size_t need = (size_t)2 * count + 4 * (size_t)nblk + 8 + (size_t)count / 2 + 1 + 2 * (size_t)nblk + 2;
    if (c->wscratch_cap < need) {
      if (c->d_wscratch) cudaFree(c->d_wscratch);
      c->d_wscratch = dalloc<double>(need);
      c->wscratch_cap = need;
    }
    double* d_costs = c->d_wscratch;
    double* d_w = d_costs + count;
    double* d_bmin = d_w + count;
    long long* d_barg = reinterpret_cast<long long*>(d_bmin + nblk);
    double* d_eta = reinterpret_cast<double*>(d_barg + nblk);
    double* d_nz = d_eta + nblk;
    double* d_g1 = d_nz + nblk;  // [2]
    double* d_g2 = d_g1 + 2;     // [2]
    int* d_cand = reinterpret_cast<int*>(d_g2 + 2);                         // [count]
    int* d_ccnt = d_cand + count + (count & 1);                            // [nblk]
    long long* d_coff = reinterpret_cast<long long*>(d_ccnt + nblk + (nblk & 1));  // [nblk+1]
    CK(cudaMemcpyAsync(d_costs, costs, sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
    CK(launch_begin_solve(c->header(), c->stream));
    CK(launch_min_only(d_costs, count, d_bmin, d_barg, nblk, c->d_counters + 8, d_g1,
                       reinterpret_cast<long long*>(d_g1 + 1), c->stream));
    IterArgs a = c->base;
    a.S = 1;
    a.world = 1;
    a.rank = 0;
    a.M_local = (int)count;
    a.costs = d_costs;
    a.weights = d_w;
    a.lambda = lambda;
    a.inv_lambda_pow2 = exact_inverse_pow2(lambda);
    a.gather1 = d_g1;
    a.gather2 = d_g2;
    a.n_w_blocks = nblk;
    a.blk_eta = d_eta;
    a.blk_nz = reinterpret_cast<long long*>(d_nz);
    a.cand = d_cand;
    a.cand_e = nullptr;  // weights only: no update follows
    a.cem_k = 0.0;       // plain softmin weights e/eta even on a CEM context (engine.cpp:342-363)
    a.skip_w = 0.0;
    a.cand_cnt = d_ccnt;
    a.cand_off = d_coff;
    CK(launch_weights(a, c->stream));
    CK(launch_normalize_weights(a, c->stream));
    double g1[2], g2[2];
    if (weights_out) CK(cudaMemcpyAsync(weights_out, d_w, sizeof(double) * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g1, d_g1, sizeof g1, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(g2, d_g2, sizeof g2, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (summary) {
      summary->baseline = g1[0];
      long long am;
      memcpy(&am, &g1[1], sizeof am);
      summary->argmin = am;
      summary->normalizer = g2[0];
      summary->nonzero = (int64_t)g2[1];
    }
  });
}

smpc_status smpc_sorted_samples(smpc_ctx* c, int32_t system, int64_t count, int64_t* order_out, double* costs_out) {
  if (!c || !order_out || system < 0 || system >= c->S || count < 1 || count > c->M_local) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    if (c->world > 1 || c->M_local != c->M) throw ConfigError{"smpc_sorted_samples: single-shard contexts only"};
    IterArgs a = c->base;
    a.S = 1;
    a.costs = c->d_costs + (size_t)system * c->M_local;
    a.weights = c->d_weights + (size_t)system * c->M_local;
    long long n_pad = 1;
    while (n_pad < count) n_pad <<= 1;
    unsigned long long* keys = dalloc<unsigned long long>((size_t)n_pad + 1);
    long long* idx = dalloc<long long>((size_t)n_pad);
    CK(launch_select(a, c->d_select, count, c->d_counters + 8, c->d_eq_cnt, c->d_eq_off, c->stream));
    CK(launch_sort_selected(a, count, keys, idx, keys + n_pad, c->stream));
    std::vector<unsigned long long> hk((size_t)count);
    CK(cudaMemcpyAsync(order_out, idx, sizeof(long long) * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(hk.data(), keys, sizeof(unsigned long long) * count, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(keys);
    cudaFree(idx);
    if (costs_out) {
      for (int64_t i = 0; i < count; ++i) {  // invert select.cu:cost_key
        const unsigned long long k = hk[(size_t)i];
        const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
        memcpy(&costs_out[i], &b, sizeof b);
      }
    }
  });
}

smpc_status smpc_export_sample_trajectories(smpc_ctx* c, const float* x0, const float* mean, const float* eps,
                                            uint32_t stream, double fraction, int64_t* k_out, int64_t* order_out,
                                            float* outputs_out) {
  if (!c || !x0 || !mean || !k_out) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    if (!(fraction >= 0.0 && fraction <= 1.0)) throw RuntimeError{"export_sample_trajectories: fraction must be in [0, 1]"};
    if (c->world > 1 || c->M_local != c->M) throw ConfigError{"export_sample_trajectories: single-shard contexts only"};
    const long long k = (long long)std::ceil(fraction * (double)c->M);  // engine.cpp:417
    *k_out = k;
    if (k == 0) return;
    const size_t TU = (size_t)c->T * c->nu;
    if (!c->d_ro_mean) c->d_ro_mean = dalloc<float>(2 * TU);
    if (!c->d_ro_x0) c->d_ro_x0 = dalloc<float>(2 * kMaxNX);
    CK(cudaMemcpyAsync(c->d_ro_mean, mean, sizeof(float) * TU, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_ro_x0, x0, sizeof(float) * c->nx, cudaMemcpyHostToDevice, c->stream));
    IterArgs a = c->base;
    a.S = 1;
    a.solve_count = nullptr;
    a.stream = stream;
    a.iter = 0;
    a.mean_in = c->d_ro_mean;
    a.x0 = c->d_ro_x0;
    a.rank = 0;
    a.world = 1;
    // RolloutEngine::rollout takes its cost adjustments from the sampler
    // config whatever controller owns the engine (only CemController's own
    // compute_control drops them, controllers.cpp:155-162)
    a.importance = c->p.importance_sampling != 0;
    if (eps) {
      const size_t n = (size_t)c->M_local * TU;
      if (c->eps_cap < n) {
        if (c->d_eps) cudaFree(c->d_eps);
        c->d_eps = dalloc<float>(n);
        c->eps_cap = n;
        c->eps_tma = false;  // re-encode for the new buffer
      }
      CK(cudaMemcpyAsync(c->d_eps, eps, sizeof(float) * n, cudaMemcpyHostToDevice, c->stream));
      if (!c->eps_tma) c->eps_tma = encode_eps_map(&c->eps_map, c->d_eps, c->M_local, (int)TU);
      a.eps_in = c->d_eps;
      a.eps_tma = c->eps_tma;
      a.eps_map = &c->eps_map;
    }
    // 1) the fused rollout (RolloutResult::costs, system 0)
    CK(launch_begin_solve(c->header(), c->stream));
    CK(c->ops.rollout(a, c->p.cost_kind, c->stream));
    // 2) the k lowest (cost, index) samples in partial_sort order (engine.cpp:419-426)
    long long n_pad = 1;
    while (n_pad < k) n_pad <<= 1;
    unsigned long long* keys = dalloc<unsigned long long>((size_t)n_pad + 1);
    long long* idx = dalloc<long long>((size_t)n_pad);
    CK(launch_select(a, c->d_select, k, c->d_counters + 8, c->d_eq_cnt, c->d_eq_off, c->stream));
    CK(launch_sort_selected(a, k, keys, idx, keys + n_pad, c->stream));
    // 3) re-roll just the chosen samples with stored outputs (engine.cpp:435-453)
    float* outs = dalloc<float>((size_t)k * c->T * c->ny);
    double* costs = dalloc<double>((size_t)k);
    const int nblk = (int)((k + kRolloutThreads - 1) / kRolloutThreads);
    double* bmin = dalloc<double>((size_t)nblk);
    long long* barg = dalloc<long long>((size_t)nblk);
    IterArgs b = a;
    b.sample_idx = idx;
    b.M_local = (int)k;
    b.costs = costs;
    b.outputs = outs;
    b.n_roll_blocks = nblk;
    b.blk_min = bmin;
    b.blk_arg = barg;
    CK(c->ops.rollout(b, c->p.cost_kind, c->stream));
    ResultHeader h;
    if (order_out) CK(cudaMemcpyAsync(order_out, idx, sizeof(long long) * k, cudaMemcpyDeviceToHost, c->stream));
    if (outputs_out)
      CK(cudaMemcpyAsync(outputs_out, outs, sizeof(float) * k * c->T * c->ny, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(&h, c->header(), sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    void* tmp[] = {keys, idx, outs, costs, bmin, barg};
    for (void* q : tmp) cudaFree(q);
    if (h.err_key != kNoError && (h.err_key >> 62) == 0) {
      decode_error(c, h.err_key);
      throw RuntimeError{c->err};
    }
  });
}

// RolloutEngine::auto_select (engine.cpp:281-320) for the device's two noise
// strategies (split = materialised normals, fused = in-register Philox): a
// scratch budget first, then medians of timed runs, fused only if strictly
// faster (ties -> split).
extern "C" int32_t smpc_noise_strategy_rule(double split_bytes, double split_budget_bytes, double split_median_ms,
                                            double fused_median_ms) {
  if (split_bytes > split_budget_bytes) return SMPC_NOISE_FUSED;
  return fused_median_ms < split_median_ms ? SMPC_NOISE_FUSED : SMPC_NOISE_SPLIT;
}


smpc_status smpc_select_noise_strategy(smpc_ctx* c, int32_t kind, int32_t trials, double split_budget_bytes,
                                       const float* x0, smpc_noise_choice* out) {
  if (!c || kind < SMPC_NOISE_AUTO || kind > SMPC_NOISE_FUSED || (kind == SMPC_NOISE_AUTO && !x0))
    return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    smpc_noise_choice ch = {kind, 0.0, 0.0, 0};
    if (kind == SMPC_NOISE_AUTO) {
      upload_x0(c, x0, c->S);
      ch = auto_select_noise(c, trials, split_budget_bytes);
    } else {
      set_noise(c, kind == SMPC_NOISE_SPLIT);
      c->noise_choice = ch;
      c->noise_resolved = true;
    }
    if (out) *out = ch;
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_set_x0(smpc_ctx* c, const float* x0) {
  if (!c || !x0) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    upload_x0(c, x0, c->S);
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_launch_iteration(smpc_ctx* c) {
  if (!c) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] { launch_solve(c); });
}

smpc_status smpc_synchronize(smpc_ctx* c) {
  if (!c) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    CK(cudaMemcpyAsync(c->h_result, c->d_result, sizeof(ResultHeader), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    collect_timing(c);
    const ResultHeader* h = c->h_header();
    if (h->err_key != kNoError) {
      decode_error(c, h->err_key);
      throw RuntimeError{c->err};
    }
    c->solve_count = h->solve_count;
  });
}

void* smpc_stream(smpc_ctx* c) { return c ? (void*)c->stream : nullptr; }

int32_t smpc_kernels_per_solve(const smpc_ctx* c) {
  if (!c) return 0;
  const int zq = c->use_zq ? 1 : 0;  // gen_zq_kernel per iteration in split-noise mode
  const int rm = c->p.controller_kind == SMPC_CTRL_RMPPI ? 1 : 0;
  // begin_solve (folded into the first gen_zq in small-N mode) + per iteration
  // (the clean-solve count is kept by the last update / combine)
  const int begin = c->use_zq && !c->d_inj && !rm ? 0 : 1;
  if (c->p.controller_kind == SMPC_CTRL_CEM) return begin + c->I * (1 + 11 + 1 + zq);  // rollout, select (init+8+2), update
  return begin + rm + c->I * (3 + zq + (c->world > 1 ? 1 : 0));
}

smpc_status smpc_icdf_table(smpc_ctx* c, float* out) {
  if (!c || !out) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    const float* d;
    {
      std::lock_guard<std::mutex> lk(g_full_mu);
      d = g_full[c->p.device & 63].d;
    }
    if (!d) throw RuntimeError{"icdf table not built"};
    CK(cudaMemcpyAsync(out, d, sizeof(float) << 23, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

smpc_status smpc_icdf_domain(smpc_ctx* c, float* out) {
  if (!c || !out) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    float* d = dalloc<float>(1u << 23);
    CK(launch_icdf_domain(c->base, d, c->stream));
    CK(cudaMemcpyAsync(out, d, sizeof(float) << 23, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d);
  });
}

smpc_status smpc_rollout_kernel_ms(smpc_ctx* c, int32_t enable, double* total_ms, int64_t* launches) {
  if (!c) return SMPC_ERR_ARGUMENT;
  if (total_ms) *total_ms = c->rollout_ms_total;
  if (launches) *launches = c->rollout_launches;
  if (enable >= 0) {
    c->timing = enable != 0;
    c->rollout_ms_total = 0.0;
    c->rollout_launches = 0;
  }
  return SMPC_OK;
}

smpc_status smpc_group_init(smpc_ctx** ctxs, int32_t n) {
  if (!ctxs || n < 1 || n > 8) return SMPC_ERR_ARGUMENT;
  for (int r = 0; r < n; ++r)
    if (!ctxs[r]) return SMPC_ERR_ARGUMENT;
  return guarded(ctxs[0], [&] {
    for (int r = 0; r < n; ++r) {
      smpc_ctx* c = ctxs[r];
      if (n > 1 && c->p.controller_kind == SMPC_CTRL_CEM) throw ConfigError{"cem: multi-GPU sharding is not supported"};
      // the in-process group runs plain compute_control solves: no per-solve
      // nominal-state choice (RMPPI) and no Tube nominal bookkeeping
      if (c->p.controller_kind == SMPC_CTRL_RMPPI || c->p.controller_kind == SMPC_CTRL_TUBE)
        throw ConfigError{"smpc_group_init: tube and rmppi controllers are not supported by the in-process group"};
      if (c->M != ctxs[0]->M || c->T != ctxs[0]->T || c->S != ctxs[0]->S || c->I != ctxs[0]->I ||
          c->comm_mode != ctxs[0]->comm_mode)
        throw ConfigError{"smpc_group_init: contexts describe different problems"};
      c->rank = r;
      c->world = n;
      fill_args(c);
      if (c->graph) {
        cudaGraphExecDestroy(c->graph);
        c->graph = nullptr;
      }
    }
  });
}

smpc_status smpc_group_compute_control(smpc_ctx** ctxs, int32_t n, const float* x0, smpc_solution* out) {
  if (!ctxs || n < 1 || !x0) return SMPC_ERR_ARGUMENT;
  return guarded(ctxs[0], [&] {
    const double t0 = now_ms();
    for (int r = 0; r < n; ++r) {
      if (ctxs[r]->world != n || ctxs[r]->rank != r) throw ConfigError{"smpc_group_compute_control: call smpc_group_init first"};
      upload_x0(ctxs[r], x0, ctxs[r]->S);
    }
    enqueue_group_solve(ctxs, n);
    for (int r = 0; r < n; ++r) fetch_results(ctxs[r]);
    for (int r = 0; r < n; ++r) {
      if (out) {
        copy_solution(ctxs[r], 0, &out[r]);
        out[r].solve_time_ms = now_ms() - t0;
      }
    }
  });
}

// ---- closed loop ------------------------------------------------------------

namespace {

// Host side of one Plant::run_control_loop (plant.cpp:133-181): the replan
// schedule depends only on t, so the host walks it and enqueues, per step,
// [shift + solve] on replans and one plant step; nothing is synchronised
// until the end. Several loops are advanced in lockstep (one stream each).
struct LoopState {
  smpc_ctx* c;
  smpc_plant_config pc;
  long long steps = 0;
  double dt = 0.0, interval = 0.0, next_replan_t = 0.0, solution_t = 0.0;
  bool solved_once = false;
  long long solves = 0;
  float* d_x = nullptr;
  double* d_log = nullptr;
  std::vector<cudaEvent_t> ev;  // per solve: start, end
  PlantStepArgs p{};
};

void loop_begin(LoopState& L, smpc_ctx* c, const smpc_plant_config* pc, const float* x0, double duration_s,
                bool want_log) {
  L.c = c;
  L.pc = *pc;
  if (c->S != 1) throw ConfigError{"run_control_loop: tube controllers are not supported"};
  if (!(pc->replan_rate > 0.0)) throw RuntimeError{"plant: replan_rate must be > 0"};
  if (!(pc->dt_min > 0.0)) throw RuntimeError{"plant: dt_min must be > 0"};
  if (!(pc->disturbance_std >= 0.0)) throw RuntimeError{"simulated system: disturbance_std must be >= 0"};
  if (!(duration_s > 0.0)) throw RuntimeError{"plant: loop duration must be > 0"};
  for (int i = 0; i < c->nx; ++i)
    if (!std::isfinite(x0[i])) throw RuntimeError{"state vector has non-finite entry at channel " + std::to_string(i)};
  L.dt = c->p.dt;
  L.steps = std::llround(duration_s / L.dt);
  L.interval = 1.0 / pc->replan_rate;
  L.d_x = dalloc<float>(kMaxNX);
  CK(cudaMemcpyAsync(L.d_x, x0, sizeof(float) * c->nx, cudaMemcpyHostToDevice, c->stream));
  upload_x0(c, x0, 1);
  if (want_log) L.d_log = dalloc<double>((size_t)std::max(1LL, L.steps) * (2 + c->nx + c->nu));
  // loop_err / loop_cost live in the result header
  const unsigned long long no_err = kNoError;
  const double zero = 0.0;
  CK(cudaMemcpyAsync(&c->header()->loop_err, &no_err, sizeof no_err, cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->header()->loop_cost, &zero, sizeof zero, cudaMemcpyHostToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));  // the pageable H2D sources above are locals
  PlantStepArgs& p = L.p;
  p.x = L.d_x;
  p.x0_out = c->d_x0;
  p.controls = reinterpret_cast<const float*>(c->d_result + c->off_controls);
  p.dt = (float)L.dt;
  p.scale = (float)(pc->disturbance_std * std::sqrt(L.dt));  // plant.cpp:35
  const uint64_t sim_seed = pc->rng_seed ^ 0x9E3779B97F4A7C15ull;  // plant.cpp:228-229
  for (int r = 0; r < 10; ++r) {
    p.rk.k0[r] = (uint32_t)sim_seed + (uint32_t)r * 0x9E3779B9u;
    p.rk.k1[r] = (uint32_t)(sim_seed >> 32) + (uint32_t)r * 0xBB67AE85u;
  }
  p.log = L.d_log;
  if (!c->graph) build_graph(c);
}

void loop_step(LoopState& L, long long step) {
  smpc_ctx* c = L.c;
  const double t = (double)step * L.dt;
  if (!L.solved_once || t >= L.next_replan_t - 1e-9) {
    if (L.solved_once) {  // shift_control_sequence(t - solution_t, dt_min) (controllers.cpp:68-84)
      const double elapsed = t - L.solution_t;
      if (elapsed > 0.0) {
        const double quantized = (double)std::llrint(elapsed / L.pc.dt_min) * L.pc.dt_min;
        const long long k = std::llrint(quantized / c->p.dt);
        if (k > 0) CK(launch_shift_mean(c->d_mean, c->S, c->T, c->nu, k, c->stream));
      }
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    L.ev.push_back(e0);
    L.ev.push_back(e1);
    CK(cudaEventRecord(e0, c->stream));
    CK(cudaGraphLaunch(c->graph, c->stream));  // compute_control(x) with x = the sim snapshot (d_x0)
    CK(cudaEventRecord(e1, c->stream));
    L.solution_t = t;
    ++L.solves;
    L.solved_once = true;
    while (L.next_replan_t <= t + 1e-9) L.next_replan_t += L.interval;
  }
  // control_for_time (plant.cpp:106-115)
  const long long raw = (long long)std::floor((t - L.solution_t) / c->p.dt);
  L.p.idx = (int)std::min<long long>(std::max<long long>(raw, 0), c->T - 1);
  L.p.step = (uint32_t)step;
  L.p.t = t;
  IterArgs a = c->base;
  CK(c->ops.plant_step(a, c->p.cost_kind, L.p, c->stream));
}

void loop_end(LoopState& L, smpc_loop_result* out, double* log_out) {
  smpc_ctx* c = L.c;
  CK(cudaMemcpyAsync(c->h_result, c->d_result, c->result_bytes, cudaMemcpyDeviceToHost, c->stream));
  if (log_out && L.d_log)
    CK(cudaMemcpyAsync(log_out, L.d_log, sizeof(double) * L.steps * (2 + c->nx + c->nu), cudaMemcpyDeviceToHost,
                       c->stream));
  CK(cudaStreamSynchronize(c->stream));
  double total_ms = 0.0;
  for (size_t i = 0; i + 1 < L.ev.size(); i += 2) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, L.ev[i], L.ev[i + 1]));
    total_ms += ms;
  }
  for (auto e : L.ev) cudaEventDestroy(e);
  L.ev.clear();
  cudaFree(L.d_x);
  if (L.d_log) cudaFree(L.d_log);
  const ResultHeader* h = c->h_header();
  c->solve_count = h->solve_count;
  if (h->loop_err != kNoError) {
    decode_error(c, h->loop_err);
    throw RuntimeError{c->err};
  }
  if (out) {
    out->accumulated_cost = h->loop_cost;
    out->solve_count = L.solves;
    out->mean_solve_ms = L.solves ? total_ms / (double)L.solves : 0.0;
    out->steps = L.steps;
  }
}

}  // namespace

smpc_status smpc_run_control_loop(smpc_ctx* c, const smpc_plant_config* pc, const float* x0, double duration_s,
                                  smpc_loop_result* out, double* log_out) {
  if (!c || !pc || !x0) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    LoopState L;
    loop_begin(L, c, pc, x0, duration_s, log_out != nullptr);
    for (long long step = 0; step < L.steps; ++step) loop_step(L, step);
    loop_end(L, out, log_out);
  });
}

smpc_status smpc_run_control_loops(smpc_ctx** cs, int32_t n, const smpc_plant_config* pcs, const float* x0s,
                                   double duration_s, smpc_loop_result* outs) {
  if (!cs || n < 1 || !pcs || !x0s) return SMPC_ERR_ARGUMENT;
  for (int i = 0; i < n; ++i)
    if (!cs[i]) return SMPC_ERR_ARGUMENT;
  std::vector<LoopState> L((size_t)n);
  smpc_ctx* failed = cs[0];
  return guarded(cs[0], [&] {
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
      failed = cs[i];
      loop_begin(L[i], cs[i], &pcs[i], x0s + off, duration_s, false);
      off += (size_t)cs[i]->nx;
    }
    long long steps = 0;
    for (int i = 0; i < n; ++i) steps = std::max(steps, L[i].steps);
    for (long long step = 0; step < steps; ++step)
      for (int i = 0; i < n; ++i)
        if (step < L[i].steps) loop_step(L[i], step);
    for (int i = 0; i < n; ++i) {
      failed = cs[i];
      loop_end(L[i], outs ? &outs[i] : nullptr, nullptr);
    }
    (void)failed;
  });
}

smpc_status smpc_comm_unique_id(uint8_t id_out[128]) {
  NcclApi* api = nccl();
  if (!api) {
    g_create_error = "NCCL (libnccl.so.2) could not be loaded";
    return SMPC_ERR_CUDA;
  }
  ncclUniqueId id;
  if (api->GetUniqueId(&id) != 0) return SMPC_ERR_CUDA;
  memcpy(id_out, id.internal, 128);
  return SMPC_OK;
}

smpc_status smpc_set_injected_noise(smpc_ctx* c, const float* d_eps) {
  if (!c) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    if (c->p.controller_kind == SMPC_CTRL_CEM || c->p.dynamics_kind == SMPC_DYN_MLP)
      throw ConfigError{"injected noise: supported for mppi / dmd / tube / rmppi on the SIMT models"};
    c->d_inj = d_eps;
    c->inj_tma = d_eps ? encode_eps_map(&c->inj_map, d_eps, c->M_local, c->T * c->nu) : false;
    if (c->graph) {
      cudaGraphExecDestroy(c->graph);
      c->graph = nullptr;
    }
  });
}

smpc_status smpc_comm_set_mode(smpc_ctx* c, int32_t mode) {
  if (!c || (mode != SMPC_COMM_SINGLE && mode != SMPC_COMM_EXACT)) return SMPC_ERR_ARGUMENT;
  c->comm_mode = mode;
  fill_args(c);
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  return SMPC_OK;
}

smpc_status smpc_comm_init(smpc_ctx* c, const uint8_t id[128], int32_t rank, int32_t world) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world || world > 8) return SMPC_ERR_ARGUMENT;
  return guarded(c, [&] {
    if (world == 1) return;
    if (c->p.controller_kind == SMPC_CTRL_CEM) throw ConfigError{"cem: multi-GPU sharding is not supported"};
    NcclApi* api = nccl();
    if (!api) throw CudaError{"NCCL (libnccl.so.2) could not be loaded"};
    ncclUniqueId uid;
    memcpy(uid.internal, id, 128);
    CK(cudaSetDevice(c->p.device));
    const ncclResult_t r = api->CommInitRank(&c->comm, world, uid, rank);
    if (r != 0) throw CudaError{std::string("ncclCommInitRank: ") + (api->GetErrorString ? api->GetErrorString(r) : "")};
    c->rank = rank;
    c->world = world;
    fill_args(c);
    if (c->graph) {
      cudaGraphExecDestroy(c->graph);
      c->graph = nullptr;
    }
  });
}

}  // extern "C"
