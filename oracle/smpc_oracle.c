/*
 * smpc_oracle.c — CPU restatement of the reference MPPI iteration.
 * TEST INFRASTRUCTURE ONLY (see smpc_oracle.h). Build: oracle/Makefile
 * (gcc -O2 -ffp-contract=off; no -march, no -ffast-math), which is how the
 * reference's own Release build evaluates float expressions on x86-64
 * (unfused mulss/addss).
 *
 * Each function cites the reference lines it restates
 * (paths relative to /root/reference/proj/core).
 */
#include "smpc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KMAX SMPC_MAX_DIM

static int fail(oracle_error* err, const char* msg) {
  if (err) {
    snprintf(err->message, sizeof(err->message), "%s", msg);
    err->sample = -1;
    err->timestep = -1;
    err->channel = -1;
  }
  return SMPC_ERR_RUNTIME;
}

/* ---- rng.hpp ------------------------------------------------------------ */

/* philox::round_once / block (rng.hpp:14-31). */
void oracle_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int i = 0; i < 10; ++i) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* NormalStream::to_open_unit (rng.hpp:52-54). */
float oracle_to_open_unit(uint32_t x) { return (float)(x >> 9) * 0x1.0p-23f + 0x1.0p-24f; }

/* NormalStream::normal_icdf (rng.hpp:56-96), Acklam's rational approximation. */
float oracle_normal_icdf(float p) {
  const float kLow = 0.02425f;
  if (p >= kLow && p <= 1.0f - kLow) {
    const float q = p - 0.5f;
    const float r = q * q;
    return q *
           (((((-3.969683028665376e+01f * r + 2.209460984245205e+02f) * r -
               2.759285104469687e+02f) *
                  r +
              1.383577518672690e+02f) *
                 r -
             3.066479806614716e+01f) *
                r +
            2.506628277459239e+00f) /
           (((((-5.447609879822406e+01f * r + 1.615858368580409e+02f) * r -
               1.556989798598866e+02f) *
                  r +
              6.680131188771972e+01f) *
                 r -
             1.328068155288572e+01f) *
                r +
            1.0f);
  }
  const int lower = p < kLow;
  const float q = sqrtf(-2.0f * logf(lower ? p : 1.0f - p));
  const float x = (((((-7.784894002430293e-03f * q - 3.223964580411365e-01f) * q -
                      2.400758277161838e+00f) *
                         q -
                     2.549732539343734e+00f) *
                        q +
                    4.374664141464968e+00f) *
                       q +
                   2.938163982698783e+00f) /
                  ((((7.784695709041462e-03f * q + 3.224671290700398e-01f) * q +
                     2.445134137142996e+00f) *
                        q +
                    3.754408661907416e+00f) *
                       q +
                   1.0f);
  return lower ? x : -x;
}

void oracle_icdf_domain(float* out) {
  for (uint32_t k = 0; k < (1u << 23); ++k) out[k] = oracle_normal_icdf(oracle_to_open_unit(k << 9));
}

/* NormalStream ctor + quad (rng.hpp:41-48). */
void oracle_quad(uint64_t seed, uint32_t a, uint32_t b, uint32_t c, float out[4]) {
  const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  const uint32_t ctr[4] = {a, b, c, 0u};
  uint32_t w[4];
  oracle_philox(ctr, key, w);
  for (int i = 0; i < 4; ++i) out[i] = oracle_normal_icdf(oracle_to_open_unit(w[i]));
}

/* ---- types.hpp / dynamics.cpp ------------------------------------------- */

/* wrap_angle (types.hpp:36-42). */
static float wrap_angle(float a) {
  const float kTwoPi = 6.283185307179586f;
  a = fmodf(a, kTwoPi);
  if (a <= -3.14159265358979f) a += kTwoPi;
  if (a > 3.14159265358979f) a -= kTwoPi;
  return a;
}

int oracle_dims_of(const smpc_problem* p, oracle_dims* d, oracle_error* err) {
  switch (p->dynamics_kind) {
    case SMPC_DYN_UNICYCLE:
    case SMPC_DYN_DIFF_DRIVE:
      d->n_x = 3, d->n_u = 2, d->n_y = 3;
      return 0;
    case SMPC_DYN_CARTPOLE:
      d->n_x = 4, d->n_u = 1, d->n_y = 4;
      return 0;
    case SMPC_DYN_DOUBLE_INTEGRATOR:
      d->n_x = 4, d->n_u = 2, d->n_y = 4;
      return 0;
    case SMPC_DYN_QUADROTOR:
      d->n_x = 13, d->n_u = 4, d->n_y = 13;
      return 0;
    case SMPC_DYN_BICYCLE:
      d->n_x = 3, d->n_u = 2, d->n_y = 3;
      return 0;
    case SMPC_DYN_MLP:
      if (!p->dyn_tensor || p->dyn_tensor_len != 1412) return fail(err, "mlp: dyn_tensor must hold 1412 floats");
      d->n_x = 7, d->n_u = 2, d->n_y = 7;
      return 0;
    default:
      return fail(err, "dynamics.kind is not recognized");
  }
}

static double dparam(const smpc_problem* p, int i, double dflt) {
  return i < p->n_dyn_params ? p->dyn_params[i] : dflt;
}
static double cparam(const smpc_problem* p, int i, double dflt) {
  return i < p->n_cost_params ? p->cost_params[i] : dflt;
}

/* Builder-defined quadrotor (no reference counterpart; paper_2409_07563_b200/
 * csrc/models.cuh:QuadrotorDyn is the device twin — parity unpinned by the
 * reference). params {mass, gravity, tau, thrust_max, rate_max}. */
typedef struct quad_params {
  float inv_mass, gravity, inv_tau, hover, lo[4], hi[4];
} quad_params;

static quad_params quadrotor_params(const smpc_problem* p) {
  quad_params q;
  const float mass = (float)dparam(p, 0, 1.0), g = (float)dparam(p, 1, 9.81), tau = (float)dparam(p, 2, 0.05);
  const float tmax = (float)dparam(p, 3, 39.24), rmax = (float)dparam(p, 4, 5.0);
  q.inv_mass = 1.0f / mass;
  q.inv_tau = 1.0f / tau;
  q.gravity = g;
  q.hover = mass * g;
  for (int i = 0; i < 3; ++i) q.lo[i] = -rmax, q.hi[i] = rmax;
  q.lo[3] = -q.hover;
  q.hi[3] = tmax - q.hover;
  return q;
}

static void quadrotor_derivative(const smpc_problem* p, const float* x, const float* u, float* dx) {
  const quad_params q = quadrotor_params(p);
  const float qw = x[6], qx = x[7], qy = x[8], qz = x[9];
  const float wx = x[10], wy = x[11], wz = x[12];
  const float acc = (q.hover + u[3]) * q.inv_mass;
  const float zx = 2.0f * (qx * qz + qw * qy);
  const float zy = 2.0f * (qy * qz - qw * qx);
  const float zz = 1.0f - 2.0f * (qx * qx + qy * qy);
  dx[0] = x[3];
  dx[1] = x[4];
  dx[2] = x[5];
  dx[3] = acc * zx;
  dx[4] = acc * zy;
  dx[5] = acc * zz - q.gravity;
  dx[6] = -0.5f * (qx * wx + qy * wy + qz * wz);
  dx[7] = 0.5f * (qw * wx + qy * wz - qz * wy);
  dx[8] = 0.5f * (qw * wy - qx * wz + qz * wx);
  dx[9] = 0.5f * (qw * wz + qx * wy - qy * wx);
  dx[10] = (u[0] - wx) * q.inv_tau;
  dx[11] = (u[1] - wy) * q.inv_tau;
  dx[12] = (u[2] - wz) * q.inv_tau;
}

/* quaternion re-normalisation after the Euler step */
static void quadrotor_post_step(float* x) {
  const float n = sqrtf(x[6] * x[6] + x[7] * x[7] + x[8] * x[8] + x[9] * x[9]);
  for (int i = 6; i < 10; ++i) x[i] = x[i] / n;
}

/* Builder-defined AutoRally-style neural dynamics (device twin: csrc/models.cuh
 * MlpDyn + csrc/mlp.cu; parity is tolerance-based: the device runs layer 2 in
 * 3xTF32 on the tensor cores and uses an exp-based tanh). Blob layout
 * W1[32][6] b1[32] W2[32][32] b2[32] W3[4][32] b3[4]. */
static void mlp_derivative(const smpc_problem* p, const float* x, const float* u, float* dx) {
  const float* w = p->dyn_tensor;
  const float *W1 = w, *b1 = W1 + 192, *W2 = b1 + 32, *b2 = W2 + 1024, *W3 = b2 + 32, *b3 = W3 + 128;
  const float in[6] = {x[3], x[4], x[5], x[6], u[0], u[1]};
  float h1[32], h2[32];
  for (int j = 0; j < 32; ++j) {
    float acc = b1[j];
    for (int k = 0; k < 6; ++k) acc += W1[j * 6 + k] * in[k];
    h1[j] = tanhf(acc);
  }
  for (int j = 0; j < 32; ++j) {
    float acc = b2[j];
    for (int k = 0; k < 32; ++k) acc += W2[j * 32 + k] * h1[k];
    h2[j] = tanhf(acc);
  }
  const float c = cosf(x[2]), s = sinf(x[2]);
  dx[0] = x[4] * c - x[5] * s;
  dx[1] = x[4] * s + x[5] * c;
  dx[2] = x[6];
  for (int q = 0; q < 4; ++q) {
    float acc = b3[q];
    for (int j = 0; j < 32; ++j) acc += W3[q * 32 + j] * h2[j];
    dx[3 + q] = acc;
  }
}

/* state_derivative overrides: unicycle dynamics.cpp:127-131, cartpole :143-156,
 * diff-drive :167-171, double integrator :176-181. */
static void state_derivative(const smpc_problem* p, const float* x, const float* u, float* dx) {
  switch (p->dynamics_kind) {
    case SMPC_DYN_UNICYCLE:
    case SMPC_DYN_DIFF_DRIVE:
      dx[0] = u[0] * cosf(x[2]);
      dx[1] = u[0] * sinf(x[2]);
      dx[2] = u[1];
      break;
    case SMPC_DYN_CARTPOLE: {
      const float mc = (float)dparam(p, 0, 1.0), mp = (float)dparam(p, 1, 1.0);
      const float l = (float)dparam(p, 2, 1.0), g = (float)dparam(p, 3, 9.81);
      const float sin_t = sinf(x[2]);
      const float cos_t = cosf(x[2]);
      const float omega = x[3];
      const float denom = mc + mp * sin_t * sin_t;
      const float x_acc = (u[0] + mp * sin_t * (l * omega * omega + g * cos_t)) / denom;
      dx[0] = x[1];
      dx[1] = x_acc;
      dx[2] = omega;
      dx[3] = -(x_acc * cos_t + g * sin_t) / l;
      break;
    }
    case SMPC_DYN_DOUBLE_INTEGRATOR:
      dx[0] = x[2];
      dx[1] = x[3];
      dx[2] = u[0];
      dx[3] = u[1];
      break;
    case SMPC_DYN_QUADROTOR:
      quadrotor_derivative(p, x, u, dx);
      break;
    case SMPC_DYN_MLP:
      mlp_derivative(p, x, u, dx);
      break;
    case SMPC_DYN_BICYCLE: { /* builder-defined kinematic bicycle (device twin: models.cuh BicycleDyn) */
      dx[0] = u[0] * cosf(x[2]);
      dx[1] = u[0] * sinf(x[2]);
      const float tan_d = sinf(u[1]) / cosf(u[1]);
      dx[2] = (u[0] * tan_d) / (float)dparam(p, 0, 0.5);
      break;
    }
  }
}

/* clamp_control (dynamics.cpp:31-39); only diff-drive is bounded (:164). */
static void clamp_control(const smpc_problem* p, const float* u, float* out, int n_u) {
  if (p->dynamics_kind == SMPC_DYN_DIFF_DRIVE) {
    const float lo[2] = {(float)dparam(p, 2, -0.35), (float)dparam(p, 4, -0.5)};
    const float hi[2] = {(float)dparam(p, 3, 0.5), (float)dparam(p, 5, 0.5)};
    for (int i = 0; i < 2; ++i) {
      const float a = u[i] < lo[i] ? lo[i] : u[i]; /* std::max(u, lo) */
      out[i] = hi[i] < a ? hi[i] : a;              /* std::min(., hi) */
    }
    return;
  }
  if (p->dynamics_kind == SMPC_DYN_BICYCLE) {
    const float lo[2] = {(float)dparam(p, 1, -0.35), (float)dparam(p, 3, -0.6)};
    const float hi[2] = {(float)dparam(p, 2, 0.5), (float)dparam(p, 4, 0.6)};
    for (int i = 0; i < 2; ++i) {
      const float a = u[i] < lo[i] ? lo[i] : u[i];
      out[i] = hi[i] < a ? hi[i] : a;
    }
    return;
  }
  if (p->dynamics_kind == SMPC_DYN_MLP) { /* steering, throttle in [-1, 1] */
    for (int i = 0; i < 2; ++i) {
      const float a = u[i] < -1.0f ? -1.0f : u[i];
      out[i] = 1.0f < a ? 1.0f : a;
    }
    return;
  }
  if (p->dynamics_kind == SMPC_DYN_QUADROTOR) {
    const quad_params q = quadrotor_params(p);
    for (int i = 0; i < 4; ++i) {
      const float a = u[i] < q.lo[i] ? q.lo[i] : u[i];
      out[i] = q.hi[i] < a ? q.hi[i] : a;
    }
    return;
  }
  for (int i = 0; i < n_u; ++i) out[i] = u[i];
}

static int angular_channel(const smpc_problem* p) {
  return (p->dynamics_kind == SMPC_DYN_DOUBLE_INTEGRATOR || p->dynamics_kind == SMPC_DYN_QUADROTOR) ? -1 : 2;
}

/* step_raw (dynamics.cpp:45-54) with the default observe (:41-43). */
static void step_raw(const smpc_problem* p, const oracle_dims* d, const float* x, const float* u,
                     float dt, float* x_next, float* y) {
  float u_c[KMAX], dx[KMAX];
  clamp_control(p, u, u_c, d->n_u);
  state_derivative(p, x, u_c, dx);
  for (int i = 0; i < d->n_x; ++i) x_next[i] = x[i] + dt * dx[i];
  if (p->dynamics_kind == SMPC_DYN_QUADROTOR) quadrotor_post_step(x_next);
  const int ang = angular_channel(p);
  if (ang >= 0) x_next[ang] = wrap_angle(x_next[ang]);
  for (int i = 0; i < d->n_y; ++i) y[i] = x_next[i];
}

int oracle_step(const smpc_problem* p, const float* x, const float* u, float dt, float* x_next,
                float* y, oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  step_raw(p, &d, x, u, dt, x_next, y);
  return 0;
}

/* ---- costs.cpp / costmap.hpp -------------------------------------------- */

/* Costmap2D::occupancy (costmap.hpp:34-41). */
static float occupancy(const smpc_problem* p, float x, float y) {
  const float inv_res = (float)(1.0 / p->costmap_resolution);
  const float fx = (x - (float)p->costmap_origin_x) * inv_res;
  const float fy = (y - (float)p->costmap_origin_y) * inv_res;
  const float flx = floorf(fx), fly = floorf(fy);
  /* static_cast<int> of an out-of-range float is INT_MIN on x86 (cvttss2si). */
  const int ix = (flx >= -2147483648.0f && flx < 2147483648.0f) ? (int)flx : INT32_MIN;
  const int iy = (fly >= -2147483648.0f && fly < 2147483648.0f) ? (int)fly : INT32_MIN;
  if (ix < 0 || iy < 0 || ix >= p->costmap_cells_x || iy >= p->costmap_cells_y) return 1.0f;
  if (!p->costmap) return 0.0f;
  return p->costmap[(size_t)iy * p->costmap_cells_x + ix] ? 1.0f : 0.0f;
}

/* running_cost_raw: road costs.cpp:33-41, circle :54-65, nav :75-82, quadratic :98-105. */
static double running_cost(const smpc_problem* p, const float* y) {
  switch (p->cost_kind) {
    case SMPC_COST_ROAD: {
      const float hw = (float)cparam(p, 0, 1.0), lin = (float)cparam(p, 1, 1.0),
                  quad = (float)cparam(p, 2, 10.0);
      const float offset = fabsf(y[1]);
      if (offset <= hw) return (double)lin * offset;
      const float excess = offset - hw;
      return (double)lin * hw + (double)quad * excess * excess;
    }
    case SMPC_COST_CIRCLE_TRACK: {
      const float inner = (float)cparam(p, 0, 1.875), outer = (float)cparam(p, 1, 2.125);
      const float crash = (float)cparam(p, 2, 1000.0), speed_target = (float)cparam(p, 3, 2.0);
      const float speed_coeff = (float)cparam(p, 4, 2.0), am_target = (float)cparam(p, 5, 4.0);
      const float am_coeff = (float)cparam(p, 6, 2.0);
      const float inner_sq = inner * inner, outer_sq = outer * outer; /* costs.cpp:50-51 */
      const float r_sq = y[0] * y[0] + y[1] * y[1];
      double cost = 0.0;
      if (r_sq <= inner_sq) cost += crash;
      if (r_sq >= outer_sq) cost += crash;
      const float speed = sqrtf(y[2] * y[2] + y[3] * y[3]);
      cost += (double)speed_coeff * fabsf(speed_target - speed);
      const float am = y[0] * y[3] - y[1] * y[2];
      cost += (double)am_coeff * fabsf(am_target - am);
      return cost;
    }
    case SMPC_COST_DIFF_DRIVE_NAV: {
      const float gx = (float)cparam(p, 0, 2.0), gy = (float)cparam(p, 1, 2.0),
                  gyaw = (float)cparam(p, 2, 0.0);
      const float dist = (float)cparam(p, 3, 5.0), yawc = (float)cparam(p, 4, 5.0),
                  obst = (float)cparam(p, 5, 20.0);
      const float dx = y[0] - gx;
      const float dy = y[1] - gy;
      const float dyaw = wrap_angle(y[2] - gyaw);
      return (double)dist * (dx * dx + dy * dy) + (double)yawc * dyaw * dyaw +
             (double)obst * occupancy(p, y[0], y[1]);
    }
    case SMPC_COST_QUADRATIC: {
      double cost = 0.0;
      for (int i = 0; i < p->n_quad; ++i) {
        const double d = (double)y[i] - p->quad_target[i];
        cost += p->quad_weights[i] * d * d;
      }
      return cost;
    }
  }
  return NAN;
}

/* terminal_cost_raw: 0 except quadratic (costs.cpp:43, :67, :84, :107-109). */
static double terminal_cost(const smpc_problem* p, const float* y) {
  return p->cost_kind == SMPC_COST_QUADRATIC ? running_cost(p, y) : 0.0;
}

/* ---- sampling.cpp -------------------------------------------------------- */

static float std_at(const smpc_problem* p, int t, int c, int n_u) {
  if (p->std_per_step) return p->std_per_step[(size_t)t * n_u + c];
  return p->n_control_std == 1 ? p->control_std[0] : p->control_std[c];
}

/* GaussianSampler::generate_samples (sampling.cpp:32-96). */
int oracle_generate_samples(const smpc_problem* p, const float* mean, int64_t m_begin,
                            int64_t m_end, uint32_t stream, float* eps, uint8_t* flags,
                            oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  const int M = p->num_samples, T = p->horizon, n_u = d.n_u;
  const int with_mean = p->include_mean_sample != 0;
  int n_zero = (int)ceil(p->zero_mean_fraction * M);
  const int cap = with_mean ? M - 1 : M;
  if (n_zero > cap) n_zero = cap;
  const int zero_begin = M - n_zero;
  const int per_sample = T * n_u;
  for (int64_t m = m_begin; m < m_end; ++m) {
    float* row = &eps[(size_t)(m - m_begin) * per_sample];
    const int is_mean = with_mean && m == 0;
    const int zero_mean = m >= zero_begin;
    if (flags) flags[m - m_begin] = (uint8_t)((is_mean ? 1 : 0) | (zero_mean ? 2 : 0));
    if (is_mean) {
      for (int k = 0; k < per_sample; ++k) row[k] = 0.0f;
      continue;
    }
    for (int q = 0; q * 4 < per_sample; ++q) {
      float z[4];
      oracle_quad(p->seed, stream, (uint32_t)m, (uint32_t)q, z);
      const int base = q * 4;
      const int lanes = per_sample - base < 4 ? per_sample - base : 4;
      for (int lane = 0; lane < lanes; ++lane) {
        const int k = base + lane;
        const int t = k / n_u, c = k % n_u;
        float e = std_at(p, t, c, n_u) * z[lane];
        if (zero_mean) e -= mean[(size_t)t * n_u + c];
        row[k] = e;
      }
    }
  }
  return 0;
}

/* GaussianSampler::importance_weight_adjustment (sampling.cpp:111-130). */
void oracle_importance(const smpc_problem* p, const float* eps, int64_t count,
                       const float* mean, double* adj) {
  oracle_dims d;
  oracle_dims_of(p, &d, NULL);
  const int T = p->horizon, n_u = d.n_u;
  for (int64_t m = 0; m < count; ++m) {
    if (!p->importance_sampling) {
      adj[m] = 0.0;
      continue;
    }
    double acc = 0.0;
    for (int t = 0; t < T; ++t) {
      for (int c = 0; c < n_u; ++c) {
        const double sigma = std_at(p, t, c, n_u);
        acc += (double)mean[(size_t)t * n_u + c] * eps[((size_t)m * T + t) * n_u + c] /
               (sigma * sigma);
      }
    }
    adj[m] = p->lambda * acc;
  }
}

/* ---- engine.cpp ---------------------------------------------------------- */

static int rollout_error(oracle_error* err, const char* what, int channel, int64_t m, int t) {
  if (err) {
    if (channel >= 0) {
      snprintf(err->message, sizeof(err->message),
               "rollout produced non-finite state channel %d at sample %lld timestep %d", channel,
               (long long)m, t);
    } else {
      snprintf(err->message, sizeof(err->message), "rollout produced %s at sample %lld timestep %d",
               what, (long long)m, t);
    }
    err->sample = m;
    err->timestep = t;
    err->channel = channel;
  }
  return SMPC_ERR_RUNTIME;
}

/* run_sample_fused (engine.cpp:211-239) over every (s, m), then + adjustment
 * (engine.cpp:263-265). Samples are visited in (s, m) order, so the first
 * error reported is the one a single worker would throw. */
int oracle_rollout(const smpc_problem* p, int32_t S, const float* x0s, const float* means,
                   const float* eps, int64_t m_begin, int64_t count, const double* adj,
                   double* costs, float* outputs, oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  const int T = p->horizon, n_u = d.n_u;
  const float dt = (float)p->dt; /* engine.cpp:216 */
  for (int s = 0; s < S; ++s) {
    const float* mean_base = &means[(size_t)s * T * n_u];
    for (int64_t i = 0; i < count; ++i) {
      float x[KMAX], x_next[KMAX], y[KMAX], u[KMAX];
      for (int ch = 0; ch < d.n_x; ++ch) x[ch] = x0s[(size_t)s * d.n_x + ch];
      double total = 0.0;
      for (int t = 0; t < T; ++t) {
        const float* e = &eps[((size_t)i * T + t) * n_u];
        for (int c = 0; c < n_u; ++c) u[c] = mean_base[(size_t)t * n_u + c] + e[c];
        step_raw(p, &d, x, u, dt, x_next, y);
        for (int ch = 0; ch < d.n_x; ++ch) {
          if (!isfinite(x_next[ch])) return rollout_error(err, NULL, ch, m_begin + i, t);
        }
        const double c_t = running_cost(p, y);
        if (!isfinite(c_t) || c_t < 0.0) {
          return rollout_error(err, "invalid running cost", -1, m_begin + i, t);
        }
        total += c_t;
        if (outputs) {
          memcpy(&outputs[(((size_t)s * count + i) * T + t) * d.n_y], y, sizeof(float) * d.n_y);
        }
        memcpy(x, x_next, sizeof(float) * d.n_x);
      }
      const double terminal = terminal_cost(p, y);
      if (!isfinite(terminal) || terminal < 0.0) {
        return rollout_error(err, "invalid running cost", -1, m_begin + i, T - 1);
      }
      total = total + terminal;
      if (adj) total += adj[(size_t)s * count + i];
      costs[(size_t)s * count + i] = total;
    }
  }
  return 0;
}

/* RolloutEngine::compute_weights (engine.cpp:342-363). */
int oracle_compute_weights(const double* costs, int64_t n, double lambda, double* weights,
                           double* baseline, double* normalizer, int64_t* argmin,
                           oracle_error* err) {
  if (!(lambda > 0.0)) return fail(err, "compute_weights: lambda must be > 0");
  if (n <= 0) return fail(err, "compute_weights: cost list is empty");
  for (int64_t m = 0; m < n; ++m) {
    if (!isfinite(costs[m])) {
      char buf[128];
      snprintf(buf, sizeof(buf), "compute_weights: non-finite cost at sample %lld", (long long)m);
      return fail(err, buf);
    }
  }
  int64_t best = 0; /* std::min_element: first minimum */
  for (int64_t m = 1; m < n; ++m)
    if (costs[m] < costs[best]) best = m;
  const double rho = costs[best];
  double eta = 0.0;
  for (int64_t m = 0; m < n; ++m) {
    const double e = exp(-(costs[m] - rho) / lambda);
    weights[m] = e;
    eta += e;
  }
  for (int64_t m = 0; m < n; ++m) weights[m] /= eta;
  *baseline = rho;
  *normalizer = eta;
  if (argmin) *argmin = best;
  return 0;
}

/* RolloutEngine::weighted_update (engine.cpp:365-409). */
int oracle_weighted_update(const float* mean, int32_t T, int32_t n_u, const float* eps,
                           int64_t M, const double* weights, const float* steps,
                           int32_t n_steps, float* out, oracle_error* err) {
  if (!(n_steps == 0 || n_steps == 1 || n_steps == T)) {
    return fail(err, "weighted_update: step sizes must be empty, scalar, or one per timestep");
  }
  for (int i = 0; i < n_steps; ++i) {
    if (!(steps[i] > 0.0f && steps[i] <= 1.0f)) {
      return fail(err, "weighted_update: step sizes must be in (0, 1]");
    }
  }
  const size_t K = (size_t)T * n_u;
  double* acc = (double*)calloc(K, sizeof(double));
  for (int64_t m = 0; m < M; ++m) {
    const double w = weights[m];
    const float* row = &eps[(size_t)m * K];
    for (size_t k = 0; k < K; ++k) acc[k] += w * row[k];
  }
  for (int t = 0; t < T; ++t) {
    const double gamma = n_steps == 0 ? 1.0 : (double)steps[n_steps == 1 ? 0 : t];
    for (int c = 0; c < n_u; ++c) {
      const size_t k = (size_t)t * n_u + c;
      out[k] = (float)(mean[k] + gamma * acc[k]);
    }
  }
  free(acc);
  return 0;
}

/* ---- controllers.cpp ----------------------------------------------------- */

/* Controller::finish_solution (controllers.cpp:86-104): checked typed steps. */
static int finish_solution(const smpc_problem* p, const oracle_dims* d, const float* mean,
                           const float* x0, float* states, float* outputs, oracle_error* err) {
  const int T = p->horizon;
  const float dt = (float)p->dt;
  float x[KMAX], xn[KMAX], y[KMAX];
  memcpy(x, x0, sizeof(float) * d->n_x);
  if (states) memcpy(states, x0, sizeof(float) * d->n_x);
  for (int t = 0; t < T; ++t) {
    step_raw(p, d, x, &mean[(size_t)t * d->n_u], dt, xn, y);
    for (int ch = 0; ch < d->n_x; ++ch) {
      if (!isfinite(xn[ch])) {
        char buf[96];
        snprintf(buf, sizeof(buf), "state vector has non-finite entry at channel %d", ch);
        return fail(err, buf);
      }
    }
    if (states) memcpy(&states[(size_t)(t + 1) * d->n_x], xn, sizeof(float) * d->n_x);
    if (outputs) memcpy(&outputs[(size_t)t * d->n_y], y, sizeof(float) * d->n_y);
    memcpy(x, xn, sizeof(float) * d->n_x);
  }
  return 0;
}

/* One iteration shared by MPPI and Tube: S systems over one noise batch drawn
 * about means[0] (controllers.cpp:116-131, :229-253). */
static int iterate(const smpc_problem* p, const oracle_dims* d, int S, const float* x0s,
                   float* means, uint32_t stream, double* last_weights,
                   smpc_weight_summary* summaries, oracle_error* err) {
  const int M = p->num_samples, T = p->horizon, n_u = d->n_u;
  const size_t K = (size_t)T * n_u;
  float* eps = (float*)malloc(sizeof(float) * (size_t)M * K);
  double* adj = p->importance_sampling ? (double*)malloc(sizeof(double) * (size_t)S * M) : NULL;
  double* costs = (double*)malloc(sizeof(double) * (size_t)S * M);
  double* w = (double*)malloc(sizeof(double) * (size_t)M);
  float* updated = (float*)malloc(sizeof(float) * K);
  int rc = oracle_generate_samples(p, means, 0, M, stream, eps, NULL, err);
  if (!rc && adj) {
    for (int s = 0; s < S; ++s) oracle_importance(p, eps, M, &means[s * K], &adj[(size_t)s * M]);
  }
  if (!rc) rc = oracle_rollout(p, S, x0s, means, eps, 0, M, adj, costs, NULL, err);
  /* controllers.cpp:130-131 (MPPI); :248-252 (Tube: both weights, then both updates). */
  for (int s = 0; !rc && s < S; ++s) {
    smpc_weight_summary* sm = &summaries[s];
    rc = oracle_compute_weights(&costs[(size_t)s * M], M, p->lambda, w, &sm->baseline,
                                &sm->normalizer, &sm->argmin, err);
    if (rc) break;
    int64_t nz = 0;
    for (int m = 0; m < M; ++m) nz += w[m] != 0.0;
    sm->nonzero = nz;
    rc = oracle_weighted_update(&means[s * K], T, n_u, eps, M, w, p->step_sizes, p->n_step_sizes,
                                updated, err);
    if (rc) break;
    if (s == 0 && last_weights) memcpy(last_weights, w, sizeof(double) * M);
    memcpy(&means[s * K], updated, sizeof(float) * K);
  }
  free(eps);
  free(adj);
  free(costs);
  free(w);
  free(updated);
  return rc;
}

/* The CEM comparator (controllers.cpp:165-171): cost, then lower index. */
static const double* g_sort_costs; /* qsort has no context argument; test-only, single-threaded */
static int cem_cmp(const void* pa, const void* pb) {
  const int64_t a = *(const int64_t*)pa, b = *(const int64_t*)pb;
  const double ca = g_sort_costs[a], cb = g_sort_costs[b];
  if (ca != cb) return ca < cb ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* std::partial_sort(order, order + k, order + n, cmp) (controllers.cpp:165-171):
 * the comparator is a strict total order, so the first k of a full sort are
 * exactly partial_sort's first k. */
void oracle_partial_sort(const double* costs, int64_t n, int64_t k, int64_t* order_out) {
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  g_sort_costs = costs;
  qsort(order, (size_t)n, sizeof(int64_t), cem_cmp);
  memcpy(order_out, order, sizeof(int64_t) * (size_t)k);
  free(order);
}

/* One CemController iteration (controllers.cpp:153-199): rollout without the
 * importance adjustment, elite average of the noise in sorted-elite order. */
static int iterate_cem(const smpc_problem* p, const oracle_dims* d, const float* x0, float* mean,
                       uint32_t stream, double* weights, smpc_weight_summary* sm, oracle_error* err) {
  const int M = p->num_samples, T = p->horizon, n_u = d->n_u;
  const size_t K = (size_t)T * n_u;
  float* eps = (float*)malloc(sizeof(float) * (size_t)M * K);
  double* costs = (double*)malloc(sizeof(double) * (size_t)M);
  int rc = oracle_generate_samples(p, mean, 0, M, stream, eps, NULL, err);
  if (!rc) rc = oracle_rollout(p, 1, x0, mean, eps, 0, M, NULL, costs, NULL, err);
  if (!rc) {
    int k = (int)ceil(p->elite_fraction * M); /* std::max(1, (int)std::ceil(f * M)) (:164) */
    if (k < 1) k = 1;
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    oracle_partial_sort(costs, M, k, order);
    double* acc = (double*)calloc(K, sizeof(double));
    for (int i = 0; i < k; ++i) {
      const float* row = &eps[(size_t)order[i] * K];
      for (size_t j = 0; j < K; ++j) acc[j] += row[j];
    }
    for (size_t j = 0; j < K; ++j) mean[j] = (float)(mean[j] + acc[j] / k);
    sm->baseline = costs[order[0]];
    sm->normalizer = (double)k;
    sm->argmin = order[0];
    sm->nonzero = k;
    if (weights) {
      for (int m = 0; m < M; ++m) weights[m] = 0.0;
      for (int i = 0; i < k; ++i) weights[order[i]] = 1.0 / k;
    }
    free(acc);
    free(order);
  }
  free(eps);
  free(costs);
  return rc;
}

/* MppiController::compute_control (controllers.cpp:113-135); CemController
 * (controllers.cpp:149-203) when p->controller_kind == SMPC_CTRL_CEM. */
int oracle_compute_control(const smpc_problem* p, float* mean, uint64_t* solve_count,
                           const float* x0, float* controls, float* states, float* outputs,
                           double* weights, smpc_weight_summary* summary, oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  const size_t K = (size_t)p->horizon * d.n_u;
  smpc_weight_summary sm = {0};
  for (int iter = 0; iter < p->iterations; ++iter) {
    const uint32_t stream = (uint32_t)(*solve_count * 256u + (uint64_t)iter); /* :63-66 */
    const int rc = p->controller_kind == SMPC_CTRL_CEM
                       ? iterate_cem(p, &d, x0, mean, stream, weights, &sm, err)
                       : iterate(p, &d, 1, x0, mean, stream, weights, &sm, err);
    if (rc) return rc;
  }
  ++*solve_count;
  if (summary) *summary = sm;
  if (controls) memcpy(controls, mean, sizeof(float) * K);
  return finish_solution(p, &d, mean, x0, states, outputs, err);
}

/* TubeMppiController::tube_compute_control (controllers.cpp:219-279) minus PID. */
int oracle_tube_compute_control(const smpc_problem* p, float* nominal_mean, float* real_mean,
                                float* nominal_state, int32_t* nominal_started,
                                uint64_t* solve_count, const float* x_real,
                                float* nominal_controls, float* nominal_states,
                                float* real_controls, float* real_states,
                                smpc_weight_summary* nominal_summary,
                                smpc_weight_summary* real_summary, oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  const size_t K = (size_t)p->horizon * d.n_u;
  if (!*nominal_started) {
    memcpy(nominal_state, x_real, sizeof(float) * d.n_x);
    *nominal_started = 1;
  } else if (isfinite(p->nominal_reset_bound)) {
    float acc = 0.0f; /* Eigen norm() of the float difference (controllers.cpp:225) */
    for (int i = 0; i < d.n_x; ++i) {
      const float diff = x_real[i] - nominal_state[i];
      acc += diff * diff;
    }
    if ((double)sqrtf(acc) > p->nominal_reset_bound)
      memcpy(nominal_state, x_real, sizeof(float) * d.n_x);
  }
  float* means = (float*)malloc(sizeof(float) * 2 * K);
  memcpy(means, nominal_mean, sizeof(float) * K);
  memcpy(means + K, real_mean, sizeof(float) * K);
  float x0s[2 * KMAX];
  memcpy(x0s, nominal_state, sizeof(float) * d.n_x);
  memcpy(x0s + d.n_x, x_real, sizeof(float) * d.n_x);
  smpc_weight_summary sm[2] = {{0}, {0}};
  int rc = 0;
  for (int iter = 0; !rc && iter < p->iterations; ++iter) {
    const uint32_t stream = (uint32_t)(*solve_count * 256u + (uint64_t)iter);
    rc = iterate(p, &d, 2, x0s, means, stream, NULL, sm, err);
  }
  if (rc) {
    free(means);
    return rc;
  }
  ++*solve_count;
  memcpy(nominal_mean, means, sizeof(float) * K);
  memcpy(real_mean, means + K, sizeof(float) * K);
  free(means);
  if (nominal_summary) *nominal_summary = sm[0];
  if (real_summary) *real_summary = sm[1];
  if (nominal_controls) memcpy(nominal_controls, nominal_mean, sizeof(float) * K);
  if (real_controls) memcpy(real_controls, real_mean, sizeof(float) * K);
  rc = finish_solution(p, &d, nominal_mean, nominal_state, nominal_states, NULL, err);
  if (!rc) rc = finish_solution(p, &d, real_mean, x_real, real_states, NULL, err);
  if (rc) return rc;
  /* nominal_state_ = dynamics_->step(nominal_state_, mean_.at(0), dt).first (:276-277) */
  float xn[KMAX], y[KMAX];
  step_raw(p, &d, nominal_state, nominal_mean, (float)p->dt, xn, y);
  memcpy(nominal_state, xn, sizeof(float) * d.n_x);
  return 0;
}

/* DynamicsModel::clamp_control (dynamics.cpp:31-39) and wrap_angle (types.hpp:36-42) for the closed-loop checker. */
void oracle_clamp_control(const smpc_problem* p, const float* u, float* out) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, NULL)) return;
  clamp_control(p, u, out, d.n_u);
}
float oracle_wrap_angle(float a) { return wrap_angle(a); }
int oracle_angular_channel(const smpc_problem* p) { return angular_channel(p); }

/* ---- RMPPI (builder-defined: PAPER.md:150-151; device twin smpc_capi.cu /
 * kernels.cuh rmppi_select_kernel + the S = 2 rollout with feedback) ------- */

/* DynamicsModel::interpolate_states (dynamics.cpp:106-120). */
static void interpolate_states(const smpc_problem* p, const oracle_dims* d, const float* a, const float* b,
                               float alpha, float* out) {
  const int ang = angular_channel(p);
  for (int i = 0; i < d->n_x; ++i) out[i] = a[i] + alpha * (b[i] - a[i]);
  if (ang >= 0) out[ang] = wrap_angle(a[ang] + alpha * wrap_angle(b[ang] - a[ang]));
}

/* Cost of the mean rolled out from z (running + terminal; non-finite -> inf). */
static double mean_trajectory_cost(const smpc_problem* p, const oracle_dims* d, const float* z, const float* mean) {
  float x[KMAX], xn[KMAX], y[KMAX];
  memcpy(x, z, sizeof(float) * d->n_x);
  double total = 0.0;
  for (int t = 0; t < p->horizon; ++t) {
    step_raw(p, d, x, &mean[(size_t)t * d->n_u], (float)p->dt, xn, y);
    total += running_cost(p, y);
    memcpy(x, xn, sizeof(float) * d->n_x);
  }
  const double J = total + terminal_cost(p, y);
  return J == J ? J : INFINITY;
}

int oracle_rmppi_compute_control(const smpc_problem* p, float* mean, float* nominal_state,
                                 int32_t* nominal_started, uint64_t* solve_count, const float* x_real,
                                 float* controls, float* nominal_states, float* real_states,
                                 float* chosen_nominal, int32_t* choice, smpc_weight_summary* summary,
                                 oracle_error* err) {
  oracle_dims d;
  if (oracle_dims_of(p, &d, err)) return SMPC_ERR_CONFIG;
  const int M = p->num_samples, T = p->horizon, n_u = d.n_u, n_x = d.n_x;
  const size_t K = (size_t)T * n_u;
  float prev[KMAX], z[KMAX];
  memcpy(prev, *nominal_started ? nominal_state : x_real, sizeof(float) * n_x);
  *nominal_started = 1;
  /* candidate nominal states: the largest i with J(z_i) <= alpha, else i = 0 */
  const int n = p->num_candidates;
  int best = 0;
  for (int i = n - 1; i > 0; --i) {
    interpolate_states(p, &d, prev, x_real, (float)i / (float)(n - 1), z);
    if (mean_trajectory_cost(p, &d, z, mean) <= p->cost_threshold) {
      best = i;
      break;
    }
  }
  interpolate_states(p, &d, prev, x_real, n > 1 ? (float)best / (float)(n - 1) : 1.0f, z);
  if (chosen_nominal) memcpy(chosen_nominal, z, sizeof(float) * n_x);
  if (choice) *choice = best;
  float* eps = (float*)malloc(sizeof(float) * (size_t)M * K);
  double* costs = (double*)malloc(sizeof(double) * 2 * (size_t)M);
  double* adj = (double*)malloc(sizeof(double) * (size_t)M);
  double* w = (double*)malloc(sizeof(double) * (size_t)M);
  float* updated = (float*)malloc(sizeof(float) * K);
  const float dt = (float)p->dt;
  int rc = 0;
  smpc_weight_summary sm = {0};
  for (int iter = 0; !rc && iter < p->iterations; ++iter) {
    const uint32_t stream = (uint32_t)(*solve_count * 256u + (uint64_t)iter);
    rc = oracle_generate_samples(p, mean, 0, M, stream, eps, NULL, err);
    if (rc) break;
    oracle_importance(p, eps, M, mean, adj); /* both systems sample about the one mean */
    /* coupled rollout: first failure in (system, sample, timestep) order */
    int fail_s = 2, fail_ch = -1, fail_t = -1, fail_kind = 0;
    int64_t fail_m = -1;
    for (int64_t m = 0; m < M; ++m) {
      float xs[2][KMAX], xn[KMAX], y[2][KMAX], u[2][KMAX];
      memcpy(xs[0], z, sizeof(float) * n_x);
      memcpy(xs[1], x_real, sizeof(float) * n_x);
      double total[2] = {0.0, 0.0};
      int dead[2] = {0, 0};
      for (int t = 0; t < T; ++t) {
        const float* e = &eps[((size_t)m * T + t) * n_u];
        for (int c = 0; c < n_u; ++c) {
          float fb = 0.0f;
          if (p->feedback_gain)
            for (int j = 0; j < n_x; ++j) fb += p->feedback_gain[c * n_x + j] * (xs[1][j] - xs[0][j]);
          u[0][c] = mean[(size_t)t * n_u + c] + e[c];
          u[1][c] = u[0][c] + fb;
        }
        for (int s = 0; s < 2; ++s) {
          step_raw(p, &d, xs[s], u[s], dt, xn, y[s]);
          const double ct = running_cost(p, y[s]);
          if (!dead[s]) {
            int ch = -1;
            for (int c = n_x - 1; c >= 0; --c)
              if (!isfinite(xn[c])) ch = c;
            if (ch >= 0 || !(ct >= 0.0 && isfinite(ct))) {
              dead[s] = 1;
              if (s < fail_s || (s == fail_s && m < fail_m)) {
                fail_s = s, fail_m = m, fail_t = t, fail_ch = ch, fail_kind = ch >= 0 ? 0 : 1;
              }
            }
          }
          total[s] += ct;
          memcpy(xs[s], xn, sizeof(float) * n_x);
        }
      }
      for (int s = 0; s < 2; ++s) {
        double J = total[s] + terminal_cost(p, y[s]);
        if (p->importance_sampling) J += adj[m];
        costs[(size_t)s * M + m] = J;
      }
    }
    if (fail_s < 2) {
      rc = rollout_error(err, fail_kind ? "invalid running cost" : NULL, fail_kind ? -1 : fail_ch, fail_m, fail_t);
      break;
    }
    /* one control sequence, updated with the real (feedback) system's weights */
    rc = oracle_compute_weights(&costs[M], M, p->lambda, w, &sm.baseline, &sm.normalizer, &sm.argmin, err);
    if (rc) break;
    int64_t nz = 0;
    for (int m = 0; m < M; ++m) nz += w[m] != 0.0;
    sm.nonzero = nz;
    rc = oracle_weighted_update(mean, T, n_u, eps, M, w, p->step_sizes, p->n_step_sizes, updated, err);
    if (rc) break;
    memcpy(mean, updated, sizeof(float) * K);
  }
  free(eps);
  free(costs);
  free(adj);
  free(w);
  free(updated);
  if (rc) return rc;
  ++*solve_count;
  if (summary) *summary = sm;
  if (controls) memcpy(controls, mean, sizeof(float) * K);
  rc = finish_solution(p, &d, mean, z, nominal_states, NULL, err);
  if (!rc) rc = finish_solution(p, &d, mean, x_real, real_states, NULL, err);
  if (rc) return rc;
  float xn[KMAX], y[KMAX];
  step_raw(p, &d, z, mean, dt, xn, y); /* the nominal system advances through the model */
  memcpy(nominal_state, xn, sizeof(float) * n_x);
  return 0;
}

/* CostFunction::running_cost_raw / terminal_cost_raw (costs.hpp:24-25) for unit tests. */
double oracle_running_cost(const smpc_problem* p, const float* y) { return running_cost(p, y); }
double oracle_terminal_cost(const smpc_problem* p, const float* y) { return terminal_cost(p, y); }
