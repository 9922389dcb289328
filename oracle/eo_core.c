/* eo_core.c -- TEST INFRASTRUCTURE (parity oracle, see evorl_oracle.h).
 * RNG, environments, MLP forward, observation normalisation, optimizers.
 * Restates proj/src/rng.cpp, env.cpp, net.cpp, obs_norm.cpp, optim.cpp. */
#define _GNU_SOURCE
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "evorl_oracle.h"

static __thread char g_err[512];

const char* eo_last_error(void) { return g_err; }

int eo_set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

/* ================================================================== rng */
/* proj/src/rng.cpp:9-10 */
static const uint64_t kParity = 0x1BD11BDAA9FC1A22ull;
static const int kRot[8] = {16, 42, 12, 31, 16, 32, 24, 21};

static inline uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

/* proj/src/rng.cpp:18-34 */
void eo_threefry2x64(const uint64_t key[2], const uint64_t ctr[2], uint64_t out[2]) {
  const uint64_t ks[3] = {key[0], key[1], kParity ^ key[0] ^ key[1]};
  uint64_t x0 = ctr[0] + ks[0];
  uint64_t x1 = ctr[1] + ks[1];
  for (int r = 0; r < 20; ++r) {
    x0 += x1;
    x1 = rotl64(x1, kRot[r % 8]);
    x1 ^= x0;
    if ((r + 1) % 4 == 0) {
      const uint64_t j = (uint64_t)(r + 1) / 4;
      x0 += ks[j % 3];
      x1 += ks[(j + 1) % 3] + j;
    }
  }
  out[0] = x0;
  out[1] = x1;
}

/* proj/src/rng.cpp:36-41 */
eo_key eo_key_from_seed(uint64_t seed) {
  const uint64_t k[2] = {0x9E3779B97F4A7C15ull, 0xBB67AE8584CAA73Bull};
  const uint64_t c[2] = {0, seed};
  uint64_t o[2];
  eo_threefry2x64(k, c, o);
  eo_key r = {o[0], o[1]};
  return r;
}

/* proj/src/rng.cpp:43-46 */
eo_key eo_fold_in(eo_key key, uint64_t index) {
  const uint64_t k[2] = {key.hi, key.lo};
  const uint64_t c[2] = {0, index};
  uint64_t o[2];
  eo_threefry2x64(k, c, o);
  eo_key r = {o[0], o[1]};
  return r;
}

void eo_stream_init(eo_stream* s, eo_key key) {
  memset(s, 0, sizeof *s);
  s->key = key;
}

/* proj/src/rng.cpp:54-63 */
uint64_t eo_next_u64(eo_stream* s) {
  if (s->has_pending_word) {
    s->has_pending_word = 0;
    return s->pending_word;
  }
  const uint64_t k[2] = {s->key.hi, s->key.lo};
  const uint64_t c[2] = {1, s->block++};
  uint64_t o[2];
  eo_threefry2x64(k, c, o);
  s->pending_word = o[1];
  s->has_pending_word = 1;
  return o[0];
}

/* proj/src/rng.cpp:65-72 */
double eo_uniform(eo_stream* s) { return (double)(eo_next_u64(s) >> 11) * 0x1.0p-53; }
double eo_uniform_range(eo_stream* s, double lo, double hi) {
  return lo + (hi - lo) * eo_uniform(s);
}

/* proj/src/rng.cpp:74-87 */
double eo_normal(eo_stream* s) {
  if (s->has_pending_normal) {
    s->has_pending_normal = 0;
    return s->pending_normal;
  }
  const double u1 = (double)((eo_next_u64(s) >> 11) + 1) * 0x1.0p-53;
  const double u2 = eo_uniform(s);
  const double r = sqrt(-2.0 * log(u1));
  const double a = 2.0 * M_PI * u2;
  s->pending_normal = r * sin(a);
  s->has_pending_normal = 1;
  return r * cos(a);
}

/* proj/src/rng.cpp:89-96 */
uint64_t eo_randint(eo_stream* s, uint64_t n) {
  const uint64_t m = (~(uint64_t)0 % n + 1) % n; /* 2^64 mod n */
  for (;;) {
    const uint64_t x = eo_next_u64(s);
    if (m == 0 || x < (uint64_t)0 - m) return x % n;
  }
}

/* proj/src/ec.cpp:22-28 */
void eo_gaussian_matrix(eo_key key, int64_t rows, int64_t cols, double* out) {
  eo_stream st;
  eo_stream_init(&st, key);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) out[r * cols + c] = eo_normal(&st);
}

/* ================================================================== env */
/* proj/src/env.cpp:10-25 */
#define kGravity 9.8
#define kCartMass 1.0
#define kPoleMass 0.1
#define kTotalMass (kCartMass + kPoleMass)
#define kPoleHalfLength 0.5
#define kPoleMassLength (kPoleMass * kPoleHalfLength)
#define kForceMag 10.0
#define kCartDt 0.02
#define kXLimit 2.4
#define kThetaLimit (12.0 * M_PI / 180.0)
#define kPenG 10.0
#define kPenDt 0.05
#define kMaxSpeed 8.0
#define kMaxTorque 2.0

static inline double clampd(double x, double lo, double hi) {
  /* std::clamp semantics: v < lo ? lo : hi < v ? hi : v */
  return x < lo ? lo : (hi < x ? hi : x);
}

/* proj/src/env.cpp:28-32 */
static double wrap_angle(double th) {
  double w = fmod(th + M_PI, 2.0 * M_PI);
  if (w <= 0.0) w += 2.0 * M_PI;
  return w - M_PI;
}

/* proj/src/env.cpp:46-51 */
void eo_pendulum_physics(double* th, double* thdot, double torque, double dt) {
  *thdot += (1.5 * kPenG * sin(*th) + 3.0 * torque) * dt;
  *thdot = clampd(*thdot, -kMaxSpeed, kMaxSpeed);
  *th += *thdot * dt;
}

/* proj/src/env.cpp:55-81 */
eo_env_spec eo_env_cartpole(int fixed_horizon, int max_episode_steps) {
  eo_env_spec s;
  memset(&s, 0, sizeof s);
  s.id = EO_CARTPOLE;
  s.obs_dim = 4;
  s.discrete = 1;
  s.num_actions = 2;
  s.act_dim = 1;
  s.act_low = 0.0;
  s.act_high = 0.0;
  s.max_episode_steps = max_episode_steps > 0 ? max_episode_steps : 500;
  s.fixed_horizon = fixed_horizon;
  return s;
}

eo_env_spec eo_env_pendulum(int fixed_horizon, int max_episode_steps) {
  eo_env_spec s;
  memset(&s, 0, sizeof s);
  s.id = EO_PENDULUM;
  s.obs_dim = 3;
  s.discrete = 0;
  s.num_actions = 0;
  s.act_dim = 1;
  s.act_low = -kMaxTorque;
  s.act_high = kMaxTorque;
  s.max_episode_steps = max_episode_steps > 0 ? max_episode_steps : 200;
  s.fixed_horizon = fixed_horizon;
  return s;
}

/* proj/src/env.cpp:87-97 */
void eo_observe(const eo_env_spec* spec, const eo_env_state* s, double obs[4]) {
  if (spec->id == EO_CARTPOLE) {
    for (int i = 0; i < 4; ++i) obs[i] = s->phys[i];
  } else {
    obs[0] = cos(s->phys[0]);
    obs[1] = sin(s->phys[0]);
    obs[2] = s->phys[1];
    obs[3] = 0.0;
  }
}

/* proj/src/env.cpp:99-111 */
void eo_env_reset(const eo_env_spec* spec, eo_key key, eo_env_state* out, double obs[4]) {
  eo_stream st;
  eo_stream_init(&st, eo_fold_in(key, 0));
  memset(out, 0, sizeof *out);
  if (spec->id == EO_CARTPOLE) {
    for (int i = 0; i < 4; ++i) out->phys[i] = eo_uniform_range(&st, -0.05, 0.05);
  } else {
    out->phys[0] = eo_uniform_range(&st, -M_PI, M_PI);
    out->phys[1] = eo_uniform_range(&st, -1.0, 1.0);
  }
  out->step_count = 0;
  out->rng = eo_fold_in(key, 1);
  if (obs) eo_observe(spec, out, obs);
}

/* proj/src/env.cpp:113-155 */
int eo_env_step(const eo_env_spec* spec, const eo_env_state* s, const double* action,
                eo_env_state* next_out, double* reward, int* terminated, int* truncated,
                double obs[4]) {
  const int nphys = spec->id == EO_CARTPOLE ? 4 : 2;
  /* check_finite, proj/src/env.cpp:34-42 */
  for (int i = 0; i < nphys; ++i)
    if (!isfinite(s->phys[i]))
      return eo_set_error(EO_E_ENV_FAULT,
                          "env_step: non-finite state value (numeric divergence)");
  for (int i = 0; i < spec->act_dim; ++i)
    if (!isfinite(action[i]))
      return eo_set_error(EO_E_ENV_FAULT,
                          "env_step: non-finite action value (numeric divergence)");
  eo_env_state next = *s;
  double r = 0.0;
  int term = 0;
  if (spec->id == EO_CARTPOLE) {
    const double force = action[0] > 0.5 ? kForceMag : -kForceMag;
    const double x = s->phys[0], xdot = s->phys[1];
    const double th = s->phys[2], thdot = s->phys[3];
    const double costh = cos(th), sinth = sin(th);
    const double temp = (force + kPoleMassLength * thdot * thdot * sinth) / kTotalMass;
    const double thacc = (kGravity * sinth - costh * temp) /
                         (kPoleHalfLength * (4.0 / 3.0 - kPoleMass * costh * costh / kTotalMass));
    const double xacc = temp - kPoleMassLength * thacc * costh / kTotalMass;
    next.phys[0] = x + kCartDt * xdot;
    next.phys[1] = xdot + kCartDt * xacc;
    next.phys[2] = th + kCartDt * thdot;
    next.phys[3] = thdot + kCartDt * thacc;
    r = 1.0;
    if (!spec->fixed_horizon)
      term = fabs(next.phys[0]) > kXLimit || fabs(next.phys[2]) > kThetaLimit;
  } else {
    const double u = clampd(action[0], -kMaxTorque, kMaxTorque);
    const double th = s->phys[0], thdot = s->phys[1];
    const double w = wrap_angle(th);
    r = -(w * w + 0.1 * thdot * thdot + 0.001 * u * u);
    next.phys[0] = th;
    next.phys[1] = thdot;
    eo_pendulum_physics(&next.phys[0], &next.phys[1], u, kPenDt);
  }
  next.step_count = s->step_count + 1;
  const int trunc = next.step_count >= spec->max_episode_steps && !term;
  for (int i = 0; i < nphys; ++i)
    if (!isfinite(next.phys[i]))
      return eo_set_error(EO_E_ENV_FAULT,
                          "env_step: non-finite successor state (numeric divergence)");
  if (obs) eo_observe(spec, &next, obs);
  *next_out = next;
  *reward = r;
  *terminated = term;
  *truncated = trunc;
  return EO_OK;
}

/* proj/src/env.cpp:157-175 (one lane; the lane index inside batched_step is
 * always 0 when called from rollout_lane, proj/src/rollout.cpp:131) */
int eo_env_step_autoreset(const eo_env_spec* spec, eo_env_state* s, const double* action,
                          double* reward, int* terminated, int* truncated, double obs[4],
                          double final_obs[4]) {
  eo_env_state next;
  double o[4];
  int rc = eo_env_step(spec, s, action, &next, reward, terminated, truncated, o);
  if (rc != EO_OK) {
    char msg[512];
    snprintf(msg, sizeof msg, "%s [lane 0]", eo_last_error());
    return eo_set_error(rc, "%s", msg);
  }
  if (final_obs) memcpy(final_obs, o, sizeof o);
  if (*terminated || *truncated) {
    eo_env_state fresh;
    eo_env_reset(spec, next.rng, &fresh, o);
    next = fresh;
  }
  *s = next;
  if (obs) memcpy(obs, o, sizeof o);
  return EO_OK;
}

/* ================================================================== net */
/* proj/src/net.cpp:26-48 */
int eo_param_layout(const eo_mlp_spec* spec, eo_segment* segs, int max_segs, int64_t* total) {
  if (spec->n_hidden <= 0 && !spec->allow_linear)
    return -eo_set_error(EO_E_INVALID_ARGUMENT, "MlpSpec.hidden must be nonempty");
  int dims[EO_MAX_HIDDEN + 2];
  int nd = 0;
  dims[nd++] = spec->input_dim;
  for (int i = 0; i < spec->n_hidden; ++i) dims[nd++] = spec->hidden[i];
  dims[nd++] = spec->output_dim;
  const int nlayers = nd - 1;
  int64_t off = 0;
  int ns = 0;
#define PUSH(L, K, R, C)                                             \
  do {                                                               \
    if (ns < max_segs && segs) {                                     \
      segs[ns].layer = (L);                                          \
      segs[ns].kind = (K);                                           \
      segs[ns].offset = off;                                         \
      segs[ns].rows = (R);                                           \
      segs[ns].cols = (C);                                           \
    }                                                                \
    ++ns;                                                            \
    off += (int64_t)(R) * (C);                                       \
  } while (0)
  for (int l = 0; l < nlayers; ++l) {
    const int fan_in = dims[l], fan_out = dims[l + 1];
    PUSH(l, 0, fan_out, fan_in);
    PUSH(l, 1, fan_out, 1);
    if (spec->layer_norm && l < nlayers - 1) {
      PUSH(l, 2, fan_out, 1);
      PUSH(l, 3, fan_out, 1);
    }
  }
  if (spec->head == EO_HEAD_GAUSSIAN) PUSH(nlayers, 4, spec->output_dim, 1);
#undef PUSH
  if (total) *total = off;
  return ns;
}

int64_t eo_param_count(const eo_mlp_spec* spec) {
  int64_t total = 0;
  if (eo_param_layout(spec, NULL, 0, &total) < 0) return -1;
  return total;
}

/* proj/src/net.cpp:52-68 */
int eo_init_params(const eo_mlp_spec* spec, eo_key key, double* p) {
  eo_segment segs[4 * (EO_MAX_HIDDEN + 2) + 1];
  int64_t total;
  const int ns = eo_param_layout(spec, segs, (int)(sizeof segs / sizeof segs[0]), &total);
  if (ns < 0) return -ns;
  memset(p, 0, sizeof(double) * (size_t)total);
  eo_stream st;
  eo_stream_init(&st, key);
  for (int i = 0; i < ns; ++i) {
    const eo_segment* s = &segs[i];
    if (s->kind == 0) {
      const double limit = sqrt(6.0 / (s->cols + s->rows));
      for (int c = 0; c < s->cols; ++c)
        for (int r = 0; r < s->rows; ++r)
          p[s->offset + (int64_t)c * s->rows + r] = eo_uniform_range(&st, -limit, limit);
    } else if (s->kind == 2) {
      for (int r = 0; r < s->rows; ++r) p[s->offset + r] = 1.0;
    }
  }
  return EO_OK;
}

#define kLnEps 1e-5

/* proj/src/net.cpp:77-136 for a single row.  GEMV accumulation is sequential
 * in the column index (Eigen's order is unpinned). */
int eo_forward(const eo_mlp_spec* spec, const double* params, const double* xin, double* out) {
  eo_segment segs[4 * (EO_MAX_HIDDEN + 2) + 1];
  int64_t total;
  const int ns = eo_param_layout(spec, segs, (int)(sizeof segs / sizeof segs[0]), &total);
  if (ns < 0) return -ns;
  int dims[EO_MAX_HIDDEN + 2];
  int nd = 0;
  dims[nd++] = spec->input_dim;
  for (int i = 0; i < spec->n_hidden; ++i) dims[nd++] = spec->hidden[i];
  dims[nd++] = spec->output_dim;
  const int nlayers = nd - 1;
  int maxw = 0;
  for (int i = 0; i < nd; ++i)
    if (dims[i] > maxw) maxw = dims[i];
  double* x = (double*)malloc(sizeof(double) * (size_t)maxw);
  double* z = (double*)malloc(sizeof(double) * (size_t)maxw);
  for (int i = 0; i < dims[0]; ++i) x[i] = xin[i];
  int si = 0;
  for (int l = 0; l < nlayers; ++l) {
    const eo_segment* sw = &segs[si++];
    const eo_segment* sb = &segs[si++];
    const double* w = params + sw->offset;
    const double* b = params + sb->offset;
    const int rows = sw->rows, cols = sw->cols;
    for (int r = 0; r < rows; ++r) {
      double acc = 0.0;
      for (int c = 0; c < cols; ++c) acc += w[(int64_t)c * rows + r] * x[c];
      z[r] = acc + b[r];
    }
    const int hidden = l < nlayers - 1;
    if (hidden) {
      if (spec->layer_norm) {
        const double* gain = params + segs[si++].offset;
        const double* offs = params + segs[si++].offset;
        double mean = 0.0;
        for (int r = 0; r < rows; ++r) mean += z[r];
        mean /= rows;
        double var = 0.0;
        for (int r = 0; r < rows; ++r) var += (z[r] - mean) * (z[r] - mean);
        var /= rows;
        const double inv_std = 1.0 / sqrt(var + kLnEps);
        for (int r = 0; r < rows; ++r) z[r] = ((z[r] - mean) * inv_std) * gain[r] + offs[r];
      }
      for (int r = 0; r < rows; ++r) x[r] = z[r] > 0.0 ? z[r] : 0.0; /* cwiseMax(0) */
    } else {
      for (int r = 0; r < rows; ++r) x[r] = z[r];
    }
    for (int r = 0; r < rows; ++r)
      if (!isfinite(x[r])) {
        free(x);
        free(z);
        return eo_set_error(EO_E_NET_FAULT, "forward: non-finite activations at layer %d", l);
      }
  }
  const int od = dims[nd - 1];
  if (spec->head == EO_HEAD_TANH) {
    for (int i = 0; i < od; ++i) out[i] = spec->tanh_scale * tanh(x[i]);
  } else {
    for (int i = 0; i < od; ++i) out[i] = x[i];
  }
  free(x);
  free(z);
  return EO_OK;
}

/* proj/src/workflow.cpp:87-101 */
eo_mlp_spec eo_policy_net_spec(const eo_env_spec* env, const int* hidden, int n_hidden,
                               int layer_norm) {
  eo_mlp_spec s;
  memset(&s, 0, sizeof s);
  s.input_dim = env->obs_dim;
  s.n_hidden = n_hidden;
  for (int i = 0; i < n_hidden && i < EO_MAX_HIDDEN; ++i) s.hidden[i] = hidden[i];
  s.layer_norm = layer_norm;
  s.tanh_scale = 1.0;
  s.min_logstd = -20.0;
  s.max_logstd = 2.0;
  if (env->discrete) {
    s.output_dim = env->num_actions;
    s.head = EO_HEAD_CATEGORICAL;
  } else {
    s.output_dim = env->act_dim;
    s.head = EO_HEAD_TANH;
    s.tanh_scale = env->act_high;
  }
  return s;
}

/* ============================================================ obs norm */
/* proj/src/obs_norm.cpp:7-18 */
void eo_welford_add(eo_welford* w, const double* row, int dim) {
  if (w->count == 0.0) {
    w->dim = dim;
    for (int i = 0; i < dim; ++i) {
      w->mean[i] = row[i];
      w->m2[i] = 0.0;
    }
    w->count = 1.0;
    return;
  }
  w->count += 1.0;
  for (int i = 0; i < dim; ++i) {
    const double delta = row[i] - w->mean[i];
    w->mean[i] += delta / w->count;
    w->m2[i] += delta * (row[i] - w->mean[i]);
  }
}

/* proj/src/obs_norm.cpp:20-31 */
void eo_welford_merge(eo_welford* w, const eo_welford* o) {
  if (o->count == 0.0) return;
  if (w->count == 0.0) {
    *w = *o;
    return;
  }
  const double total = w->count + o->count;
  const double s = w->count * o->count / total;
  const double f = o->count / total;
  for (int i = 0; i < w->dim; ++i) {
    const double delta = o->mean[i] - w->mean[i];
    w->m2[i] += o->m2[i] + delta * delta * s;
    w->mean[i] += delta * f;
  }
  w->count = total;
}

void eo_welford_variance(const eo_welford* w, double* var) {
  for (int i = 0; i < w->dim; ++i) var[i] = w->count == 0.0 ? w->mean[i] : w->m2[i] / w->count;
}

eo_obs_norm eo_obs_norm_none(void) {
  eo_obs_norm s;
  memset(&s, 0, sizeof s);
  s.mode = EO_NORM_NONE;
  return s;
}

/* proj/src/obs_norm.cpp:38-45 */
eo_obs_norm eo_obs_norm_running_stats(int dim) {
  eo_obs_norm s;
  memset(&s, 0, sizeof s);
  s.mode = EO_NORM_RS;
  s.dim = dim;
  for (int i = 0; i < dim; ++i) {
    s.mean[i] = 0.0;
    s.var[i] = 1.0;
  }
  s.count = 0.0;
  return s;
}

/* proj/src/obs_norm.cpp:47-54 */
eo_obs_norm eo_obs_norm_from_stats(int mode, const eo_welford* w) {
  eo_obs_norm s;
  memset(&s, 0, sizeof s);
  s.mode = mode;
  s.dim = w->dim;
  for (int i = 0; i < w->dim; ++i) s.mean[i] = w->mean[i];
  eo_welford_variance(w, s.var);
  s.count = w->count;
  return s;
}

/* proj/src/obs_norm.cpp:56-68 */
void eo_rs_update(eo_obs_norm* s, const eo_welford* batch) {
  if (s->mode != EO_NORM_RS || batch->count == 0.0) return;
  eo_welford cur;
  memset(&cur, 0, sizeof cur);
  if (s->count > 0.0) {
    cur.count = s->count;
    cur.dim = s->dim;
    for (int i = 0; i < s->dim; ++i) {
      cur.mean[i] = s->mean[i];
      cur.m2[i] = s->var[i] * s->count;
    }
  }
  eo_welford_merge(&cur, batch);
  s->dim = cur.dim;
  for (int i = 0; i < cur.dim; ++i) s->mean[i] = cur.mean[i];
  eo_welford_variance(&cur, s->var);
  s->count = cur.count;
}

/* proj/src/obs_norm.cpp:76-79 */
void eo_normalize(const eo_obs_norm* s, const double* obs, int dim, double* out) {
  if (s == NULL || s->mode == EO_NORM_NONE || s->count == 0.0) {
    for (int i = 0; i < dim; ++i) out[i] = obs[i];
    return;
  }
  for (int i = 0; i < dim; ++i) {
    const double sd = sqrt(s->var[i]);
    const double den = sd > 1e-8 ? sd : 1e-8; /* Eigen .max(1e-8) */
    out[i] = (obs[i] - s->mean[i]) / den;
  }
}

/* ================================================================ optim */
eo_adam_cfg eo_adam_default(void) {
  eo_adam_cfg c = {1e-3, 0.9, 0.999, 1e-8, 0.0};
  return c;
}

/* proj/src/optim.cpp:7-17 */
void eo_adam_step(double* p, const double* g, double* m, double* v, int64_t* t, int64_t n,
                  const eo_adam_cfg* cfg) {
  *t += 1;
  const double b1 = cfg->beta1, b2 = cfg->beta2;
  const double omb1 = 1.0 - b1, omb2 = 1.0 - b2;
  const double bc1 = 1.0 - pow(b1, (double)*t);
  const double bc2 = 1.0 - pow(b2, (double)*t);
  const double lrwd = cfg->lr * cfg->weight_decay;
  for (int64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + omb1 * g[i];
    v[i] = b2 * v[i] + omb2 * (g[i] * g[i]);
    p[i] -= cfg->lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + cfg->eps);
  }
  if (cfg->weight_decay != 0.0)
    for (int64_t i = 0; i < n; ++i) p[i] -= lrwd * p[i];
}

/* proj/src/optim.cpp:19-21 */
void eo_sgd_step(double* p, const double* g, int64_t n, double lr) {
  for (int64_t i = 0; i < n; ++i) p[i] -= lr * g[i];
}
