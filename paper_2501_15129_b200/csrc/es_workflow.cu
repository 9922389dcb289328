// es_workflow.cu -- device-resident EsWorkflow behind the C ABI
// (include/evorl_b200.h).  Host orchestration of one generation
// (proj/src/workflow_es.cpp:87-172):
//
//   step_key k = fold_in(fold_in(rng, 0), iteration)
//   ask  (implicit: perturbations regenerated in-kernel from fold_in(k, 0))
//   rollout of agents [a0, a1) keyed fold_in(k, 1)          -> K2 rollout
//   fitness reduction                                       -> k_fitness
//   [caller all-gathers fitness across ranks]               (C1)
//   RunningStats merge + rs_update (ARS)                    -> k_rs_update
//   ranks / elites                                          -> k_rank
//   tell on coordinates [p0, p1) (+ Adam for OpenES)        -> K4 tell
//   [caller all-gathers mean slices across ranks]           (C2)
//
// Nothing on this path runs on the CPU except key derivation (two Threefry
// blocks per generation) and launch orchestration; there is no CPU fallback:
// a missing device or a failed launch is an EVORL_E_CUDA error.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "../../include/evorl_b200.h"
#include "cma.cuh"
#include "kernels.cuh"

using namespace evorl_b200;

namespace evorl_b200 {
long long kernel_launch_count();
}

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                       \
  do {                                                                                 \
    cudaError_t _e = (call);                                                           \
    if (_e != cudaSuccess)                                                             \
      return set_err(EVORL_E_CUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(_e), \
                     __FILE__, __LINE__, #call);                                        \
  } while (0)

extern "C" const char* evorl_last_error(void) { return g_err.c_str(); }
extern "C" int evorl_abi_version(void) { return EVORL_B200_ABI_VERSION; }
extern "C" int64_t evorl_kernel_launches(void) { return kernel_launch_count(); }

static DKey mk(uint64_t hi, uint64_t lo) { return DKey{hi, lo}; }

// -------------------------------------------------------- spec builders
static EnvDesc make_env(int env_id, int fixed_horizon, int max_steps) {
  EnvDesc e{};
  e.id = env_id;
  if (env_id == ENV_CARTPOLE) {  // EnvSpec::cartpole, proj/src/env.cpp:55-66
    e.obs_dim = 4;
    e.discrete = 1;
    e.num_actions = 2;
    e.act_dim = 1;
    e.act_low = 0.0;
    e.act_high = 0.0;
    e.max_episode_steps = max_steps > 0 ? max_steps : 500;
  } else {  // EnvSpec::pendulum, proj/src/env.cpp:68-81
    e.obs_dim = 3;
    e.discrete = 0;
    e.num_actions = 0;
    e.act_dim = 1;
    e.act_low = -2.0;
    e.act_high = 2.0;
    e.max_episode_steps = max_steps > 0 ? max_steps : 200;
  }
  e.fixed_horizon = fixed_horizon;
  return e;
}

// param_layout (proj/src/net.cpp:26-48) without layer norm / logstd.
static int make_net(const evorl_mlp_desc& m, NetDesc* out) {
  if (m.layer_norm)
    return set_err(EVORL_E_UNSUPPORTED, "net.layer_norm is not supported on the B200 device path");
  if (m.n_hidden <= 0 && !m.allow_linear) return set_err(EVORL_E_INVALID_ARGUMENT, "MlpSpec.hidden must be nonempty");
  if (m.n_hidden > EVORL_MAX_HIDDEN) return set_err(EVORL_E_INVALID_ARGUMENT, "too many hidden layers");
  if (m.head == EVORL_HEAD_GAUSSIAN)
    return set_err(EVORL_E_UNSUPPORTED, "Gaussian head is not on the ES path");
  NetDesc n{};
  n.nlayers = m.n_hidden + 1;
  n.dims[0] = m.input_dim;
  for (int i = 0; i < m.n_hidden; ++i) n.dims[i + 1] = m.hidden[i];
  n.dims[n.nlayers] = m.output_dim;
  long long off = 0;
  for (int l = 0; l < n.nlayers; ++l) {
    n.w_off[l] = off;
    off += (long long)n.dims[l] * n.dims[l + 1];
    n.b_off[l] = off;
    off += n.dims[l + 1];
  }
  n.d = off;
  n.head = m.head;
  n.tanh_scale = m.tanh_scale;
  *out = n;
  return EVORL_OK;
}

// policy_net_spec (proj/src/workflow.cpp:87-101)
static evorl_mlp_desc policy_net(const EnvDesc& env, const int* hidden, int nh, int allow_linear) {
  evorl_mlp_desc m{};
  m.input_dim = env.obs_dim;
  m.n_hidden = nh;
  for (int i = 0; i < nh && i < EVORL_MAX_HIDDEN; ++i) m.hidden[i] = hidden[i];
  m.allow_linear = allow_linear;
  if (env.discrete) {
    m.output_dim = env.num_actions;
    m.head = EVORL_HEAD_CATEGORICAL;
    m.tanh_scale = 1.0;
  } else {
    m.output_dim = env.act_dim;
    m.head = EVORL_HEAD_TANH;
    m.tanh_scale = env.act_high;
  }
  return m;
}

static int fault_to_error(unsigned long long code) {
  const unsigned kind = (unsigned)((code >> 4) & 15u);
  const unsigned layer = (unsigned)(code & 15u);
  // EnvFault from batched_step inside rollout_lane always carries "[lane 0]"
  // (proj/src/env.cpp:170-172 with a one-state batch, proj/src/rollout.cpp:131)
  switch (kind) {
    case FAULT_ENV_STATE:
      return set_err(EVORL_E_ENV_FAULT, "env_step: non-finite state value (numeric divergence) [lane 0]");
    case FAULT_ENV_ACTION:
      return set_err(EVORL_E_ENV_FAULT, "env_step: non-finite action value (numeric divergence) [lane 0]");
    case FAULT_ENV_SUCCESSOR:
      return set_err(EVORL_E_ENV_FAULT,
                     "env_step: non-finite successor state (numeric divergence) [lane 0]");
    case FAULT_TC_RANGE:
      return set_err(EVORL_E_UNSUPPORTED,
                     "precision tc: an activation of layer %u exceeds the fp16 hi/lo operand range "
                     "(|h| > 60000); use EVORL_PREC_F32 or EVORL_PREC_F64",
                     layer);
    default:
      return set_err(EVORL_E_NET_FAULT, "forward: non-finite activations at layer %u", layer);
  }
}

// ------------------------------------------------------------ the handle
struct Pinned {
  double metrics[3];
  unsigned long long steps;
  unsigned long long fault;
  ArsSel sel;
  double eval[2];
};

struct evorl_es {
  evorl_es_config cfg{};
  EnvDesc env{};
  NetDesc net{};
  int norm_mode = 0;
  long long d = 0;
  int e = 1, count = 1;
  SmemPlan plan{};
  int groups = 1;
  bool warp_path = false;  // small policies: warp-per-lane rollout (rollout_warp.cu)
  WarpPlanOut wplan{};
  double* d_cand = nullptr;  // materialised candidates for the warp path
  // fp32 policy paths (tc / f32 teams): the generation's candidates rounded to
  // fp32, materialised once by a fully parallel ask instead of being
  // regenerated in every CTA's prologue (null: regenerate, e.g. over the cap)
  float* d_cand_f32 = nullptr;
  unsigned char* d_tc_blocks = nullptr;  // tc team: pre-split layer-1 weights (cand_cap agents)
  int cand_cap = 0;               // agents per materialised chunk (team path)
  bool cma_only = false;          // evorl_cma_create: a CmaState of dimension d, no env / policy
  // OpenES noise-table mode (proj/src/ec.cpp:50-86): the shared table and
  // this generation's window offsets
  double* d_table = nullptr;
  long long* d_offsets = nullptr;
  uint64_t table_seed = 0;
  std::vector<long long> h_offsets;
  double* d_tell_part = nullptr;  // OpenES tell: per-row-chunk partial contractions
  long long tell_part_cap = 0;
  // OpenES: this generation's sampled noise rows (base x d), written by the
  // ask when one rank materialises every row, read by the tell instead of
  // regenerating them (valid between phase_rollout and phase_tell)
  double* d_eps_rows = nullptr;
  bool eps_rows_valid = false;
  bool eps_rows_failed = false;
  // ... and the NEXT generation's noise rows, generated beside this rollout on
  // a low-priority stream (one small block per SM next to the team CTA), so
  // the next ask only adds the mean (valid while its key is the next ask key)
  double* d_eps_next = nullptr;
  bool eps_next_valid = false, eps_next_failed = false;
  DKey eps_next_key{};
  long long eps_next_r0 = 0, eps_next_r1 = 0;  // rows the kept-ahead buffer holds
  // coordinate-sharded tell: the noise columns [p0, p1) of every row, generated
  // beside the previous rollout (cur: this generation's tell; next: being filled)
  double *d_cols_cur = nullptr, *d_cols_next = nullptr;
  bool cols_cur_valid = false, cols_next_valid = false, cols_failed = false;
  DKey cols_cur_key{}, cols_next_key{};
  long long cols_cur_p0 = 0, cols_cur_p1 = 0, cols_next_p0 = 0, cols_next_p1 = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_noise = nullptr;
  int n_sms = 0;
  // evorl_es_step_host: pinned staging of the host-resident state (3 d + 1)
  double* h_stage = nullptr;
  cudaStream_t stream = nullptr;
  // WorkflowState (proj/include/evorl/workflow.hpp:31-36)
  DKey rng{};
  long long iteration = 0, env_steps = 0, episodes = 0;
  bool initialised = false;
  // EsState on the device
  double *d_mean = nullptr, *d_m = nullptr, *d_v = nullptr, *d_var = nullptr;
  long long* d_t = nullptr;
  long long adam_t_host = 0;
  long long cem_iter = 0;
  DevNorm* d_norm = nullptr;
  NormParams* d_normp = nullptr;
  // generation buffers
  double *d_fitness = nullptr, *d_ep_returns = nullptr, *d_lane_stats = nullptr, *d_agent_stats = nullptr;
  long long* d_lane_steps = nullptr;
  int *d_rank = nullptr, *d_order = nullptr, *d_elite_idx = nullptr;
  double *d_shaped = nullptr, *d_scores = nullptr, *d_elite_diff = nullptr, *d_metrics = nullptr;
  ArsSel* d_sel = nullptr;
  unsigned long long *d_steps = nullptr, *d_fault = nullptr;
  double* d_adam_bc = nullptr;
  long long adam_bc_len = 0;
  double* d_ves_w = nullptr;
  Pinned* h = nullptr;
  // sharding
  int rank = 0, world = 1, a0 = 0, a1 = 0;
  long long p0 = 0, p1 = 0;
  // timing
  cudaEvent_t ev_r0 = nullptr, ev_r1 = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
  cudaEvent_t ev_a0 = nullptr, ev_a1 = nullptr;  // around the materialised ask (one chunk)
  float last_rollout_ms = 0.f, last_step_ms = 0.f, last_ask_ms = -1.f;
  bool ask_timed = false;
  // per-step keys
  DKey step_key{}, ask_key{}, rollout_key{};
  // CmaState (proj/include/evorl/ec.hpp:107-122): scalars on the host (the
  // reference's std:: math, bit-identical), matrices on the device
  struct {
    int mu = 0;
    std::vector<double> w;
    double mueff = 0, cs = 0, ds = 0, cc = 0, c1 = 0, cmu = 0, chi_n = 0, sigma = 0;
    long long generation = 0, recondition_count = 0;
    int last_sweeps = 0;
    double* d_w = nullptr;
    CmaDev dev{};
  } cma;
};

extern "C" void evorl_es_default_config(evorl_es_config* c) {
  // registry defaults, proj/src/config.cpp:23-70
  std::memset(c, 0, sizeof *c);
  c->algo = EVORL_ALGO_OPENES;
  c->env_id = EVORL_ENV_CARTPOLE;
  c->fixed_horizon = 0;
  c->max_episode_steps = 0;
  c->n_hidden = 2;
  c->hidden[0] = 64;
  c->hidden[1] = 64;
  c->pop = 128;
  c->fitness_episodes = 1;
  c->obs_norm_mode = EVORL_NORM_AUTO;
  c->vbn_samples = 10000;
  c->openes_sigma = 0.02;
  c->openes_lr = 0.01;
  c->openes_weight_decay = 0.005;
  c->openes_mirrored = 1;
  c->openes_noise_table = 0;
  c->openes_noise_table_size = 4194304;
  c->ars_sigma = 0.03;
  c->ars_lr = 0.02;
  c->ars_elites = 16;
  c->ves_sigma = 0.02;
  c->ves_elites = 16;
  c->ves_mirrored = 1;
  c->cmaes_sigma0 = 0.1;
  c->cmaes_elites = 64;
  c->cmaes_max_dim = 4096;
  c->cem_elites = 5;
  c->cem_var_init = 1e-3;
  c->cem_noise_start = 1e-3;
  c->cem_noise_end = 1e-5;
  c->cem_decay_iters = 2000;
  c->precision = EVORL_PREC_F64;
  c->device = 0;
  c->cmaes_eig_every = 1;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, sizeof(T) * (n ? n : 1));
}

static void free_all(evorl_es* s) {
  void* ptrs[] = {s->d_mean, s->d_m, s->d_v, s->d_var, s->d_t, s->d_norm, s->d_normp, s->d_fitness,
                  s->d_ep_returns, s->d_lane_stats, s->d_agent_stats, s->d_lane_steps, s->d_rank,
                  s->d_order, s->d_elite_idx, s->d_shaped, s->d_scores, s->d_elite_diff, s->d_metrics,
                  s->d_sel, s->d_steps, s->d_fault, s->d_adam_bc, s->d_ves_w, s->d_cand,
                  s->d_cand_f32, s->d_tell_part, s->d_table, s->d_offsets, s->d_tc_blocks, s->d_eps_rows,
                  s->d_eps_next, s->d_cols_cur, s->d_cols_next};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (s->h) cudaFreeHost(s->h);
  if (s->h_stage) cudaFreeHost(s->h_stage);
  for (cudaEvent_t ev : {s->ev_r0, s->ev_r1, s->ev_s0, s->ev_s1, s->ev_a0, s->ev_a1, s->ev_noise})
    if (ev) cudaEventDestroy(ev);
  void* cm[] = {s->cma.d_w, s->cma.dev.C, s->cma.dev.B, s->cma.dev.D, s->cma.dev.ps, s->cma.dev.pc,
                s->cma.dev.W, s->cma.dev.V, s->cma.dev.Bt, s->cma.dev.Tt, s->cma.dev.U, s->cma.dev.skipf, s->cma.dev.evals, s->cma.dev.order, s->cma.dev.zD,
                s->cma.dev.ytT, s->cma.dev.wyT, s->cma.dev.yw, s->cma.dev.t1, s->cma.dev.cih, s->cma.dev.red};
  for (void* p : cm)
    if (p) cudaFree(p);
  if (s->stream) cudaStreamDestroy(s->stream);
  if (s->side) cudaStreamDestroy(s->side);
}

static int resolve_norm(const evorl_es_config& c) {  // proj/src/workflow.cpp:131-144
  if (c.obs_norm_mode >= 0) return c.obs_norm_mode;
  if (c.algo == EVORL_ALGO_ARS) return EVORL_NORM_RS;
  if (c.algo == EVORL_ALGO_CEM) return EVORL_NORM_NONE;
  return EVORL_NORM_VBN;
}

static int es_create(const evorl_es_config* cfg, long long forced_d, evorl_es** out);
extern "C" int evorl_es_create(const evorl_es_config* cfg, evorl_es** out) { return es_create(cfg, 0, out); }

static int es_create(const evorl_es_config* cfg, long long forced_d, evorl_es** out) {
  *out = nullptr;
  if (cfg->algo < 0 || cfg->algo > EVORL_ALGO_CEM) return set_err(EVORL_E_CONFIG, "ec.algo: unknown algorithm");
  if (cfg->env_id != EVORL_ENV_CARTPOLE && cfg->env_id != EVORL_ENV_PENDULUM)
    return set_err(EVORL_E_INVALID_ARGUMENT, "unknown env id");
  if (cfg->precision < EVORL_PREC_F64 || cfg->precision > EVORL_PREC_OZ)
    return set_err(EVORL_E_INVALID_ARGUMENT,
                   "precision must be EVORL_PREC_F64, EVORL_PREC_F32, EVORL_PREC_TC or EVORL_PREC_OZ");
  if (cfg->pop < 1 || cfg->fitness_episodes < 1)
    return set_err(EVORL_E_INVALID_ARGUMENT, "ec.pop and ec.fitness_episodes must be positive");
  auto* s = new evorl_es();
  s->cfg = *cfg;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    delete s;
    return set_err(EVORL_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (cudaSetDevice(cfg->device) != cudaSuccess) {
    delete s;
    return set_err(EVORL_E_CUDA, "cudaSetDevice(%d) failed", cfg->device);
  }
  s->env = make_env(cfg->env_id, cfg->fixed_horizon, cfg->max_episode_steps);
  const evorl_mlp_desc md = policy_net(s->env, cfg->hidden, cfg->n_hidden, cfg->allow_linear);
  int rc = make_net(md, &s->net);
  if (rc) {
    delete s;
    return rc;
  }
  s->d = s->net.d;
  if (forced_d > 0) {  // CMA-ES free functions: the state's own dimension
    s->d = forced_d;
    s->cma_only = true;
  }
  const bool table = cfg->algo == EVORL_ALGO_OPENES && cfg->openes_noise_table;
  if (table && cfg->openes_noise_table_size < s->d) {  // the reference's span = size - d would wrap (UB)
    delete s;
    return set_err(EVORL_E_INVALID_ARGUMENT, "openes noise table (%lld entries) smaller than the parameter count (%lld)",
                   (long long)cfg->openes_noise_table_size, (long long)s->net.d);
  }
  s->norm_mode = resolve_norm(*cfg);
  s->e = cfg->fitness_episodes;
  s->count = cfg->fitness_episodes;  // RolloutMode::episodes(fitness_episodes)
  const bool cta_ok = plan_rollout(s->net, s->env.obs_dim, s->e, cfg->precision, &s->plan);
  // warp-per-lane only pays when there are enough lanes to fill the SMs
  // (>= 512 lanes); fewer lanes get a whole CTA each to cut step latency.
  s->warp_path = !(cta_ok && (s->plan.tc || s->plan.oz)) && (long long)cfg->pop * s->e >= 512 &&
                 plan_rollout_warp(s->net, s->env.obs_dim, s->e, cfg->precision, &s->wplan);
  if (!cta_ok && !s->warp_path) {
    delete s;
    return set_err(EVORL_E_UNSUPPORTED, "policy too large for a shared-memory resident team");
  }
  s->groups = (s->e + s->plan.ET - 1) / s->plan.ET;
  s->a0 = 0;
  s->a1 = cfg->pop;
  s->p0 = 0;
  s->p1 = s->d;
  const int n = cfg->pop;
  const long long d = s->d;
#define A(call)                \
  do {                         \
    cudaError_t _e = (call);   \
    if (_e != cudaSuccess) {   \
      free_all(s);             \
      delete s;                \
      return set_err(EVORL_E_CUDA, "allocation failed: %s", cudaGetErrorString(_e)); \
    }                          \
  } while (0)
  {
    // the generation's stream at the highest priority, so the rollout's team
    // CTAs are placed before the low-priority noise-ahead blocks (side stream)
    int least = 0, greatest = 0;
    A(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    A(cudaStreamCreateWithPriority(&s->stream, cudaStreamNonBlocking, greatest));
  }
  A(dalloc(&s->d_mean, d));
  A(dalloc(&s->d_m, d));
  A(dalloc(&s->d_v, d));
  A(dalloc(&s->d_var, d));
  A(dalloc(&s->d_t, 1));
  A(dalloc(&s->d_norm, 1));
  A(dalloc(&s->d_normp, 1));
  A(dalloc(&s->d_fitness, n));
  A(dalloc(&s->d_ep_returns, (size_t)n * s->count));
  A(dalloc(&s->d_lane_stats, (size_t)n * s->e * 9));
  A(dalloc(&s->d_agent_stats, (size_t)n * 9));
  A(dalloc(&s->d_lane_steps, (size_t)n * s->e));
  A(dalloc(&s->d_rank, n));
  A(dalloc(&s->d_order, n));
  A(dalloc(&s->d_elite_idx, n));
  A(dalloc(&s->d_shaped, n));
  A(dalloc(&s->d_scores, n));
  A(dalloc(&s->d_elite_diff, n));
  A(dalloc(&s->d_metrics, 4));
  A(dalloc(&s->d_sel, 1));
  // materialised ask: the warp path always; the CTA teams when the candidate
  // matrix fits the cap (fp32 for the fp32 policy paths, fp64 for parity) --
  // one fully parallel pass instead of every CTA regenerating its slice
  // (chunks of cand_cap agents when the whole population exceeds the cap;
  // the global-weights plan reads its weights from this buffer)
  // (EVORL_CAND_CAP_BYTES overrides the 8 GiB cap -- used by the chunking test)
  static const double kCandCap =
      getenv("EVORL_CAND_CAP_BYTES") ? atof(getenv("EVORL_CAND_CAP_BYTES")) : 8.0 * (1ull << 30);
  const bool team_mat = !s->warp_path && cfg->algo != EVORL_ALGO_CMAES;
  if (s->warp_path) A(dalloc(&s->d_cand, (size_t)n * d));
  if (cfg->algo == EVORL_ALGO_OPENES && cfg->openes_noise_table) {
    A(dalloc(&s->d_table, (size_t)cfg->openes_noise_table_size));
    A(dalloc(&s->d_offsets, (size_t)n));
  }
  if (team_mat) {
    const bool f64 = cfg->precision == EVORL_PREC_F64 || cfg->precision == EVORL_PREC_OZ;  // fp64 candidates
    const size_t tsz = f64 ? sizeof(double) : sizeof(float);
    s->cand_cap = (int)std::max(1.0, std::min((double)n, std::floor(kCandCap / ((double)d * tsz))));
    if (f64) {
      A(dalloc(&s->d_cand, (size_t)s->cand_cap * d));
      if (s->plan.oz)
        A(dalloc(&s->d_tc_blocks, (size_t)s->cand_cap * s->plan.tcp.data[0] * oz_block_bytes(s->plan.tcp)));
    } else {
      A(dalloc(&s->d_cand_f32, (size_t)s->cand_cap * d));
      if (s->plan.tc)
        A(dalloc(&s->d_tc_blocks, (size_t)s->cand_cap * s->plan.tcp.data[0] * tc_block_bytes(s->plan.tcp)));
    }
  }
  if (cfg->algo == EVORL_ALGO_CMAES) {
    // CmaState::init (proj/src/ec.cpp:191-224)
    if (d > cfg->cmaes_max_dim) {
      free_all(s);
      delete s;
      return set_err(EVORL_E_LENGTH,
                     "cmaes: genotype dimension %lld exceeds the full-covariance capacity cap %d",
                     (long long)d, cfg->cmaes_max_dim);
    }
    const int mu = cfg->cmaes_elites;
    if (mu < 1 || mu > n) {  // the reference indexes order[i < mu] unchecked (UB when mu > pop)
      free_all(s);
      delete s;
      return set_err(EVORL_E_INVALID_ARGUMENT, "cmaes_tell: elites (%d) exceed population (%d)", mu, n);
    }
    auto& c = s->cma;
    c.mu = mu;
    c.w.resize(mu);
    double sum = 0.0;
    for (int i = 0; i < mu; ++i) {
      double wi = std::log((cfg->pop + 1) / 2.0) - std::log(i + 1.0);
      if (wi < 0) wi = 0.0;
      c.w[i] = wi;
      sum += wi;
    }
    double sq = 0.0;
    for (int i = 0; i < mu; ++i) {
      c.w[i] /= sum;
      sq += c.w[i] * c.w[i];
    }
    c.mueff = 1.0 / sq;
    const double dd = (double)d;
    c.cs = (c.mueff + 2.0) / (dd + c.mueff + 5.0);
    c.ds = 1.0 + 2.0 * std::max(0.0, std::sqrt((c.mueff - 1.0) / (dd + 1.0)) - 1.0) + c.cs;
    c.cc = (4.0 + c.mueff / dd) / (dd + 4.0 + 2.0 * c.mueff / dd);
    c.c1 = 2.0 / ((dd + 1.3) * (dd + 1.3) + c.mueff);
    c.cmu = std::min(1.0 - c.c1, 2.0 * (c.mueff - 2.0 + 1.0 / c.mueff) / ((dd + 2.0) * (dd + 2.0) + c.mueff));
    c.chi_n = std::sqrt(dd) * (1.0 - 1.0 / (4.0 * dd) + 1.0 / (21.0 * dd * dd));
    CmaDev& v = c.dev;
    v.d = (int)d;
    v.dp = (int)((d + 63) / 64 * 64);
    const size_t dp2 = (size_t)v.dp * v.dp;
    A(dalloc(&c.d_w, mu));
    A(cudaMemcpy(c.d_w, c.w.data(), sizeof(double) * mu, cudaMemcpyHostToDevice));
    A(dalloc(&v.C, dp2));
    A(dalloc(&v.B, dp2));
    A(dalloc(&v.W, dp2));
    A(dalloc(&v.V, dp2));
    A(dalloc(&v.Bt, dp2));
    A(dalloc(&v.Tt, dp2));
    A(dalloc(&v.U, (size_t)(v.dp / 64) * 64 * 64));
    A(dalloc(&v.skipf, (size_t)(v.dp / 64)));
    A(dalloc(&v.D, v.dp));
    A(dalloc(&v.ps, v.dp));
    A(dalloc(&v.pc, v.dp));
    A(dalloc(&v.evals, v.dp));
    A(dalloc(&v.order, v.dp));
    A(dalloc(&v.zD, (size_t)n * d));
    A(dalloc(&v.ytT, (size_t)d * mu));
    A(dalloc(&v.wyT, (size_t)d * mu));
    A(dalloc(&v.yw, v.dp));
    A(dalloc(&v.t1, v.dp));
    A(dalloc(&v.cih, v.dp));
    A(dalloc(&v.red, 8));
    if (!s->d_cand) A(dalloc(&s->d_cand, (size_t)n * d));
  }
  A(dalloc(&s->d_steps, 1));
  A(dalloc(&s->d_fault, 1));
  A(cudaMallocHost((void**)&s->h, sizeof(Pinned)));
  A(cudaEventCreate(&s->ev_r0));
  A(cudaEventCreate(&s->ev_r1));
  A(cudaEventCreate(&s->ev_s0));
  A(cudaEventCreate(&s->ev_s1));
  A(cudaEventCreate(&s->ev_a0));
  A(cudaEventCreate(&s->ev_a1));
  // Adam bias corrections 1 - beta^t with the host libm pow (the reference's
  // std::pow, proj/src/optim.cpp:12-13), t = 1..65536.
  s->adam_bc_len = 65536;
  std::vector<double> bc(2 * s->adam_bc_len);
  for (long long t = 1; t <= s->adam_bc_len; ++t) {
    bc[2 * (t - 1)] = 1.0 - std::pow(0.9, (double)t);
    bc[2 * (t - 1) + 1] = 1.0 - std::pow(0.999, (double)t);
  }
  A(dalloc(&s->d_adam_bc, bc.size()));
  A(cudaMemcpy(s->d_adam_bc, bc.data(), sizeof(double) * bc.size(), cudaMemcpyHostToDevice));
  if (cfg->algo == EVORL_ALGO_VES) {  // canonical_es_weights (proj/src/ec.cpp:158-162)
    const int mu = std::min(cfg->ves_elites, n);
    std::vector<double> w(mu);
    double sum = 0.0;
    for (int i = 0; i < mu; ++i) {
      w[i] = std::log(mu + 0.5) - std::log(i + 1.0);
      sum += w[i];
    }
    for (auto& x : w) x /= sum;
    A(dalloc(&s->d_ves_w, mu));
    A(cudaMemcpy(s->d_ves_w, w.data(), sizeof(double) * mu, cudaMemcpyHostToDevice));
  }
#undef A
  *out = s;
  return EVORL_OK;
}

extern "C" void evorl_es_destroy(evorl_es* s) {
  if (!s) return;
  cudaSetDevice(s->cfg.device);
  cudaStreamSynchronize(s->stream);
  if (s->side) cudaStreamSynchronize(s->side);
  free_all(s);
  delete s;
}

extern "C" int64_t evorl_es_dim(const evorl_es* s) { return s->d; }

static DKey init_key(DKey run, uint64_t i) { return fold_in(fold_in(run, 2), i); }

// key_from_seed (proj/src/rng.cpp:36-41)
static DKey key_from_seed(uint64_t seed) {
  DKey k;
  threefry2x64(0x9E3779B97F4A7C15ull, 0xBB67AE8584CAA73Bull, 0, seed, k.hi, k.lo);
  return k;
}
// openes_rebuild_table (proj/src/ec.cpp:63-69): normals #0.. of
// RandomStream(key_from_seed(table_seed)), counter-addressed on the device
static cudaError_t rebuild_table(evorl_es* s) {
  return run_gaussian_matrix(key_from_seed(s->table_seed), 1, s->cfg.openes_noise_table_size, s->d_table,
                             s->stream);
}
// this generation's window offsets (proj/src/ec.cpp:79-84): RandomStream(ask
// key).randint(span + 1) per sampled row, with the rejection of
// proj/src/rng.cpp:89-96 -- sequential, so drawn on the host (base words)
static cudaError_t table_offsets(evorl_es* s, int base) {
  const uint64_t nn = (uint64_t)(s->cfg.openes_noise_table_size - s->d) + 1;
  const uint64_t m = (~0ull % nn + 1) % nn;
  s->h_offsets.resize(base);
  uint64_t w = 0;
  for (int i = 0; i < base; ++i) {
    for (;;) {
      const uint64_t x = stream_word(s->ask_key, w++);
      if (m == 0 || x < 0ull - m) {
        s->h_offsets[i] = (long long)(x % nn);
        break;
      }
    }
  }
  return cudaMemcpyAsync(s->d_offsets, s->h_offsets.data(), sizeof(long long) * base, cudaMemcpyHostToDevice,
                         s->stream);
}

// EsWorkflow::init (proj/src/workflow_es.cpp:68-85)
// CmaState::init's matrices (proj/src/ec.cpp:214-223): C = B = I, D = 1, ps = pc = 0
static int cma_state_init(evorl_es* s) {
  CmaDev& v = s->cma.dev;
  const size_t dp2 = (size_t)v.dp * v.dp;
  std::vector<double> eye(dp2, 0.0);
  for (int i = 0; i < v.dp; ++i) eye[(size_t)i * v.dp + i] = 1.0;
  CK(cudaMemcpy(v.C, eye.data(), sizeof(double) * dp2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v.B, eye.data(), sizeof(double) * dp2, cudaMemcpyHostToDevice));
  std::vector<double> ones(v.dp, 1.0);
  CK(cudaMemcpy(v.D, ones.data(), sizeof(double) * v.dp, cudaMemcpyHostToDevice));
  CK(cudaMemset(v.ps, 0, sizeof(double) * v.dp));
  CK(cudaMemset(v.pc, 0, sizeof(double) * v.dp));
  s->cma.sigma = s->cfg.cmaes_sigma0;
  s->cma.generation = 0;
  s->cma.recondition_count = 0;
  return EVORL_OK;
}

extern "C" int evorl_es_init(evorl_es* s, uint64_t key_hi, uint64_t key_lo) {
  if (s->cma_only) return set_err(EVORL_E_INVALID_ARGUMENT, "cma-only handle: use evorl_cma_ask / evorl_cma_tell");
  CK(cudaSetDevice(s->cfg.device));
  const DKey key = mk(key_hi, key_lo);
  s->rng = key;
  s->iteration = s->env_steps = s->episodes = 0;
  s->adam_t_host = 0;
  s->cem_iter = 0;
  CK(run_init_params(s->net, init_key(key, 1), s->d_mean, s->stream));
  if (s->d_table) {  // OpenEsState::init (proj/src/ec.cpp:50-61) with init_key(key, 2)
    s->table_seed = fold_in(init_key(key, 2), 0x7ab1e).lo;
    CK(rebuild_table(s));
  }
  CK(cudaMemsetAsync(s->d_m, 0, sizeof(double) * s->d, s->stream));
  CK(cudaMemsetAsync(s->d_v, 0, sizeof(double) * s->d, s->stream));
  CK(cudaMemsetAsync(s->d_t, 0, sizeof(long long), s->stream));
  if (s->cfg.algo == EVORL_ALGO_CMAES)
    if (int rc = cma_state_init(s)) return rc;
  if (s->cfg.algo == EVORL_ALGO_CEM) {
    std::vector<double> v(s->d, s->cfg.cem_var_init);
    CK(cudaMemcpyAsync(s->d_var, v.data(), sizeof(double) * s->d, cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
  }
  DevNorm nm{};
  nm.mode = s->norm_mode;
  nm.dim = s->env.obs_dim;
  if (s->norm_mode == EVORL_NORM_VBN) {
    CK(run_vbn_fit(s->env, init_key(key, 0), s->cfg.vbn_samples, s->d_norm, s->d_normp, s->stream));
  } else {
    if (s->norm_mode == EVORL_NORM_RS)  // ObsNormState::running_stats
      for (int i = 0; i < nm.dim; ++i) {
        nm.mean[i] = 0.0;
        nm.var[i] = 1.0;
      }
    CK(cudaMemcpyAsync(s->d_norm, &nm, sizeof nm, cudaMemcpyHostToDevice, s->stream));
    CK(run_norm_params(s->d_norm, s->d_normp, s->stream));
  }
  CK(cudaStreamSynchronize(s->stream));
  s->initialised = true;
  return EVORL_OK;
}

static ParamDesc param_desc(const evorl_es* s) {
  ParamDesc p{};
  p.mean = s->d_mean;
  p.ask_key = s->ask_key;
  switch (s->cfg.algo) {
    case EVORL_ALGO_OPENES:
      p.src = s->d_table ? SRC_OPENES_TABLE : SRC_OPENES;
      p.sigma = s->cfg.openes_sigma;
      p.mirrored = s->cfg.openes_mirrored;
      p.base = p.mirrored ? s->cfg.pop / 2 : s->cfg.pop;
      p.table = s->d_table;
      p.offsets = s->d_offsets;
      break;
    case EVORL_ALGO_VES:
      p.src = SRC_OPENES;
      p.sigma = s->cfg.ves_sigma;
      p.mirrored = s->cfg.ves_mirrored;
      p.base = p.mirrored ? s->cfg.pop / 2 : s->cfg.pop;
      break;
    case EVORL_ALGO_ARS:
      p.src = SRC_ARS;
      p.sigma = s->cfg.ars_sigma;
      break;
    case EVORL_ALGO_CEM:
      p.src = SRC_CEM;
      p.var = s->d_var;
      break;
  }
  return p;
}

static int check_ask(const evorl_es* s) {  // the ask-side argument checks
  const int n = s->cfg.pop;
  switch (s->cfg.algo) {
    case EVORL_ALGO_OPENES:
      if (n < 2) return set_err(EVORL_E_INVALID_ARGUMENT, "openes_ask: population must be at least 2");
      if (s->cfg.openes_mirrored && n % 2)
        return set_err(EVORL_E_INVALID_ARGUMENT, "openes_ask: mirrored sampling needs an even population");
      break;
    case EVORL_ALGO_ARS:
      if (n < 2 || n % 2) return set_err(EVORL_E_INVALID_ARGUMENT, "ars_ask: population must be even");
      break;
    case EVORL_ALGO_VES:
      if (n < 2) return set_err(EVORL_E_INVALID_ARGUMENT, "ves_ask: population must be at least 2");
      if (s->cfg.ves_mirrored && n % 2)
        return set_err(EVORL_E_INVALID_ARGUMENT, "ves_ask: mirrored sampling needs an even population");
      break;
  }
  return EVORL_OK;
}

// The buffer the ask keeps this generation's OpenES noise rows in (the rows
// this rank's agents use, from its first row on), or null: regenerated-noise
// mode, under a 4 GiB cap (EVORL_EPS_ROWS_CAP_BYTES overrides it; 0 disables
// -- used by the tests).  The tell reads it only when the rank holds every
// row (unsharded); sharded, the tell regenerates its coordinate slice.
static double* eps_rows_buffer(evorl_es* s) {
  if (s->cfg.algo != EVORL_ALGO_OPENES || s->d_table || s->eps_rows_failed) return nullptr;
  static const double kCap =
      getenv("EVORL_EPS_ROWS_CAP_BYTES") ? atof(getenv("EVORL_EPS_ROWS_CAP_BYTES")) : 4.0 * (1ull << 30);
  const long long rows = s->cfg.openes_mirrored ? s->cfg.pop / 2 : s->cfg.pop;
  const double bytes = (double)rows * (double)s->d * sizeof(double);
  if (bytes <= 0 || bytes > kCap) return nullptr;
  if (!s->d_eps_rows && cudaMalloc((void**)&s->d_eps_rows, (size_t)bytes) != cudaSuccess) {
    cudaGetLastError();  // out of memory: keep regenerating
    s->d_eps_rows = nullptr;
    s->eps_rows_failed = true;
  }
  return s->d_eps_rows;
}

// The buffer for the next generation's noise rows (same size as
// eps_rows_buffer's), the low-priority stream and event, or null
// (EVORL_NO_NOISE_AHEAD=1 disables it -- used by the tests).
static double* eps_next_buffer(evorl_es* s) {
  static const bool off = getenv("EVORL_NO_NOISE_AHEAD") && atoi(getenv("EVORL_NO_NOISE_AHEAD")) != 0;
  if (off || s->eps_next_failed || !s->d_eps_rows) return nullptr;
  if (!s->d_eps_next) {
    const long long rows = s->cfg.openes_mirrored ? s->cfg.pop / 2 : s->cfg.pop;
    int least = 0, greatest = 0;
    bool ok = cudaMalloc((void**)&s->d_eps_next, sizeof(double) * (size_t)rows * (size_t)s->d) == cudaSuccess;
    ok = ok && cudaDeviceGetStreamPriorityRange(&least, &greatest) == cudaSuccess;
    ok = ok && cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, least) == cudaSuccess;
    ok = ok && cudaEventCreateWithFlags(&s->ev_noise, cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaDeviceGetAttribute(&s->n_sms, cudaDevAttrMultiProcessorCount, s->cfg.device) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      s->eps_next_failed = true;
      return nullptr;
    }
  }
  return s->d_eps_next;
}

static long long rows_of(const evorl_es* s) { return s->cfg.openes_mirrored ? s->cfg.pop / 2 : s->cfg.pop; }
static int sms_of(evorl_es* s) {
  if (s->n_sms <= 0 && cudaDeviceGetAttribute(&s->n_sms, cudaDevAttrMultiProcessorCount, s->cfg.device) != cudaSuccess)
    s->n_sms = 148;
  return s->n_sms;
}
// EVORL_NO_FUSED_ASK=1: the oz ask as materialise + pre-split (used by the tests)
static bool no_fused_ask() {
  static const bool off = getenv("EVORL_NO_FUSED_ASK") && atoi(getenv("EVORL_NO_FUSED_ASK")) != 0;
  return off;
}

static RolloutArgs rollout_args(const evorl_es* s) {
  RolloutArgs a{};
  a.env = s->env;
  a.net = s->net;
  a.par = param_desc(s);
  a.plan = s->plan;
  a.norm = s->d_normp;
  a.n_agents = s->a1 - s->a0;
  a.agent_offset = s->a0;
  a.e = s->e;
  a.count = s->count;
  a.groups = s->groups;
  a.rollout_key = s->rollout_key;
  a.track_stats = s->norm_mode == EVORL_NORM_RS;
  const int per_lane = (s->count + s->e - 1) / s->e;
  a.max_iters = per_lane * s->env.max_episode_steps + 1;
  a.ep_returns = s->d_ep_returns + (long long)s->a0 * s->count;
  a.ep_lengths = nullptr;
  a.lane_steps = s->d_lane_steps + (long long)s->a0 * s->e;
  a.lane_stats = s->d_lane_stats + (long long)s->a0 * s->e * 9;
  a.fault = s->d_fault;
  return a;
}

// cmaes_tell (proj/src/ec.cpp:236-288) on the device state: d_fitness (n) and
// d_cand (n x d) in, mean / paths / C / sigma updated, B and D re-factorised
// every k-th generation
static int cma_tell_device(evorl_es* s, int n, cudaStream_t st) {
  auto& c = s->cma;
  CmaDev& v = c.dev;
  const int d = (int)s->d, mu = c.mu, dp = v.dp;
  CK(run_rank(s->d_fitness, n, 1, s->d_rank, st));
  CK(run_order_from_rank(s->d_rank, n, s->d_order, st));
  CK(run_cma_ytop(s->d_cand, s->d_order, mu, d, s->d_mean, c.sigma, c.d_w, v.ytT, v.wyT, st));
  CK(run_cma_yw_mean(v.ytT, c.d_w, mu, d, c.sigma, v.yw, s->d_mean, st));
  CK(run_cma_gemv_t(v.B, dp, d, v.yw, v.D, v.t1, st));
  CK(run_cma_gemv(v.B, dp, d, v.t1, v.cih, st));
  const double cps = std::sqrt(c.cs * (2.0 - c.cs) * c.mueff);
  CK(run_cma_ps(v.ps, v.cih, d, c.cs, cps, v.red, st));
  double nrm2 = 0.0;
  CK(cudaMemcpyAsync(&nrm2, v.red, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double gen1 = (double)(c.generation + 1);
  const double ps_norm = std::sqrt(nrm2);
  const bool hsig = ps_norm / std::sqrt(1.0 - std::pow(1.0 - c.cs, 2.0 * gen1)) <
                    (1.4 + 2.0 / ((double)d + 1.0)) * c.chi_n;
  const double cpc = hsig ? std::sqrt(c.cc * (2.0 - c.cc) * c.mueff) : 0.0;
  CK(run_cma_pc(v.pc, v.yw, d, c.cc, cpc, st));
  // C' = (1-c1-cmu) C + c1 (pc pc^T + dhsig C) + cmu sum_i w_i y_i y_i^T,
  // the rank-mu sum as a K = mu DMMA GEMM with the blend in its epilogue
  GemmEpi epi{};
  epi.mode = GEMM_RANKMU;
  epi.out = v.W;
  epi.ldo = dp;
  epi.Cold = v.C;
  epi.pc = v.pc;
  epi.a = 1.0 - c.c1 - c.cmu;
  epi.c1 = c.c1;
  epi.dh = (hsig ? 0.0 : 1.0) * c.cc * (2.0 - c.cc);
  epi.cmu = c.cmu;
  CK(run_gemm_nt(d, d, mu, v.wyT, mu, v.ytT, mu, epi, st));
  CK(run_cma_symmetrize(v.W, v.C, d, dp, st));
  c.sigma *= std::exp((c.cs / c.ds) * (ps_norm / c.chi_n - 1.0));
  c.generation += 1;
  // re-factorise; re-condition when eigenvalues fall to <= 0
  // (EXTENSION: only every cmaes_eig_every-th generation; 1 = reference)
  // k = 0: Hansen's lazy gap max(1, floor(1 / (10 d (c1 + cmu)))), which
  // keeps the amortised eigendecomposition at O(d^2) per generation
  const int k_eig = s->cfg.cmaes_eig_every > 0
                        ? s->cfg.cmaes_eig_every
                        : std::max(1, (int)std::floor(1.0 / (10.0 * d * (c.c1 + c.cmu))));
  if (c.generation % k_eig != 0) return EVORL_OK;
  double evmin = 0.0;
  int sw = sym_eig_jacobi(v, v.C, d, &evmin, v.B, v.evals, st, v.B);
  if (sw < 0) return set_err(EVORL_E_CUDA, "cmaes: eigensolver failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (evmin <= 0.0) {
    CK(run_cma_add_diag(v.C, d, dp, 1e-10 - evmin, st));
    sw = sym_eig_jacobi(v, v.C, d, &evmin, v.B, v.evals, st, v.B);
    if (sw < 0) return set_err(EVORL_E_CUDA, "cmaes: eigensolver failed");
    c.recondition_count += 1;
  }
  c.last_sweeps = sw;
  CK(run_cma_sqrt_pos(v.evals, v.D, d, st));
  return EVORL_OK;
}

// cmaes_ask (proj/src/ec.cpp:226-234): d_cand = ((z .* D^T) B^T) sigma + mean
static int cma_ask_device(evorl_es* s, DKey key, int n, cudaStream_t st) {
  CmaDev& v = s->cma.dev;
  CK(run_cma_zD(key, n, (int)s->d, v.D, v.zD, st));
  GemmEpi epi{};
  epi.mode = GEMM_ASK;
  epi.out = s->d_cand;
  epi.ldo = s->d;
  epi.sigma = s->cma.sigma;
  epi.mean = s->d_mean;
  CK(run_gemm_nt(n, (int)s->d, (int)s->d, v.zD, s->d, v.B, v.dp, epi, st));
  return EVORL_OK;
}

// ask + rollout + fitness of agents [a0, a1)
extern "C" int evorl_es_phase_rollout(evorl_es* s) {
  if (s->cma_only) return set_err(EVORL_E_INVALID_ARGUMENT, "cma-only handle: use evorl_cma_ask / evorl_cma_tell");
  if (!s->initialised) return set_err(EVORL_E_INVALID_ARGUMENT, "evorl_es_step before evorl_es_init");
  CK(cudaSetDevice(s->cfg.device));
  int rc = check_ask(s);
  if (rc) return rc;
  // WorkflowState::step_key (proj/include/evorl/workflow.hpp:41)
  s->step_key = fold_in(fold_in(s->rng, 0), (uint64_t)s->iteration);
  s->ask_key = fold_in(s->step_key, 0);      // proj/src/workflow_es.cpp:94
  s->rollout_key = fold_in(s->step_key, 1);  // proj/src/workflow_es.cpp:125
  if (s->d_table) CK(table_offsets(s, s->cfg.openes_mirrored ? s->cfg.pop / 2 : s->cfg.pop));
  s->eps_rows_valid = false;
  s->ask_timed = false;
  CK(cudaEventRecord(s->ev_s0, s->stream));
  CK(cudaMemsetAsync(s->d_steps, 0, sizeof(unsigned long long), s->stream));
  CK(cudaMemsetAsync(s->d_fault, 0xFF, sizeof(unsigned long long), s->stream));
  RolloutArgs a = rollout_args(s);
  if (s->cfg.algo == EVORL_ALGO_CMAES) {
    // cmaes_ask (proj/src/ec.cpp:226-234): all n candidates (every rank needs
    // the elites' rows for the tell), Y = ((z .* D^T) B^T) sigma + mean
    if (int rc = cma_ask_device(s, s->ask_key, s->cfg.pop, s->stream)) return rc;
    a.par.src = SRC_EXPLICIT;
    a.par.params = s->d_cand + (long long)s->a0 * s->d;
    CK(cudaEventRecord(s->ev_r0, s->stream));
    if (s->warp_path) {
      CK(launch_rollout_warp(a, s->wplan, s->cfg.precision, s->stream));
    } else {
      CK(launch_rollout(a, s->cfg.precision, s->stream));
      count_launch();
    }
  } else if (s->warp_path) {
    // small policy: materialise the shard's candidates (fully parallel ask),
    // then one warp per lane with the weights resident in shared memory
    double* er = a.par.src == SRC_OPENES ? eps_rows_buffer(s) : nullptr;
    long long r0 = 0, r1 = 0;
    if (er) openes_row_range(a.par, s->a0, s->a1, &r0, &r1);
    CK(cudaEventRecord(s->ev_a0, s->stream));
    CK(run_materialize(a.par, s->d, s->a0, s->a1, s->d_cand, s->stream, er, r0));
    CK(cudaEventRecord(s->ev_a1, s->stream));
    s->ask_timed = true;
    s->eps_rows_valid = er != nullptr && r0 == 0 && r1 == rows_of(s);
    count_launch();
    a.par.src = SRC_EXPLICIT;
    a.par.params = s->d_cand;
    CK(cudaEventRecord(s->ev_r0, s->stream));
    CK(launch_rollout_warp(a, s->wplan, s->cfg.precision, s->stream));
  } else {
    // team path: materialise the shard's candidates (chunks of cand_cap
    // agents), then roll each chunk out
    double* er = a.par.src == SRC_OPENES ? eps_rows_buffer(s) : nullptr;
    long long r0 = 0, r1 = 0;  // noise rows of this shard: er holds rows [r0, r1)
    if (er) openes_row_range(a.par, s->a0, s->a1, &r0, &r1);
    const bool whole = s->cand_cap >= s->a1 - s->a0;  // one materialised chunk
    bool kept = false;  // this ask's noise rows were generated beside the last rollout
    if (er && whole && s->eps_next_valid && s->eps_next_key.hi == s->ask_key.hi &&
        s->eps_next_key.lo == s->ask_key.lo && s->eps_next_r0 == r0 && s->eps_next_r1 == r1) {
      CK(cudaStreamWaitEvent(s->stream, s->ev_noise, 0));
      std::swap(s->d_eps_rows, s->d_eps_next);
      er = s->d_eps_rows;
      kept = true;
    }
    s->eps_next_valid = false;
    for (int c0 = s->a0; c0 < s->a1; c0 += s->cand_cap) {
      const int c1 = std::min(s->a1, c0 + s->cand_cap);
      RolloutArgs ac = a;
      ac.n_agents = c1 - c0;
      ac.agent_offset = c0;
      ac.ep_returns = s->d_ep_returns + (long long)c0 * s->count;
      ac.lane_steps = s->d_lane_steps + (long long)c0 * s->e;
      ac.lane_stats = s->d_lane_stats + (long long)c0 * s->e * 9;
      const bool one_chunk = c0 == s->a0 && c1 == s->a1;
      if (one_chunk) CK(cudaEventRecord(s->ev_a0, s->stream));
      if (s->d_cand_f32) {
        if (kept) {
          CK(run_cand_from_eps_f32(a.par, s->d, c0, c1, er, r0, s->d_cand_f32, s->stream));
        } else {
          CK(run_materialize_f32(a.par, s->d, c0, c1, s->d_cand_f32, s->stream, er, r0));
        }
        if (one_chunk) CK(cudaEventRecord(s->ev_a1, s->stream));
        ac.par.src = SRC_EXPLICIT_F32;
        ac.par.params_f32 = s->d_cand_f32;
        if (s->d_tc_blocks) {  // the tc team's layer-1 weights, pre-split (bulk-copied by its prologue)
          CK(run_tc_split(s->d_cand_f32, s->net, s->plan.tcp, c1 - c0, s->d_tc_blocks, s->stream));
          count_launch();
          ac.tc_blocks = s->d_tc_blocks;
          ac.tc_block_bytes = tc_block_bytes(s->plan.tcp);
        }
      } else {
        const bool fused = s->d_tc_blocks && er && whole && !no_fused_ask();
        if (fused) {
          // oz: the ask fused with the pre-split from the noise rows (generated
          // here on the first generation, else kept from beside the last rollout)
          if (!kept) CK(run_noise_rows(s->ask_key, r0 * s->d, (r1 - r0) * s->d, er, 16 * sms_of(s), s->stream));
          CK(run_oz_ask_split(a.par, s->net, s->plan.tcp, c0, c1, er, r0, s->d_cand, s->d_tc_blocks, s->stream));
          count_launch();
        } else if (kept) {
          CK(run_cand_from_eps(a.par, s->d, c0, c1, er, r0, s->d_cand, s->stream));
        } else {
          CK(run_materialize(a.par, s->d, c0, c1, s->d_cand, s->stream, er, r0));
        }
        if (one_chunk) CK(cudaEventRecord(s->ev_a1, s->stream));
        ac.par.src = SRC_EXPLICIT;
        ac.par.params = s->d_cand;
        if (s->d_tc_blocks) {  // the oz team's layer-1 weights, pre-split into fixed-point byte slices
          if (!fused) {
            CK(run_oz_split(s->d_cand, s->net, s->plan.tcp, c1 - c0, s->d_tc_blocks, s->stream));
            count_launch();
          }
          ac.tc_blocks = s->d_tc_blocks;
          ac.tc_block_bytes = oz_block_bytes(s->plan.tcp);
        }
      }
      count_launch();
      s->ask_timed = one_chunk;
      if (c0 == s->a0) CK(cudaEventRecord(s->ev_r0, s->stream));
      CK(launch_rollout(ac, s->cfg.precision, s->stream));
      count_launch();
    }
    // the tell reads the kept rows only when they are every row (unsharded)
    s->eps_rows_valid = er != nullptr && s->a1 > s->a0 && r0 == 0 && r1 == rows_of(s);
    if (er && s->world > 1 && s->p1 > s->p0 && s->a1 > s->a0 && eps_next_buffer(s) && !s->cols_failed) {
      // the next generation's tell noise (every row, this rank's coordinates)
      const long long span = s->p1 - s->p0, cap = rows_of(s) * ((s->d + s->world - 1) / s->world);
      if (!s->d_cols_next) {
        bool ok = cudaMalloc((void**)&s->d_cols_next, sizeof(double) * (size_t)cap) == cudaSuccess;
        ok = ok && cudaMalloc((void**)&s->d_cols_cur, sizeof(double) * (size_t)cap) == cudaSuccess;
        if (!ok) {
          cudaGetLastError();
          s->cols_failed = true;
        }
      }
      if (!s->cols_failed && rows_of(s) * span <= cap) {
        const DKey next = fold_in(fold_in(fold_in(s->rng, 0), (uint64_t)(s->iteration + 1)), 0);
        CK(cudaStreamWaitEvent(s->side, s->ev_r0, 0));
        CK(run_noise_cols(next, s->d, s->p0, s->p1, rows_of(s), s->d_cols_next, s->n_sms, s->side));
        CK(cudaEventRecord(s->ev_noise, s->side));
        count_launch();
        s->cols_next_valid = true;
        s->cols_next_key = next;
        s->cols_next_p0 = s->p0;
        s->cols_next_p1 = s->p1;
      }
    }
    if (er && whole && s->a1 > s->a0) {
      if (double* nx = eps_next_buffer(s)) {  // the next generation's noise, beside this rollout
        const DKey next = fold_in(fold_in(fold_in(s->rng, 0), (uint64_t)(s->iteration + 1)), 0);
        CK(cudaStreamWaitEvent(s->side, s->ev_r0, 0));
        CK(run_noise_rows(next, r0 * s->d, (r1 - r0) * s->d, nx, s->n_sms, s->side));
        CK(cudaEventRecord(s->ev_noise, s->side));
        count_launch();
        s->eps_next_valid = true;
        s->eps_next_key = next;
        s->eps_next_r0 = r0;
        s->eps_next_r1 = r1;
      }
    }
  }
  CK(cudaEventRecord(s->ev_r1, s->stream));
  CK(run_fitness(a.ep_returns, s->count, a.n_agents, s->a0, s->d_fitness, a.lane_steps, s->e, s->d_steps,
                 s->stream));
  CK(cudaMemcpyAsync(&s->h->steps, s->d_steps, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(&s->h->fault, s->d_fault, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (s->h->fault != ~0ull) return fault_to_error(s->h->fault);
  return EVORL_OK;
}

static double cem_floor(const evorl_es* s) {  // CemState::noise_floor, proj/src/ec.cpp:292-298
  const double frac = s->cfg.cem_decay_iters > 0
                          ? std::min(1.0, (double)s->cem_iter / (double)s->cfg.cem_decay_iters)
                          : 1.0;
  return s->cfg.cem_noise_start * std::pow(s->cfg.cem_noise_end / s->cfg.cem_noise_start, frac);
}

static int cem_sigma_metric(evorl_es* s, double* sigma);

// ranks + tell on [p0, p1) + metrics; expects the full fitness vector.
extern "C" int evorl_es_phase_tell(evorl_es* s, evorl_step_metrics* out) {
  CK(cudaSetDevice(s->cfg.device));
  const int n = s->cfg.pop;
  const cudaStream_t st = s->stream;
  if (s->norm_mode == EVORL_NORM_RS)  // proj/src/workflow_es.cpp:136-138
    CK(run_rs_merge(s->d_lane_stats, n, s->e, s->d_norm, s->d_normp, s->d_agent_stats, st));
  double sigma = 0.0;
  bool ars = false;
  switch (s->cfg.algo) {
    case EVORL_ALGO_OPENES: {
      CK(run_rank(s->d_fitness, n, 0, s->d_rank, st));
      CK(run_shaped_from_rank(s->d_rank, n, s->d_shaped, st));
      OpenEsTellArgs t{};
      t.mean = s->d_mean;
      t.m = s->d_m;
      t.v = s->d_v;
      t.t_dev = s->d_t;
      t.d = s->d;
      t.p0 = s->p0;
      t.p1 = s->p1;
      t.sigma = s->cfg.openes_sigma;
      t.lr = s->cfg.openes_lr;
      t.weight_decay = s->cfg.openes_weight_decay;
      t.lrwd = s->cfg.openes_lr * s->cfg.openes_weight_decay;
      t.beta1 = 0.9;
      t.beta2 = 0.999;
      t.omb1 = 1.0 - 0.9;
      t.omb2 = 1.0 - 0.999;
      t.eps = 1e-8;
      t.n = n;
      t.mirrored = s->cfg.openes_mirrored;
      t.base = t.mirrored ? n / 2 : n;
      t.ask_key = s->ask_key;
      t.shaped = s->d_shaped;
      t.adam_bc = s->d_adam_bc;
      t.adam_bc_len = s->adam_bc_len;
      t.table = s->d_table;
      t.offsets = s->d_offsets;
      t.eps_rows = s->eps_rows_valid ? s->d_eps_rows : nullptr;
      t.eps_ld = s->d;
      t.eps_p0 = 0;
      s->eps_rows_valid = false;
      if (!t.eps_rows && !t.table && s->cols_cur_valid && s->cols_cur_key.hi == s->ask_key.hi &&
          s->cols_cur_key.lo == s->ask_key.lo && s->cols_cur_p0 == s->p0 && s->cols_cur_p1 == s->p1) {
        CK(cudaStreamWaitEvent(st, s->ev_noise, 0));  // the side stream filled them beside the last rollout
        t.eps_rows = s->d_cols_cur;
        t.eps_ld = s->p1 - s->p0;
        t.eps_p0 = s->p0;
      }
      {
        const long long need = (long long)openes_tell_chunks(t.base, s->d) * (s->p1 - s->p0);
        if (need > s->tell_part_cap) {
          if (s->d_tell_part) cudaFree(s->d_tell_part);
          s->d_tell_part = nullptr;
          s->tell_part_cap = 0;
          CK(cudaMalloc((void**)&s->d_tell_part, sizeof(double) * need));
          s->tell_part_cap = need;
        }
      }
      t.partial = s->d_tell_part;
      CK(run_openes_tell(t, st));
      // the columns filled beside this generation's rollout serve the next tell
      std::swap(s->d_cols_cur, s->d_cols_next);
      s->cols_cur_valid = s->cols_next_valid;
      s->cols_cur_key = s->cols_next_key;
      s->cols_cur_p0 = s->cols_next_p0;
      s->cols_cur_p1 = s->cols_next_p1;
      s->cols_next_valid = false;
      CK(run_inc_counter(s->d_t, st));
      s->adam_t_host += 1;
      sigma = s->cfg.openes_sigma;
      break;
    }
    case EVORL_ALGO_ARS: {
      const int half = n / 2;
      CK(run_ars_scores(s->d_fitness, half, s->d_scores, st));
      CK(run_rank(s->d_scores, half, 1, s->d_rank, st));
      CK(run_ars_select(s->d_fitness, s->d_rank, half, s->cfg.ars_elites, s->cfg.ars_lr, s->d_elite_idx,
                        s->d_elite_diff, s->d_sel, st));
      CK(run_ars_update(s->d_mean, s->d, s->p0, s->p1, s->ask_key, s->d_elite_idx, s->d_elite_diff, s->d_sel,
                        st));
      CK(cudaMemcpyAsync(&s->h->sel, s->d_sel, sizeof(ArsSel), cudaMemcpyDeviceToHost, st));
      sigma = s->cfg.ars_sigma;
      ars = true;
      break;
    }
    case EVORL_ALGO_VES: {
      CK(run_rank(s->d_fitness, n, 1, s->d_rank, st));
      CK(run_order_from_rank(s->d_rank, n, s->d_order, st));
      const int mu = std::min(s->cfg.ves_elites, n);
      const int base = s->cfg.ves_mirrored ? n / 2 : n;
      CK(run_ves_tell(s->d_mean, s->d, s->p0, s->p1, s->cfg.ves_sigma, s->cfg.ves_mirrored, base,
                      s->ask_key, s->d_order, s->d_ves_w, mu, st));
      sigma = s->cfg.ves_sigma;
      break;
    }
    case EVORL_ALGO_CMAES: {  // cmaes_tell (proj/src/ec.cpp:236-288), replicated on every rank
      if (int rc = cma_tell_device(s, n, st)) return rc;
      sigma = s->cma.sigma;
      break;
    }
    case EVORL_ALGO_CEM: {
      CK(run_rank(s->d_fitness, n, 1, s->d_rank, st));
      CK(run_order_from_rank(s->d_rank, n, s->d_order, st));
      const int h = std::min(s->cfg.cem_elites, n);
      CK(run_cem_tell(s->d_mean, s->d_var, s->d, s->p0, s->p1, s->ask_key, s->d_order, h, cem_floor(s), st));
      s->cem_iter += 1;
      break;
    }
  }
  CK(run_metrics(s->d_fitness, n, s->d_metrics, st));
  CK(cudaMemcpyAsync(s->h->metrics, s->d_metrics, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(s->ev_s1, st));
  CK(cudaStreamSynchronize(st));
  // es/sigma = sqrt(diag_var.mean()) (proj/src/workflow_es.cpp:162); a sharded
  // handle holds only its [p0, p1) slice of the new variance here, so the
  // caller gathers it and asks evorl_es_cem_sigma (NaN until then)
  if (s->cfg.algo == EVORL_ALGO_CEM) {
    if (s->world == 1) {
      if (int rc = cem_sigma_metric(s, &sigma)) return rc;
    } else {
      sigma = std::numeric_limits<double>::quiet_NaN();
    }
  }
  cudaEventElapsedTime(&s->last_rollout_ms, s->ev_r0, s->ev_r1);
  cudaEventElapsedTime(&s->last_step_ms, s->ev_s0, s->ev_s1);
  s->last_ask_ms = -1.f;
  if (s->ask_timed) cudaEventElapsedTime(&s->last_ask_ms, s->ev_a0, s->ev_a1);
  s->env_steps += (long long)s->h->steps;
  s->episodes += (long long)n * s->count;
  s->iteration += 1;
  if (out) {
    out->fitness_mean = s->h->metrics[0];
    out->fitness_max = s->h->metrics[1];
    out->fitness_min = s->h->metrics[2];
    out->sigma = sigma;
    out->update_skipped = ars && s->h->sel.skipped ? 1.0 : 0.0;
  }
  return EVORL_OK;
}

// ------------------------------------------------- CMA-ES free functions
// CmaState::init / cmaes_ask / cmaes_tell (proj/src/ec.cpp:191-288) on a device
// state of dimension d with no env or policy attached (the free-function seam,
// proj/include/evorl/ec.hpp:107-125).  The state (mean, sigma, C, B, D, ps, pc,
// generation, recondition_count) is read / written with evorl_es_get/set_mean
// and evorl_es_cma_get/set; release with evorl_es_destroy.
extern "C" int evorl_cma_create(int64_t d, int32_t pop, int32_t elites, double sigma0, int32_t max_dim,
                                int32_t eig_every, evorl_es** out) {
  *out = nullptr;
  if (d < 1) return set_err(EVORL_E_INVALID_ARGUMENT, "cmaes: dimension must be positive");
  evorl_es_config cfg;
  evorl_es_default_config(&cfg);
  cfg.algo = EVORL_ALGO_CMAES;
  cfg.env_id = EVORL_ENV_PENDULUM;  // not used by a cma-only handle
  cfg.n_hidden = 0;
  cfg.allow_linear = 1;
  cfg.pop = pop;
  cfg.cmaes_elites = elites;
  cfg.cmaes_sigma0 = sigma0;
  cfg.cmaes_max_dim = max_dim;
  cfg.cmaes_eig_every = eig_every;
  cfg.obs_norm_mode = EVORL_NORM_NONE;
  evorl_es* s = nullptr;
  if (int rc = es_create(&cfg, d, &s)) return rc;
  if (int rc = cma_state_init(s)) {
    evorl_es_destroy(s);
    return rc;
  }
  CK(cudaMemset(s->d_mean, 0, sizeof(double) * d));
  s->initialised = true;
  *out = s;
  return EVORL_OK;
}

extern "C" int evorl_cma_ask(evorl_es* s, uint64_t key_hi, uint64_t key_lo, double* candidates) {
  if (!s->cma_only) return set_err(EVORL_E_INVALID_ARGUMENT, "evorl_cma_ask needs an evorl_cma_create handle");
  CK(cudaSetDevice(s->cfg.device));
  const int n = s->cfg.pop;
  if (int rc = cma_ask_device(s, mk(key_hi, key_lo), n, s->stream)) return rc;
  CK(cudaMemcpyAsync(candidates, s->d_cand, sizeof(double) * n * s->d, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}

extern "C" int evorl_cma_tell(evorl_es* s, const double* candidates, const double* fitness) {
  if (!s->cma_only) return set_err(EVORL_E_INVALID_ARGUMENT, "evorl_cma_tell needs an evorl_cma_create handle");
  CK(cudaSetDevice(s->cfg.device));
  const int n = s->cfg.pop;
  CK(cudaMemcpyAsync(s->d_cand, candidates, sizeof(double) * n * s->d, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(s->d_fitness, fitness, sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
  if (int rc = cma_tell_device(s, n, s->stream)) return rc;
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}

// Workflow::step on one GPU: both phases with the full ranges.
extern "C" int evorl_es_step(evorl_es* s, evorl_step_metrics* out) {
  if (s->world != 1) return set_err(EVORL_E_INVALID_ARGUMENT, "sharded handle: use the phase API");
  int rc = evorl_es_phase_rollout(s);
  if (rc) return rc;
  return evorl_es_phase_tell(s, out);
}

// Workflow::step with the EsState on the host (the reference's own layout:
// mean and the Adam moments live with the caller): the state is staged through
// pinned memory and copied with stream-ordered async copies around the two
// phases, one synchronisation at the end instead of one per transfer call.
extern "C" int evorl_es_step_host(evorl_es* s, const double* mean_in, const double* m_in, const double* v_in,
                                  int64_t t_in, double* mean_out, double* m_out, double* v_out, int64_t* t_out,
                                  evorl_step_metrics* out) {
  if (s->world != 1) return set_err(EVORL_E_INVALID_ARGUMENT, "sharded handle: use the phase API");
  if (!mean_in || !mean_out) return set_err(EVORL_E_INVALID_ARGUMENT, "step_host: mean buffers are required");
  if ((m_in == nullptr) != (v_in == nullptr))
    return set_err(EVORL_E_INVALID_ARGUMENT, "step_host: the Adam moments come as a pair");
  CK(cudaSetDevice(s->cfg.device));
  const size_t d = (size_t)s->d;
  if (!s->h_stage) CK(cudaMallocHost((void**)&s->h_stage, sizeof(double) * (3 * d + 1)));
  long long* st_t = reinterpret_cast<long long*>(s->h_stage + 3 * d);
  // a caller buffer in page-locked memory (evorl_host_alloc) is copied directly
  // by the DMA engines; a pageable one goes through the handle's pinned stage
  auto pinned = [](const void* p) {
    cudaPointerAttributes a{};
    const bool ok = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
    cudaGetLastError();
    return ok;
  };
  auto up = [&](double* dev, const double* host, size_t k) -> cudaError_t {
    const double* src = host;
    if (!pinned(host)) {
      std::memcpy(s->h_stage + k * d, host, sizeof(double) * d);
      src = s->h_stage + k * d;
    }
    return cudaMemcpyAsync(dev, src, sizeof(double) * d, cudaMemcpyHostToDevice, s->stream);
  };
  double* direct[3] = {nullptr, nullptr, nullptr};  // outputs written by DMA in place
  auto down = [&](double* host, const double* dev, size_t k) -> cudaError_t {
    double* dst = pinned(host) ? host : s->h_stage + k * d;
    if (dst == host) direct[k] = host;
    return cudaMemcpyAsync(dst, dev, sizeof(double) * d, cudaMemcpyDeviceToHost, s->stream);
  };
  CK(up(s->d_mean, mean_in, 0));
  if (m_in) {
    CK(up(s->d_m, m_in, 1));
    CK(up(s->d_v, v_in, 2));
    *st_t = t_in;
    CK(cudaMemcpyAsync(s->d_t, st_t, sizeof(long long), cudaMemcpyHostToDevice, s->stream));
    s->adam_t_host = t_in;
  }
  if (int rc = evorl_es_phase_rollout(s)) return rc;  // (both phases order after the copies on the stream)
  if (int rc = evorl_es_phase_tell(s, out)) return rc;
  CK(down(mean_out, s->d_mean, 0));
  if (m_out) CK(down(m_out, s->d_m, 1));
  if (v_out) CK(down(v_out, s->d_v, 2));
  if (t_out) CK(cudaMemcpyAsync(st_t, s->d_t, sizeof(long long), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (!direct[0]) std::memcpy(mean_out, s->h_stage, sizeof(double) * d);
  if (m_out && !direct[1]) std::memcpy(m_out, s->h_stage + d, sizeof(double) * d);
  if (v_out && !direct[2]) std::memcpy(v_out, s->h_stage + 2 * d, sizeof(double) * d);
  if (t_out) *t_out = *st_t;
  return EVORL_OK;
}

// Page-locked host memory for the host-state calls (freed by evorl_host_free).
extern "C" int evorl_host_alloc(int64_t bytes, void** out) {
  *out = nullptr;
  if (bytes <= 0) return set_err(EVORL_E_INVALID_ARGUMENT, "host_alloc: bytes must be positive");
  CK(cudaMallocHost(out, (size_t)bytes));
  return EVORL_OK;
}
extern "C" void evorl_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

extern "C" int evorl_es_set_shard(evorl_es* s, int32_t rank, int32_t world) {
  if (world < 1 || rank < 0 || rank >= world) return set_err(EVORL_E_INVALID_ARGUMENT, "bad shard");
  const long long n = s->cfg.pop;
  // Equal contiguous chunks of ceil(n / world) agents and ceil(d / world)
  // coordinates (paper_2501_15129_b200/dist.py:shard_range); every rank
  // regenerates the noise rows it needs, so no pairing constraint applies.
  const long long acs = (n + world - 1) / world, pcs = (s->d + world - 1) / world;
  s->rank = rank;
  s->world = world;
  s->a0 = (int)std::min(n, acs * rank);
  s->a1 = (int)std::min(n, acs * (rank + 1));
  s->p0 = std::min(s->d, pcs * rank);
  s->p1 = std::min(s->d, pcs * (rank + 1));
  return EVORL_OK;
}

extern "C" int evorl_es_shard_ranges(const evorl_es* s, int32_t* a0, int32_t* a1, int64_t* p0, int64_t* p1) {
  *a0 = s->a0;
  *a1 = s->a1;
  *p0 = s->p0;
  *p1 = s->p1;
  return EVORL_OK;
}

extern "C" int evorl_es_device_buffers(evorl_es* s, void** fitness, void** mean, void** lane_stats) {
  if (fitness) *fitness = s->d_fitness;
  if (mean) *mean = s->d_mean;
  if (lane_stats) *lane_stats = s->d_lane_stats;
  return EVORL_OK;
}

// CEM's diagonal variance (CemState::diag_var, proj/include/evorl/ec.hpp:129-135):
// k_cem_tell updates it on [p0, p1) only, so a sharded caller gathers it like
// the mean (the next ask reads every coordinate).
extern "C" int evorl_es_device_var(evorl_es* s, void** var) {
  if (var) *var = s->d_var;
  return EVORL_OK;
}

// The resolved obs_norm mode (EVORL_NORM_NONE/VBN/RS): per-lane RunningStats
// are tracked (and must be gathered by a sharded caller) iff it is RS.
extern "C" int evorl_es_norm_mode(const evorl_es* s, int32_t* mode) {
  *mode = s->norm_mode;
  return EVORL_OK;
}

// The WorkflowState root key (state.rng) the workflow was initialised or
// loaded with; learn() derives eval keys from it (proj/include/evorl/workflow.hpp:42).
extern "C" int evorl_es_get_rng(const evorl_es* s, uint64_t* hi, uint64_t* lo) {
  *hi = s->rng.hi;
  *lo = s->rng.lo;
  return EVORL_OK;
}

// es/sigma of a CEM workflow = sqrt(diag_var.mean()) (proj/src/workflow_es.cpp:162),
// summed sequentially over the FULL variance (a sharded caller calls it after
// gathering the variance slices).
static int cem_sigma_metric(evorl_es* s, double* sigma) {
  std::vector<double> v(s->d);
  CK(cudaMemcpy(v.data(), s->d_var, sizeof(double) * s->d, cudaMemcpyDeviceToHost));
  double acc = 0.0;
  for (double x : v) acc += x;
  *sigma = std::sqrt(acc / (double)s->d);
  return EVORL_OK;
}
extern "C" int evorl_es_cem_sigma(evorl_es* s, double* sigma) {
  if (s->cfg.algo != EVORL_ALGO_CEM) return set_err(EVORL_E_INVALID_ARGUMENT, "not a cem workflow");
  CK(cudaSetDevice(s->cfg.device));
  return cem_sigma_metric(s, sigma);
}
extern "C" void* evorl_es_stream(evorl_es* s) { return (void*)s->stream; }

extern "C" int evorl_es_last_timings(const evorl_es* s, float* rollout_ms, float* step_ms) {
  if (rollout_ms) *rollout_ms = s->last_rollout_ms;
  if (step_ms) *step_ms = s->last_step_ms;
  return EVORL_OK;
}

extern "C" int evorl_es_last_ask_ms(const evorl_es* s, float* ask_ms) {
  if (ask_ms) *ask_ms = s->last_ask_ms;
  return EVORL_OK;
}

extern "C" int evorl_es_counters(const evorl_es* s, int64_t* it, int64_t* steps, int64_t* eps) {
  if (it) *it = s->iteration;
  if (steps) *steps = s->env_steps;
  if (eps) *eps = s->episodes;
  return EVORL_OK;
}
extern "C" int evorl_es_set_counters(evorl_es* s, int64_t it, int64_t steps, int64_t eps) {
  s->iteration = it;
  s->env_steps = steps;
  s->episodes = eps;
  return EVORL_OK;
}

extern "C" int evorl_es_get_mean(evorl_es* s, double* mean) {
  CK(cudaSetDevice(s->cfg.device));
  CK(cudaMemcpyAsync(mean, s->d_mean, sizeof(double) * s->d, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}
extern "C" int evorl_es_set_mean(evorl_es* s, const double* mean) {
  CK(cudaSetDevice(s->cfg.device));
  CK(cudaMemcpyAsync(s->d_mean, mean, sizeof(double) * s->d, cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}
extern "C" int evorl_es_get_adam(evorl_es* s, double* m, double* v, int64_t* t) {
  CK(cudaSetDevice(s->cfg.device));
  if (m) CK(cudaMemcpyAsync(m, s->d_m, sizeof(double) * s->d, cudaMemcpyDeviceToHost, s->stream));
  if (v) CK(cudaMemcpyAsync(v, s->d_v, sizeof(double) * s->d, cudaMemcpyDeviceToHost, s->stream));
  long long tt = 0;
  CK(cudaMemcpyAsync(&tt, s->d_t, sizeof tt, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (t) *t = tt;
  return EVORL_OK;
}
extern "C" int evorl_es_set_adam(evorl_es* s, const double* m, const double* v, int64_t t) {
  CK(cudaSetDevice(s->cfg.device));
  long long tt = t;
  CK(cudaMemcpyAsync(s->d_m, m, sizeof(double) * s->d, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(s->d_v, v, sizeof(double) * s->d, cudaMemcpyHostToDevice, s->stream));
  CK(cudaMemcpyAsync(s->d_t, &tt, sizeof tt, cudaMemcpyHostToDevice, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  s->adam_t_host = t;
  return EVORL_OK;
}
// CmaState transfer (proj/include/evorl/ec.hpp:107-122; checkpoint segments
// ec/C, ec/B, ec/D, ec/ps, ec/pc, ec/sigma, ec/generation,
// ec/recondition_count of proj/src/workflow_es.cpp:194-203).  C and B are
// d x d row-major (B[p*d + j] = component p of eigenvector j); any pointer may
// be NULL.
extern "C" int evorl_es_cma_get(evorl_es* s, double* C, double* B, double* D, double* ps, double* pc,
                                double* sigma, int64_t* generation, int64_t* recondition_count) {
  if (s->cfg.algo != EVORL_ALGO_CMAES) return set_err(EVORL_E_INVALID_ARGUMENT, "not a cmaes workflow");
  CK(cudaSetDevice(s->cfg.device));
  const CmaDev& v = s->cma.dev;
  const int d = (int)s->d;
  if (C) CK(cudaMemcpy2D(C, sizeof(double) * d, v.C, sizeof(double) * v.dp, sizeof(double) * d, d,
                         cudaMemcpyDeviceToHost));
  if (B) CK(cudaMemcpy2D(B, sizeof(double) * d, v.B, sizeof(double) * v.dp, sizeof(double) * d, d,
                         cudaMemcpyDeviceToHost));
  if (D) CK(cudaMemcpy(D, v.D, sizeof(double) * d, cudaMemcpyDeviceToHost));
  if (ps) CK(cudaMemcpy(ps, v.ps, sizeof(double) * d, cudaMemcpyDeviceToHost));
  if (pc) CK(cudaMemcpy(pc, v.pc, sizeof(double) * d, cudaMemcpyDeviceToHost));
  if (sigma) *sigma = s->cma.sigma;
  if (generation) *generation = s->cma.generation;
  if (recondition_count) *recondition_count = s->cma.recondition_count;
  return EVORL_OK;
}

extern "C" int evorl_es_cma_set(evorl_es* s, const double* C, const double* B, const double* D,
                                const double* ps, const double* pc, double sigma, int64_t generation,
                                int64_t recondition_count) {
  if (s->cfg.algo != EVORL_ALGO_CMAES) return set_err(EVORL_E_INVALID_ARGUMENT, "not a cmaes workflow");
  CK(cudaSetDevice(s->cfg.device));
  CmaDev& v = s->cma.dev;
  const int d = (int)s->d;
  if (C) CK(cudaMemcpy2D(v.C, sizeof(double) * v.dp, C, sizeof(double) * d, sizeof(double) * d, d,
                         cudaMemcpyHostToDevice));
  if (B) CK(cudaMemcpy2D(v.B, sizeof(double) * v.dp, B, sizeof(double) * d, sizeof(double) * d, d,
                         cudaMemcpyHostToDevice));
  if (D) CK(cudaMemcpy(v.D, D, sizeof(double) * d, cudaMemcpyHostToDevice));
  if (ps) CK(cudaMemcpy(v.ps, ps, sizeof(double) * d, cudaMemcpyHostToDevice));
  if (pc) CK(cudaMemcpy(v.pc, pc, sizeof(double) * d, cudaMemcpyHostToDevice));
  s->cma.sigma = sigma;
  s->cma.generation = generation;
  s->cma.recondition_count = recondition_count;
  return EVORL_OK;
}

extern "C" int evorl_es_get_fitness(evorl_es* s, double* f) {
  CK(cudaSetDevice(s->cfg.device));
  CK(cudaMemcpyAsync(f, s->d_fitness, sizeof(double) * s->cfg.pop, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}
extern "C" int evorl_es_get_obs_norm(evorl_es* s, evorl_obs_norm* o) {
  CK(cudaSetDevice(s->cfg.device));
  DevNorm nm{};
  CK(cudaMemcpyAsync(&nm, s->d_norm, sizeof nm, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  o->mode = nm.mode;
  o->dim = nm.dim;
  for (int i = 0; i < 4; ++i) {
    o->mean[i] = nm.mean[i];
    o->var[i] = nm.var[i];
  }
  o->count = nm.count;
  return EVORL_OK;
}
extern "C" int evorl_es_set_obs_norm(evorl_es* s, const evorl_obs_norm* o) {
  CK(cudaSetDevice(s->cfg.device));
  DevNorm nm{};
  nm.mode = o->mode;
  nm.dim = o->dim;
  for (int i = 0; i < 4; ++i) {
    nm.mean[i] = o->mean[i];
    nm.var[i] = o->var[i];
  }
  nm.count = o->count;
  CK(cudaMemcpyAsync(s->d_norm, &nm, sizeof nm, cudaMemcpyHostToDevice, s->stream));
  CK(run_norm_params(s->d_norm, s->d_normp, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  return EVORL_OK;
}

// Workflow::evaluate -> eval_params(m=1, e=episodes) (proj/src/workflow.cpp:103-129)
extern "C" int evorl_es_evaluate(evorl_es* s, int32_t episodes, uint64_t key_hi, uint64_t key_lo,
                                 double* mean_return, double* return_std) {
  if (s->cma_only) return set_err(EVORL_E_INVALID_ARGUMENT, "cma-only handle has no policy to evaluate");
  CK(cudaSetDevice(s->cfg.device));
  if (episodes < 1) return set_err(EVORL_E_INVALID_ARGUMENT, "episodes must be positive");
  SmemPlan plan{};
  if (!plan_rollout(s->net, s->env.obs_dim, episodes, s->cfg.precision, &plan))
    return set_err(EVORL_E_UNSUPPORTED, "policy too large for a shared-memory resident team");
  double* rets = nullptr;
  long long* steps = nullptr;
  double* out2 = nullptr;
  CK(cudaMallocAsync((void**)&rets, sizeof(double) * episodes, s->stream));
  CK(cudaMallocAsync((void**)&steps, sizeof(long long) * episodes, s->stream));
  CK(cudaMallocAsync((void**)&out2, sizeof(double) * 2, s->stream));
  CK(cudaMemsetAsync(s->d_fault, 0xFF, sizeof(unsigned long long), s->stream));
  RolloutArgs a{};
  a.env = s->env;
  a.net = s->net;
  a.par.src = SRC_EXPLICIT;
  a.par.params = s->d_mean;
  a.plan = plan;
  a.norm = s->d_normp;
  a.n_agents = 1;
  a.agent_offset = 0;
  a.e = episodes;
  a.count = episodes;
  a.groups = (episodes + plan.ET - 1) / plan.ET;
  a.rollout_key = mk(key_hi, key_lo);
  a.track_stats = 0;
  a.max_iters = s->env.max_episode_steps + 1;
  a.ep_returns = rets;
  a.lane_steps = steps;
  a.fault = s->d_fault;
  float* mean_f32 = nullptr;
  if (plan.gw && s->cfg.precision != EVORL_PREC_F64 && s->cfg.precision != EVORL_PREC_OZ) {  // fp32 gw team: fp32 row
    CK(cudaMallocAsync((void**)&mean_f32, sizeof(float) * s->d, s->stream));
    CK(run_materialize_f32(a.par, s->d, 0, 1, mean_f32, s->stream));
    a.par.src = SRC_EXPLICIT_F32;
    a.par.params_f32 = mean_f32;
  }
  CK(launch_rollout(a, s->cfg.precision, s->stream));
  if (mean_f32) CK(cudaFreeAsync(mean_f32, s->stream));
  count_launch();
  CK(run_eval_reduce(rets, episodes, out2, s->stream));
  CK(cudaMemcpyAsync(s->h->eval, out2, sizeof(double) * 2, cudaMemcpyDeviceToHost, s->stream));
  CK(cudaMemcpyAsync(&s->h->fault, s->d_fault, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s->stream));
  CK(cudaFreeAsync(rets, s->stream));
  CK(cudaFreeAsync(steps, s->stream));
  CK(cudaFreeAsync(out2, s->stream));
  CK(cudaStreamSynchronize(s->stream));
  if (s->h->fault != ~0ull) return fault_to_error(s->h->fault);
  *mean_return = s->h->eval[0];
  *return_std = s->h->eval[1];
  return EVORL_OK;
}

// ================================================================ stateless
// Scratch device buffers for the stateless (host-buffer) entry points.
struct Scratch {
  void* p = nullptr;
  ~Scratch() {
    if (p) cudaFree(p);
  }
};
template <typename T>
static int up(Scratch& s, const T* host, size_t n, T** dev) {
  CK(cudaMalloc(&s.p, sizeof(T) * (n ? n : 1)));
  *dev = (T*)s.p;
  if (host && n) CK(cudaMemcpy(*dev, host, sizeof(T) * n, cudaMemcpyHostToDevice));
  return EVORL_OK;
}
static int ensure_device() {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
    return set_err(EVORL_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  return EVORL_OK;
}
#define DEV_OR_RETURN()        \
  do {                         \
    int _rc = ensure_device(); \
    if (_rc) return _rc;       \
  } while (0)

extern "C" int evorl_threefry2x64(const uint64_t* keys, const uint64_t* ctrs, uint64_t* out, int64_t n) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  Scratch a, b, c;
  uint64_t *dk, *dc, *dout;
  if (int rc = up(a, keys, 2 * n, &dk)) return rc;
  if (int rc = up(b, ctrs, 2 * n, &dc)) return rc;
  if (int rc = up(c, (const uint64_t*)nullptr, 2 * n, &dout)) return rc;
  CK(run_threefry_batch(dk, dc, dout, n, 0));
  CK(cudaMemcpy(out, dout, sizeof(uint64_t) * 2 * n, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_stream_words(uint64_t hi, uint64_t lo, int64_t first, int64_t n, uint64_t* out) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  Scratch a;
  uint64_t* d;
  if (int rc = up(a, (const uint64_t*)nullptr, n, &d)) return rc;
  CK(run_stream_words(mk(hi, lo), first, n, d, 0));
  CK(cudaMemcpy(out, d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_gaussian_matrix(uint64_t hi, uint64_t lo, int64_t rows, int64_t cols, double* out) {
  DEV_OR_RETURN();
  if (rows * cols <= 0) return EVORL_OK;
  Scratch a;
  double* d;
  if (int rc = up(a, (const double*)nullptr, rows * cols, &d)) return rc;
  CK(run_gaussian_matrix(mk(hi, lo), rows, cols, d, 0));
  CK(cudaMemcpy(out, d, sizeof(double) * rows * cols, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_centered_ranks(const double* f, int64_t n, double* shaped) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  Scratch a, b, c;
  double *df, *ds;
  int* dr;
  if (int rc = up(a, f, n, &df)) return rc;
  if (int rc = up(b, (const int*)nullptr, n, &dr)) return rc;
  if (int rc = up(c, (const double*)nullptr, n, &ds)) return rc;
  CK(run_rank(df, (int)n, 0, dr, 0));
  CK(run_shaped_from_rank(dr, (int)n, ds, 0));
  CK(cudaMemcpy(shaped, ds, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_rank_desc(const double* f, int64_t n, int32_t* order) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  Scratch a, b, c;
  double* df;
  int *dr, *dord;
  if (int rc = up(a, f, n, &df)) return rc;
  if (int rc = up(b, (const int*)nullptr, n, &dr)) return rc;
  if (int rc = up(c, (const int*)nullptr, n, &dord)) return rc;
  CK(run_rank(df, (int)n, 1, dr, 0));
  CK(run_order_from_rank(dr, (int)n, dord, 0));
  CK(cudaMemcpy(order, dord, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_env_step_batch(int env_id, int fixed_horizon, int max_episode_steps, int64_t n,
                                    double* phys, int32_t* step_count, const double* action, double* reward,
                                    int32_t* terminated, int32_t* truncated, int32_t* fault) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  const EnvDesc env = make_env(env_id, fixed_horizon, max_episode_steps);
  Scratch a, b, c, d, e, f, g;
  double *dp, *da, *dr;
  int *dsc, *dt, *dtr, *df;
  if (int rc = up(a, phys, 4 * n, &dp)) return rc;
  if (int rc = up(b, step_count, n, &dsc)) return rc;
  if (int rc = up(c, action, n, &da)) return rc;
  if (int rc = up(d, (const double*)nullptr, n, &dr)) return rc;
  if (int rc = up(e, (const int*)nullptr, n, &dt)) return rc;
  if (int rc = up(f, (const int*)nullptr, n, &dtr)) return rc;
  if (int rc = up(g, (const int*)nullptr, n, &df)) return rc;
  CK(run_env_step_batch(env, n, dp, dsc, da, dr, dt, dtr, df, 0));
  CK(cudaMemcpy(phys, dp, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(step_count, dsc, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(reward, dr, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(terminated, dt, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(truncated, dtr, sizeof(int) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(fault, df, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

// transition outputs of evorl_batched_rollout_transitions (host pointers)
struct TransHost {
  long long row_cap;
  double *obs, *act, *rew, *next;
  uint8_t *term, *trunc;
  int64_t* lane_rows;
};

static int batched_rollout_impl(const evorl_env_desc* envd, const evorl_mlp_desc* netd,
                                const evorl_obs_norm* norm, const double* params, int32_t m, int32_t e,
                                int32_t count, uint64_t key_hi, uint64_t key_lo, int32_t precision,
                                double* returns, int64_t* steps, double* obs_stats, const TransHost* tr) {
  DEV_OR_RETURN();
  if (m <= 0) return EVORL_OK;
  if (e < 1 || count < 0) return set_err(EVORL_E_INVALID_ARGUMENT, "envs_per_agent must be positive");
  const EnvDesc env = make_env(envd->env_id, envd->fixed_horizon, envd->max_episode_steps);
  NetDesc net{};
  if (int rc = make_net(*netd, &net)) return rc;
  if (netd->input_dim != env.obs_dim) return set_err(EVORL_E_INVALID_ARGUMENT, "net input_dim != obs_dim");
  SmemPlan plan{};
  WarpPlanOut wplan{};
  if (precision < EVORL_PREC_F64 || precision > EVORL_PREC_OZ)
    return set_err(EVORL_E_INVALID_ARGUMENT, "unknown precision");
  // transitions are written by the cluster team (the tc team evaluates as f32)
  const bool cta_ok = plan_rollout(net, env.obs_dim, e, tr && precision == EVORL_PREC_TC ? EVORL_PREC_F32 : precision,
                                   &plan, tr != nullptr);
  if (tr) plan.trn = 1;
  const bool use_warp =
      !tr && !(cta_ok && (plan.tc || plan.oz)) && plan_rollout_warp(net, env.obs_dim, e, precision, &wplan);
  if (!cta_ok && !use_warp)
    return set_err(EVORL_E_UNSUPPORTED, "policy too large for a shared-memory resident team");
  const long long d = net.d;
  const long long max_iters = (long long)((count + e - 1) / e) * env.max_episode_steps;
  if (tr && tr->row_cap < max_iters)
    return set_err(EVORL_E_INVALID_ARGUMENT, "row_cap (%lld) below episodes per lane x max_episode_steps (%lld)",
                   tr->row_cap, max_iters);
  Scratch sp, sr, ss, sst, sag, sn, sf;
  double *dparams, *drets, *dstats, *dagent;
  long long* dsteps;
  NormParams* dnorm = nullptr;
  unsigned long long* dfault;
  if (int rc = up(sp, params, (size_t)m * d, &dparams)) return rc;
  if (int rc = up(sr, (const double*)nullptr, (size_t)m * std::max(count, 1), &drets)) return rc;
  if (int rc = up(ss, (const long long*)nullptr, (size_t)m * e, &dsteps)) return rc;
  if (int rc = up(sst, (const double*)nullptr, (size_t)m * e * 9, &dstats)) return rc;
  if (int rc = up(sag, (const double*)nullptr, (size_t)m * 9, &dagent)) return rc;
  if (int rc = up(sf, (const unsigned long long*)nullptr, 1, &dfault)) return rc;
  if (norm && norm->mode != EVORL_NORM_NONE) {
    NormParams np{};
    np.active = norm->count != 0.0;
    np.dim = norm->dim;
    for (int i = 0; i < 4; ++i) {
      np.mean[i] = norm->mean[i];
      const double sd = std::sqrt(norm->var[i]);
      np.den[i] = sd > 1e-8 ? sd : 1e-8;
    }
    if (int rc = up(sn, &np, 1, &dnorm)) return rc;
  }
  CK(cudaMemset(dfault, 0xFF, sizeof(unsigned long long)));
  CK(cudaMemset(dstats, 0, sizeof(double) * m * e * 9));
  RolloutArgs a{};
  a.env = env;
  a.net = net;
  a.par.src = SRC_EXPLICIT;
  a.par.params = dparams;
  a.plan = plan;
  a.norm = dnorm;
  a.n_agents = m;
  a.e = e;
  a.count = count;
  a.groups = (e + plan.ET - 1) / plan.ET;
  a.rollout_key = mk(key_hi, key_lo);
  a.track_stats = obs_stats != nullptr;
  a.max_iters = ((count + e - 1) / e) * env.max_episode_steps + 1;
  a.ep_returns = drets;
  a.lane_steps = dsteps;
  a.lane_stats = dstats;
  a.fault = dfault;
  Scratch st_o, st_a, st_r, st_n, st_t, st_u;
  if (tr) {
    const size_t rows = (size_t)m * e * tr->row_cap;
    if (int rc = up(st_o, (const double*)nullptr, rows * env.obs_dim, &a.t_obs)) return rc;
    if (int rc = up(st_n, (const double*)nullptr, rows * env.obs_dim, &a.t_next)) return rc;
    if (int rc = up(st_a, (const double*)nullptr, rows, &a.t_act)) return rc;
    if (int rc = up(st_r, (const double*)nullptr, rows, &a.t_rew)) return rc;
    if (int rc = up(st_t, (const unsigned char*)nullptr, rows, &a.t_term)) return rc;
    if (int rc = up(st_u, (const unsigned char*)nullptr, rows, &a.t_trunc)) return rc;
    a.t_cap = tr->row_cap;
  }
  Scratch sf32;
  if (!use_warp && plan.gw && precision != EVORL_PREC_F64 && precision != EVORL_PREC_OZ) {  // fp32 gw team
    float* pf = nullptr;
    if (int rc = up(sf32, (const float*)nullptr, (size_t)m * d, &pf)) return rc;
    CK(run_materialize_f32(a.par, d, 0, m, pf, 0));
    a.par.src = SRC_EXPLICIT_F32;
    a.par.params_f32 = pf;
  }
  if (use_warp) {
    CK(launch_rollout_warp(a, wplan, precision, 0));
  } else {
    CK(launch_rollout(a, precision, 0));
    count_launch();
  }
  if (obs_stats) CK(run_agent_stats(dstats, m, e, dagent, 0));
  CK(cudaDeviceSynchronize());
  unsigned long long fault = 0;
  CK(cudaMemcpy(&fault, dfault, sizeof fault, cudaMemcpyDeviceToHost));
  if (fault != ~0ull) return fault_to_error(fault);
  if (returns) CK(cudaMemcpy(returns, drets, sizeof(double) * m * count, cudaMemcpyDeviceToHost));
  if (steps) {
    std::vector<long long> ls((size_t)m * e);
    CK(cudaMemcpy(ls.data(), dsteps, sizeof(long long) * m * e, cudaMemcpyDeviceToHost));
    for (int i = 0; i < m; ++i) {
      long long acc = 0;
      for (int j = 0; j < e; ++j) acc += ls[(size_t)i * e + j];
      steps[i] = acc;
    }
  }
  if (obs_stats) CK(cudaMemcpy(obs_stats, dagent, sizeof(double) * m * 9, cudaMemcpyDeviceToHost));
  if (tr) {
    const size_t rows = (size_t)m * e * tr->row_cap;
    CK(cudaMemcpy(tr->obs, a.t_obs, sizeof(double) * rows * env.obs_dim, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->next, a.t_next, sizeof(double) * rows * env.obs_dim, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->act, a.t_act, sizeof(double) * rows, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->rew, a.t_rew, sizeof(double) * rows, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->term, a.t_term, rows, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->trunc, a.t_trunc, rows, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tr->lane_rows, dsteps, sizeof(long long) * m * e, cudaMemcpyDeviceToHost));
  }
  return EVORL_OK;
}

extern "C" int evorl_batched_rollout(const evorl_env_desc* envd, const evorl_mlp_desc* netd,
                                     const evorl_obs_norm* norm, const double* params, int32_t m, int32_t e,
                                     int32_t count, uint64_t key_hi, uint64_t key_lo, int32_t precision,
                                     double* returns, int64_t* steps, double* obs_stats) {
  return batched_rollout_impl(envd, netd, norm, params, m, e, count, key_hi, key_lo, precision, returns, steps,
                              obs_stats, nullptr);
}

extern "C" int evorl_batched_rollout_transitions(const evorl_env_desc* envd, const evorl_mlp_desc* netd,
                                                 const evorl_obs_norm* norm, const double* params, int32_t m,
                                                 int32_t e, int32_t count, uint64_t key_hi, uint64_t key_lo,
                                                 int32_t precision, double* returns, int64_t* steps,
                                                 int64_t row_cap, double* t_obs, double* t_act, double* t_rew,
                                                 uint8_t* t_term, uint8_t* t_trunc, double* t_next,
                                                 int64_t* lane_rows) {
  const TransHost tr{row_cap, t_obs, t_act, t_rew, t_next, t_term, t_trunc, lane_rows};
  return batched_rollout_impl(envd, netd, norm, params, m, e, count, key_hi, key_lo, precision, returns, steps,
                              nullptr, &tr);
}

extern "C" int evorl_openes_ask(const double* mean, int64_t d, double sigma, int32_t mirrored, uint64_t hi,
                                uint64_t lo, int32_t n, double* cand, double* eps) {
  DEV_OR_RETURN();
  if (n < 2) return set_err(EVORL_E_INVALID_ARGUMENT, "openes_ask: population must be at least 2");
  if (mirrored && n % 2)
    return set_err(EVORL_E_INVALID_ARGUMENT, "openes_ask: mirrored sampling needs an even population");
  Scratch a, b, c;
  double *dm, *dc, *de;
  if (int rc = up(a, mean, d, &dm)) return rc;
  if (int rc = up(b, (const double*)nullptr, (size_t)n * d, &dc)) return rc;
  if (int rc = up(c, (const double*)nullptr, (size_t)n * d, &de)) return rc;
  CK(run_openes_ask(dm, d, sigma, mirrored, mk(hi, lo), n, dc, de, 0));
  if (cand) CK(cudaMemcpy(cand, dc, sizeof(double) * n * d, cudaMemcpyDeviceToHost));
  if (eps) CK(cudaMemcpy(eps, de, sizeof(double) * n * d, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_openes_tell(double* mean, double* m, double* v, int64_t* t, int64_t d, double sigma,
                                 double lr, double wd, int32_t mirrored, uint64_t hi, uint64_t lo,
                                 const double* fitness, int32_t n) {
  DEV_OR_RETURN();
  if (n < 1) return set_err(EVORL_E_INVALID_ARGUMENT, "openes_tell: eps/fitness size mismatch");
  if (mirrored && n % 2)
    return set_err(EVORL_E_INVALID_ARGUMENT, "openes_ask: mirrored sampling needs an even population");
  Scratch a, b, c, f, r, sh, tt, bc, pt;
  double *dmean, *dm, *dv, *df, *dsh, *dbc;
  int* dr;
  long long* dt;
  long long th = *t;
  if (int rc = up(a, mean, d, &dmean)) return rc;
  if (int rc = up(b, m, d, &dm)) return rc;
  if (int rc = up(c, v, d, &dv)) return rc;
  if (int rc = up(f, fitness, n, &df)) return rc;
  if (int rc = up(r, (const int*)nullptr, n, &dr)) return rc;
  if (int rc = up(sh, (const double*)nullptr, n, &dsh)) return rc;
  if (int rc = up(tt, &th, 1, &dt)) return rc;
  const double bch[2] = {1.0 - std::pow(0.9, (double)(th + 1)), 1.0 - std::pow(0.999, (double)(th + 1))};
  if (int rc = up(bc, bch, 2, &dbc)) return rc;
  CK(run_rank(df, n, 0, dr, 0));
  CK(run_shaped_from_rank(dr, n, dsh, 0));
  OpenEsTellArgs ta{};
  ta.mean = dmean;
  ta.m = dm;
  ta.v = dv;
  ta.t_dev = dt;
  ta.d = d;
  ta.p0 = 0;
  ta.p1 = d;
  ta.sigma = sigma;
  ta.lr = lr;
  ta.weight_decay = wd;
  ta.lrwd = lr * wd;
  ta.beta1 = 0.9;
  ta.beta2 = 0.999;
  ta.omb1 = 1.0 - 0.9;
  ta.omb2 = 1.0 - 0.999;
  ta.eps = 1e-8;
  ta.n = n;
  ta.mirrored = mirrored;
  ta.base = mirrored ? n / 2 : n;
  ta.ask_key = mk(hi, lo);
  ta.shaped = dsh;
  // single-entry table holding exactly this step's corrections
  ta.adam_bc = dbc - 2 * th;  // index 2*(t-1) with t = th+1 -> dbc[0]
  ta.adam_bc_len = th + 1;
  double* dpart = nullptr;
  const long long part_n = (long long)openes_tell_chunks(ta.base, d) * d;
  if (int rc = up(pt, (const double*)nullptr, (size_t)part_n, &dpart)) return rc;
  ta.partial = dpart;
  CK(run_openes_tell(ta, 0));
  CK(cudaMemcpy(mean, dmean, sizeof(double) * d, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(m, dm, sizeof(double) * d, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(v, dv, sizeof(double) * d, cudaMemcpyDeviceToHost));
  *t = th + 1;
  return EVORL_OK;
}

extern "C" int evorl_ars_ask(const double* mean, int64_t d, double sigma, uint64_t hi, uint64_t lo, int32_t n,
                             double* deltas, double* cand) {
  DEV_OR_RETURN();
  if (n < 2 || n % 2) return set_err(EVORL_E_INVALID_ARGUMENT, "ars_ask: population must be even");
  Scratch a, b, c;
  double *dm, *dd, *dc;
  if (int rc = up(a, mean, d, &dm)) return rc;
  if (int rc = up(b, (const double*)nullptr, (size_t)(n / 2) * d, &dd)) return rc;
  if (int rc = up(c, (const double*)nullptr, (size_t)n * d, &dc)) return rc;
  CK(run_ars_ask(dm, d, sigma, mk(hi, lo), n, dd, dc, 0));
  if (deltas) CK(cudaMemcpy(deltas, dd, sizeof(double) * (n / 2) * d, cudaMemcpyDeviceToHost));
  if (cand) CK(cudaMemcpy(cand, dc, sizeof(double) * n * d, cudaMemcpyDeviceToHost));
  return EVORL_OK;
}

extern "C" int evorl_ars_tell(double* mean, int64_t d, int32_t elites, double lr, uint64_t hi, uint64_t lo,
                              const double* fitness, int32_t n, int32_t* updated) {
  DEV_OR_RETURN();
  if (n < 2 || n % 2) return set_err(EVORL_E_INVALID_ARGUMENT, "ars_tell: reward/direction size mismatch");
  const int half = n / 2;
  Scratch a, f, sc, r, ei, ed, se;
  double *dm, *df, *dsc, *ded;
  int *dr, *dei;
  ArsSel* dsel;
  if (int rc = up(a, mean, d, &dm)) return rc;
  if (int rc = up(f, fitness, n, &df)) return rc;
  if (int rc = up(sc, (const double*)nullptr, half, &dsc)) return rc;
  if (int rc = up(r, (const int*)nullptr, half, &dr)) return rc;
  if (int rc = up(ei, (const int*)nullptr, half, &dei)) return rc;
  if (int rc = up(ed, (const double*)nullptr, half, &ded)) return rc;
  if (int rc = up(se, (const ArsSel*)nullptr, 1, &dsel)) return rc;
  CK(run_ars_scores(df, half, dsc, 0));
  CK(run_rank(dsc, half, 1, dr, 0));
  CK(run_ars_select(df, dr, half, elites, lr, dei, ded, dsel, 0));
  CK(run_ars_update(dm, d, 0, d, mk(hi, lo), dei, ded, dsel, 0));
  ArsSel hs{};
  CK(cudaMemcpy(&hs, dsel, sizeof hs, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mean, dm, sizeof(double) * d, cudaMemcpyDeviceToHost));
  if (updated) *updated = hs.skipped ? 0 : 1;
  return EVORL_OK;
}

extern "C" int evorl_measure_dmma_peak(double* tflops) {
  DEV_OR_RETURN();
  *tflops = measure_dmma_peak_tflops();
  CK(cudaGetLastError());
  return EVORL_OK;
}

// The ask's noise generator at full machine occupancy: n normals of a fixed
// key by k_noise_rows (16 blocks per SM), device ms of the second of two runs.
extern "C" int evorl_measure_noise_rate(int64_t n, float* ms) {
  DEV_OR_RETURN();
  if (n <= 0) return set_err(EVORL_E_INVALID_ARGUMENT, "measure_noise_rate: n must be positive");
  int dev = 0, sms = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  Scratch buf;
  double* eps;
  if (int rc = up(buf, (const double*)nullptr, (size_t)n, &eps)) return rc;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const DKey key{0x9E3779B97F4A7C15ull, 0xBB67AE8584CAA73Bull};
  cudaError_t err = run_noise_rows(key, 0, n, eps, 16 * sms, 0);
  if (err == cudaSuccess) err = cudaEventRecord(e0, 0);
  if (err == cudaSuccess) err = run_noise_rows(key, 0, n, eps, 16 * sms, 0);
  if (err == cudaSuccess) err = cudaEventRecord(e1, 0);
  if (err == cudaSuccess) err = cudaEventSynchronize(e1);
  if (err == cudaSuccess) err = cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(err);
  return EVORL_OK;
}

extern "C" int evorl_measure_fp64_peak(double* tflops) {
  DEV_OR_RETURN();
  *tflops = measure_fp64_peak_tflops();
  CK(cudaGetLastError());
  return EVORL_OK;
}

// Symmetric eigendecomposition on the device (the K7 Jacobi eigensolver,
// replacing Eigen::SelfAdjointEigenSolver at proj/src/ec.cpp:278-287):
// A is n x n row-major symmetric; evals ascending; vecs[p*n + j] = component
// p of eigenvector j (largest-|.| component positive).  Returns the sweeps in
// *sweeps.
extern "C" int evorl_sym_eig(const double* A, int32_t n, double* evals, double* vecs, int32_t* sweeps) {
  DEV_OR_RETURN();
  if (n <= 0) return EVORL_OK;
  CmaDev v{};
  v.d = n;
  v.dp = (n + 63) / 64 * 64;
  const size_t dp2 = (size_t)v.dp * v.dp;
  Scratch a, b, w, vv, u, ev, od, t1, red, sk;
  double *dA, *dB;
  if (int rc = up(a, (const double*)nullptr, dp2, &dA)) return rc;
  if (int rc = up(b, (const double*)nullptr, dp2, &dB)) return rc;
  if (int rc = up(w, (const double*)nullptr, dp2, &v.W)) return rc;
  if (int rc = up(vv, (const double*)nullptr, dp2, &v.V)) return rc;
  if (int rc = up(u, (const double*)nullptr, (size_t)(v.dp / 64) * 4096, &v.U)) return rc;
  if (int rc = up(ev, (const double*)nullptr, v.dp, &v.evals)) return rc;
  if (int rc = up(od, (const int*)nullptr, v.dp, &v.order)) return rc;
  if (int rc = up(t1, (const double*)nullptr, v.dp, &v.t1)) return rc;
  if (int rc = up(red, (const double*)nullptr, 8, &v.red)) return rc;
  if (int rc = up(sk, (const int*)nullptr, v.dp / 64, &v.skipf)) return rc;
  CK(cudaMemset(dA, 0, sizeof(double) * dp2));
  CK(cudaMemcpy2D(dA, sizeof(double) * v.dp, A, sizeof(double) * n, sizeof(double) * n, n, cudaMemcpyHostToDevice));
  double evmin = 0.0;
  const int sw = sym_eig_jacobi(v, dA, n, &evmin, dB, v.evals, 0);
  if (sw < 0) return set_err(EVORL_E_CUDA, "eigensolver failed");
  CK(cudaMemcpy(evals, v.evals, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy2D(vecs, sizeof(double) * n, dB, sizeof(double) * v.dp, sizeof(double) * n, n,
                  cudaMemcpyDeviceToHost));
  if (sweeps) *sweeps = sw;
  return EVORL_OK;
}


// ====================================================== checkpoint interop
// EVORL1 files (proj/src/checkpoint.cpp:6-212): magic "EVORL1", u32 version 1,
// length-prefixed workflow id, u32 segment count, then segments {u32 name
// length, name, u8 type (0 f64, 1 i64), u64 count, little-endian 64-bit words}.
// EsWorkflow::save/load (proj/src/workflow_es.cpp:181-249) with the base
// segments of proj/src/workflow.cpp:11-25 and the obs_norm / adam helpers of
// proj/src/workflow.cpp:146-174, in the same order, so files are
// interchangeable with the reference's.
namespace {

struct SegWriter {
  std::string buf;
  uint32_t count = 0;
  static void u32(std::string& b, uint32_t v) {
    for (int i = 0; i < 4; ++i) b.push_back((char)((v >> (8 * i)) & 0xff));
  }
  static void u64(std::string& b, uint64_t v) {
    for (int i = 0; i < 8; ++i) b.push_back((char)((v >> (8 * i)) & 0xff));
  }
  void head(const std::string& name, uint8_t type, uint64_t n) {
    u32(buf, (uint32_t)name.size());
    buf += name;
    buf.push_back((char)type);
    u64(buf, n);
    ++count;
  }
  void f64(const std::string& name, const double* p, size_t n) {
    head(name, 0, n);
    for (size_t i = 0; i < n; ++i) {
      uint64_t w;
      std::memcpy(&w, p + i, 8);
      u64(buf, w);
    }
  }
  void f64(const std::string& name, double v) { f64(name, &v, 1); }
  void i64(const std::string& name, const int64_t* p, size_t n) {
    head(name, 1, n);
    for (size_t i = 0; i < n; ++i) u64(buf, (uint64_t)p[i]);
  }
  void i64(const std::string& name, int64_t v) { i64(name, &v, 1); }
};

struct SegReader {
  std::vector<std::pair<std::string, std::vector<double>>> f;
  std::vector<std::pair<std::string, std::vector<int64_t>>> i;
  const std::vector<double>* fv(const std::string& n) const {
    for (auto& x : f)
      if (x.first == n) return &x.second;
    return nullptr;
  }
  const std::vector<int64_t>* iv(const std::string& n) const {
    for (auto& x : i)
      if (x.first == n) return &x.second;
    return nullptr;
  }
};

int ckpt_err(const char* fmt, const std::string& a = "", const std::string& b = "") {
  return set_err(EVORL_E_CHECKPOINT, fmt, a.c_str(), b.c_str());
}

// parse (proj/src/checkpoint.cpp:72-118): later segments of the same name
// replace earlier ones, as std::map::operator[] does
int ckpt_parse(const std::string& bytes, std::string* id, SegReader* r) {
  size_t pos = 0;
  bool ok = true;
  auto need = [&](size_t n) {
    if (pos + n > bytes.size()) ok = false;
    return ok;
  };
  auto u32 = [&]() -> uint32_t {
    if (!need(4)) return 0;
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) v |= (uint32_t)(unsigned char)bytes[pos + k] << (8 * k);
    pos += 4;
    return v;
  };
  auto u64 = [&]() -> uint64_t {
    if (!need(8)) return 0;
    uint64_t v = 0;
    for (int k = 0; k < 8; ++k) v |= (uint64_t)(unsigned char)bytes[pos + k] << (8 * k);
    pos += 8;
    return v;
  };
  auto str = [&](size_t n) -> std::string {
    if (!need(n)) return std::string();
    std::string s = bytes.substr(pos, n);
    pos += n;
    return s;
  };
  const std::string magic = str(6);
  if (!ok) return ckpt_err("incompatible checkpoint: truncated file");
  if (magic != "EVORL1") return ckpt_err("incompatible checkpoint: bad magic");
  const uint32_t version = u32();
  if (!ok) return ckpt_err("incompatible checkpoint: truncated file");
  if (version != 1)
    return set_err(EVORL_E_CHECKPOINT, "incompatible checkpoint: format version %u", (unsigned)version);
  *id = str(u32());
  const uint32_t nseg = u32();
  if (!ok) return ckpt_err("incompatible checkpoint: truncated file");
  for (uint32_t sgi = 0; sgi < nseg; ++sgi) {
    const std::string name = str(u32());
    if (!need(1)) return ckpt_err("incompatible checkpoint: truncated file");
    const uint8_t type = (uint8_t)bytes[pos++];
    const uint64_t n = u64();
    if (!ok) return ckpt_err("incompatible checkpoint: truncated file");
    if (type > 1) return ckpt_err("incompatible checkpoint: unknown segment type");
    if (n > (bytes.size() - pos) / 8) return ckpt_err("incompatible checkpoint: truncated file");
    if (type == 0) {
      std::vector<double> v(n);
      for (uint64_t k = 0; k < n; ++k) {
        const uint64_t w = u64();
        std::memcpy(&v[k], &w, 8);
      }
      bool replaced = false;
      for (auto& x : r->f)
        if (x.first == name) {
          x.second = std::move(v);
          replaced = true;
          break;
        }
      if (!replaced) r->f.emplace_back(name, std::move(v));
    } else {
      std::vector<int64_t> v(n);
      for (uint64_t k = 0; k < n; ++k) v[k] = (int64_t)u64();
      bool replaced = false;
      for (auto& x : r->i)
        if (x.first == name) {
          x.second = std::move(v);
          replaced = true;
          break;
        }
      if (!replaced) r->i.emplace_back(name, std::move(v));
    }
  }
  if (pos != bytes.size()) return ckpt_err("incompatible checkpoint: trailing bytes after last segment");
  return EVORL_OK;
}

}  // namespace

extern "C" int evorl_es_save(evorl_es* s, const char* path) {
  if (!s->initialised) return set_err(EVORL_E_INVALID_ARGUMENT, "evorl_es_save before evorl_es_init");
  const long long d = s->d;
  SegWriter w;
  // WorkflowState::save_base (proj/src/workflow.cpp:11-17)
  w.i64("iteration", (int64_t)s->iteration);
  const int64_t key[2] = {(int64_t)s->rng.hi, (int64_t)s->rng.lo};
  w.i64("rng", key, 2);
  w.i64("env_steps", (int64_t)s->env_steps);
  w.i64("episodes", (int64_t)s->episodes);
  w.i64("rl_updates", (int64_t)0);
  // save_obs_norm (proj/src/workflow.cpp:160-165); ObsNormState::none() has
  // empty mean/var (proj/include/evorl/obs_norm.hpp:27)
  evorl_obs_norm on{};
  if (int rc = evorl_es_get_obs_norm(s, &on)) return rc;
  const int nd = on.mode == EVORL_NORM_NONE ? 0 : on.dim;
  w.i64("obs_norm/mode", (int64_t)on.mode);
  w.f64("obs_norm/mean", on.mean, nd);
  w.f64("obs_norm/var", on.var, nd);
  w.f64("obs_norm/count", on.count);
  std::vector<double> mean(d);
  if (int rc = evorl_es_get_mean(s, mean.data())) return rc;
  switch (s->cfg.algo) {
    case EVORL_ALGO_OPENES: {
      std::vector<double> m(d), v(d);
      int64_t t = 0;
      if (int rc = evorl_es_get_adam(s, m.data(), v.data(), &t)) return rc;
      w.f64("ec/mean", mean.data(), d);
      w.f64("ec/sigma", s->cfg.openes_sigma);
      w.f64("ec/adam/m", m.data(), d);
      w.f64("ec/adam/v", v.data(), d);
      w.i64("ec/adam/t", t);
      w.i64("ec/table_seed", s->d_table ? (int64_t)s->table_seed : (int64_t)0);
      break;
    }
    case EVORL_ALGO_ARS:
    case EVORL_ALGO_VES:
      w.f64("ec/mean", mean.data(), d);
      break;
    case EVORL_ALGO_CMAES: {
      std::vector<double> C(d * d), B(d * d), Bc(d * d), D(d), ps(d), pc(d);
      double sigma = 0;
      int64_t gen = 0, rec = 0;
      if (int rc = evorl_es_cma_get(s, C.data(), B.data(), D.data(), ps.data(), pc.data(), &sigma, &gen, &rec))
        return rc;
      for (long long p = 0; p < d; ++p)  // row-major B[p][j] -> Eigen column-major flat[j*d + p]
        for (long long j = 0; j < d; ++j) Bc[j * d + p] = B[p * d + j];
      w.f64("ec/mean", mean.data(), d);
      w.f64("ec/sigma", sigma);
      w.f64("ec/C", C.data(), d * d);  // symmetric: row- and column-major coincide
      w.f64("ec/B", Bc.data(), d * d);
      w.f64("ec/D", D.data(), d);
      w.f64("ec/ps", ps.data(), d);
      w.f64("ec/pc", pc.data(), d);
      w.i64("ec/generation", gen);
      w.i64("ec/recondition_count", rec);
      break;
    }
    default: {  // CEM
      std::vector<double> var(d);
      CK(cudaMemcpy(var.data(), s->d_var, sizeof(double) * d, cudaMemcpyDeviceToHost));
      w.f64("ec/mean", mean.data(), d);
      w.f64("ec/var", var.data(), d);
      w.i64("ec/iter", (int64_t)s->cem_iter);
      break;
    }
  }
  // checkpoint_save (proj/src/checkpoint.cpp:180-198): header, then tmp + rename
  std::string out = "EVORL1";
  SegWriter::u32(out, 1);
  const std::string id = "es";
  SegWriter::u32(out, (uint32_t)id.size());
  out += id;
  SegWriter::u32(out, w.count);
  out += w.buf;
  const std::string fpath(path), tmp = fpath + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return ckpt_err("cannot write checkpoint: %s", tmp);
  const size_t wr = std::fwrite(out.data(), 1, out.size(), f);
  const int cl = std::fclose(f);
  if (wr != out.size() || cl != 0) return ckpt_err("short write to checkpoint: %s", tmp);
  std::remove(fpath.c_str());
  if (std::rename(tmp.c_str(), fpath.c_str()) != 0) return ckpt_err("cannot finalize checkpoint: %s", fpath);
  return EVORL_OK;
}

extern "C" int evorl_es_load(evorl_es* s, const char* path) {
  CK(cudaSetDevice(s->cfg.device));
  std::string bytes;
  {
    FILE* f = std::fopen(path, "rb");
    if (!f) return ckpt_err("cannot open checkpoint: %s", path);
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) bytes.append(buf, n);
    std::fclose(f);
  }
  std::string id;
  SegReader r;
  if (int rc = ckpt_parse(bytes, &id, &r)) return rc;
  if (id != "es") return ckpt_err("incompatible checkpoint: workflow '%s', expected '%s'", id, "es");
  const long long d = s->d;
  auto scal_i = [&](const char* n, int64_t* out) -> int {
    const auto* v = r.iv(n);
    if (!v || v->size() != 1) return ckpt_err("checkpoint: missing integer segment '%s'", n);
    *out = (*v)[0];
    return EVORL_OK;
  };
  auto scal_f = [&](const char* n, double* out) -> int {
    const auto* v = r.fv(n);
    if (!v || v->size() != 1) return ckpt_err("checkpoint: missing scalar segment '%s'", n);
    *out = (*v)[0];
    return EVORL_OK;
  };
  auto vec = [&](const char* n, long long len, const std::vector<double>** out) -> int {
    const auto* v = r.fv(n);
    if (!v) return ckpt_err("checkpoint: missing segment '%s'", n);
    if (len >= 0 && (long long)v->size() != len) return ckpt_err("checkpoint: segment '%s' has wrong size", n);
    *out = v;
    return EVORL_OK;
  };
  // load_base (proj/src/workflow.cpp:19-25)
  int64_t it = 0, steps = 0, eps = 0, rl = 0;
  if (int rc = scal_i("iteration", &it)) return rc;
  const auto* key = r.iv("rng");
  if (!key || key->size() != 2) return ckpt_err("checkpoint: missing key segment '%s'", "rng");
  if (int rc = scal_i("env_steps", &steps)) return rc;
  if (int rc = scal_i("episodes", &eps)) return rc;
  if (int rc = scal_i("rl_updates", &rl)) return rc;
  // load_obs_norm (proj/src/workflow.cpp:167-174)
  int64_t mode = 0;
  double count = 0;
  const std::vector<double>*nmean, *nvar;
  if (int rc = scal_i("obs_norm/mode", &mode)) return rc;
  if (int rc = vec("obs_norm/mean", -1, &nmean)) return rc;
  if (int rc = vec("obs_norm/var", (long long)nmean->size(), &nvar)) return rc;
  if (int rc = scal_f("obs_norm/count", &count)) return rc;
  if (mode < 0 || mode > 2 || nmean->size() > 4 || (mode != 0 && (int)nmean->size() != s->env.obs_dim))
    return ckpt_err("checkpoint: segment '%s' has wrong size", "obs_norm/mean");
  const std::vector<double>* mean;
  if (int rc = vec("ec/mean", d, &mean)) return rc;
  // Every segment is parsed and validated before the handle is touched; the
  // device setters below can then only fail on a CUDA error, and the host-side
  // scalars (OpenES sigma / table seed, CEM iteration, keys, counters) are
  // applied last, once every device write has succeeded.
  double os_sigma = 0;
  int64_t os_seed = 0, cem_iter = 0;
  switch (s->cfg.algo) {
    case EVORL_ALGO_OPENES: {
      int64_t t = 0;
      const std::vector<double>*m, *v;
      if (int rc = scal_f("ec/sigma", &os_sigma)) return rc;
      if (int rc = vec("ec/adam/m", d, &m)) return rc;
      if (int rc = vec("ec/adam/v", d, &v)) return rc;
      if (int rc = scal_i("ec/adam/t", &t)) return rc;
      if (int rc = scal_i("ec/table_seed", &os_seed)) return rc;
      if (int rc = evorl_es_set_adam(s, m->data(), v->data(), t)) return rc;
      break;
    }
    case EVORL_ALGO_ARS:
    case EVORL_ALGO_VES:
      break;
    case EVORL_ALGO_CMAES: {
      double sigma = 0;
      int64_t gen = 0, rec = 0;
      const std::vector<double>*C, *B, *D, *ps, *pc;
      if (int rc = scal_f("ec/sigma", &sigma)) return rc;
      if (int rc = vec("ec/C", d * d, &C)) return rc;
      if (int rc = vec("ec/B", d * d, &B)) return rc;
      if (int rc = vec("ec/D", d, &D)) return rc;
      if (int rc = vec("ec/ps", d, &ps)) return rc;
      if (int rc = vec("ec/pc", d, &pc)) return rc;
      if (int rc = scal_i("ec/generation", &gen)) return rc;
      if (int rc = scal_i("ec/recondition_count", &rec)) return rc;
      std::vector<double> Br(d * d);
      for (long long p = 0; p < d; ++p)
        for (long long j = 0; j < d; ++j) Br[p * d + j] = (*B)[j * d + p];
      if (int rc = evorl_es_cma_set(s, C->data(), Br.data(), D->data(), ps->data(), pc->data(), sigma, gen, rec))
        return rc;
      break;
    }
    default: {  // CEM
      const std::vector<double>* var;
      if (int rc = vec("ec/var", d, &var)) return rc;
      if (int rc = scal_i("ec/iter", &cem_iter)) return rc;
      CK(cudaMemcpy(s->d_var, var->data(), sizeof(double) * d, cudaMemcpyHostToDevice));
      break;
    }
  }
  if (int rc = evorl_es_set_mean(s, mean->data())) return rc;
  evorl_obs_norm on{};
  on.mode = (int32_t)mode;
  on.dim = mode == 0 ? s->env.obs_dim : (int32_t)nmean->size();
  for (int k = 0; k < 4; ++k) {
    on.mean[k] = k < (int)nmean->size() ? (*nmean)[k] : 0.0;
    on.var[k] = k < (int)nvar->size() ? (*nvar)[k] : 1.0;
  }
  on.count = count;
  if (int rc = evorl_es_set_obs_norm(s, &on)) return rc;
  if (s->cfg.algo == EVORL_ALGO_OPENES) {
    const double old_sigma = s->cfg.openes_sigma;
    const uint64_t old_seed = s->table_seed;
    s->cfg.openes_sigma = os_sigma;
    if (s->d_table) {  // openes_rebuild_table (proj/src/workflow_es.cpp:223-224)
      s->table_seed = (uint64_t)os_seed;
      const cudaError_t e = rebuild_table(s);
      if (e != cudaSuccess) {
        s->cfg.openes_sigma = old_sigma;
        s->table_seed = old_seed;
        CK(e);
      }
    }
  } else if (s->cfg.algo == EVORL_ALGO_CEM) {
    s->cem_iter = cem_iter;
  }
  s->rng = DKey{(uint64_t)(*key)[0], (uint64_t)(*key)[1]};
  s->iteration = it;
  s->env_steps = steps;
  s->episodes = eps;
  s->initialised = true;
  return EVORL_OK;
}
