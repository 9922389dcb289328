/*
 * evorl_oracle.h -- CPU restatement of the EvoRL reference ES generation path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 implementation (paper_2501_15129_b200/).  Only tests/, the smoke()
 * entry of __graft_entry__.py and the cpu_baseline / --impl reference legs
 * of bench.py may load it.  The product path never links or calls it.
 *
 * Every function restates the reference C++ (/root/reference/proj, cited as
 * path:line) in plain C11, fp64, sequential accumulation order, no FMA
 * (built with -ffp-contract=off and no -march, like the reference Release
 * build, proj/CMakeLists.txt:8-15).  Parity is pinned against the reference's
 * own known-answer tests (proj/tests/test_rng.cpp, test_env.cpp, test_ec.cpp,
 * test_optim.cpp, test_obs_norm.cpp, test_net.cpp) and, for the RNG, against
 * the reference's rng.cpp compiled unchanged into oracle/_ref/ (see Makefile).
 * Eigen reduction orders (GEMV, .sum(), .mean()) are unpinned by the reference
 * tests (1e-12..1e-15); this oracle uses sequential order.
 */
#ifndef EVORL_ORACLE_H
#define EVORL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- errors */
enum {
  EO_OK = 0,
  EO_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  EO_E_LENGTH = 2,           /* std::length_error (CMA capacity cap) */
  EO_E_ENV_FAULT = 3,        /* evorl::EnvFault */
  EO_E_NET_FAULT = 4,        /* evorl::NetFault */
  EO_E_CONFIG = 5,           /* evorl::ConfigError */
  EO_E_NOMEM = 6
};
const char* eo_last_error(void);

/* ------------------------------------------------------------------ rng
 * proj/include/evorl/rng.hpp, proj/src/rng.cpp */
typedef struct {
  uint64_t hi, lo;
} eo_key;

void eo_threefry2x64(const uint64_t key[2], const uint64_t ctr[2], uint64_t out[2]);
eo_key eo_key_from_seed(uint64_t seed);
eo_key eo_fold_in(eo_key key, uint64_t index);

typedef struct {
  eo_key key;
  uint64_t block;
  uint64_t pending_word;
  int has_pending_word;
  double pending_normal;
  int has_pending_normal;
} eo_stream;

void eo_stream_init(eo_stream* s, eo_key key);
uint64_t eo_next_u64(eo_stream* s);
double eo_uniform(eo_stream* s);
double eo_uniform_range(eo_stream* s, double lo, double hi);
double eo_normal(eo_stream* s);
uint64_t eo_randint(eo_stream* s, uint64_t n);
/* proj/src/ec.cpp:22-28: row-major normals from ONE stream; out is rows x cols row-major */
void eo_gaussian_matrix(eo_key key, int64_t rows, int64_t cols, double* out);

/* ------------------------------------------------------------------ env
 * proj/include/evorl/env.hpp, proj/src/env.cpp */
enum { EO_CARTPOLE = 0, EO_PENDULUM = 1 };
typedef struct {
  int id;
  int obs_dim;
  int discrete;
  int num_actions;
  int act_dim;
  double act_low, act_high;
  int max_episode_steps;
  int fixed_horizon;
} eo_env_spec;

typedef struct {
  double phys[4];
  int step_count;
  eo_key rng;
} eo_env_state;

eo_env_spec eo_env_cartpole(int fixed_horizon, int max_episode_steps);
eo_env_spec eo_env_pendulum(int fixed_horizon, int max_episode_steps);
void eo_observe(const eo_env_spec* spec, const eo_env_state* s, double obs[4]);
void eo_env_reset(const eo_env_spec* spec, eo_key key, eo_env_state* out, double obs[4]);
/* returns EO_OK or EO_E_ENV_FAULT */
int eo_env_step(const eo_env_spec* spec, const eo_env_state* s, const double* action,
                eo_env_state* next, double* reward, int* terminated, int* truncated,
                double obs[4]);
void eo_pendulum_physics(double* th, double* thdot, double torque, double dt);
/* batched_step for a single lane (proj/src/env.cpp:157-175): env_step then
 * auto-reset from next.rng.  obs receives the post-reset observation,
 * final_obs the true successor. */
int eo_env_step_autoreset(const eo_env_spec* spec, eo_env_state* s, const double* action,
                          double* reward, int* terminated, int* truncated, double obs[4],
                          double final_obs[4]);

/* ------------------------------------------------------------------ net
 * proj/include/evorl/net.hpp, proj/src/net.cpp */
enum { EO_HEAD_TANH = 0, EO_HEAD_GAUSSIAN = 1, EO_HEAD_CATEGORICAL = 2, EO_HEAD_LINEAR = 3 };
#define EO_MAX_HIDDEN 8
typedef struct {
  int input_dim;
  int n_hidden;
  int hidden[EO_MAX_HIDDEN];
  int output_dim;
  int layer_norm;
  int head;
  double tanh_scale;
  double min_logstd, max_logstd;
  /* EXTENSION (not reference behaviour): allow n_hidden == 0, i.e. a linear
   * policy. The reference throws at proj/src/net.cpp:27. */
  int allow_linear;
} eo_mlp_spec;

typedef struct {
  int layer;
  int kind; /* 0 w, 1 b, 2 ln_gain, 3 ln_offset, 4 logstd */
  int64_t offset;
  int rows, cols;
} eo_segment;

/* returns number of segments written, or -1 (EO_E_INVALID_ARGUMENT set) */
int eo_param_layout(const eo_mlp_spec* spec, eo_segment* segs, int max_segs, int64_t* total);
int64_t eo_param_count(const eo_mlp_spec* spec);
int eo_init_params(const eo_mlp_spec* spec, eo_key key, double* params);
/* One row (proj/src/net.cpp:77-136).  out has output_dim entries; returns
 * EO_OK or EO_E_NET_FAULT. */
int eo_forward(const eo_mlp_spec* spec, const double* params, const double* x, double* out);
eo_mlp_spec eo_policy_net_spec(const eo_env_spec* env, const int* hidden, int n_hidden,
                               int layer_norm);

/* ------------------------------------------------------- obs normalisation
 * proj/include/evorl/obs_norm.hpp, proj/src/obs_norm.cpp */
enum { EO_NORM_NONE = 0, EO_NORM_VBN = 1, EO_NORM_RS = 2 };
typedef struct {
  double count;
  int dim; /* 0 until first add */
  double mean[4];
  double m2[4];
} eo_welford;
typedef struct {
  int mode;
  int dim;
  double mean[4], var[4];
  double count;
} eo_obs_norm;

void eo_welford_add(eo_welford* w, const double* row, int dim);
void eo_welford_merge(eo_welford* w, const eo_welford* other);
void eo_welford_variance(const eo_welford* w, double* var);
eo_obs_norm eo_obs_norm_none(void);
eo_obs_norm eo_obs_norm_running_stats(int dim);
eo_obs_norm eo_obs_norm_from_stats(int mode, const eo_welford* w);
void eo_rs_update(eo_obs_norm* s, const eo_welford* batch);
void eo_normalize(const eo_obs_norm* s, const double* obs, int dim, double* out);

/* ---------------------------------------------------------------- optim
 * proj/include/evorl/optim.hpp, proj/src/optim.cpp */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay;
} eo_adam_cfg;
eo_adam_cfg eo_adam_default(void);
void eo_adam_step(double* p, const double* grad, double* m, double* v, int64_t* t, int64_t n,
                  const eo_adam_cfg* cfg);
void eo_sgd_step(double* p, const double* grad, int64_t n, double lr);

/* ------------------------------------------------------------------- ec
 * proj/include/evorl/ec.hpp, proj/src/ec.cpp */
void eo_centered_ranks(const double* f, int64_t n, double* shaped);
void eo_rank_desc(const double* f, int64_t n, int32_t* idx);
void eo_rank_asc(const double* f, int64_t n, int32_t* idx);

typedef struct {
  int pop;
  double sigma, lr, weight_decay;
  int mirrored;
  int noise_table;
  int64_t noise_table_size;
} eo_openes_cfg;
eo_openes_cfg eo_openes_default(void);
/* mean0 copied; m, v zeroed; table built if cfg.noise_table (caller frees via eo_openes_free) */
typedef struct {
  eo_openes_cfg cfg;
  int64_t d;
  double* mean;
  double sigma;
  double* m;
  double* v;
  int64_t t;
  uint64_t table_seed;
  double* table;
} eo_openes_state;
int eo_openes_init(eo_openes_state* s, const eo_openes_cfg* cfg, const double* mean0, int64_t d,
                   eo_key key);
void eo_openes_free(eo_openes_state* s);
void eo_openes_rebuild_table(eo_openes_state* s);
/* candidates, eps: n x d row-major */
int eo_openes_ask(const eo_openes_state* s, eo_key key, int n, double* candidates, double* eps);
int eo_openes_tell(eo_openes_state* s, const double* eps, const double* fitness, int n);

typedef struct {
  int pop, elites;
  double sigma, lr;
} eo_ars_cfg;
eo_ars_cfg eo_ars_default(void);
/* deltas (n/2) x d, candidates n x d, row-major */
int eo_ars_ask(const double* mean, int64_t d, double sigma, eo_key key, int n, double* deltas,
               double* candidates);
/* returns 1 if updated, 0 if skipped (sigma_R == 0), <0 on error */
int eo_ars_tell(double* mean, int64_t d, const eo_ars_cfg* cfg, const double* deltas,
                const double* r_plus, const double* r_minus, int half);

typedef struct {
  int pop, elites;
  double sigma;
  int mirrored;
} eo_ves_cfg;
eo_ves_cfg eo_ves_default(void);
void eo_canonical_es_weights(int mu, double* w);
int eo_ves_ask(const double* mean, int64_t d, const eo_ves_cfg* cfg, eo_key key, int n,
               double* candidates);
int eo_ves_tell(double* mean, int64_t d, const eo_ves_cfg* cfg, const double* candidates,
                const double* fitness, int n);

typedef struct {
  int pop, elites;
  double sigma0;
  int max_dim;
} eo_cma_cfg;
eo_cma_cfg eo_cma_default(void);
typedef struct {
  eo_cma_cfg cfg;
  int dim;
  double* mean;
  double sigma;
  double* C; /* d x d (symmetric; row-major == col-major) */
  double* B; /* d x d, column j = eigenvector j (col-major like Eigen) */
  double* D; /* d */
  double* ps;
  double* pc;
  double* weights; /* mu */
  int mu;
  double mueff, cs, ds, cc, c1, cmu, chi_n;
  int64_t generation;
  int64_t recondition_count;
} eo_cma_state;
int eo_cma_init(eo_cma_state* s, const eo_cma_cfg* cfg, const double* mean0, int64_t d);
void eo_cma_free(eo_cma_state* s);
int eo_cma_ask(const eo_cma_state* s, eo_key key, int n, double* candidates);
int eo_cma_tell(eo_cma_state* s, const double* candidates, const double* fitness, int n);
/* Symmetric eigensolver (cyclic Jacobi, fp64). Eigen's SelfAdjointEigenSolver
 * is not available; eigenvalues ascending like Eigen; eigenvector signs are
 * normalised (largest |component| positive) and therefore differ from Eigen. */
int eo_sym_eig(const double* A, int n, double* evals, double* evecs_colmajor);

typedef struct {
  int pop, elites;
  double var_init, noise_start, noise_end;
  int64_t decay_iters;
} eo_cem_cfg;
eo_cem_cfg eo_cem_default(void);

/* -------------------------------------------------------------- rollout
 * proj/include/evorl/rollout.hpp, proj/src/rollout.cpp */
enum { EO_ACT_DETERMINISTIC = 0, EO_ACT_STOCHASTIC = 1, EO_ACT_UNIFORM = 2 };
typedef struct {
  const eo_mlp_spec* spec;
  const eo_obs_norm* obs_norm; /* may be NULL */
  int mode;
  double exploration_noise;
} eo_policy;

typedef struct {
  int64_t steps;
  int n_episodes;
  double* episode_returns; /* malloc'd, n_episodes */
  int* episode_lengths;
  eo_welford obs_stats;
  /* SampleBatch when collecting transitions (proj/include/evorl/sample_batch.hpp,
   * proj/src/rollout.cpp:118-170): rows lane-major; next_obs is the true
   * successor (final_obs) even across auto-resets; lane_bounds[e + 1] */
  int64_t n_rows;
  double* t_obs;      /* n_rows x obs_dim */
  double* t_act;      /* n_rows x act_dim */
  double* t_rew;      /* n_rows */
  uint8_t* t_term;    /* n_rows */
  uint8_t* t_trunc;   /* n_rows */
  double* t_next;     /* n_rows x obs_dim */
  int64_t* lane_bounds; /* e + 1 (batched results only) */
} eo_agent_rollout;
void eo_agent_rollout_free(eo_agent_rollout* r);

/* Episodes mode (count = total episodes per agent) or Steps mode. */
enum { EO_MODE_EPISODES = 0, EO_MODE_STEPS = 1 };
int eo_rollout_lane(const eo_env_spec* env, const eo_policy* pol, const double* params,
                    int mode, int count, int episodes_this_lane, eo_key lane_key,
                    int track_obs_stats, int collect_transitions, eo_agent_rollout* out);
/* agents: m pointers to d-vectors; out: m results.  workers: 0 = all cores. */
int eo_batched_rollout(int workers, const eo_env_spec* env, const eo_policy* pol,
                       const double* const* agents, int m, int envs_per_agent, int mode,
                       int count, eo_key key, int track_obs_stats, eo_agent_rollout* out);
/* RolloutOptions::collect_transitions = 1 */
int eo_batched_rollout_ex(int workers, const eo_env_spec* env, const eo_policy* pol,
                          const double* const* agents, int m, int envs_per_agent, int mode,
                          int count, eo_key key, int track_obs_stats, int collect_transitions,
                          eo_agent_rollout* out);
eo_obs_norm eo_vbn_fit(const eo_env_spec* env, eo_key key, int n);

/* ------------------------------------------------------- ES workflow
 * proj/src/workflow_es.cpp, proj/src/workflow.cpp, workflow_internal.hpp */
enum { EO_ALGO_OPENES = 0, EO_ALGO_ARS = 1, EO_ALGO_VES = 2, EO_ALGO_CMAES = 3, EO_ALGO_CEM = 4 };
typedef struct {
  int algo;
  int env_id;
  int fixed_horizon;
  int max_episode_steps; /* 0 = env default */
  int n_hidden;
  int hidden[EO_MAX_HIDDEN];
  int layer_norm;
  int allow_linear; /* extension flag, see eo_mlp_spec */
  int pop;
  int fitness_episodes;
  int obs_norm_mode; /* -1 = auto (proj/src/workflow.cpp:131-144) */
  int vbn_samples;
  eo_openes_cfg openes;
  eo_ars_cfg ars;
  eo_ves_cfg ves;
  eo_cma_cfg cma;
  eo_cem_cfg cem;
  int workers;
} eo_es_config;
/* Defaults of the reference config registry (proj/src/config.cpp:23-70). */
eo_es_config eo_es_default_config(void);

typedef struct eo_es eo_es;
typedef struct {
  double fitness_mean, fitness_max, fitness_min, sigma, update_skipped;
} eo_step_metrics;

int eo_es_create(const eo_es_config* cfg, eo_es** out);
void eo_es_destroy(eo_es* es);
int eo_es_init(eo_es* es, eo_key key);
int eo_es_step(eo_es* es, eo_step_metrics* m);
int64_t eo_es_dim(const eo_es* es);
int64_t eo_es_iteration(const eo_es* es);
int64_t eo_es_env_steps(const eo_es* es);
int64_t eo_es_episodes(const eo_es* es);
void eo_es_get_mean(const eo_es* es, double* out);
void eo_es_set_mean(eo_es* es, const double* mean);
/* OpenES only: adam m, v (d each) and t */
int eo_es_get_adam(const eo_es* es, double* m, double* v, int64_t* t);
void eo_es_get_obs_norm(const eo_es* es, eo_obs_norm* out);
void eo_es_set_obs_norm(eo_es* es, const eo_obs_norm* in);
/* last generation's fitness vector (pop entries) */
void eo_es_get_fitness(const eo_es* es, double* out);
const eo_mlp_spec* eo_es_net(const eo_es* es);
const eo_env_spec* eo_es_env(const eo_es* es);
/* CMA only: access to the internal state */
eo_cma_state* eo_es_cma(eo_es* es);
/* Workflow::evaluate (proj/src/workflow_es.cpp:174-179, workflow.cpp:103-129) */
int eo_es_evaluate(eo_es* es, int episodes, eo_key key, double* mean_return, double* return_std);
/* eval_key of WorkflowState (proj/include/evorl/workflow.hpp:42) */
eo_key eo_es_step_key(const eo_es* es);
eo_key eo_es_eval_key(const eo_es* es);
eo_key eo_init_key(eo_key run_key, uint64_t index);

#ifdef __cplusplus
}
#endif
#endif
