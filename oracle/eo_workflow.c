/* eo_workflow.c -- TEST INFRASTRUCTURE (parity oracle, see evorl_oracle.h).
 * Rollout grid (proj/src/rollout.cpp), the CPU ThreadPool semantics
 * (proj/src/thread_pool.cpp: dynamic index claiming, lowest failing index
 * wins) and the ES workflow generation step (proj/src/workflow_es.cpp). */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "evorl_oracle.h"

int eo_set_error(int code, const char* fmt, ...);

void eo_agent_rollout_free(eo_agent_rollout* r) {
  free(r->episode_returns);
  free(r->episode_lengths);
  free(r->t_obs);
  free(r->t_act);
  free(r->t_rew);
  free(r->t_term);
  free(r->t_trunc);
  free(r->t_next);
  free(r->lane_bounds);
  memset(r, 0, sizeof *r);
}

static void push_episode(eo_agent_rollout* out, int* cap, double ret, int len) {
  if (out->n_episodes == *cap) {
    *cap = *cap ? *cap * 2 : 4;
    out->episode_returns = (double*)realloc(out->episode_returns, sizeof(double) * (size_t)*cap);
    out->episode_lengths = (int*)realloc(out->episode_lengths, sizeof(int) * (size_t)*cap);
  }
  out->episode_returns[out->n_episodes] = ret;
  out->episode_lengths[out->n_episodes] = len;
  out->n_episodes++;
}

/* draw_action, proj/src/rollout.cpp:44-90 (Deterministic / UniformRandom;
 * Stochastic heads are outside the ES path). */
static int draw_action(const eo_env_spec* env, const eo_policy* pol, const double* params,
                       const double* net_in, eo_stream* st, double* a) {
  if (pol->mode == EO_ACT_UNIFORM) {
    if (env->discrete) {
      a[0] = (double)eo_randint(st, (uint64_t)env->num_actions);
    } else {
      for (int d = 0; d < env->act_dim; ++d) a[d] = eo_uniform_range(st, env->act_low, env->act_high);
    }
    return EO_OK;
  }
  if (pol->mode == EO_ACT_STOCHASTIC)
    return eo_set_error(EO_E_INVALID_ARGUMENT, "oracle: stochastic heads are not on the ES path");
  const eo_mlp_spec* spec = pol->spec;
  double out[8];
  const int rc = eo_forward(spec, params, net_in, out);
  if (rc != EO_OK) return rc;
  if (spec->head == EO_HEAD_CATEGORICAL) {
    int arg = 0;
    for (int i = 1; i < spec->output_dim; ++i)
      if (out[i] > out[arg]) arg = i; /* maxCoeff: first max */
    a[0] = (double)arg;
    return EO_OK;
  }
  for (int d = 0; d < env->act_dim; ++d) a[d] = out[d];
  if (!env->discrete && pol->exploration_noise > 0.0) {
    for (int d = 0; d < env->act_dim; ++d) {
      double v = a[d] + pol->exploration_noise * eo_normal(st);
      v = v < env->act_low ? env->act_low : (env->act_high < v ? env->act_high : v);
      a[d] = v;
    }
  }
  return EO_OK;
}

/* proj/src/rollout.cpp:94-174 */
/* append one transition row (growing the lane's SampleBatch arrays) */
static void push_row(eo_agent_rollout* o, int64_t* cap, const eo_env_spec* env, const double* raw,
                     const double* a, double r, int term, int trunc, const double* next) {
  if (o->n_rows == *cap) {
    *cap = *cap ? *cap * 2 : 64;
    o->t_obs = (double*)realloc(o->t_obs, sizeof(double) * (size_t)(*cap * env->obs_dim));
    o->t_act = (double*)realloc(o->t_act, sizeof(double) * (size_t)(*cap * env->act_dim));
    o->t_rew = (double*)realloc(o->t_rew, sizeof(double) * (size_t)*cap);
    o->t_term = (uint8_t*)realloc(o->t_term, (size_t)*cap);
    o->t_trunc = (uint8_t*)realloc(o->t_trunc, (size_t)*cap);
    o->t_next = (double*)realloc(o->t_next, sizeof(double) * (size_t)(*cap * env->obs_dim));
  }
  const int64_t i = o->n_rows++;
  memcpy(o->t_obs + i * env->obs_dim, raw, sizeof(double) * (size_t)env->obs_dim);
  memcpy(o->t_act + i * env->act_dim, a, sizeof(double) * (size_t)env->act_dim);
  o->t_rew[i] = r;
  o->t_term[i] = (uint8_t)(term ? 1 : 0);
  o->t_trunc[i] = (uint8_t)(trunc ? 1 : 0);
  memcpy(o->t_next + i * env->obs_dim, next, sizeof(double) * (size_t)env->obs_dim);
}

int eo_rollout_lane(const eo_env_spec* env, const eo_policy* pol, const double* params, int mode,
                    int count, int episodes_this_lane, eo_key lane_key, int track_obs_stats,
                    int collect_transitions, eo_agent_rollout* out) {
  int64_t rcap = 0;
  memset(out, 0, sizeof *out);
  const int by_episodes = mode == EO_MODE_EPISODES;
  if (by_episodes && episodes_this_lane <= 0) return EO_OK;
  eo_env_state state;
  double obs[4];
  eo_env_reset(env, eo_fold_in(lane_key, 0), &state, obs);
  eo_stream st;
  eo_stream_init(&st, eo_fold_in(lane_key, 1));
  double ep_return = 0.0;
  int ep_len = 0, eps_done = 0, cap = 0;
  while (by_episodes ? eps_done < episodes_this_lane : out->steps < count) {
    double raw[4], net_in[4], a[4];
    memcpy(raw, obs, sizeof raw);
    if (track_obs_stats) eo_welford_add(&out->obs_stats, raw, env->obs_dim);
    eo_normalize(pol->obs_norm, raw, env->obs_dim, net_in);
    int rc = draw_action(env, pol, params, net_in, &st, a);
    if (rc != EO_OK) return rc;
    double reward;
    int term, trunc;
    double final_obs[4];
    rc = eo_env_step_autoreset(env, &state, a, &reward, &term, &trunc, obs, final_obs);
    if (rc != EO_OK) return rc;
    if (collect_transitions) push_row(out, &rcap, env, raw, a, reward, term, trunc, final_obs);
    ep_return += reward;
    ep_len += 1;
    out->steps += 1;
    if (term || trunc) {
      push_episode(out, &cap, ep_return, ep_len);
      ep_return = 0.0;
      ep_len = 0;
      eps_done += 1;
    }
  }
  return EO_OK;
}

/* ---------------------------------------------------------- thread pool
 * proj/src/thread_pool.cpp:24-81: workers claim indices dynamically; per
 * index result slots; the lowest failing index's error wins. */
typedef struct {
  const eo_env_spec* env;
  const eo_policy* pol;
  const double* const* agents;
  int e, mode, count, track, collect;
  eo_key key;
  eo_agent_rollout* lanes;
  int* rcs;
  char (*msgs)[512];
  size_t n;
  atomic_size_t next;
} lane_job;

static void run_lane(lane_job* J, size_t li) {
  const size_t a = li / (size_t)J->e, j = li % (size_t)J->e;
  const eo_key lane_key = eo_fold_in(eo_fold_in(J->key, a), j);
  int eps_this = 0;
  if (J->mode == EO_MODE_EPISODES)
    eps_this = J->count / J->e + ((int)j < J->count % J->e ? 1 : 0);
  J->rcs[li] = eo_rollout_lane(J->env, J->pol, J->agents[a], J->mode, J->count, eps_this, lane_key,
                               J->track, J->collect, &J->lanes[li]);
  if (J->rcs[li] != EO_OK) strncpy(J->msgs[li], eo_last_error(), 511);
}

static void* worker(void* arg) {
  lane_job* J = (lane_job*)arg;
  for (;;) {
    const size_t i = atomic_fetch_add(&J->next, 1);
    if (i >= J->n) break;
    run_lane(J, i);
  }
  return NULL;
}

static int resolve_workers(int workers) {
  if (workers <= 0) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    workers = n > 0 ? (int)n : 1;
  }
  return workers;
}

/* proj/src/rollout.cpp:176-214 */
int eo_batched_rollout(int workers, const eo_env_spec* env, const eo_policy* pol,
                       const double* const* agents, int m, int e, int mode, int count, eo_key key,
                       int track_obs_stats, eo_agent_rollout* out) {
  return eo_batched_rollout_ex(workers, env, pol, agents, m, e, mode, count, key, track_obs_stats, 0, out);
}

int eo_batched_rollout_ex(int workers, const eo_env_spec* env, const eo_policy* pol,
                          const double* const* agents, int m, int e, int mode, int count, eo_key key,
                          int track_obs_stats, int collect_transitions, eo_agent_rollout* out) {
  const size_t n = (size_t)m * (size_t)e;
  lane_job J;
  memset(&J, 0, sizeof J);
  J.env = env;
  J.pol = pol;
  J.agents = agents;
  J.e = e;
  J.mode = mode;
  J.count = count;
  J.track = track_obs_stats;
  J.collect = collect_transitions;
  J.key = key;
  J.n = n;
  J.lanes = (eo_agent_rollout*)calloc(n ? n : 1, sizeof(eo_agent_rollout));
  J.rcs = (int*)calloc(n ? n : 1, sizeof(int));
  J.msgs = (char(*)[512])calloc(n ? n : 1, 512);
  atomic_init(&J.next, 0);
  workers = resolve_workers(workers);
  if (workers == 1 || n <= 1) {
    for (size_t i = 0; i < n; ++i) run_lane(&J, i);
  } else {
    const int nt = (size_t)workers < n ? workers : (int)n;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
    for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, worker, &J);
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  int rc = EO_OK;
  for (size_t i = 0; i < n; ++i)
    if (J.rcs[i] != EO_OK) {
      rc = eo_set_error(J.rcs[i], "%s", J.msgs[i]);
      break;
    }
  if (rc == EO_OK) {
    for (int a = 0; a < m; ++a) {
      eo_agent_rollout* agg = &out[a];
      memset(agg, 0, sizeof *agg);
      int cap = 0;
      for (int j = 0; j < e; ++j) {
        eo_agent_rollout* lane = &J.lanes[(size_t)a * e + j];
        for (int k = 0; k < lane->n_episodes; ++k)
          push_episode(agg, &cap, lane->episode_returns[k], lane->episode_lengths[k]);
        agg->steps += lane->steps;
        eo_welford_merge(&agg->obs_stats, &lane->obs_stats);
      }
      if (collect_transitions) {  /* lane-major concatenation + lane bounds */
        int64_t rows = 0;
        agg->lane_bounds = (int64_t*)calloc((size_t)e + 1, sizeof(int64_t));
        for (int j = 0; j < e; ++j) {
          agg->lane_bounds[j] = rows;
          rows += J.lanes[(size_t)a * e + j].n_rows;
        }
        agg->lane_bounds[e] = rows;
        int64_t cap = 0;
        for (int j = 0; j < e; ++j) {
          const eo_agent_rollout* L = &J.lanes[(size_t)a * e + j];
          for (int64_t i = 0; i < L->n_rows; ++i)
            push_row(agg, &cap, env, L->t_obs + i * env->obs_dim, L->t_act + i * env->act_dim, L->t_rew[i],
                     L->t_term[i], L->t_trunc[i], L->t_next + i * env->obs_dim);
        }
      }
    }
  }
  for (size_t i = 0; i < n; ++i) eo_agent_rollout_free(&J.lanes[i]);
  free(J.lanes);
  free(J.rcs);
  free(J.msgs);
  return rc;
}

/* proj/src/rollout.cpp:216-224 */
eo_obs_norm eo_vbn_fit(const eo_env_spec* env, eo_key key, int n) {
  eo_policy pol;
  memset(&pol, 0, sizeof pol);
  pol.mode = EO_ACT_UNIFORM;
  eo_agent_rollout r;
  eo_rollout_lane(env, &pol, NULL, EO_MODE_STEPS, n, 0, key, 1, 0, &r);
  eo_obs_norm s = eo_obs_norm_from_stats(EO_NORM_VBN, &r.obs_stats);
  eo_agent_rollout_free(&r);
  return s;
}

/* ======================================================== ES workflow */

/* proj/src/workflow_internal.hpp:35-37 */
eo_key eo_init_key(eo_key run_key, uint64_t index) { return eo_fold_in(eo_fold_in(run_key, 2), index); }

/* registry defaults, proj/src/config.cpp:23-70 */
eo_es_config eo_es_default_config(void) {
  eo_es_config c;
  memset(&c, 0, sizeof c);
  c.algo = EO_ALGO_OPENES;
  c.env_id = EO_CARTPOLE;
  c.fixed_horizon = 0;
  c.max_episode_steps = 0;
  c.n_hidden = 2;
  c.hidden[0] = 64;
  c.hidden[1] = 64;
  c.layer_norm = 0;
  c.allow_linear = 0;
  c.pop = 128;
  c.fitness_episodes = 1;
  c.obs_norm_mode = -1;
  c.vbn_samples = 10000;
  c.openes = eo_openes_default();
  c.ars = eo_ars_default();
  c.ves = eo_ves_default();
  c.cma = eo_cma_default();
  c.cem = eo_cem_default();
  c.workers = 0;
  return c;
}

struct eo_es {
  eo_es_config cfg;
  eo_env_spec env;
  eo_mlp_spec net;
  int norm_mode;
  int64_t d;
  /* WorkflowState, proj/include/evorl/workflow.hpp:31-46 */
  int64_t iteration;
  eo_key rng;
  int64_t env_steps, episodes;
  /* EsState, proj/src/workflow_es.cpp:15-20 */
  eo_openes_state openes;
  double* mean; /* ars / ves / cem mean (openes/cma keep their own) */
  double* cem_var;
  int64_t cem_iter;
  eo_cma_state cma;
  eo_obs_norm obs_norm;
  double* fitness;
};

/* proj/src/workflow.cpp:131-144 */
static int resolve_norm(const eo_es_config* c) {
  if (c->obs_norm_mode >= 0) return c->obs_norm_mode;
  if (c->algo == EO_ALGO_ARS) return EO_NORM_RS;
  if (c->algo == EO_ALGO_CEM) return EO_NORM_NONE;
  return EO_NORM_VBN;
}

/* EsWorkflow ctor, proj/src/workflow_es.cpp:28-64 */
int eo_es_create(const eo_es_config* cfg, eo_es** out) {
  eo_es* es = (eo_es*)calloc(1, sizeof(eo_es));
  es->cfg = *cfg;
  /* the ctor builds every algorithm config with pop_ = ec.pop
   * (proj/src/workflow_es.cpp:33-61); CMA's weights depend on it */
  es->cfg.openes.pop = cfg->pop;
  es->cfg.ars.pop = cfg->pop;
  es->cfg.ves.pop = cfg->pop;
  es->cfg.cma.pop = cfg->pop;
  es->cfg.cem.pop = cfg->pop;
  es->env = cfg->env_id == EO_CARTPOLE ? eo_env_cartpole(cfg->fixed_horizon, cfg->max_episode_steps)
                                       : eo_env_pendulum(cfg->fixed_horizon, cfg->max_episode_steps);
  es->net = eo_policy_net_spec(&es->env, cfg->hidden, cfg->n_hidden, cfg->layer_norm);
  es->net.allow_linear = cfg->allow_linear;
  es->norm_mode = resolve_norm(cfg);
  es->d = eo_param_count(&es->net);
  if (es->d < 0) {
    free(es);
    return EO_E_INVALID_ARGUMENT;
  }
  if (cfg->algo < 0 || cfg->algo > EO_ALGO_CEM) {
    free(es);
    return eo_set_error(EO_E_CONFIG, "ec.algo: unknown algorithm");
  }
  es->fitness = (double*)calloc((size_t)cfg->pop, sizeof(double));
  *out = es;
  return EO_OK;
}

void eo_es_destroy(eo_es* es) {
  if (!es) return;
  eo_openes_free(&es->openes);
  eo_cma_free(&es->cma);
  free(es->mean);
  free(es->cem_var);
  free(es->fitness);
  free(es);
}

/* proj/src/workflow_es.cpp:68-85 */
int eo_es_init(eo_es* es, eo_key key) {
  es->rng = key;
  es->iteration = 0;
  es->env_steps = 0;
  es->episodes = 0;
  const int64_t d = es->d;
  double* mean0 = (double*)malloc(sizeof(double) * (size_t)d);
  int rc = eo_init_params(&es->net, eo_init_key(key, 1), mean0);
  if (rc != EO_OK) {
    free(mean0);
    return rc;
  }
  switch (es->cfg.algo) {
    case EO_ALGO_OPENES:
      rc = eo_openes_init(&es->openes, &es->cfg.openes, mean0, d, eo_init_key(key, 2));
      break;
    case EO_ALGO_CMAES:
      rc = eo_cma_init(&es->cma, &es->cfg.cma, mean0, d);
      break;
    case EO_ALGO_CEM:
      es->mean = (double*)malloc(sizeof(double) * (size_t)d);
      memcpy(es->mean, mean0, sizeof(double) * (size_t)d);
      es->cem_var = (double*)malloc(sizeof(double) * (size_t)d);
      for (int64_t p = 0; p < d; ++p) es->cem_var[p] = es->cfg.cem.var_init;
      es->cem_iter = 0;
      break;
    default:
      es->mean = (double*)malloc(sizeof(double) * (size_t)d);
      memcpy(es->mean, mean0, sizeof(double) * (size_t)d);
  }
  free(mean0);
  if (rc != EO_OK) return rc;
  if (es->norm_mode == EO_NORM_VBN)
    es->obs_norm = eo_vbn_fit(&es->env, eo_init_key(key, 0), es->cfg.vbn_samples);
  else if (es->norm_mode == EO_NORM_RS)
    es->obs_norm = eo_obs_norm_running_stats(es->env.obs_dim);
  else
    es->obs_norm = eo_obs_norm_none();
  return EO_OK;
}

eo_key eo_es_step_key(const eo_es* es) {
  return eo_fold_in(eo_fold_in(es->rng, 0), (uint64_t)es->iteration);
}
eo_key eo_es_eval_key(const eo_es* es) {
  return eo_fold_in(eo_fold_in(es->rng, 1), (uint64_t)es->iteration);
}

static double* center_ptr(eo_es* es) {
  if (es->cfg.algo == EO_ALGO_OPENES) return es->openes.mean;
  if (es->cfg.algo == EO_ALGO_CMAES) return es->cma.mean;
  return es->mean;
}

static double cem_noise_floor(const eo_es* es) {
  const eo_cem_cfg* c = &es->cfg.cem;
  double frac = c->decay_iters > 0 ? (double)es->cem_iter / (double)c->decay_iters : 1.0;
  if (frac > 1.0) frac = 1.0;
  return c->noise_start * pow(c->noise_end / c->noise_start, frac);
}

/* EsWorkflow::step, proj/src/workflow_es.cpp:87-172 */
int eo_es_step(eo_es* es, eo_step_metrics* met) {
  const eo_key k = eo_es_step_key(es);
  const int n = es->cfg.pop;
  const int64_t d = es->d;
  int rc = EO_OK;
  double* cand = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
  double* eps = NULL;
  double* deltas = NULL;
  const eo_key ask_key = eo_fold_in(k, 0);
  switch (es->cfg.algo) {
    case EO_ALGO_OPENES:
      eps = (double*)malloc(sizeof(double) * (size_t)n * (size_t)d);
      rc = eo_openes_ask(&es->openes, ask_key, n, cand, eps);
      break;
    case EO_ALGO_ARS:
      deltas = (double*)malloc(sizeof(double) * (size_t)(n / 2 > 0 ? n / 2 : 1) * (size_t)d);
      rc = eo_ars_ask(es->mean, d, es->cfg.ars.sigma, ask_key, n, deltas, cand);
      break;
    case EO_ALGO_VES:
      rc = eo_ves_ask(es->mean, d, &es->cfg.ves, ask_key, n, cand);
      break;
    case EO_ALGO_CMAES:
      rc = eo_cma_ask(&es->cma, ask_key, n, cand);
      break;
    case EO_ALGO_CEM: { /* proj/src/ec.cpp:306-313 */
      eo_gaussian_matrix(ask_key, n, d, cand);
      for (int i = 0; i < n; ++i)
        for (int64_t p = 0; p < d; ++p)
          cand[(int64_t)i * d + p] = cand[(int64_t)i * d + p] * sqrt(es->cem_var[p]) + es->mean[p];
      break;
    }
  }
  if (rc != EO_OK) goto done;
  {
    const double** agents = (const double**)malloc(sizeof(double*) * (size_t)n);
    for (int i = 0; i < n; ++i) agents[i] = cand + (int64_t)i * d;
    eo_policy pol;
    memset(&pol, 0, sizeof pol);
    pol.spec = &es->net;
    pol.obs_norm = &es->obs_norm;
    pol.mode = EO_ACT_DETERMINISTIC;
    const int track = es->norm_mode == EO_NORM_RS;
    eo_agent_rollout* ro = (eo_agent_rollout*)calloc((size_t)n, sizeof(eo_agent_rollout));
    const int e = es->cfg.fitness_episodes;
    rc = eo_batched_rollout(es->cfg.workers, &es->env, &pol, agents, n, e, EO_MODE_EPISODES, e,
                            eo_fold_in(k, 1), track, ro);
    free(agents);
    if (rc != EO_OK) {
      free(ro);
      goto done;
    }
    /* proj/src/workflow_es.cpp:127-138 */
    eo_welford stats;
    memset(&stats, 0, sizeof stats);
    for (int i = 0; i < n; ++i) {
      double sum = 0.0;
      for (int q = 0; q < ro[i].n_episodes; ++q) sum += ro[i].episode_returns[q];
      es->fitness[i] = sum / (double)ro[i].n_episodes;
      es->env_steps += ro[i].steps;
      es->episodes += ro[i].n_episodes;
      if (track) eo_welford_merge(&stats, &ro[i].obs_stats);
      eo_agent_rollout_free(&ro[i]);
    }
    free(ro);
    if (track) eo_rs_update(&es->obs_norm, &stats);
  }
  {
    int skipped = 0;
    double sigma = 0.0;
    switch (es->cfg.algo) {
      case EO_ALGO_OPENES:
        rc = eo_openes_tell(&es->openes, eps, es->fitness, n);
        sigma = es->openes.sigma;
        break;
      case EO_ALGO_ARS: {
        const int half = n / 2;
        double* rp = (double*)malloc(sizeof(double) * (size_t)half);
        double* rm = (double*)malloc(sizeof(double) * (size_t)half);
        for (int i = 0; i < half; ++i) {
          rp[i] = es->fitness[2 * i];
          rm[i] = es->fitness[2 * i + 1];
        }
        const int r = eo_ars_tell(es->mean, d, &es->cfg.ars, deltas, rp, rm, half);
        skipped = r == 0;
        free(rp);
        free(rm);
        sigma = es->cfg.ars.sigma;
        break;
      }
      case EO_ALGO_VES:
        rc = eo_ves_tell(es->mean, d, &es->cfg.ves, cand, es->fitness, n);
        sigma = es->cfg.ves.sigma;
        break;
      case EO_ALGO_CMAES:
        rc = eo_cma_tell(&es->cma, cand, es->fitness, n);
        sigma = es->cma.sigma;
        break;
      case EO_ALGO_CEM: { /* proj/src/ec.cpp:315-336 */
        const int h = es->cfg.cem.elites < n ? es->cfg.cem.elites : n;
        int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
        eo_rank_desc(es->fitness, n, order);
        double* mean = (double*)calloc((size_t)d, sizeof(double));
        for (int i = 0; i < h; ++i)
          for (int64_t p = 0; p < d; ++p) mean[p] += cand[(int64_t)order[i] * d + p];
        for (int64_t p = 0; p < d; ++p) mean[p] /= h;
        const double floor_ = cem_noise_floor(es);
        for (int64_t p = 0; p < d; ++p) {
          double var = 0.0;
          for (int i = 0; i < h; ++i) {
            const double x = cand[(int64_t)order[i] * d + p] - mean[p];
            var += x * x;
          }
          var /= h;
          es->cem_var[p] = var + floor_;
        }
        memcpy(es->mean, mean, sizeof(double) * (size_t)d);
        es->cem_iter += 1;
        free(mean);
        free(order);
        double s = 0.0;
        for (int64_t p = 0; p < d; ++p) s += es->cem_var[p];
        sigma = sqrt(s / (double)d);
        break;
      }
    }
    if (rc != EO_OK) goto done;
    double s = 0.0, mx = es->fitness[0], mn = es->fitness[0];
    for (int i = 0; i < n; ++i) {
      s += es->fitness[i];
      if (es->fitness[i] > mx) mx = es->fitness[i];
      if (es->fitness[i] < mn) mn = es->fitness[i];
    }
    if (met) {
      met->fitness_mean = s / n;
      met->fitness_max = mx;
      met->fitness_min = mn;
      met->sigma = sigma;
      met->update_skipped = skipped ? 1.0 : 0.0;
    }
    es->iteration += 1;
  }
done:
  free(cand);
  free(eps);
  free(deltas);
  return rc;
}

int64_t eo_es_dim(const eo_es* es) { return es->d; }
int64_t eo_es_iteration(const eo_es* es) { return es->iteration; }
int64_t eo_es_env_steps(const eo_es* es) { return es->env_steps; }
int64_t eo_es_episodes(const eo_es* es) { return es->episodes; }
void eo_es_get_mean(const eo_es* es, double* out) {
  memcpy(out, center_ptr((eo_es*)es), sizeof(double) * (size_t)es->d);
}
void eo_es_set_mean(eo_es* es, const double* mean) {
  memcpy(center_ptr(es), mean, sizeof(double) * (size_t)es->d);
}
int eo_es_get_adam(const eo_es* es, double* m, double* v, int64_t* t) {
  if (es->cfg.algo != EO_ALGO_OPENES) return EO_E_INVALID_ARGUMENT;
  memcpy(m, es->openes.m, sizeof(double) * (size_t)es->d);
  memcpy(v, es->openes.v, sizeof(double) * (size_t)es->d);
  *t = es->openes.t;
  return EO_OK;
}
void eo_es_get_obs_norm(const eo_es* es, eo_obs_norm* out) { *out = es->obs_norm; }
void eo_es_set_obs_norm(eo_es* es, const eo_obs_norm* in) { es->obs_norm = *in; }
void eo_es_get_fitness(const eo_es* es, double* out) {
  memcpy(out, es->fitness, sizeof(double) * (size_t)es->cfg.pop);
}
const eo_mlp_spec* eo_es_net(const eo_es* es) { return &es->net; }
const eo_env_spec* eo_es_env(const eo_es* es) { return &es->env; }
eo_cma_state* eo_es_cma(eo_es* es) { return &es->cma; }

/* proj/src/workflow_es.cpp:174-179 -> proj/src/workflow.cpp:103-129 */
int eo_es_evaluate(eo_es* es, int episodes, eo_key key, double* mean_return, double* return_std) {
  const double* center = center_ptr(es);
  eo_policy pol;
  memset(&pol, 0, sizeof pol);
  pol.spec = &es->net;
  pol.obs_norm = &es->obs_norm;
  pol.mode = EO_ACT_DETERMINISTIC;
  eo_agent_rollout r;
  const double* agents[1] = {center};
  int rc = eo_batched_rollout(es->cfg.workers, &es->env, &pol, agents, 1, episodes,
                              EO_MODE_EPISODES, episodes, key, 0, &r);
  if (rc != EO_OK) return rc;
  double sum = 0.0, sq = 0.0;
  for (int q = 0; q < r.n_episodes; ++q) {
    sum += r.episode_returns[q];
    sq += r.episode_returns[q] * r.episode_returns[q];
  }
  const double nn = (double)r.n_episodes;
  *mean_return = sum / nn;
  const double var = sq / nn - (*mean_return) * (*mean_return);
  *return_std = sqrt(var > 0.0 ? var : 0.0);
  eo_agent_rollout_free(&r);
  return EO_OK;
}
