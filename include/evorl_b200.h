/*
 * evorl_b200.h -- C ABI of the B200-native EvoRL ES generation path.
 *
 * This is the drop-in boundary.  The reference (a C++20 static library,
 * /root/reference/proj) has no FFI; its seam is the C++ API listed in
 * SURVEY.md §8(b).  Each entry point below names the reference interface it
 * replaces (path:line relative to /root/reference).  INTEGRATION.md shows the
 * reference-side binding a maintainer adds.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or CUDA types cross the ABI.
 *  - Every function returns an int status: EVORL_OK (0) or one of the codes
 *    below, which map 1:1 to the reference's exception types.  No exception
 *    crosses the ABI.  evorl_last_error() returns the message of the last
 *    failure on the calling thread (the reference's what() text, e.g.
 *    "openes_ask: mirrored sampling needs an even population").
 *  - "Host" arrays are caller-owned host memory, copied in/out during the call
 *    and never retained.  Matrices are row-major (row i = candidate i), the
 *    transpose-free view of the reference's Eigen row access.
 *  - Calls are synchronous with respect to their outputs (like the reference).
 *  - One host thread per handle (the reference's Workflow::step is called from
 *    one orchestrating thread, proj/include/evorl/thread_pool.hpp:27-29).
 *  - Precision: EVORL_PREC_F64 evaluates the policy in fp64 (parity mode, same
 *    arithmetic type as the reference); EVORL_PREC_F32 evaluates the policy
 *    GEMMs in fp32 (env dynamics, returns, noise and the EC update stay fp64);
 *    EVORL_PREC_TC runs the dense hidden layer of obs -> W1 -> W2 -> O policies
 *    (W2 a multiple of 128, W1 <= 256) on the tcgen05 tensor cores as a
 *    3-pass fp16 hi/lo split with fp32 accumulation in TMEM (fp32-level
 *    accuracy) and the other layers in fp32; other shapes run as EVORL_PREC_F32.
 *    EVORL_PREC_OZ keeps fp64-level accuracy on the tensor cores: the dense
 *    hidden layer of obs -> W1 -> W2 -> O policies (W1 <= 256) runs as exact
 *    int8 tcgen05 MMAs over 6 byte slices of per-row / per-lane fixed-point
 *    operands (Ozaki scheme, ~47 bits per operand, int32 accumulation), every
 *    other layer, the head and the env in fp64; other shapes run as F64.
 */
#ifndef EVORL_B200_H
#define EVORL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVORL_B200_ABI_VERSION 1

/* status codes (proj/src/runner.cpp:39-82 maps exceptions to exit codes) */
enum {
  EVORL_OK = 0,
  EVORL_E_INVALID_ARGUMENT = 1, /* std::invalid_argument (proj/src/ec.cpp:72-74 ...) */
  EVORL_E_LENGTH = 2,           /* std::length_error (proj/src/ec.cpp:193-196) */
  EVORL_E_ENV_FAULT = 3,        /* evorl::EnvFault (proj/include/evorl/env.hpp:19-21) */
  EVORL_E_NET_FAULT = 4,        /* evorl::NetFault (proj/include/evorl/net.hpp:19-21) */
  EVORL_E_CONFIG = 5,           /* evorl::ConfigError (proj/include/evorl/config.hpp:11-13) */
  EVORL_E_CUDA = 6,             /* device / driver failure */
  EVORL_E_UNSUPPORTED = 7,      /* valid reference input the device path refuses */
  EVORL_E_CHECKPOINT = 8        /* evorl::CheckpointError (proj/include/evorl/checkpoint.hpp:14-16) */
};

enum { EVORL_PREC_F64 = 0, EVORL_PREC_F32 = 1, EVORL_PREC_TC = 2, EVORL_PREC_OZ = 3 };
enum { EVORL_ENV_CARTPOLE = 0, EVORL_ENV_PENDULUM = 1 };
enum { EVORL_ALGO_OPENES = 0, EVORL_ALGO_ARS = 1, EVORL_ALGO_VES = 2, EVORL_ALGO_CMAES = 3,
       EVORL_ALGO_CEM = 4 };
enum { EVORL_NORM_AUTO = -1, EVORL_NORM_NONE = 0, EVORL_NORM_VBN = 1, EVORL_NORM_RS = 2 };
enum { EVORL_HEAD_TANH = 0, EVORL_HEAD_GAUSSIAN = 1, EVORL_HEAD_CATEGORICAL = 2,
       EVORL_HEAD_LINEAR = 3 };
#define EVORL_MAX_HIDDEN 8

const char* evorl_last_error(void);
int evorl_abi_version(void);
/* Number of CUDA kernels this library launched since load (for accounting). */
int64_t evorl_kernel_launches(void);

/* ---------------------------------------------------------------- RNG
 * replaces threefry2x64 / key_from_seed / fold_in (proj/src/rng.cpp:18-46)
 * and RandomStream draws (proj/src/rng.cpp:54-87), counter-addressed. */
int evorl_threefry2x64(const uint64_t* keys /* 2n */, const uint64_t* ctrs /* 2n */,
                       uint64_t* out /* 2n */, int64_t n);
/* words [first, first+n) of RandomStream(key) */
int evorl_stream_words(uint64_t key_hi, uint64_t key_lo, int64_t first, int64_t n,
                       uint64_t* out);
/* replaces gaussian_matrix (proj/src/ec.cpp:22-28): rows x cols row-major */
int evorl_gaussian_matrix(uint64_t key_hi, uint64_t key_lo, int64_t rows, int64_t cols,
                          double* out);

/* --------------------------------------------------------- ranks
 * replaces centered_ranks (proj/src/ec.cpp:32-46) and rank_desc (:14-20):
 * stable (ties -> lower index). */
int evorl_centered_ranks(const double* fitness, int64_t n, double* shaped);
int evorl_rank_desc(const double* fitness, int64_t n, int32_t* order);

/* ---------------------------------------------------- env / policy units
 * replaces env_step (proj/src/env.cpp:113-155) for n independent states.
 * phys: n x 4, step_count: n; outputs written in place plus reward/flags.
 * fault: per-state 0 or EVORL_E_ENV_FAULT (no exception for batch use). */
int evorl_env_step_batch(int env_id, int fixed_horizon, int max_episode_steps, int64_t n,
                         double* phys, int32_t* step_count, const double* action,
                         double* reward, int32_t* terminated, int32_t* truncated,
                         int32_t* fault);

/* MLP description = policy_net_spec (proj/src/workflow.cpp:87-101). */
typedef struct {
  int32_t input_dim;
  int32_t n_hidden;
  int32_t hidden[EVORL_MAX_HIDDEN];
  int32_t output_dim;
  int32_t layer_norm;   /* must be 0 on the device path */
  int32_t head;         /* EVORL_HEAD_* */
  double tanh_scale;
  int32_t allow_linear; /* EXTENSION: n_hidden == 0 (reference throws, proj/src/net.cpp:27) */
} evorl_mlp_desc;

typedef struct {
  int32_t env_id;
  int32_t fixed_horizon;
  int32_t max_episode_steps; /* 0 = env default */
} evorl_env_desc;

/* Observation normaliser (ObsNormState, proj/include/evorl/obs_norm.hpp:22-30) */
typedef struct {
  int32_t mode; /* EVORL_NORM_* (NONE/VBN/RS) */
  int32_t dim;
  double mean[4];
  double var[4];
  double count;
} evorl_obs_norm;

/* replaces batched_rollout (proj/src/rollout.cpp:176-214) for deterministic
 * policies in Episodes mode: m agents (params m x d row-major), e lanes per
 * agent, `count` episodes per agent spread over the lanes, lane (a, j) keyed
 * fold_in(fold_in(key, a), j).  Outputs: returns m x count (lane-major episode
 * order, as AgentRollout::episode_returns), steps per agent, and (if
 * obs_stats != NULL) per-agent Welford stats (m x 9: count, mean[4], m2[4]). */
int evorl_batched_rollout(const evorl_env_desc* env, const evorl_mlp_desc* net,
                          const evorl_obs_norm* norm, const double* params, int32_t m,
                          int32_t e, int32_t count, uint64_t key_hi, uint64_t key_lo,
                          int32_t precision, double* returns, int64_t* steps,
                          double* obs_stats);

/* batched_rollout with RolloutOptions::collect_transitions -- the ERL / CEM-RL
 * population evaluation (proj/src/workflow_erl.cpp:104-110,
 * proj/src/workflow_cemrl.cpp:176-182; SampleBatch rows of
 * proj/src/rollout.cpp:132-170).  As evorl_batched_rollout, plus every lane's
 * transitions in padded per-lane buffers: lane l = a * e + j owns rows
 * [l * row_cap, l * row_cap + lane_rows[l]) (lane-major concatenation per agent
 * gives the reference's AgentRollout::batch, lane_bounds = prefix sums of
 * lane_rows).  row_cap >= ceil(count / e) * max_episode_steps.  t_obs / t_next:
 * rows x obs_dim (t_next = the successor observation before any auto-reset),
 * t_act: rows x 1, t_term / t_trunc: 0/1 bytes.  Evaluated by the cluster
 * team (precision tc evaluates as f32). */
int evorl_batched_rollout_transitions(const evorl_env_desc* env, const evorl_mlp_desc* net,
                                      const evorl_obs_norm* norm, const double* params, int32_t m,
                                      int32_t e, int32_t count, uint64_t key_hi, uint64_t key_lo,
                                      int32_t precision, double* returns, int64_t* steps,
                                      int64_t row_cap, double* t_obs, double* t_act,
                                      double* t_rew, uint8_t* t_term, uint8_t* t_trunc,
                                      double* t_next, int64_t* lane_rows);

/* -------------------------------------------------------- EC updates
 * replaces openes_tell (proj/src/ec.cpp:99-109) + adam_step
 * (proj/src/optim.cpp:7-17).  The perturbations are NOT passed: they are
 * regenerated from the ask key exactly as openes_ask drew them
 * (proj/src/ec.cpp:79-90), which is the point of the B200 design.  mean, m, v
 * (d each) and *t are updated in place. */
int evorl_openes_tell(double* mean, double* m, double* v, int64_t* t, int64_t d,
                      double sigma, double lr, double weight_decay, int32_t mirrored,
                      uint64_t ask_hi, uint64_t ask_lo, const double* fitness, int32_t n);
/* replaces openes_ask (proj/src/ec.cpp:71-97), materialising the sample
 * (candidates / eps may be NULL). */
int evorl_openes_ask(const double* mean, int64_t d, double sigma, int32_t mirrored,
                     uint64_t ask_hi, uint64_t ask_lo, int32_t n, double* candidates,
                     double* eps);
/* replaces ars_ask / ars_tell (proj/src/ec.cpp:113-154); returns 1 in
 * *updated, or 0 when sigma_R == 0 (update skipped). */
int evorl_ars_ask(const double* mean, int64_t d, double sigma, uint64_t ask_hi,
                  uint64_t ask_lo, int32_t n, double* deltas, double* candidates);
int evorl_ars_tell(double* mean, int64_t d, int32_t elites, double lr, uint64_t ask_hi,
                   uint64_t ask_lo, const double* fitness /* n, interleaved +/- */, int32_t n,
                   int32_t* updated);

/* ------------------------------------------ the generation (Workflow seam)
 * Device-resident EsWorkflow: replaces EsWorkflow (proj/src/workflow_es.cpp)
 * init (:68-85), step (:87-172) and evaluate (:174-179) behind
 * Workflow (proj/include/evorl/workflow.hpp:48-70).  Config fields use the
 * reference config-registry keys and defaults (proj/src/config.cpp:23-70). */
typedef struct {
  int32_t algo;              /* ec.algo */
  int32_t env_id;            /* env.id */
  int32_t fixed_horizon;     /* env.fixed_horizon */
  int32_t max_episode_steps; /* env.max_episode_steps (0 = env default) */
  int32_t n_hidden;          /* net.hidden */
  int32_t hidden[EVORL_MAX_HIDDEN];
  int32_t layer_norm;        /* net.layer_norm (device path: must be 0) */
  int32_t allow_linear;      /* EXTENSION: linear policy, see evorl_mlp_desc */
  int32_t pop;               /* ec.pop */
  int32_t fitness_episodes;  /* ec.fitness_episodes */
  int32_t obs_norm_mode;     /* obs_norm.mode (EVORL_NORM_AUTO = "auto") */
  int32_t vbn_samples;       /* obs_norm.vbn_samples */
  double openes_sigma, openes_lr, openes_weight_decay;
  int32_t openes_mirrored, openes_noise_table;
  int64_t openes_noise_table_size;
  double ars_sigma, ars_lr;
  int32_t ars_elites;
  double ves_sigma;
  int32_t ves_elites, ves_mirrored;
  double cmaes_sigma0;
  int32_t cmaes_elites, cmaes_max_dim;
  int32_t cem_elites;
  double cem_var_init, cem_noise_start, cem_noise_end;
  int64_t cem_decay_iters;
  int32_t precision; /* EVORL_PREC_* (not a reference key) */
  int32_t device;    /* CUDA ordinal (not a reference key) */
  /* EXTENSION (BASELINE config 4): re-factorise C every k-th generation
   * (lazy CMA-ES).  k = 1 (default) is the reference behaviour
   * (proj/src/ec.cpp:276-287); B and D stay fixed in between; k = 0 picks
   * the standard lazy gap max(1, floor(1 / (10 d (c1 + cmu)))). */
  int32_t cmaes_eig_every;
} evorl_es_config;

/* StepMetrics of EsWorkflow::step (proj/src/workflow_es.cpp:140-169) */
typedef struct {
  double fitness_mean, fitness_max, fitness_min, sigma, update_skipped;
} evorl_step_metrics;

typedef struct evorl_es evorl_es;

void evorl_es_default_config(evorl_es_config* cfg);
int evorl_es_create(const evorl_es_config* cfg, evorl_es** out);
void evorl_es_destroy(evorl_es* es);
int64_t evorl_es_dim(const evorl_es* es);
/* Workflow::init(key) */
int evorl_es_init(evorl_es* es, uint64_t key_hi, uint64_t key_lo);
/* Workflow::step: one full generation on the device. */
int evorl_es_step(evorl_es* es, evorl_step_metrics* out);
/* Workflow::step with a host-resident EsState (the reference's layout): uploads
 * mean (and the Adam moments m, v and step count t -- pass NULL for m_in/v_in
 * to keep the device's), runs the generation, downloads the updated state
 * (NULL outputs are skipped); one synchronisation, staged through pinned
 * memory.  Unsharded handles only. */
int evorl_es_step_host(evorl_es* es, const double* mean_in, const double* m_in, const double* v_in, int64_t t_in,
                       double* mean_out, double* m_out, double* v_out, int64_t* t_out, evorl_step_metrics* out);
/* Page-locked host buffers: evorl_es_step_host copies them with the DMA engines
 * directly (no staging copy); in and out may be the same buffer. */
int evorl_host_alloc(int64_t bytes, void** out);
void evorl_host_free(void* p);
/* Workflow::evaluate (centre evaluation, proj/src/workflow.cpp:103-129) */
int evorl_es_evaluate(evorl_es* es, int32_t episodes, uint64_t key_hi, uint64_t key_lo,
                      double* mean_return, double* return_std);
/* Workflow::save / load + checkpoint_save / checkpoint_load
 * (proj/src/workflow.cpp:70-80, proj/src/checkpoint.cpp:180-212,
 * proj/src/workflow_es.cpp:181-249): EVORL1 files, workflow id "es", the
 * reference's segment names, order and encoding -- interchangeable with the
 * reference's checkpoints.  load() needs a handle created with the same config
 * and leaves it initialised; errors are EVORL_E_CHECKPOINT with the reference's
 * messages. */
int evorl_es_save(evorl_es* es, const char* path);
int evorl_es_load(evorl_es* es, const char* path);
/* WorkflowState counters (proj/include/evorl/workflow.hpp:31-36) */
int evorl_es_counters(const evorl_es* es, int64_t* iteration, int64_t* env_steps,
                      int64_t* episodes);
/* host <-> device state transfer (EsState, proj/src/workflow_es.cpp:15-20) */
int evorl_es_get_mean(evorl_es* es, double* mean);
int evorl_es_set_mean(evorl_es* es, const double* mean);
int evorl_es_get_adam(evorl_es* es, double* m, double* v, int64_t* t);
int evorl_es_set_adam(evorl_es* es, const double* m, const double* v, int64_t t);
int evorl_es_get_fitness(evorl_es* es, double* fitness);
int evorl_es_get_obs_norm(evorl_es* es, evorl_obs_norm* out);
int evorl_es_set_obs_norm(evorl_es* es, const evorl_obs_norm* in);
/* WorkflowState::rng (the root key of init / the loaded checkpoint); eval keys
 * are fold_in(fold_in(rng, 1), iteration) (proj/include/evorl/workflow.hpp:42) */
int evorl_es_get_rng(const evorl_es* es, uint64_t* hi, uint64_t* lo);
int evorl_es_set_counters(evorl_es* es, int64_t iteration, int64_t env_steps,
                          int64_t episodes);

/* CmaState transfer (proj/include/evorl/ec.hpp:107-122; the ec/C, ec/B, ec/D,
 * ec/ps, ec/pc, ec/sigma, ec/generation, ec/recondition_count checkpoint
 * segments of proj/src/workflow_es.cpp:194-203).  C, B: d x d row-major,
 * B[p*d + j] = component p of eigenvector j (Eigen's column j).  Any pointer
 * may be NULL. */
int evorl_es_cma_get(evorl_es* es, double* C, double* B, double* D, double* ps, double* pc,
                     double* sigma, int64_t* generation, int64_t* recondition_count);
int evorl_es_cma_set(evorl_es* es, const double* C, const double* B, const double* D,
                     const double* ps, const double* pc, double sigma, int64_t generation,
                     int64_t recondition_count);
/* CMA-ES free functions: CmaState::init / cmaes_ask / cmaes_tell
 * (proj/src/ec.cpp:191-288, proj/include/evorl/ec.hpp:107-125) on a device
 * state of dimension d with no env / policy attached: after create mean = 0,
 * C = B = I, D = 1, ps = pc = 0, sigma = sigma0.  State moves through
 * evorl_es_get/set_mean and evorl_es_cma_get/set; free with
 * evorl_es_destroy.  ask writes pop x d row-major candidates
 * (mean + sigma * B diag(D) z, z = gaussian_matrix(key, pop, d)); tell takes
 * pop x d candidates and their fitness (maximised).  eig_every as
 * evorl_es_config::cmaes_eig_every (1 = the reference's schedule). */
int evorl_cma_create(int64_t d, int32_t pop, int32_t elites, double sigma0, int32_t max_dim,
                     int32_t eig_every, evorl_es** out);
int evorl_cma_ask(evorl_es* cma, uint64_t key_hi, uint64_t key_lo, double* candidates);
int evorl_cma_tell(evorl_es* cma, const double* candidates, const double* fitness);

/* The device eigensolver (blocked Jacobi), replacing
 * Eigen::SelfAdjointEigenSolver (proj/src/ec.cpp:278-287): A n x n symmetric
 * row-major; evals ascending; vecs[p*n + j] = component p of eigenvector j,
 * normalised so its largest-|.| component is positive. */
int evorl_sym_eig(const double* A, int32_t n, double* evals, double* vecs, int32_t* sweeps);

/* ------------------------------------------- population sharding (N GPUs)
 * A generation split into the phases around the two collectives of
 * rank r rolls out agents [a0, a1), the caller all-gathers
 * the fitness vector (C1), then every rank applies the coordinate-sharded
 * tell to mean[p0, p1) and the caller all-gathers the mean slices (C2).
 * The device pointers returned by evorl_es_device_buffers let the caller run
 * the collectives (e.g. torch.distributed/NCCL) in place on the handle's
 * stream (evorl_es_stream). */
int evorl_es_set_shard(evorl_es* es, int32_t rank, int32_t world);
int evorl_es_shard_ranges(const evorl_es* es, int32_t* a0, int32_t* a1, int64_t* p0,
                          int64_t* p1);
int evorl_es_phase_rollout(evorl_es* es);            /* ask + rollout of [a0,a1) */
int evorl_es_phase_tell(evorl_es* es, evorl_step_metrics* out); /* ranks + tell of [p0,p1) */
/* fitness (pop doubles), mean (d doubles), lane stats (pop*e*9 doubles) */
int evorl_es_device_buffers(evorl_es* es, void** fitness, void** mean, void** lane_stats);
/* CEM diagonal variance (d doubles; CemState::diag_var, proj/include/evorl/ec.hpp:129-135):
 * the sharded tell updates [p0,p1) only, so the caller all-gathers it like the
 * mean, then reads the es/sigma metric with evorl_es_cem_sigma (phase_tell
 * reports NaN for it on a sharded handle). */
int evorl_es_device_var(evorl_es* es, void** var);
int evorl_es_cem_sigma(evorl_es* es, double* sigma); /* sqrt(diag_var.mean()), workflow_es.cpp:162 */
/* resolved obs_norm mode (EVORL_NORM_*): the lane stats are tracked, and must
 * be all-gathered by a sharded caller, iff it is EVORL_NORM_RS */
int evorl_es_norm_mode(const evorl_es* es, int32_t* mode);
void* evorl_es_stream(evorl_es* es);
/* device time (ms) of the last rollout launch and last full step, from CUDA
 * events on the handle's stream */
int evorl_es_last_timings(const evorl_es* es, float* rollout_ms, float* step_ms);
/* device time (ms) of the last generation's materialised ask (the candidate
 * matrix in one launch: for OpenES from the noise rows generated beside the
 * previous rollout, or with its own Threefry + Box-Muller noise on the first
 * generation / when that is off), or -1 when the ask was not one timed launch
 * (chunked candidates, CMA-ES, or before the first step) */
int evorl_es_last_ask_ms(const evorl_es* es, float* ask_ms);

/* ---------------------------------------------------------- benchmarking
 * Measured FP64 FMA peak of this GPU (TFLOP/s) by a DFMA-bound kernel; used
 * as the roofline denominator of the fp64 rollout. */
int evorl_measure_fp64_peak(double* tflops);
/* The OpenES noise generator (counter-addressed Threefry2x64 + Box-Muller)
 * at full occupancy: device ms to write n normals (second of two runs). */
int evorl_measure_noise_rate(int64_t n, float* ms);
/* Measured FP64 tensor-core (mma.sync m8n8k4 DMMA) peak, TFLOP/s. */
int evorl_measure_dmma_peak(double* tflops);

#ifdef __cplusplus
}
#endif
#endif
