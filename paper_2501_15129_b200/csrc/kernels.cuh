// kernels.cuh -- the non-rollout kernels of the generation (noise, ranks,
// fitness reduction, EC tells, observation statistics, init).
#pragma once

#include "rollout.cuh"

namespace evorl_b200 {

// Device-resident ObsNormState (proj/include/evorl/obs_norm.hpp:22-30).
struct DevNorm {
  int mode;  // 0 none, 1 vbn, 2 running stats
  int dim;
  double mean[4], var[4];
  double count;
};

struct ArsSel {  // elite selection of ars_tell (proj/src/ec.cpp:131-147)
  int b;
  int skipped;
  double scale;  // lr / (b * sigma_R)
  double sigma_r;
};

// Counter of kernel launches made by this library.
void count_launch(int n = 1);

cudaError_t run_threefry_batch(const uint64_t* keys, const uint64_t* ctrs, uint64_t* out, long long n,
                               cudaStream_t s);
cudaError_t run_stream_words(DKey key, long long first, long long n, uint64_t* out, cudaStream_t s);
cudaError_t run_gaussian_matrix(DKey key, long long rows, long long cols, double* out, cudaStream_t s);
// rank[i] = position of i in the stable ascending (desc=0) / descending order.
cudaError_t run_rank(const double* keys, int n, int desc, int* rank, cudaStream_t s);
cudaError_t run_shaped_from_rank(const int* rank, int n, double* shaped, cudaStream_t s);
cudaError_t run_order_from_rank(const int* rank, int n, int* order, cudaStream_t s);
cudaError_t run_fitness(const double* ep_returns, int count, int n_agents, int agent_offset,
                        double* fitness, const long long* lane_steps, int e,
                        unsigned long long* steps_accum, cudaStream_t s);
// metrics[0..2] = mean, max, min of fitness (deterministic order)
cudaError_t run_metrics(const double* fitness, int n, double* metrics, cudaStream_t s);
// OpenES tell + Adam over coordinates [p0, p1).  adam_bc: (1-b1^t, 1-b2^t) table.
struct OpenEsTellArgs {
  double* mean;
  double* m;
  double* v;
  const long long* t_dev;  // Adam step count before this tell
  long long d, p0, p1;
  double sigma, lr, lrwd, weight_decay, beta1, beta2, omb1, omb2, eps;
  int n, base, mirrored;
  DKey ask_key;
  const double* shaped;     // n
  const double* adam_bc;    // [2 * T_max]
  long long adam_bc_len;
  double* partial;          // scratch: openes_tell_chunks(...) x (p1 - p0) doubles
  const double* table;      // noise-table mode: eps_i[p] = table[offsets[i] + p] (else regenerated)
  const long long* offsets;
  const double* eps_rows;   // optional: eps_i[p] = eps_rows[i * eps_ld + p - eps_p0], kept by the ask
  long long eps_ld, eps_p0; // (unsharded: the ask's rows, ld = d, p0 = 0; sharded: this rank's columns)
};
// Row chunks of the tell's noise contraction for a coordinate span (so the
// grid fills the GPU; the chunk partials are summed in a fixed order).
int openes_tell_chunks(int rows, long long d);  // row chunks: a function of (rows, d) only
cudaError_t run_openes_tell(const OpenEsTellArgs& a, cudaStream_t s);
cudaError_t run_inc_counter(long long* t, cudaStream_t s);
cudaError_t run_openes_ask(const double* mean, long long d, double sigma, int mirrored, DKey key, int n,
                           double* cand, double* eps, cudaStream_t s);
cudaError_t run_ars_ask(const double* mean, long long d, double sigma, DKey key, int n, double* deltas,
                        double* cand, cudaStream_t s);
// ars: scores -> rank (caller) -> selection -> update
cudaError_t run_ars_scores(const double* fitness, int half, double* scores, cudaStream_t s);
cudaError_t run_ars_select(const double* fitness, const int* score_rank, int half, int elites,
                           double lr, int* elite_idx, double* elite_diff, ArsSel* sel, cudaStream_t s);
cudaError_t run_ars_update(double* mean, long long d, long long p0, long long p1, DKey key,
                           const int* elite_idx, const double* elite_diff, const ArsSel* sel,
                           cudaStream_t s);
// VES / CEM tells on regenerated candidates (order = stable descending)
cudaError_t run_ves_tell(double* mean, long long d, long long p0, long long p1, double sigma,
                         int mirrored, int base, DKey key, const int* order, const double* w,
                         int mu, cudaStream_t s);
cudaError_t run_cem_tell(double* mean, double* var, long long d, long long p0, long long p1, DKey key,
                         const int* order, int h, double floor_, cudaStream_t s);
// observation statistics
cudaError_t run_rs_merge(const double* lane_stats, int n_agents, int e, DevNorm* norm,
                         NormParams* params, double* agent_scratch, cudaStream_t s);
cudaError_t run_norm_params(const DevNorm* norm, NormParams* params, cudaStream_t s);
cudaError_t run_vbn_fit(const EnvDesc& env, DKey lane_key, int n, DevNorm* norm, NormParams* params,
                        cudaStream_t s);
// Glorot init (proj/src/net.cpp:52-68) of the whole parameter vector.
cudaError_t run_init_params(const NetDesc& net, DKey key, double* p, cudaStream_t s);
cudaError_t run_env_step_batch(const EnvDesc& env, long long n, double* phys, int* step_count,
                               const double* action, double* reward, int* term, int* trunc, int* fault,
                               cudaStream_t s);
cudaError_t run_eval_reduce(const double* returns, int n, double* out2, cudaStream_t s);
cudaError_t run_agent_stats(const double* lane_stats, int n_agents, int e, double* agent_stats,
                            cudaStream_t s);
double measure_fp64_peak_tflops();
double measure_dmma_peak_tflops();

}  // namespace evorl_b200
