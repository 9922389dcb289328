// rollout.cuh -- descriptors shared by the host planner and the fused
// population-rollout kernel (rollout.cu).
#pragma once

#include "common.cuh"
#include "env.cuh"

namespace evorl_b200 {

constexpr int MAXL = 9;  // up to 8 hidden layers + output layer
constexpr int ROLLOUT_THREADS = 256;

enum : int { HEAD_TANH = 0, HEAD_GAUSSIAN = 1, HEAD_CATEGORICAL = 2, HEAD_LINEAR = 3 };

// Flat parameter layout of proj/src/net.cpp:26-48 (column-major W then b per
// layer).  Layer norm is not supported on the device path (refused by the
// host planner).
struct NetDesc {
  int nlayers;  // hidden layers + 1
  int dims[MAXL + 1];
  long long w_off[MAXL];
  long long b_off[MAXL];
  int head;
  double tanh_scale;
  long long d;
};

// Where candidate i's parameters come from.  Only SRC_EXPLICIT reads a stored
// n x d matrix; the others regenerate the perturbation from the ask key
// (proj/src/ec.cpp:71-97 OpenES/VES, :113-125 ARS, :306-313 CEM).
enum : int { SRC_EXPLICIT = 0, SRC_OPENES = 1, SRC_ARS = 2, SRC_CEM = 3, SRC_EXPLICIT_F32 = 4,
             SRC_OPENES_TABLE = 5 };
struct ParamDesc {
  int src;
  const double* params;  // SRC_EXPLICIT: n_agents x d, row-major
  const float* params_f32;  // SRC_EXPLICIT_F32: n_agents x d, the fp32 policy paths' candidates
  const double* mean;    // d
  const double* var;     // CEM diagonal variance
  double sigma;
  DKey ask_key;
  int base;  // OpenES/VES: number of sampled rows (n/2 when mirrored)
  const double* table;         // SRC_OPENES_TABLE: the shared noise table
  const long long* offsets;    // SRC_OPENES_TABLE: window start of each sampled row
  int mirrored;
};

// Observation normaliser frozen for the generation: x = (o - mean) / den,
// den = max(sqrt(var), 1e-8) (proj/src/obs_norm.cpp:76-79).
struct NormParams {
  int active;
  int dim;
  double mean[4];
  double den[4];
};

// The generation's normaliser, or the identity (inactive, den = 1) when there
// is none -- every field defined, so no uninitialised value reaches the
// speculated reciprocals of the env code.
EVB_DEV NormParams load_norm(const NormParams* p) {
  if (p != nullptr) return *p;
  NormParams n{};
#pragma unroll
  for (int i = 0; i < 4; ++i) n.den[i] = 1.0;
  return n;
}

// Candidate parameter p of agent `agent` (global population index).
EVB_DEV double param_value(const ParamDesc& P, long long d, int agent_local, int agent,
                           long long p) {
  switch (P.src) {
    case SRC_OPENES: {  // proj/src/ec.cpp:87-94: (sigma * eps) + mean, rows [base,n) = -eps
      long long row = agent;
      bool neg = false;
      if (P.mirrored && agent >= P.base) {
        row = agent - P.base;
        neg = true;
      }
      double eps = normal_at(P.ask_key, (uint64_t)(row * d + p));
      if (neg) eps = -eps;
      return dadd(dmul(P.sigma, eps), P.mean[p]);
    }
    case SRC_OPENES_TABLE: {  // proj/src/ec.cpp:79-86: row i = table[off_i : off_i + d]
      long long row = agent;
      bool neg = false;
      if (P.mirrored && agent >= P.base) {
        row = agent - P.base;
        neg = true;
      }
      double eps = P.table[P.offsets[row] + p];
      if (neg) eps = -eps;
      return dadd(dmul(P.sigma, eps), P.mean[p]);
    }
    case SRC_ARS: {  // proj/src/ec.cpp:119-123: interleaved mean +/- sigma*delta_k
      const long long k = agent >> 1;
      const double sd = dmul(P.sigma, normal_at(P.ask_key, (uint64_t)(k * d + p)));
      return (agent & 1) ? dsub(P.mean[p], sd) : dadd(P.mean[p], sd);
    }
    case SRC_CEM: {  // proj/src/ec.cpp:306-313: z * sqrt(var) + mean
      const double z = normal_at(P.ask_key, (uint64_t)((long long)agent * d + p));
      return dadd(dmul(z, sqrt(P.var[p])), P.mean[p]);
    }
    case SRC_EXPLICIT_F32:
      return (double)P.params_f32[(long long)agent_local * d + p];
    default:
      return P.params[(long long)agent_local * d + p];
  }
}

struct TcPlanOut {
  int data[32];  // TcPlan (rollout_tc.cu); data[0] = cluster size
};

struct SmemPlan {
  int C;             // cluster size (CTAs per team)
  int TR;            // rows per thread
  int ET;            // lanes per team
  int RS[MAXL];      // real rows owned per CTA (hidden layers)
  int RSP[MAXL];     // padded rows per CTA
  int KS[MAXL];      // k-split per hidden layer
  int WS[MAXL];      // row stride of the k-major weight slice (RSP, +4 for DMMA)
  int REP[MAXL];     // 1: layer computed in full by every CTA (no DSMEM exchange)
  int XS;            // row stride of the activation buffers (ET; 20 on the DMMA plan)
  int mma;           // 1: hidden layers with K >= 16 use FP64 tensor cores (DMMA)
  int KS_out;        // k-split of the output layer partial
  int off_w[MAXL], off_b[MAXL];
  int off_wout, off_bout, off_x0, off_h[MAXL], off_part, off_pout, off_mask, off_bar;
  int bytes;
  int gw;         // 1: weights read from the materialised candidates in HBM/L2
                 //    (policies too large for SMEM residency; SIMT slice GEMMs)
  int trn;        // 1: collect transitions (RolloutArgs::t_*), TR = 1 SIMT plans only
  int tc;         // 1: EVORL_PREC_TC tcgen05 team (rollout_tc.cu), plan in tcp
  int pipe;       // 1: pipelined fp64 DMMA team (two 8-lane groups, env warp)
  int oz;         // 1: EVORL_PREC_OZ int8-sliced tcgen05 team (rollout_oz.cu), plan in tcp
  TcPlanOut tcp;
};

struct RolloutArgs {
  EnvDesc env;
  NetDesc net;
  ParamDesc par;
  SmemPlan plan;
  const NormParams* norm;  // device; may be null (no normalisation)
  int n_agents;            // agents in this launch
  int agent_offset;        // global index of agent 0 (population sharding)
  int e;                   // lanes per agent (envs_per_agent)
  int count;               // episodes per agent (episodes mode)
  int groups;              // teams per agent = ceil(e / ET)
  DKey rollout_key;        // fold_in(step_key, 1) (proj/src/workflow_es.cpp:125)
  int track_stats;         // RunningStats obs tracking (ARS)
  int max_iters;           // safety bound on steps per lane
  double* ep_returns;      // [n_agents][count], lane-major slot order
  int* ep_lengths;         // [n_agents][count]
  long long* lane_steps;   // [n_agents * e]
  double* lane_stats;      // [n_agents * e][9] = count, mean[4], m2[4]
  unsigned long long* fault;
  // RolloutOptions::collect_transitions (proj/src/rollout.cpp:118-170), cluster
  // team only: lane l's rows at [l * t_cap, l * t_cap + lane_steps[l]) with
  // l = agent_local * e + j; null = not collected
  double* t_obs;      // rows x obs_dim (raw observation)
  double* t_act;      // rows x 1 (act_dim of both envs)
  double* t_rew;
  unsigned char* t_term;
  unsigned char* t_trunc;
  double* t_next;     // rows x obs_dim (final_obs: successor before auto-reset)
  long long t_cap;
  // tc team: per (agent, CTA) pre-split layer-1 weights in the UMMA canonical
  // layout (A_hi then A_lo, tc_block_bytes each pair), bulk-copied by the
  // prologue; null = split in the prologue from the parameters
  const unsigned char* tc_blocks;
  long long tc_block_bytes;
};

// Host-side: launch the rollout with the plan's template instance.
cudaError_t launch_rollout(const RolloutArgs& a, int precision, cudaStream_t stream);
// Host-side: build the SMEM plan; returns false if no cluster size fits.
// simple_only: only TR = 1 SIMT plans (SMEM-resident or global-weights) -- the
// plans with a transition-collecting instantiation (SmemPlan::trn)
bool plan_rollout(const NetDesc& net, int obs_dim, int e, int precision, SmemPlan* plan,
                  bool simple_only = false);

// Warp-team rollout for small policies (rollout_warp.cu): one warp per lane.
struct WarpPlanOut {
  int data[64];
};
bool plan_rollout_warp(const NetDesc& net, int obs_dim, int e, int precision, WarpPlanOut* out);
cudaError_t launch_rollout_warp(const RolloutArgs& a, const WarpPlanOut& plan, int precision,
                                cudaStream_t stream);
// Materialise candidates [a0, a1) (row-major, d each) from a ParamDesc.
// SRC_OPENES only: eps_out (optional) receives the sampled noise entries of
// the rows these agents use, entry (row, p) at eps_out[(row - eps_row0) d + p].
cudaError_t run_materialize(const ParamDesc& par, long long d, int a0, int a1, double* out,
                            cudaStream_t stream, double* eps_out = nullptr, long long eps_row0 = 0);
// The OpenES noise rows [r0, r1) agents [a0, a1) use (row a, or a - base
// for the mirrored half).
void openes_row_range(const ParamDesc& par, int a0, int a1, long long* r0, long long* r1);

// OpenES noise kept ahead of the ask: normals [t0, t0 + n) of the ask stream
// `key` into eps[t - t0] (persistent grid of `blocks` 128-thread blocks, sized
// to share the SMs with a resident rollout), and the ask's candidates from
// such rows, eps holding rows from eps_row0 on (bit-identical to
// run_materialize / run_materialize_f32 for SRC_OPENES).
cudaError_t run_noise_rows(DKey key, long long t0, long long n, double* eps, int blocks, cudaStream_t stream);
// ... and the columns [p0, p1) of rows [0, rows) (a coordinate-sharded tell's
// noise) into out[row (p1 - p0) + p - p0]
cudaError_t run_noise_cols(DKey key, long long d, long long p0, long long p1, long long rows, double* out,
                           int blocks, cudaStream_t stream);
cudaError_t run_cand_from_eps(const ParamDesc& par, long long d, int a0, int a1, const double* eps,
                              long long eps_row0, double* out, cudaStream_t stream);
cudaError_t run_cand_from_eps_f32(const ParamDesc& par, long long d, int a0, int a1, const double* eps,
                                  long long eps_row0, float* out, cudaStream_t stream);

// Materialise candidates [a0, a1) as fp32 (the value the fp32 policy paths
// round each fp64 candidate parameter to).  OpenES: one Box-Muller pair per
// thread, shared by the mirrored agents.
cudaError_t run_materialize_f32(const ParamDesc& par, long long d, int a0, int a1, float* out,
                                cudaStream_t stream, double* eps_out = nullptr, long long eps_row0 = 0);

// Tensor-core rollout (rollout_tc.cu, precision EVORL_PREC_TC): obs -> W1 -> W2 -> O
// policies with W2 a multiple of 128; the W2 x W1 layer runs on tcgen05.
bool plan_rollout_tc(const NetDesc& net, int obs_dim, int e, TcPlanOut* out);
// bytes of one (agent, CTA) pre-split weight block of a tc plan
long long tc_block_bytes(const TcPlanOut& plan);
// the fp32 candidates [n_agents x d] -> pre-split blocks [n_agents][C]
cudaError_t run_tc_split(const float* cand, const NetDesc& net, const TcPlanOut& plan, int n_agents,
                         unsigned char* blocks, cudaStream_t stream);
cudaError_t launch_rollout_tc(const RolloutArgs& a, const TcPlanOut& plan, cudaStream_t stream);

// fp64-accurate tensor-core rollout (rollout_oz.cu, precision EVORL_PREC_OZ):
// obs -> W1 -> W2 -> O policies, W1 <= 256; the W2 x W1 layer as S byte-sliced
// fixed-point int8 tcgen05 MMAs, everything else fp64.
bool plan_rollout_oz(const NetDesc& net, int obs_dim, int e, TcPlanOut* out);
cudaError_t launch_rollout_oz(const RolloutArgs& a, const TcPlanOut& plan, cudaStream_t stream);
// bytes of one (agent, CTA) pre-split layer-1 block of an oz plan
long long oz_block_bytes(const TcPlanOut& plan);
// the fp64 candidates [n_agents x d] -> pre-split blocks [n_agents][C]
cudaError_t run_oz_split(const double* cand, const NetDesc& net, const TcPlanOut& plan, int n_agents,
                         unsigned char* blocks, cudaStream_t stream);
// The OpenES ask of agents [a0, a1) fused with the pre-split, from kept noise
// rows eps (row-major, d per row, from row eps_row0 on): the layer-1 byte-slice blocks (identical to
// run_materialize + run_oz_split), the other parameters into cand, and the
// fp64 layer-1 row of cand only where it holds a non-finite weight.
cudaError_t run_oz_ask_split(const ParamDesc& par, const NetDesc& net, const TcPlanOut& po, int a0, int a1,
                             const double* eps, long long eps_row0, double* cand, unsigned char* blocks,
                             cudaStream_t stream);

}  // namespace evorl_b200
