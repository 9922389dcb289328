// rollout_tc.cu -- the population rollout with the hidden-layer GEMM on the
// 5th-generation tensor cores (tcgen05 + TMEM): precision EVORL_PREC_TC.
//
// Same lane-team semantics as rollout_kernel (proj/src/rollout.cpp:94-174);
// what changes is the policy arithmetic of the big layer:
//   * Shape: obs -> [W1] -> [W2] -> O (two hidden layers, BASELINE config 3).
//     Layer 0 (K = obs_dim <= 4) runs replicated on the CUDA cores in fp32;
//     layer 1 (W2 x W1, the dense contraction) runs on tcgen05, M = 128 rows
//     per CTA (a cluster of W2/128 CTAs per agent), N = 16 lanes, K = W1.
//   * Precision: bf16 single pass flips ~27% of ranks on this workload
//     (measured), so each fp32 operand x is split into fp16 hi = fp16(x) and
//     lo = fp16((x - hi) * 2^11); D0 = Ahi.Bhi and D1 = Ahi.Blo + Alo.Bhi are
//     accumulated in fp32 in TMEM and combined as D0 + D1 * 2^-11 (~22
//     significant bits: fp32-level, within RTOL_F32 of the fp64 reference).
//   * Operands: A = this CTA's 128-row slice of W2 (hi and lo, 128 KB) stays in
//     shared memory for the horizon in the canonical no-swizzle K-major UMMA
//     layout (8-row x 16-byte core matrices); B = the 16-lane activation block
//     is rewritten every step by the layer-0 threads.  One thread issues the
//     3 x K/16 MMAs, tcgen05.commit arrives on an mbarrier, and four warps
//     read the accumulator lanes back with tcgen05.ld.32x32b.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>

#include "rollout.cuh"

namespace evorl_b200 {

constexpr int TC_THREADS = 256;
constexpr int TC_M = 128;  // rows per CTA (UMMA M)
constexpr int TC_N = 16;   // lanes per team (UMMA N)
constexpr float TC_LO_SCALE = 2048.0f;
constexpr int TC_RANGE_ROW = 8;  // bad-layer row value: operand out of the split's range
constexpr int TC_OK_ROW = 15;    // bad-layer row value: no fault

struct TcPlan {
  int C;       // cluster size = W2 / 128
  int W1, W2;  // hidden widths
  int KSo;     // output-layer k-split
  int off_Ahi, off_Alo, off_Bhi, off_Blo, off_W0, off_b0, off_b1, off_W2o, off_b2, off_x0, off_h2,
      off_part, off_pout, off_mask, off_bar, off_tslot;
  int bytes;
};

// byte offset of element (row r, k) of a K-major no-swizzle UMMA operand with
// R rows: core matrices of 8 rows x 8 halves (128 B), row groups 128 B apart
// (SBO), K-halves (R/8)*128 B apart (LBO)
EVB_DEV uint32_t umma_off(int r, int k, int R) {
  return (uint32_t)((k >> 3) * (R >> 3) * 128 + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
}

EVB_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}

// kind::f16, A = B = f16 (K-major), D = f32, M = 128, N = 16
constexpr uint32_t TC_IDESC = (1u << 4) | ((uint32_t)(TC_N >> 3) << 17) | ((uint32_t)(TC_M >> 4) << 24);

EVB_DEV void tc_mma(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(accumulate));
}

EVB_DEV void tc_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

EVB_DEV void split_store(unsigned char* hi_base, unsigned char* lo_base, uint32_t off, float x) {
  const __half h = __float2half_rn(x);
  const __half l = __float2half_rn((x - __half2float(h)) * TC_LO_SCALE);
  *reinterpret_cast<__half*>(hi_base + off) = h;
  *reinterpret_cast<__half*>(lo_base + off) = l;
}

template <int C>
__global__ void __launch_bounds__(TC_THREADS, 1) rollout_tc_kernel(const __grid_constant__ RolloutArgs A,
                                                                   const __grid_constant__ TcPlan P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int crank = C > 1 ? (int)cluster_ctarank() : 0;
  const int team = blockIdx.x / C;
  const int agent_local = team / A.groups;
  const int group = team % A.groups;
  const int agent = A.agent_offset + agent_local;
  const int W1 = P.W1, W2 = P.W2, O = N.dims[3];
  const int r0 = crank * TC_M;  // this CTA's rows of layer 1

  for (int i = tid; i < P.bytes / 4; i += TC_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  float* W0 = reinterpret_cast<float*>(smem + P.off_W0);   // [k][W1]
  float* b0 = reinterpret_cast<float*>(smem + P.off_b0);   // W1
  float* b1 = reinterpret_cast<float*>(smem + P.off_b1);   // TC_M (slice)
  float* W2o = reinterpret_cast<float*>(smem + P.off_W2o); // [k_local][O]
  float* b2 = reinterpret_cast<float*>(smem + P.off_b2);   // O
  const int K0 = N.dims[0];
  // ---- prologue: this agent's parameters (regenerated or explicit)
  for (int i = tid; i < K0 * W1; i += TC_THREADS) {
    const int k = i / W1, r = i % W1;
    W0[k * W1 + r] = (float)param_value(A.par, N.d, agent_local, agent, N.w_off[0] + (long long)k * W1 + r);
  }
  for (int r = tid; r < W1; r += TC_THREADS)
    b0[r] = (float)param_value(A.par, N.d, agent_local, agent, N.b_off[0] + r);
  for (int i = tid; i < TC_M * W1; i += TC_THREADS) {  // A = W2 rows [r0, r0+128) x K = W1
    const int r = i % TC_M, k = i / TC_M;
    const float w =
        (float)param_value(A.par, N.d, agent_local, agent, N.w_off[1] + (long long)k * W2 + r0 + r);
    split_store(smem + P.off_Ahi, smem + P.off_Alo, umma_off(r, k, TC_M), w);
  }
  for (int r = tid; r < TC_M; r += TC_THREADS)
    b1[r] = (float)param_value(A.par, N.d, agent_local, agent, N.b_off[1] + r0 + r);
  for (int i = tid; i < TC_M * O; i += TC_THREADS) {
    const int k = i / O, o = i % O;
    W2o[i] = (float)param_value(A.par, N.d, agent_local, agent, N.w_off[2] + (long long)(r0 + k) * O + o);
  }
  for (int o = tid; o < O; o += TC_THREADS)
    b2[o] = (float)param_value(A.par, N.d, agent_local, agent, N.b_off[2] + o);

  // ---- TMEM (32 columns: D0 at 0, D1 at 16) and the MMA-completion mbarrier
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + P.off_tslot);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if constexpr (C > 1) cluster_sync_all();

  // ---- lane state
  const int j = group * TC_N + tid;
  const bool is_env = tid < TC_N;
  const bool valid = is_env && j < A.e;
  const int per = A.count / A.e, rem = A.count % A.e;
  const int eps_this = valid ? per + (j < rem ? 1 : 0) : 0;
  const int slot0 = valid ? j * per + min(j, rem) : 0;
  LaneEnv s{};
  double ep_ret = 0.0, wc = 0.0, wmean[4] = {0, 0, 0, 0}, wm2[4] = {0, 0, 0, 0};
  int ep_len = 0, eps_done = 0;
  long long steps = 0;
  uint32_t myfault = 0, myfault_layer = 0;
  if (valid) {
    const DKey lane_key = fold_in(fold_in(A.rollout_key, (uint64_t)agent), (uint64_t)j);
    env_reset(E, fold_in(lane_key, 0), s);
  }
  NormParams nrm;
  nrm.active = 0;
  if (A.norm != nullptr) nrm = *A.norm;
  float* x0 = reinterpret_cast<float*>(smem + P.off_x0);    // [4][16]
  float* h2 = reinterpret_cast<float*>(smem + P.off_h2);    // [TC_M][16]
  float* part = reinterpret_cast<float*>(smem + P.off_part);
  float* pout_base = reinterpret_cast<float*>(smem + P.off_pout);
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem + P.off_mask);
  const int OE = O * TC_N, OE1 = (O + 1) * TC_N;
  double sin_th = 0.0;
  auto observe_into_x0 = [&](bool act) {
    double raw[4];
    observe(E, s, raw);
    sin_th = raw[1];
    if (act && A.track_stats) {
      if (wc == 0.0) {
        for (int i = 0; i < E.obs_dim; ++i) {
          wmean[i] = raw[i];
          wm2[i] = 0.0;
        }
        wc = 1.0;
      } else {
        wc = dadd(wc, 1.0);
        for (int i = 0; i < E.obs_dim; ++i) {
          const double delta = dsub(raw[i], wmean[i]);
          wmean[i] = dadd(wmean[i], ddiv(delta, wc));
          wm2[i] = dadd(wm2[i], dmul(delta, dsub(raw[i], wmean[i])));
        }
      }
    }
    for (int i = 0; i < E.obs_dim; ++i) {
      double v = raw[i];
      if (nrm.active) v = ddiv(dsub(v, nrm.mean[i]), nrm.den[i]);
      x0[i * TC_N + tid] = act ? __double2float_rn(v) : 0.0f;
    }
  };
  if (valid && eps_this > 0 && A.max_iters > 0) observe_into_x0(true);

  for (int it = 0;; ++it) {
    if (tid < MAXL) mask[tid] = 0u;
    const bool active = valid && myfault == 0 && eps_done < eps_this && it < A.max_iters;
    if (!__syncthreads_or(active)) break;
    float* pout = pout_base + (it & 1) * C * OE1;

    // layer 0, replicated: h1 = relu(W0 x0 + b0) -> B operand (fp16 hi/lo)
    {
      const int e = tid & (TC_N - 1);
      float xr[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) xr[k] = k < K0 ? x0[k * TC_N + e] : 0.0f;
      uint32_t bad = 0u, range = 0u;
      for (int r = tid >> 4; r < W1; r += TC_THREADS / TC_N) {
        float z = 0.0f;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < K0) z = fmaf(W0[k * W1 + r], xr[k], z);
        z = z + b0[r];
        const float h = z > 0.0f ? z : 0.0f;
        if (h == INFINITY) bad = 1u;
        else if (h > 60000.0f) range = 1u;  // finite but beyond the fp16 split's range
        split_store(smem + P.off_Bhi, smem + P.off_Blo, umma_off(e, r, TC_N), h);
      }
      if (bad) atomicOr(&mask[0], 1u << e);
      if (range) atomicOr(&mask[MAXL - 1], 1u << e);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // layer 1 on tcgen05: 3 passes x W1/16 k-steps, issued by one thread
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t aHi = smem_u32(smem + P.off_Ahi), aLo = smem_u32(smem + P.off_Alo);
      const uint32_t bHi = smem_u32(smem + P.off_Bhi), bLo = smem_u32(smem + P.off_Blo);
      const uint32_t a_lbo = (TC_M / 8) * 128, b_lbo = (TC_N / 8) * 128;
      for (int ks = 0; ks < W1 / 16; ++ks) {
        const uint32_t ao = ks * 2 * a_lbo, bo = ks * 2 * b_lbo;
        tc_mma(tmem, umma_desc(aHi + ao, a_lbo, 128), umma_desc(bHi + bo, b_lbo, 128), ks > 0);
        tc_mma(tmem + 16, umma_desc(aHi + ao, a_lbo, 128), umma_desc(bLo + bo, b_lbo, 128), ks > 0);
        tc_mma(tmem + 16, umma_desc(aLo + ao, a_lbo, 128), umma_desc(bHi + bo, b_lbo, 128), 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(mbar))
                   : "memory");
    }
    mbar_wait_parity(mbar, (uint32_t)(it & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: warps 0-3 own TMEM lanes 32w..32w+31 = rows of the slice
    if (warp < 4) {
      const int r = warp * 32 + lane;
      float d0[16], d1[16];
      tc_ld16(tmem + ((uint32_t)(warp * 32) << 16), d0);
      tc_ld16(tmem + ((uint32_t)(warp * 32) << 16) + 16, d1);
      uint32_t bad = 0u;
      const float bb = b1[r];
#pragma unroll
      for (int e = 0; e < TC_N; ++e) {
        const float z = (d0[e] + d1[e] * (1.0f / TC_LO_SCALE)) + bb;
        const float h = z > 0.0f ? z : 0.0f;
        if (h == INFINITY) bad |= 1u << e;
        h2[r * TC_N + e] = h;
      }
      if (bad) atomicOr(&mask[1], bad);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();

    // output layer partial over this CTA's 128 rows, reduced across the cluster
    {
      const int KSo = P.KSo;
      const int kc = (TC_M + KSo - 1) / KSo;
      for (int w = tid; w < OE * KSo; w += TC_THREADS) {
        const int oe = w % OE, ks = w / OE;
        const int o = oe / TC_N, e = oe % TC_N;
        const int k0 = ks * kc, k1 = min(TC_M, k0 + kc);
        float acc = 0.0f;
        for (int k = k0; k < k1; ++k) acc = fmaf(W2o[k * O + o], h2[k * TC_N + e], acc);
        part[w] = acc;
      }
      __syncthreads();
      for (int oe = tid; oe < OE1; oe += TC_THREADS) {
        float v;
        if (oe < OE) {
          v = part[oe];
          for (int ks = 1; ks < KSo; ++ks) v += part[ks * OE + oe];
        } else {
          const int e = oe - OE;
          int bl = (mask[MAXL - 1] >> e) & 1u ? TC_RANGE_ROW : TC_OK_ROW;
          for (int l = 1; l >= 0; --l)
            if ((mask[l] >> e) & 1u) bl = l;
          v = (float)bl;
        }
        if constexpr (C > 1) {
          const uint32_t la = smem_u32(pout + crank * OE1 + oe);
#pragma unroll
          for (int c = 0; c < C; ++c) st_cluster<float>(map_cluster(la, (uint32_t)c), v);
        } else {
          pout[oe] = v;
        }
      }
      if constexpr (C > 1) {
        cluster_sync_all();
      } else {
        __syncthreads();
      }
    }

    // head + env step (proj/src/rollout.cpp:57-90, :131-153)
    if (active) {
      double z[8];
      bool nonfinite_out = false;
      int bad_layer = TC_OK_ROW;
      for (int c = 0; c < C; ++c) bad_layer = min(bad_layer, (int)pout[c * OE1 + OE + tid]);
      for (int o = 0; o < O && o < 8; ++o) {
        float v = pout[o * TC_N + tid];
        for (int c = 1; c < C; ++c) v += pout[c * OE1 + o * TC_N + tid];
        v = v + b2[o];
        z[o] = (double)v;
        if (!isfinite(z[o])) nonfinite_out = true;
      }
      if (bad_layer == TC_OK_ROW && nonfinite_out) bad_layer = 2;
      if (bad_layer == TC_RANGE_ROW) {
        myfault = FAULT_TC_RANGE;
        myfault_layer = 0u;
      } else if (bad_layer < 3) {
        myfault = FAULT_NET;
        myfault_layer = (uint32_t)bad_layer;
      } else {
        double action;
        if (N.head == HEAD_CATEGORICAL) {
          int arg = 0;
          for (int o = 1; o < O; ++o)
            if (z[o] > z[arg]) arg = o;
          action = (double)arg;
        } else if (N.head == HEAD_TANH) {
          action = N.tanh_scale * tanh(z[0]);
        } else {
          action = z[0];
        }
        double reward = 0.0;
        bool term = false, trunc = false;
        const uint32_t f =
            env_step(E, s, action, reward, term, trunc, E.id == ENV_PENDULUM ? &sin_th : nullptr);
        if (f) {
          myfault = f;
        } else {
          ep_ret = dadd(ep_ret, reward);
          ep_len += 1;
          steps += 1;
          if (term || trunc) {
            if (crank == 0) {
              const long long sl = (long long)agent_local * A.count + slot0 + eps_done;
              A.ep_returns[sl] = ep_ret;
              if (A.ep_lengths) A.ep_lengths[sl] = ep_len;
            }
            ep_ret = 0.0;
            ep_len = 0;
            eps_done += 1;
            if (eps_done < eps_this) env_reset(E, s.rng, s);
          }
        }
      }
      const bool next = myfault == 0 && eps_done < eps_this && it + 1 < A.max_iters;
      observe_into_x0(next);
    }
  }

  if (valid && crank == 0) {
    const long long ln = (long long)agent_local * A.e + j;
    if (A.lane_steps) A.lane_steps[ln] = steps;
    if (A.track_stats && A.lane_stats) {
      double* st = A.lane_stats + ln * 9;
      st[0] = wc;
      for (int i = 0; i < 4; ++i) {
        st[1 + i] = wmean[i];
        st[5 + i] = wm2[i];
      }
    }
    if (myfault) record_fault(A.fault, (uint64_t)((long long)agent * A.e + j), myfault, myfault_layer);
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
  if constexpr (C > 1) cluster_sync_all();
}

static int al(int x, int a) { return (x + a - 1) / a * a; }

bool plan_rollout_tc(const NetDesc& net, int obs_dim, int e, TcPlanOut* out) {
  if (net.nlayers != 3 || obs_dim > 4 || e < 5) return false;  // 16-lane teams, obs -> W1 -> W2 -> O
  const int W1 = net.dims[1], W2 = net.dims[2], O = net.dims[3];
  if (W1 % 16 || W1 > 256 || W2 % TC_M || W2 / TC_M > 8 || O > 8) return false;
  TcPlan p{};
  p.C = W2 / TC_M;
  p.W1 = W1;
  p.W2 = W2;
  int off = 0;
  p.off_Ahi = off;
  off = al(off + TC_M * W1 * 2, 1024);
  p.off_Alo = off;
  off = al(off + TC_M * W1 * 2, 1024);
  p.off_Bhi = off;
  off = al(off + TC_N * W1 * 2, 1024);
  p.off_Blo = off;
  off = al(off + TC_N * W1 * 2, 1024);
  p.off_W0 = off;
  off = al(off + 4 * W1 * 4, 16);
  p.off_b0 = off;
  off = al(off + W1 * 4, 16);
  p.off_b1 = off;
  off = al(off + TC_M * 4, 16);
  p.off_W2o = off;
  off = al(off + TC_M * O * 4, 16);
  p.off_b2 = off;
  off = al(off + O * 4, 16);
  p.off_x0 = off;
  off = al(off + 4 * TC_N * 4, 16);
  p.off_h2 = off;
  off = al(off + TC_M * TC_N * 4, 16);
  int KSo = 1;
  while (KSo * 2 * O * TC_N <= TC_THREADS && TC_M / (KSo * 2) >= 4) KSo *= 2;
  p.KSo = KSo;
  p.off_part = off;
  off = al(off + KSo * O * TC_N * 4, 16);
  p.off_pout = off;
  off = al(off + 2 * p.C * (O + 1) * TC_N * 4, 16);
  p.off_mask = off;
  off = al(off + MAXL * 4, 16);
  p.off_bar = off;
  off = al(off + 16, 16);
  p.off_tslot = off;
  off = al(off + 16, 16);
  p.bytes = off;
  if (off > 227 * 1024) return false;
  static_assert(sizeof(TcPlan) <= sizeof(TcPlanOut), "plan storage");
  std::memcpy(out, &p, sizeof p);
  return true;
}

template <int C>
static cudaError_t launch_tc_c(const RolloutArgs& a, const TcPlan& p, cudaStream_t stream) {
  auto kern = rollout_tc_kernel<C>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.n_agents * a.groups * C));
  cfg.blockDim = dim3(TC_THREADS);
  cfg.dynamicSmemBytes = (size_t)p.bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a, p);
}

cudaError_t launch_rollout_tc(const RolloutArgs& a, const TcPlanOut& po, cudaStream_t stream) {
  if (a.n_agents <= 0) return cudaSuccess;
  TcPlan p;
  std::memcpy(&p, &po, sizeof p);
  switch (p.C) {
    case 1: return launch_tc_c<1>(a, p, stream);
    case 2: return launch_tc_c<2>(a, p, stream);
    case 4: return launch_tc_c<4>(a, p, stream);
    case 8: return launch_tc_c<8>(a, p, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace evorl_b200
