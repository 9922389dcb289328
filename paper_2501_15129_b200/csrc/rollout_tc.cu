// rollout_tc.cu -- the population rollout with the hidden-layer GEMM on the
// 5th-generation tensor cores (tcgen05 + TMEM): precision EVORL_PREC_TC.
//
// Same lane-team semantics as rollout_kernel (proj/src/rollout.cpp:94-174);
// what changes is the policy arithmetic of the big layer:
//   * Shape: obs -> [W1] -> [W2] -> O (two hidden layers, BASELINE config 3).
//     Layer 0 (K = obs_dim <= 4) runs replicated on the CUDA cores in fp32;
//     layer 1 (W2 x W1, the dense contraction) runs on tcgen05, M = 128 rows
//     per CTA (a cluster of C = pow2(ceil(W2/128)) CTAs per agent, zero-padded
//     rows past W2), N = 16 lanes, K = W1 rounded up to 16 (zero-padded).
//   * Precision: bf16 single pass flips ~27% of ranks on this workload
//     (measured), so each fp32 operand x is split into fp16 hi = fp16(x) and
//     lo = fp16((x - hi) * 2^11); D0 = Ahi.Bhi and D1 = Ahi.Blo + Alo.Bhi are
//     accumulated in fp32 in TMEM and combined as D0 + D1 * 2^-11 (~22
//     significant bits: fp32-level, within RTOL_F32 of the fp64 reference).
//   * Operand residency (per CTA, for the whole horizon): A_hi (this CTA's
//     128 weight rows) in TENSOR MEMORY, written once by tcgen05.st; A_lo in
//     shared memory in the canonical no-swizzle K-major layout.  TMEM holds
//     256 columns (D0, D1, A_hi) and SMEM ~100 KB, so two teams share an SM
//     and one team's env phase overlaps the other's GEMM.
//   * Per k-step of 16: one TS MMA  D[0:32] += A_hi . [B_hi | B_lo]  (N = 32,
//     A from TMEM) and one SS MMA  D[16:32] += A_lo . B_hi  (N = 16), issued
//     by one thread; tcgen05.commit arrives on an mbarrier.
//   * Epilogue on all 8 warps (tcgen05.ld.32x32b.x8: warp w reads TMEM lanes
//     32(w%4).. and lane columns 8(w/4)..), bias + ReLU, and the output layer
//     fused in: each thread's row contributes W2o[r] * h to the (o, lane)
//     outputs, reduced across the warp by a shuffle reduce-scatter and across
//     the 4 row-quadrants and the cluster in a fixed order.
#include <cuda_fp16.h>

#include <algorithm>
#include <cstring>

#include "rollout.cuh"

namespace evorl_b200 {

constexpr int TC_THREADS = 256;
constexpr int TC_M = 128;  // rows per CTA (UMMA M)
constexpr int TC_N = 16;   // lanes per team
constexpr int TC_TMEM_COLS = 256;
constexpr int TC_COL_A = 32;   // C == 1: A_hi at TMEM column 32 (D0 = 0..15, D1 = 16..31)
constexpr int TC_COL_A2 = 64;  // PAIR: A_hi at column 64 (D = 0..31 hi x [hi|lo], 32..63 lo x [hi|lo])
constexpr float TC_LO_SCALE = 2048.0f;
constexpr int TC_RANGE_ROW = 8;  // bad-layer row value: operand out of the split's range
constexpr int TC_OK_ROW = 15;    // bad-layer row value: no fault
constexpr int TC_MAXO = 8;

#ifdef EVB_TC_PROFILE
// Phase cycle counters (profiling build only, libevorl_b200_prof.so): thread 0
// of every CTA accumulates clock64() deltas per phase and adds them here once.
__device__ unsigned long long g_tc_prof[16];
#define TC_MARK(i)                      \
  do {                                  \
    const long long t_ = clock64();     \
    prof[i] += (unsigned long long)(t_ - tprev); \
    tprev = t_;                         \
  } while (0)
#else
#define TC_MARK(i) \
  do {             \
  } while (0)
#endif

struct TcPlan {
  int C;       // cluster size: the power of two >= W2 / 128 (rows past W2 are zero)
  int W1, W2;  // hidden widths
  int W1p;     // W1 rounded up to the MMA K step (16); h1 rows past W1 are zero
  int off_Alo, off_B, off_W0, off_b0, off_x0, off_red, off_pout, off_mask, off_bar, off_tslot;
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

// kind::f16 instruction descriptor: A = B = f16 (K-major), D = f32
constexpr uint32_t tc_idesc(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// whole-warp variants: one elected lane issues (the operands are warp-uniform)
EVB_DEV void tc_mma_ss_elect(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
EVB_DEV void tc_mma_ts_elect(uint32_t dtmem, uint32_t atmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
EVB_DEV void tc_mma2_ss_elect(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
EVB_DEV void tc_mma2_ts_elect(uint32_t dtmem, uint32_t atmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
// pair commit: arrives on the same-offset mbarrier of both CTAs of the pair
EVB_DEV void tc_commit2_elect(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
EVB_DEV void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

EVB_DEV void tc_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
}
EVB_DEV void tc_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

EVB_DEV void split_f16(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn((x - __half2float(h)) * TC_LO_SCALE);
}
EVB_DEV uint32_t pack2(__half a, __half b) {  // element k in the low half, k+1 in the high half
  return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

template <int C>
__global__ void __launch_bounds__(TC_THREADS, 2) rollout_tc_kernel(const __grid_constant__ RolloutArgs A,
                                                                   const __grid_constant__ TcPlan P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quad = warp & 3, half = warp >> 2;  // TMEM lane quadrant, column half
  const int crank = C > 1 ? (int)cluster_ctarank() : 0;
  const int team = blockIdx.x / C;
  const int agent_local = team / A.groups;
  const int group = team % A.groups;
  const int agent = A.agent_offset + agent_local;
  const int W1 = P.W1, W1p = P.W1p, W2 = P.W2, O = N.dims[3], K0 = N.dims[0];
  const int r0 = crank * TC_M;       // this CTA's rows of layer 1
  // C >= 2: CTA pairs (2p, 2p+1) run cta_group::2 MMAs (M = 256): each CTA
  // holds its 128 weight rows and the B columns of its 8 lanes (N-split), the
  // even CTA issues for both and the commit arrives on both
  constexpr bool PAIR = C >= 2;
  const int pv = PAIR ? (crank & 1) : 0;  // 1: the pair's odd (non-issuing) CTA
  const int row = quad * 32 + lane;  // the layer-1 row this thread owns in the epilogue

#ifdef EVB_TC_PROFILE
  unsigned long long prof[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#endif
  for (int i = tid; i < P.bytes / 4; i += TC_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before any bulk copy into the zeroed SMEM
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + P.off_tslot);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* l0bar = mbar + 1;  // layer-0 B rows stored (this CTA's warps, and the odd peer's on a pair)
  uint64_t* xbar = mbar + 2;   // [2]: partial outputs of every cluster CTA landed
  uint64_t* pbar = mbar + 4;   // prologue bulk copies of the pre-split weights
  __syncthreads();
  if (warp == 0) {
    if constexpr (PAIR) {  // both CTAs of the pair: same columns in each TMEM
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                   "n"(TC_TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                   "n"(TC_TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    // layer-0 rows stored: every warp of this CTA (and, on a pair's even CTA,
    // of its odd peer) arrives once per step
    mbar_init(l0bar, (PAIR ? 2 : 1) * (TC_THREADS / 32));
    mbar_init(&xbar[0], 1);  // output exchange, double-buffered by step parity
    mbar_init(&xbar[1], 1);
    mbar_init(pbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  float* W0 = reinterpret_cast<float*>(smem + P.off_W0);  // [k][W1p], zero past W1
  float* b0 = reinterpret_cast<float*>(smem + P.off_b0);  // W1p, zero past W1
  unsigned char* Alo = smem + P.off_Alo;
  // B (K-major, K = W1): C == 1: 32 rows = B_hi of lanes 0..15, then B_lo;
  // PAIR: 16 rows = B_hi of this CTA's lanes 8pv..8pv+7, then their B_lo
  unsigned char* Bs = smem + P.off_B;
  // ---- prologue: this agent's parameters (regenerated or explicit)
  for (int i = tid; i < K0 * W1; i += TC_THREADS) {
    const int k = i / W1, r = i % W1;
    W0[k * W1p + r] = (float)param_value(A.par, N.d, agent_local, agent, N.w_off[0] + (long long)k * W1 + r);
  }
  const bool row_ok = r0 + row < W2;  // zero-padded rows of the last CTA
  for (int r = tid; r < W1; r += TC_THREADS)
    b0[r] = (float)param_value(A.par, N.d, agent_local, agent, N.b_off[0] + r);
  // layer-1 weights of row `row`: A_hi -> TMEM (lanes = rows, 2 halves per
  // column), A_lo -> SMEM.  Warp halves take alternate 16-wide k chunks.
  if (A.tc_blocks != nullptr) {
    // pre-split block (materialised ask): bulk-copy A_hi into the A_lo region,
    // move it to TMEM, then bulk-copy A_lo in place (cp.async.bulk, mbarrier)
    const unsigned char* blk = A.tc_blocks + ((long long)agent_local * C + crank) * A.tc_block_bytes;
    const uint32_t hb = (uint32_t)(A.tc_block_bytes / 2);
    if (tid == 0) {
      mbar_arrive_expect_tx(pbar, hb);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(Alo)),
                   "l"(blk), "r"(hb), "r"(smem_u32(pbar))
                   : "memory");
    }
    mbar_wait_parity_cta(pbar, 0);
    __syncwarp();
    for (int c = half; c < W1p / 16; c += 2) {
      uint32_t packed[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) packed[q] = *reinterpret_cast<const uint32_t*>(Alo + umma_off(row, c * 16 + 2 * q, TC_M));
      tc_st8(tmem + ((uint32_t)(quad * 32) << 16) + (PAIR ? TC_COL_A2 : TC_COL_A) + c * 8, packed);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    __syncthreads();  // every thread done with A_hi in the region
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(pbar, hb);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(Alo)),
                   "l"(blk + hb), "r"(hb), "r"(smem_u32(pbar))
                   : "memory");
    }
    mbar_wait_parity_cta(pbar, 1);
    __syncwarp();
  }
  for (int c = half; c < W1p / 16 && A.tc_blocks == nullptr; c += 2) {
    uint32_t packed[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      __half h[2], l[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int k = c * 16 + 2 * q + u;
        const float w = (row_ok && k < W1) ? (float)param_value(A.par, N.d, agent_local, agent,
                                                                 N.w_off[1] + (long long)k * W2 + r0 + row)
                                           : 0.0f;
        split_f16(w, h[u], l[u]);
        *reinterpret_cast<__half*>(Alo + umma_off(row, k, TC_M)) = l[u];
      }
      packed[q] = pack2(h[0], h[1]);
    }
    tc_st8(tmem + ((uint32_t)(quad * 32) << 16) + (PAIR ? TC_COL_A2 : TC_COL_A) + c * 8, packed);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const float b1r = row_ok ? (float)param_value(A.par, N.d, agent_local, agent, N.b_off[1] + r0 + row) : 0.0f;
  float w2r[TC_MAXO];
#pragma unroll
  for (int o = 0; o < TC_MAXO; ++o)
    w2r[o] = (o < O && row_ok) ? (float)param_value(A.par, N.d, agent_local, agent,
                                                    N.w_off[2] + (long long)(r0 + row) * O + o)
                               : 0.0f;
  float b2[TC_MAXO];
#pragma unroll
  for (int o = 0; o < TC_MAXO; ++o)
    b2[o] = o < O ? (float)param_value(A.par, N.d, agent_local, agent, N.b_off[2] + o) : 0.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A_lo visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
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
  const NormParams nrm = load_norm(A.norm);
  double inv_den[4];
  for (int i = 0; i < 4; ++i) inv_den[i] = nrm.active ? 1.0 / nrm.den[i] : 1.0;
  float* x0 = reinterpret_cast<float*>(smem + P.off_x0);    // [4][16]
  float* red = reinterpret_cast<float*>(smem + P.off_red);  // [4 quadrants][O][16]
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
    // normalised policy input (policy arithmetic, fp32 tolerance): multiply by
    // the reciprocal instead of the IEEE division the fp64 team uses
    for (int i = 0; i < E.obs_dim; ++i) {
      double v = raw[i];
      if (nrm.active) v = (v - nrm.mean[i]) * inv_den[i];
      x0[i * TC_N + tid] = act ? __double2float_rn(v) : 0.0f;
    }
  };
  if (valid && eps_this > 0 && A.max_iters > 0) observe_into_x0(true);

  constexpr uint32_t id32 = tc_idesc(TC_M, 32), id16 = tc_idesc(TC_M, 16), id2 = tc_idesc(2 * TC_M, 32);
  TC_MARK(0);  // prologue
  for (int it = 0;; ++it) {
    if (tid < MAXL) mask[tid] = 0u;
    const bool active = valid && myfault == 0 && eps_done < eps_this && it < A.max_iters;
    // warp-level vote first: __any_sync waits for all 32 lanes, so the warp
    // reaches the block-wide reduction barrier converged (the env lanes run
    // extra code; a partially arrived warp at BAR.RED is an illegal instruction)
    const bool wact = __any_sync(0xffffffffu, active);
    if (!__syncthreads_or(wact)) break;
    TC_MARK(1);  // loop-top barrier
    float* pout = pout_base + (it & 1) * C * OE1;
    if (C > 1 && tid == 0) mbar_arrive_expect_tx(&xbar[it & 1], (uint32_t)(C * OE1 * sizeof(float)));

    // layer 0: h1 = relu(W0 x0 + b0) -> B operand (fp16 hi/lo).  C == 1: all
    // 16 lanes; PAIR: the 8 lanes of this CTA's B columns.  k-step ks (16 rows
    // of h1) goes to warp ks % 8; a warp stores each 8-lane x 8-row core
    // matrix as 32 packed words (one per bank): lane -> (lane j = lane&7,
    // row pair = lane>>3).  Warp 7 (of the pair's even CTA) issues layer 1
    // once every warp (of both CTAs) has arrived.
    {
      constexpr int NB = PAIR ? 16 : 32;      // B rows (N) held by this CTA
      constexpr int EH = PAIR ? 1 : 2;        // 8-lane halves computed here
      const int KS = W1p / 16;
      uint32_t bad = 0u, range = 0u;
      const int el = lane & 7, rp = lane >> 3;
      float xr[EH][4];
#pragma unroll
      for (int eh = 0; eh < EH; ++eh)
#pragma unroll
        for (int k = 0; k < 4; ++k) xr[eh][k] = k < K0 ? x0[k * TC_N + (eh + pv) * 8 + el] : 0.0f;
      // (pipelining layer 0 against the MMAs in rounds of 8 k-steps measured
      // slower: the pair's tensor pipe is shared with the SM's other team)
      for (int ks = warp; ks < KS; ks += TC_THREADS / 32) {
        // this k-step's two row groups: weights and biases of rows r, r+1
        float2 wv[2][4], bv[2];
#pragma unroll
        for (int gi = 0; gi < 2; ++gi) {
          const int r = (ks * 2 + gi) * 8 + rp * 2;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            wv[gi][k] = k < K0 ? *reinterpret_cast<const float2*>(W0 + k * W1p + r) : make_float2(0.f, 0.f);
          bv[gi] = *reinterpret_cast<const float2*>(b0 + r);
        }
#pragma unroll
        for (int u = 0; u < 2 * EH; ++u) {  // (lane half eh, row group gi)
          const int eh = u % EH, gi = u / EH;
          const int e = (eh + pv) * 8 + el, r = (ks * 2 + gi) * 8 + rp * 2;
          float z0 = 0.0f, z1 = 0.0f;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k < K0) {
              z0 = fmaf(wv[gi][k].x, xr[eh][k], z0);
              z1 = fmaf(wv[gi][k].y, xr[eh][k], z1);
            }
          }
          z0 = z0 + bv[gi].x;
          z1 = z1 + bv[gi].y;
          const float h0 = z0 > 0.0f ? z0 : 0.0f;  // ReLU (NaN -> 0, as cwiseMax)
          const float h1 = z1 > 0.0f ? z1 : 0.0f;
          if (fmaxf(h0, h1) > 60000.0f) {
            if (h0 == INFINITY || h1 == INFINITY) bad |= 1u << e;
            else range |= 1u << e;  // finite but beyond the fp16 split's range
          }
          const __half2 hi = __floats2half2_rn(h0, h1);
          const float2 hf = __half22float2(hi);
          const __half2 lo = __floats2half2_rn((h0 - hf.x) * TC_LO_SCALE, (h1 - hf.y) * TC_LO_SCALE);
          const int nh = PAIR ? el : eh * 8 + el;  // B row of (lane e, hi); lo rows follow NB/2 later
          *reinterpret_cast<__half2*>(Bs + umma_off(nh, r, NB)) = hi;
          *reinterpret_cast<__half2*>(Bs + umma_off(nh + NB / 2, r, NB)) = lo;
        }
      }
      if (tid == 0) TC_MARK(12);  // layer-0 math + stores
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR && pv) {
          mbar_arrive_remote(l0bar, (uint32_t)(crank - 1));
        } else {
          mbar_arrive_local(l0bar);
        }
      }
      if (warp == TC_THREADS / 32 - 1 && !(PAIR && pv)) {  // layer 1 on tcgen05
        if constexpr (PAIR) {
          mbar_wait_parity(l0bar, (uint32_t)(it & 1));
        } else {
          mbar_wait_parity_cta(l0bar, (uint32_t)(it & 1));
        }
        __syncwarp();  // reconverge after the spin loop (elect.sync / tcgen05 below)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t aLo = smem_u32(Alo), bS = smem_u32(Bs);
        constexpr uint32_t a_lbo = (TC_M / 8) * 128, b_lbo = (NB / 8) * 128;
        for (int k = 0; k < KS; ++k) {
          const uint64_t bd = umma_desc(bS + k * 2 * b_lbo, b_lbo, 128);
          const uint64_t ad = umma_desc(aLo + k * 2 * a_lbo, a_lbo, 128);
          if constexpr (PAIR) {
            // D[0:32] += Ahi.[Bhi|Blo] (per CTA v: cols 16v..16v+7 hi.hi, +8 hi.lo);
            // D[32:64] += Alo.[Bhi|Blo] (cols 32+16v.. lo.hi; the lo.lo half is unused)
            tc_mma2_ts_elect(tmem, tmem + TC_COL_A2 + k * 8, bd, id2, k > 0);
            tc_mma2_ss_elect(tmem + 32, ad, bd, id2, k > 0);
          } else {
            tc_mma_ts_elect(tmem, tmem + TC_COL_A + k * 8, bd, id32, k > 0);  // D[0:32] += Ahi.[Bhi|Blo]
            tc_mma_ss_elect(tmem + 16, ad, bd, id16, 1);                      // D1 += Alo.Bhi
          }
        }
        if constexpr (PAIR) {
          tc_commit2_elect(mbar, (uint16_t)(3u << crank));  // crank is the pair's even rank
        } else {
          tc_commit_elect(mbar);
        }
      }
      bad = __reduce_or_sync(0xffffffffu, bad);
      range = __reduce_or_sync(0xffffffffu, range);
      if (lane == 0 && bad) atomicOr(&mask[0], bad);
      if (lane == 0 && range) atomicOr(&mask[MAXL - 1], range);
    }
    TC_MARK(2);  // layer 0 (+ waiting for the MMA issue)
    mbar_wait_parity(mbar, (uint32_t)(it & 1));
    __syncwarp();  // reconverge after the spin loop: tcgen05.ld below is .sync.aligned
    TC_MARK(3);  // MMA completion wait
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // epilogue: row `row`, lanes 8*half .. 8*half+7; output layer fused
    {
      uint32_t d0[8], d1[8], d2[8];
      const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16);
      if constexpr (PAIR) {  // lane e = 8*half + q: hi.hi col 16h+q, hi.lo 16h+8+q, lo.hi 32+16h+q
        tc_ld8(tl + half * 16, d0);
        tc_ld8(tl + half * 16 + 8, d1);
        tc_ld8(tl + 32 + half * 16, d2);
      } else {
        tc_ld8(tl + half * 8, d0);
        tc_ld8(tl + 16 + half * 8, d1);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float h[8];
      uint32_t bad = 0u;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float cross = PAIR ? __uint_as_float(d1[q]) + __uint_as_float(d2[q]) : __uint_as_float(d1[q]);
        const float z = (__uint_as_float(d0[q]) + cross * (1.0f / TC_LO_SCALE)) + b1r;
        h[q] = z > 0.0f ? z : 0.0f;
        if (h[q] == INFINITY) bad |= 1u << (half * 8 + q);
      }
      bad = __reduce_or_sync(0xffffffffu, bad);
      if (lane == 0 && bad) atomicOr(&mask[1], bad);
      // per output o: v[q] = w2[row][o] * h[q], summed over the warp's 32 rows
      // by a reduce-scatter (lane bits 4,3,2 select the lane q it ends on)
      const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1, bb2 = (lane >> 2) & 1;
#pragma unroll
      for (int o = 0; o < TC_MAXO; ++o) {
        if (o >= O) break;
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = w2r[o] * h[q];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float send = b4 ? v[i] : v[i + 4];
          const float keep = b4 ? v[i + 4] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const float send = b3 ? v[i] : v[i + 2];
          const float keep = b3 ? v[i + 2] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
        {
          const float send = bb2 ? v[0] : v[1];
          const float keep = bb2 ? v[1] : v[0];
          v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        if ((lane & 3) == 0) red[(quad * O + o) * TC_N + half * 8 + b4 * 4 + b3 * 2 + bb2] = v[0];
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    TC_MARK(4);  // epilogue
    // this CTA's partial outputs (fixed quadrant order) -> every CTA of the cluster
    for (int oe = tid; oe < OE1; oe += TC_THREADS) {
      float v;
      if (oe < OE) {
        v = ((red[oe] + red[OE + oe]) + red[2 * OE + oe]) + red[3 * OE + oe];
      } else {
        const int e = oe - OE;
        int bl = (mask[MAXL - 1] >> e) & 1u ? TC_RANGE_ROW : TC_OK_ROW;
        for (int l = 1; l >= 0; --l)
          if ((mask[l] >> e) & 1u) bl = l;
        v = (float)bl;
      }
      if constexpr (C > 1) {
        const uint32_t la = smem_u32(pout + crank * OE1 + oe), lb = smem_u32(&xbar[it & 1]);
#pragma unroll
        for (int c = 0; c < C; ++c) st_async(map_cluster(la, (uint32_t)c), v, map_cluster(lb, (uint32_t)c));
      } else {
        pout[oe] = v;
      }
    }
    if constexpr (C > 1) {
      // st.async + mbarrier: only the env threads wait for the cluster's
      // partial outputs.  This also orders the pair's B reuse: a CTA reaches
      // the next step's layer 0 only after its env threads saw the leader's
      // outputs, which the leader sends after its MMA completed.
      if (tid < TC_N) mbar_wait_parity(&xbar[it & 1], (uint32_t)((it >> 1) & 1));
    } else {
      __syncthreads();
    }

    TC_MARK(5);  // cluster exchange
    // head + env step (proj/src/rollout.cpp:57-90, :131-153)
    if (active) {
      double z[TC_MAXO];
      bool nonfinite_out = false;
      int bad_layer = TC_OK_ROW;
      for (int c = 0; c < C; ++c) bad_layer = min(bad_layer, (int)pout[c * OE1 + OE + tid]);
      for (int o = 0; o < O; ++o) {
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
        } else if (N.head == HEAD_TANH) {  // fp32 head: part of the fp32-tolerance policy
          action = N.tanh_scale * (double)tanhf((float)z[0]);
        } else {
          action = z[0];
        }
        double reward = 0.0;
        bool term = false, trunc = false;
        TC_MARK(10);  // head (output sum + tanh)
        const uint32_t f =
            env_step(E, s, action, reward, term, trunc, E.id == ENV_PENDULUM ? &sin_th : nullptr);
        TC_MARK(11);  // env_step
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
    TC_MARK(6);  // env phase
  }
#ifdef EVB_TC_PROFILE
  if (tid == 0) {
    for (int i = 0; i < 7; ++i) atomicAdd(&g_tc_prof[i], prof[i]);
    atomicAdd(&g_tc_prof[7], prof[7]);
    atomicAdd(&g_tc_prof[9], prof[9]);
    atomicAdd(&g_tc_prof[10], prof[10]);
    atomicAdd(&g_tc_prof[11], prof[11]);
    atomicAdd(&g_tc_prof[12], prof[12]);
    atomicAdd(&g_tc_prof[8], 1ull);
  }
#endif

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
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if constexpr (PAIR) {
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS));
    } else {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS));
    }
  }
  if constexpr (C > 1) cluster_sync_all();
}

static int al(int x, int a) { return (x + a - 1) / a * a; }

long long tc_block_bytes(const TcPlanOut& po) {
  TcPlan p;
  std::memcpy(&p, &po, sizeof p);
  return 2LL * TC_M * p.W1p * 2;
}

// one thread per (agent, CTA, 8-wide k chunk, row): reads 8 weights of the
// row (coalesced over rows), writes 16 B of A_hi and 16 B of A_lo -- the
// rows of a k chunk are contiguous in the canonical layout
__global__ void k_tc_split(const float* __restrict__ cand, long long d, long long w_off1, int W1, int W2, int W1p,
                           int C, long long total, unsigned char* __restrict__ blocks) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int row = (int)(idx % TC_M);
  const long long rest = idx / TC_M;
  const int kc = (int)(rest % (W1p / 8));
  const long long ac = rest / (W1p / 8);  // agent * C + crank
  const int crank = (int)(ac % C);
  const long long agent = ac / C;
  const int r = crank * TC_M + row;
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    __half h[2], l[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int k = kc * 8 + 2 * q + u;
      const float w = (r < W2 && k < W1) ? cand[agent * d + w_off1 + (long long)k * W2 + r] : 0.0f;
      split_f16(w, h[u], l[u]);
    }
    hi[q] = pack2(h[0], h[1]);
    lo[q] = pack2(l[0], l[1]);
  }
  const long long half_bytes = (long long)TC_M * W1p * 2;
  unsigned char* blk = blocks + ac * 2 * half_bytes;
  const uint32_t off = umma_off(row, kc * 8, TC_M);
  *reinterpret_cast<uint4*>(blk + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  *reinterpret_cast<uint4*>(blk + half_bytes + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

cudaError_t run_tc_split(const float* cand, const NetDesc& net, const TcPlanOut& po, int n_agents,
                         unsigned char* blocks, cudaStream_t stream) {
  TcPlan p;
  std::memcpy(&p, &po, sizeof p);
  const long long total = (long long)n_agents * p.C * (p.W1p / 8) * TC_M;
  if (total <= 0) return cudaSuccess;
  k_tc_split<<<(unsigned)((total + 255) / 256), 256, 0, stream>>>(cand, net.d, net.w_off[1], p.W1, p.W2, p.W1p, p.C,
                                                                   total, blocks);
  return cudaGetLastError();
}

bool plan_rollout_tc(const NetDesc& net, int obs_dim, int e, TcPlanOut* out) {
  if (net.nlayers != 3 || obs_dim > 4 || e < 5) return false;  // 16-lane teams, obs -> W1 -> W2 -> O
  const int W1 = net.dims[1], W2 = net.dims[2], O = net.dims[3];
  const int W1p = (W1 + 15) / 16 * 16;
  int C = 1;
  while (C * TC_M < W2) C *= 2;
  if (C > 8 || O > TC_MAXO || W1p > 2 * (TC_TMEM_COLS - (C >= 2 ? TC_COL_A2 : TC_COL_A))) return false;
  TcPlan p{};
  p.C = C;
  p.W1 = W1;
  p.W1p = W1p;
  p.W2 = W2;
  int off = 0;
  p.off_Alo = off;
  off = al(off + TC_M * W1p * 2, 1024);
  p.off_B = off;
  off = al(off + (p.C >= 2 ? 16 : 32) * W1p * 2, 1024);
  p.off_W0 = off;
  off = al(off + 4 * W1p * 4, 16);
  p.off_b0 = off;
  off = al(off + W1p * 4, 16);
  p.off_x0 = off;
  off = al(off + 4 * TC_N * 4, 16);
  p.off_red = off;
  off = al(off + 4 * O * TC_N * 4, 16);
  p.off_pout = off;
  off = al(off + 2 * p.C * (O + 1) * TC_N * 4, 16);
  p.off_mask = off;
  off = al(off + MAXL * 4, 16);
  p.off_bar = off;
  off = al(off + 8 * 5, 16);  // mbar, l0bar, xbar[2], pbar
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

#ifdef EVB_TC_PROFILE
extern "C" int evorl_debug_tc_profile(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, g_tc_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 6;
  static const unsigned long long zero[16] = {};
  return cudaMemcpyToSymbol(g_tc_prof, zero, sizeof zero) == cudaSuccess ? 0 : 6;
}
#endif

}  // namespace evorl_b200
