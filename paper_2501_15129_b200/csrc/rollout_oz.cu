// rollout_oz.cu -- the population rollout with the hidden-layer GEMM on the
// int8 tensor cores (tcgen05 kind::i8) at fp64-level accuracy: precision
// EVORL_PREC_OZ (sliced fixed point, the Ozaki scheme).
//
// Same lane-team semantics as rollout_kernel (proj/src/rollout.cpp:94-174,
// one team per (agent, group of 16 lanes)); the env, the observation
// normaliser, layer 0, the output layer and the head stay fp64 on the CUDA
// cores in the fp64 team's operation order.  What changes is the dense
// W2 x W1 layer (proj/src/net.cpp:96, z = W h + b):
//   * Each weight row r is a signed fixed-point integer W_int = floor(W 2^F_r)
//     with |W_int| < 2^(8S-1) (F_r from the row's largest |w|), cut into S
//     bytes from the top: A_0 = W_int >> 8(S-1) (s8), A_i = byte i (u8).
//     Each activation column (lane) e is h_int = rn(h 2^G_e) <= 2^(8S-1)
//     (h >= 0 after ReLU; G_e from a per-lane bound), bytes B_j (u8).
//   * W_int h_int = sum_{i,j} A_i B_j 2^(8(2S-2-i-j)); the terms i + j < S are
//     kept: D_t = sum_{i+j=t} A_i B_j, t < S, exact in int32 (|D_t| < S 2^24).
//     z = 2^(8(S-1) - F_r - G_e) sum_t D_t 2^(8(S-1-t)), combined exactly in two
//     44-bit integers and converted to fp64 once.
//     S = 6 keeps ~47 bits of every operand: the policy output differs from
//     fp64 arithmetic by ~1e-13 relative (fitness differences at the level of
//     the fp64 path's own libm/ordering differences from the reference CPU).
//   * One accumulator per lane group for all t: the B operand is the S slice
//     blocks of 8 lanes [B_0 .. B_(S-1)] in SMEM, and MMA i (A_i from TMEM)
//     writes D from column block i on with N = 8 (S - i) rounded up to 16, so
//     column block c of D receives A_i B_(c-i): D[:, 8t..8t+7] = D_t (the
//     rounding spills into block S, never read).  Per k-step of 32: S TS MMAs
//     of M = 128, K = 32, N = 48, 48, 32, 32, 16, 16 (tools/umma_i8_bench.cu
//     checks the scheme and times it: 48 MMAs in ~920 cycles).
//   * TMEM (512 columns, one team CTA per SM): A slices at columns 512 - S W1p/4
//     (written once by tcgen05.st from pre-split blocks), D_g at columns 8 (S+1) g.
//   * Per env step (one CTA = 128 weight rows; C = W2/128 CTAs per agent) the
//     16 lanes are two groups of 8 whose chains -- layer 0 (fp64, replicated)
//     -> per-lane bound, fixed point, bytes -> B_g | MMAs (MMA warp) | epilogue:
//     tcgen05.ld of D_0..D_(S-1), exact integer combine, fp64 scale, bias, ReLU,
//     output-layer partial (warp reduce-scatter) | st.async partial outputs to
//     every CTA of the cluster | env warp: head, fp64 env step, observe -- run
//     half a period apart (rollout_ozp_kernel below).
//   * Rows holding a non-finite weight (a diverged mean) are computed by an
//     fp64 dot product instead (IEEE propagation and NetFault as the fp64 team).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>

#include "rollout.cuh"

namespace evorl_b200 {

constexpr int OZ_M = 128;  // weight rows per CTA (UMMA M)
constexpr int OZ_N = 16;   // lanes per team
constexpr int OZ_MAXO = 8;
constexpr int OZ_TMEM_COLS = 512;
constexpr int OZ_MIN_SMEM = 120 * 1024;  // > half an SM's shared memory: one team CTA per SM (TMEM)

#ifdef EVB_TC_PROFILE
__device__ unsigned long long g_oz_prof[16];
#define OZ_MARK(i)                               \
  do {                                           \
    const long long t_ = clock64();              \
    prof[i] += (unsigned long long)(t_ - tprev); \
    tprev = t_;                                  \
  } while (0)
#else
#define OZ_MARK(i) \
  do {             \
  } while (0)
#endif

struct OzPlan {
  int C;       // CTAs per agent (cluster): power of two >= W2 / 128
  int S;       // byte slices per operand
  int W1, W2;  // hidden widths
  int W1p;     // W1 rounded up to the MMA K step (32)
  int off_B, off_W0, off_b0, off_mk, off_x0, off_red, off_pout, off_mask, off_bar, off_tslot, off_rmax;
  int used;   // bytes of the layout (zeroed by the prologue)
  int bytes;  // dynamic SMEM requested: >= OZ_MIN_SMEM
};

EVB_DEV uint64_t oz_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);  // version 1, SWIZZLE_NONE
}
// kind::i8 instruction descriptor: D = s32 (c_format 2), A = s8 (1) or u8 (0),
// B = u8, both K-major
constexpr uint32_t oz_idesc(int M, int N, bool a_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
EVB_DEV void oz_mma_ts_elect(uint32_t dtmem, uint32_t atmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
// single-thread forms (the caller elects the issuing lane once per group-step)
EVB_DEV bool elect_one() {
  uint32_t p;
  asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}"
               : "=r"(p));
  return p != 0;
}
EVB_DEV void oz_mma_ts(uint32_t dtmem, uint32_t atmem, uint64_t bdesc, uint32_t idesc, bool acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dtmem),
      "r"(atmem), "l"(bdesc), "r"(idesc), "r"((uint32_t)acc));
}
EVB_DEV void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
EVB_DEV void oz_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
EVB_DEV void oz_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
}
EVB_DEV void oz_ld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
EVB_DEV void named_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EVB_DEV void oz_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
// The oz teams always read materialised candidates (SRC_EXPLICIT: the
// workflow's fp64 ask, evaluate's centre, batched_rollout's params; checked by
// launch_rollout_oz), so a parameter is one load -- no inlined noise
// regeneration in the prologue (kernel size, compile time).
EVB_DEV double oz_param(const ParamDesc& P, long long d, int agent_local, long long p) {
  return P.params[(long long)agent_local * d + p];
}
// fmax over finite values only (NaN / inf weights are handled by the fp64 row path)
EVB_DEV double fin_abs(double v) { return isfinite(v) ? fabs(v) : 0.0; }
// the power-of-two exponent e with |v| < 2^e (v finite, >= 0), clamped so that
// 2^(+-(8S + e)) stays a normal double
EVB_DEV int bound_exp(double v) {
  int e = 0;
  if (v > 0.0) frexp(v, &e);
  return max(-960, min(960, e));
}
// exact int64 -> double for |x| < 2^51 without the (slow) conversion pipe:
// the integer lands in the mantissa of 1.5 * 2^52 + x
EVB_DEV double i51_to_double(long long x) {
  return __longlong_as_double(x + 0x4338000000000000LL) - 6755399441055744.0;
}
// byte b (0..3) of each of a0..a3 packed into one word (a0's in the low byte)
EVB_DEV uint32_t gather_byte(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, int b) {
  const uint32_t sel = (uint32_t)b | ((uint32_t)(b + 4) << 4);
  return __byte_perm(__byte_perm(a0, a1, sel), __byte_perm(a2, a3, sel), 0x5410);
}
// the frexp exponent of a finite v >= 0 from its bit field (v < 2^e; zero and
// subnormals give -1022), clamped like bound_exp
EVB_DEV int bound_exp_bits(double v) {
  const int e = ((__double2hiint(v) >> 20) & 0x7FF) - 1022;
  return max(-960, min(960, e));
}
// 2^g for |g| <= 1000 (a normal double), built from the exponent field
EVB_DEV double pow2(int g) { return __hiloint2double((g + 1023) << 20, 0); }
// The S bytes of 32 consecutive weights of one row, W_int = floor(w 2^F) in
// offset binary: t = w 2^F + 2^52 + 2^(8S-1) (rounded toward zero) carries
// U = W_int + 2^(8S-1) in [0, 2^(8S)) in its mantissa, so the bytes are byte
// permutes of its two words (no float->int conversion, no 64-bit shifts); the
// top byte of U minus 128 is the signed A_0 (an XOR with 0x80).  Non-finite
// weights slice as 0 (their rows take the fp64 path).
template <int S>
EVB_DEV void oz_slice32(const double* w, double wscale, uint32_t (&out)[S][8]) {
  static_assert(S <= 6, "U must fit the 52-bit mantissa with room for the offset");
  const double off = 0x1p52 + (double)(1ull << (8 * S - 1));
  uint32_t lo[32], hi[32];
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const double t = __fma_rz(isfinite(w[q]) ? w[q] : 0.0, wscale, off);
    lo[q] = (uint32_t)__double2loint(t);
    hi[q] = (uint32_t)__double2hiint(t);
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const int Pb = 8 * (S - 1 - i);
    const bool H = Pb >= 32;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t v = gather_byte(H ? hi[4 * u] : lo[4 * u], H ? hi[4 * u + 1] : lo[4 * u + 1],
                                     H ? hi[4 * u + 2] : lo[4 * u + 2], H ? hi[4 * u + 3] : lo[4 * u + 3],
                                     (Pb & 31) >> 3);
      out[i][u] = i == 0 ? v ^ 0x80808080u : v;
    }
  }
}
// The same for 16 consecutive weights: out[i] holds bytes 0..15 of slice i's
// 32-byte record half (k order as oz_slice32).
template <int S>
EVB_DEV void oz_slice16(const double* w, double wscale, uint32_t (&out)[S][4]) {
  const double off = 0x1p52 + (double)(1ull << (8 * S - 1));
  uint32_t lo[16], hi[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const double t = __fma_rz(isfinite(w[q]) ? w[q] : 0.0, wscale, off);
    lo[q] = (uint32_t)__double2loint(t);
    hi[q] = (uint32_t)__double2hiint(t);
  }
#pragma unroll
  for (int i = 0; i < S; ++i) {
    const int Pb = 8 * (S - 1 - i);
    const bool H = Pb >= 32;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t v = gather_byte(H ? hi[4 * u] : lo[4 * u], H ? hi[4 * u + 1] : lo[4 * u + 1],
                                     H ? hi[4 * u + 2] : lo[4 * u + 2], H ? hi[4 * u + 3] : lo[4 * u + 3],
                                     (Pb & 31) >> 3);
      out[i][u] = i == 0 ? v ^ 0x80808080u : v;
    }
  }
}
// atomic max of a non-negative double (bit patterns order like the values)
EVB_DEV void smem_max_nonneg(double* p, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------------------
// Pipelined team (the default oz kernel): the 16 lanes are two groups of 8 whose
// step chains -- layer 0 -> MMA -> epilogue -> cluster exchange -> env -- run
// half a period apart, so one group's MMAs (tensor core) and env step (2 env
// warps, latency-bound fp64 transcendentals) overlap the other group's layer 0
// and epilogue (8 compute warps).  Warps: 0-7 compute, 8-9 env (group 0 / 1),
// 10 MMA issue.  Per group g: B_g (zero-padded windows of 8-lane blocks, N = 8 S),
// accumulator D_g at TMEM columns 8 S g.. (A slices shared).  Handshakes are
// mbarriers: x0full[g] (env -> compute), bfull[g] (compute -> MMA, 8 warp
// arrivals), dfull[g] (tcgen05.commit -> compute), xbar[g][parity] (st.async
// partial outputs -> env).  NetFault bookkeeping uses step stamps (no resets).
constexpr int OZP_CW = 8;                         // compute warps
constexpr int OZP_THREADS = 32 * (OZP_CW + 3);    // + 2 env warps + 1 MMA warp
constexpr int OZP_G = 8;                          // lanes per group

template <int S, int C>
__global__ void __launch_bounds__(OZP_THREADS, 1) rollout_ozp_kernel(const __grid_constant__ RolloutArgs A,
                                                                     const __grid_constant__ OzPlan P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool compute = warp < OZP_CW;
  const int quad = warp & 3, half = (warp >> 2) & 1;  // compute warps: TMEM lane quadrant, lane half
  const int crank = C > 1 ? (int)cluster_ctarank() : 0;
  const int team = blockIdx.x / C;
  const int agent_local = team / A.groups;
  const int group = team % A.groups;
  const int agent = A.agent_offset + agent_local;
  const int W1 = P.W1, W1p = P.W1p, W2 = P.W2, O = N.dims[3];
  const int r0 = crank * OZ_M;
  const int row = quad * 32 + lane;
  constexpr int RB = OZP_G * (S + 1);             // rows (N) of one B buffer: S data blocks + a spill block
  const uint32_t LBO = (uint32_t)(RB / 8) * 128;  // K-direction core-matrix stride
  const int BBYTES = RB * W1p;                    // one group's B buffer
  const uint32_t colA = (uint32_t)(OZ_TMEM_COLS - S * (W1p / 4));
  constexpr int NG = OZP_G * (S + 1);             // accumulator columns per group (D_0..D_(S-1) + spill)

#ifdef EVB_TC_PROFILE
  unsigned long long prof[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tprev = clock64();
#endif
  for (int i = tid; i < P.used / 4; i += OZP_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + P.off_tslot);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* x0full = bars;      // [2]
  uint64_t* bfull = bars + 2;   // [2]
  uint64_t* dfull = bars + 4;   // [2]
  uint64_t* xbar = bars + 6;    // [2 groups][2 parities]
  __syncthreads();
  if (warp == OZP_CW + 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(OZ_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int g = 0; g < 2; ++g) {
      mbar_init(&x0full[g], 1);
      mbar_init(&bfull[g], OZP_CW);
      mbar_init(&dfull[g], 1);
      mbar_init(&xbar[2 * g], 1);
      mbar_init(&xbar[2 * g + 1], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  double* W0 = reinterpret_cast<double*>(smem + P.off_W0);
  double* b0 = reinterpret_cast<double*>(smem + P.off_b0);
  double* mk = reinterpret_cast<double*>(smem + P.off_mk);
  double* rmax = reinterpret_cast<double*>(smem + P.off_rmax);
  // ---- prologue (compute warps): layer 0 to SMEM, layer-1 slices to TMEM
  const bool row_ok = compute && r0 + row < W2;
  auto w1 = [&](int k) -> double {
    return (row_ok && k < W1) ? oz_param(A.par, N.d, agent_local, N.w_off[1] + (long long)k * W2 + r0 + row)
                              : 0.0;
  };
  const int K0 = N.dims[0];
  if (compute) {
    for (int i = tid; i < K0 * W1; i += 32 * OZP_CW) {
      const int k = i / W1, r = i % W1;
      const double w = oz_param(A.par, N.d, agent_local, N.w_off[0] + (long long)k * W1 + r);
      W0[k * W1p + r] = w;
      smem_max_nonneg(&mk[k], fin_abs(w));
    }
    for (int r = tid; r < W1; r += 32 * OZP_CW) {
      const double b = oz_param(A.par, N.d, agent_local, N.b_off[0] + r);
      b0[r] = b;
      smem_max_nonneg(&mk[4], fin_abs(b));
    }
  }
  // pre-split blocks (materialised ask): the row's exponent and slices are
  // ready-made -- coalesced 16-byte loads, then tcgen05.st
  const unsigned char* blk =
      A.tc_blocks != nullptr ? A.tc_blocks + ((long long)agent_local * C + crank) * A.tc_block_bytes : nullptr;
  double rm = 0.0;
  bool rfin = true;
  int meta = 0;
  if (compute && blk != nullptr) {
    meta = reinterpret_cast<const int*>(blk + (size_t)S * W1p * OZ_M)[row];
    rfin = (meta >> 16) == 0;
  } else if (compute) {
    for (int c = half; c < W1p / 32; c += 2)
      for (int q = 0; q < 32; ++q) {
        const double w = w1(c * 32 + q);
        rm = fmax(rm, fin_abs(w));
        rfin = rfin && isfinite(w);
      }
    rmax[half * OZ_M + row] = rm;
  }
  const bool slow_cta = __syncthreads_or(!rfin) != 0;
  int Fr = 0;
  bool rbad = false;
  double rscale = 0.0, b1r = 0.0;
  double w2r[OZ_MAXO], b2[OZ_MAXO];
#pragma unroll
  for (int o = 0; o < OZ_MAXO; ++o) {
    w2r[o] = 0.0;
    b2[o] = (!compute && o < O) ? oz_param(A.par, N.d, agent_local, N.b_off[2] + o) : 0.0;
  }
  if (compute && blk != nullptr) {
    Fr = (int)(short)(meta & 0xFFFF);
    for (int c = half; c < W1p / 32; c += 2)
#pragma unroll
      for (int i = 0; i < S; ++i) {
        const uint4* src = reinterpret_cast<const uint4*>(blk + (((size_t)i * (W1p / 32) + c) * OZ_M + row) * 32);
        const uint4 a = __ldg(src), b = __ldg(src + 1);
        const uint32_t packed[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        oz_st8(tmem + ((uint32_t)(quad * 32) << 16) + colA + (uint32_t)(i * (W1p / 4) + c * 8), packed);
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    rbad = !rfin;
  } else if (compute) {
    rm = fmax(rmax[row], rmax[OZ_M + row]);
    Fr = 8 * S - 1 - bound_exp(rm);  // |W_int| < 2^(8S-1)
    const double wscale = ldexp(1.0, Fr);
    for (int c = half; c < W1p / 32; c += 2) {
      double w[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) w[q] = w1(c * 32 + q);
      uint32_t sl[S][8];
      oz_slice32<S>(w, wscale, sl);
#pragma unroll
      for (int i = 0; i < S; ++i)
        oz_st8(tmem + ((uint32_t)(quad * 32) << 16) + colA + (uint32_t)(i * (W1p / 4) + c * 8), sl[i]);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (slow_cta)
      for (int k = 0; k < W1; ++k) rbad = rbad || !isfinite(w1(k));
  }
  if (compute) {
    rscale = ldexp(1.0, 8 * (S - 1) - Fr);
    b1r = row_ok ? oz_param(A.par, N.d, agent_local, N.b_off[1] + r0 + row) : 0.0;
#pragma unroll
    for (int o = 0; o < OZ_MAXO; ++o)
      w2r[o] = (o < O && row_ok)
                   ? oz_param(A.par, N.d, agent_local, N.w_off[2] + (long long)(r0 + row) * O + o)
                   : 0.0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (C > 1) cluster_sync_all();

  double* x0 = reinterpret_cast<double*>(smem + P.off_x0);     // [2][4][8]
  double* red = reinterpret_cast<double*>(smem + P.off_red);   // [2][4 quadrants][O][8]
  double* pout = reinterpret_cast<double*>(smem + P.off_pout); // [2 groups][2 parities][C][(O+1) 8]
  uint32_t* flags = reinterpret_cast<uint32_t*>(smem + P.off_mask);
  uint32_t* bad0 = flags;       // [2][8] step stamps: lane's layer-0 activation infinite at step t (= t + 1)
  uint32_t* bad1 = flags + 16;  // [2][8] the same for layer 1
  uint32_t* alive = flags + 32; // [2] group has an active lane at this step
  uint32_t* gdone = flags + 34; // [2] group finished (compute -> MMA warp)
  int* gexp = reinterpret_cast<int*>(flags + 36);  // [2][8] lane exponent G of layer 0's fixed point (env -> compute)
  const int OEg = O * OZP_G, OE1g = (O + 1) * OZP_G;
  OZ_MARK(0);  // prologue

  if (warp == OZP_CW || warp == OZP_CW + 1) {
    // ================================================= env warp of group lg
    const int lg = warp - OZP_CW;
    const int l = lane;
    const int j = group * OZ_N + lg * OZP_G + l;  // lane index within the agent
    const bool valid = l < OZP_G && j < A.e;
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
      env_reset(E, fold_in(lane_key, 0), s);  // proj/src/rollout.cpp:104
    }
    const NormParams nrm = load_norm(A.norm);
    // (every loop over the obs / output dimension is unrolled to its compile-time
    // bound with a predicate, so these arrays stay in registers: a dynamic
    // index would put them in local memory on the env chain's critical path)
    double inv_den[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) inv_den[i] = nrm.active ? 1.0 / nrm.den[i] : 1.0;
    double* xg = x0 + lg * 4 * OZP_G;
    double sin_th = 0.0;
    auto observe_into_x0 = [&](bool act) {  // proj/src/rollout.cpp:124-126
      double raw[4];
      observe(E, s, raw);
      sin_th = raw[1];
      if (act && A.track_stats) {  // WelfordStats::add, proj/src/obs_norm.cpp:7-18
        if (wc == 0.0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= E.obs_dim) break;
            wmean[i] = raw[i];
            wm2[i] = 0.0;
          }
          wc = 1.0;
        } else {
          wc = dadd(wc, 1.0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i >= E.obs_dim) break;
            const double delta = dsub(raw[i], wmean[i]);
            wmean[i] = dadd(wmean[i], ddiv(delta, wc));
            wm2[i] = dadd(wm2[i], dmul(delta, dsub(raw[i], wmean[i])));
          }
        }
      }
      // (o - mean) * (1 / den): within an ulp of the fp64 team's IEEE division,
      // far below this team's ~1e-13 policy tolerance, and off the divide latency
      double bnd = mk[4];  // the lane's fixed-point exponent G for layer 0's output:
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // bound = max|b0| + sum_k max|W0[.][k]| |x_k|
        if (i >= E.obs_dim) break;
        double v = raw[i];
        if (nrm.active) v = dmul(dsub(v, nrm.mean[i]), inv_den[i]);
        v = act ? v : 0.0;
        bnd = fma(mk[i], fabs(v), bnd);
        if (l < OZP_G) xg[i * OZP_G + l] = v;
      }
      bnd = bnd * (1.0 + 0x1.0p-40);  // covers the rounding of layer 0's fma chains
      if (l < OZP_G) gexp[lg * OZP_G + l] = 8 * S - 1 - bound_exp_bits(bnd);
    };
    bool act = valid && eps_this > 0 && A.max_iters > 0;
    if (act) observe_into_x0(true);
    for (int it = 0;; ++it) {
      const bool any = __any_sync(0xffffffffu, act);
      __syncwarp();  // every lane's x0 stores before lane 0's (release) arrival
      if (lane == 0) {
        alive[lg] = any ? 1u : 0u;
        mbar_arrive_local(&x0full[lg]);  // x0 (and the alive flag) of step it
      }
      if (!any) break;
      // the action-independent part of the reward, while this step's layers run
      double rpre = 0.0;
      if (act && E.id == ENV_PENDULUM) rpre = pendulum_reward_pre(s);
      uint64_t* xb = &xbar[2 * lg + (it & 1)];
      if (C > 1 && lane == 0) mbar_arrive_expect_tx(xb, (uint32_t)(C * OE1g * sizeof(double)));
      OZ_MARK(7);  // env warp: own work (reward pre-term, arming)
      if constexpr (C > 1) {
        mbar_wait_parity(xb, (uint32_t)((it >> 1) & 1));
      } else {
        mbar_wait_parity_cta(xb, (uint32_t)((it >> 1) & 1));
      }
      OZ_MARK(6);  // env warp: waiting for the partial outputs
      const double* pg = pout + (size_t)(lg * 2 + (it & 1)) * C * OE1g;
      if (act) {
        double z[OZ_MAXO];
        bool nonfinite_out = false;
        int bad_layer = 3;
        for (int c = 0; c < C; ++c) bad_layer = min(bad_layer, (int)pg[c * OE1g + OEg + l]);
#pragma unroll
        for (int o = 0; o < OZ_MAXO; ++o) {
          if (o >= O) break;
          double v = pg[o * OZP_G + l];
#pragma unroll
          for (int c = 1; c < C; ++c) v += pg[c * OE1g + o * OZP_G + l];
          v = v + b2[o];
          z[o] = v;
          if (!isfinite(v)) nonfinite_out = true;
        }
        if (bad_layer == 3 && nonfinite_out) bad_layer = 2;
        if (bad_layer < 3) {  // NetFault: the lowest layer with a non-finite activation
          myfault = FAULT_NET;
          myfault_layer = (uint32_t)bad_layer;
        } else {
          double action;
          if (N.head == HEAD_CATEGORICAL) {
            int arg = 0;
            double best = z[0];
#pragma unroll
            for (int o = 1; o < OZ_MAXO; ++o)
              if (o < O && z[o] > best) {  // maxCoeff: first maximum
                best = z[o];
                arg = o;
              }
            action = (double)arg;
          } else if (N.head == HEAD_TANH) {
            action = N.tanh_scale * tanh(z[0]);
          } else {
            action = z[0];
          }
          double reward = 0.0;
          bool term = false, trunc = false;
          OZ_MARK(11);  // env warp: head (output sum + tanh)
          const uint32_t f = env_step(E, s, action, reward, term, trunc, E.id == ENV_PENDULUM ? &sin_th : nullptr,
                                      E.id == ENV_PENDULUM ? &rpre : nullptr);
          OZ_MARK(12);  // env warp: env_step
          if (f) {
            myfault = f;
          } else {
            ep_ret = dadd(ep_ret, reward);  // proj/src/rollout.cpp:143
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
              if (eps_done < eps_this) env_reset(E, s.rng, s);  // auto-reset, env.cpp:163-167
            }
          }
        }
        const bool next = myfault == 0 && eps_done < eps_this && it + 1 < A.max_iters;
        OZ_MARK(13);  // env warp: bookkeeping
        observe_into_x0(next);
        act = next;
      }
      __syncwarp();
      OZ_MARK(14);  // env warp: observe
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
  } else if (warp == OZP_CW + 2) {
    // ================================================= MMA issue warp
    uint32_t live = 3u;  // bit g: group g still running (a mask, not an array: registers)
    const uint32_t bS = smem_u32(smem + P.off_B);
    for (int it = 0; live != 0u; ++it) {
      for (int g = 0; g < 2; ++g) {
        if (!((live >> g) & 1u)) continue;
        OZ_MARK(10);  // MMA warp: issue
        mbar_wait_parity_cta(&bfull[g], (uint32_t)(it & 1));
        __syncwarp();  // reconverge after the spin loop (elect.sync / tcgen05 below)
        OZ_MARK(9);  // MMA warp: waiting for B
        if (gdone[g]) {
          live &= ~(1u << g);
          continue;
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // one elected lane issues the whole group-step: descriptors advance by
        // constant strides (the B start address field by 2 LBO >> 4 per k-step,
        // the A TMEM column by 8), so each MMA is an add or two plus the issue
        if (elect_one()) {
          const uint64_t bd0 = oz_desc(bS + (uint32_t)(g * BBYTES), LBO, 128);
          const uint32_t dg = tmem + (uint32_t)(g * NG);
          const uint32_t aS = (uint32_t)(W1p / 4);
          const int KS = W1p / 32;
          for (int ks = 0; ks < KS; ++ks) {
            const uint64_t bd = bd0 + (uint64_t)((uint32_t)ks * ((2 * LBO) >> 4));
            const uint32_t a0 = tmem + colA + (uint32_t)ks * 8;
#pragma unroll
            for (int i = 0; i < S; ++i)  // D blocks i .. += A_i [B_0 B_1 ..]; N = 8 (S - i) rounded up to 16
              oz_mma_ts(dg + (uint32_t)(OZP_G * i), a0 + (uint32_t)i * aS, bd,
                        oz_idesc(OZ_M, (OZP_G * (S - i) + 15) / 16 * 16, i == 0), (ks | i) != 0);
          }
          oz_commit(&dfull[g]);
        }
        __syncwarp();
      }
    }
  } else {
    // ================================================= compute warps (0-7)
    uint32_t live = 3u;  // bit g: group g still running (a mask, not an array: registers)
    // layer-0 thread map: lane le of the group, 8 consecutive k rows (half a
    // 16-byte K row of a B core matrix)
    const int le = tid & 7, rg = tid >> 3;  // rg: 32 row groups of 8
    const bool l0_active = rg * 8 < W1p;
    for (int it = 0; live != 0u; ++it) {
      for (int g = 0; g < 2; ++g) {
        if (!((live >> g) & 1u)) continue;
        OZ_MARK(5);  // compute: publish (+ named barrier) / group switch
        mbar_wait_parity_cta(&x0full[g], (uint32_t)(it & 1));
        __syncwarp();
        OZ_MARK(1);  // compute: waiting for x0
        if (!alive[g]) {
          live &= ~(1u << g);
          if (tid == 0) gdone[g] = 1u;
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&bfull[g]);
          continue;
        }
        // ---- layer 0 of group g (fp64) -> fixed point -> S bytes -> B_g
        {
          const double* xg = x0 + g * 4 * OZP_G;
          if (l0_active) {
            double xr[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) xr[k] = xg[k * OZP_G + le];
            const double hscale = pow2(gexp[g * OZP_G + le]);  // 2^G, G from the env warp
            // z = W0 x + b0 as one fma chain from the bias (k = 0..3; W0 and x
            // are zero past obs_dim)
            double z[8];
            const double* __restrict__ w0r = W0 + rg * 8;
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
              const double2 b = *reinterpret_cast<const double2*>(b0 + rg * 8 + u);
              z[u] = b.x;
              z[u + 1] = b.y;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
#pragma unroll
              for (int u = 0; u < 8; u += 2) {
                const double2 w = *reinterpret_cast<const double2*>(w0r + k * W1p + u);
                z[u] = fma(w.x, xr[k], z[u]);
                z[u + 1] = fma(w.y, xr[k], z[u + 1]);
              }
            }
            uint32_t qlo[8], qhi[8], hor = 0u;
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const double h = fmax(z[u + v], 0.0);  // ReLU (NaN -> 0, as cwiseMax)
                const double t = fma(h, hscale, 0x1p52);
                qlo[u + v] = (uint32_t)__double2loint(t);
                qhi[u + v] = (uint32_t)__double2hiint(t);
                hor |= qhi[u + v];
              }
            }
            if ((hor & 0x7FF00000u) != 0x43300000u) bad0[g * OZP_G + le] = (uint32_t)it + 1u;  // h = +inf
            unsigned char* Bme = smem + P.off_B + g * BBYTES + (size_t)(rg >> 1) * LBO + le * 16 + (rg & 1) * 8;
#pragma unroll
            for (int jj = 0; jj < S; ++jj) {
              const int Pb = 8 * (S - 1 - jj);
              const bool H = Pb >= 32;
              uint32_t wv[2];
#pragma unroll
              for (int w = 0; w < 2; ++w)
                wv[w] = gather_byte(H ? qhi[4 * w] : qlo[4 * w], H ? qhi[4 * w + 1] : qlo[4 * w + 1],
                                    H ? qhi[4 * w + 2] : qlo[4 * w + 2], H ? qhi[4 * w + 3] : qlo[4 * w + 3],
                                    (Pb & 31) >> 3);
              *reinterpret_cast<uint2*>(Bme + (size_t)jj * 128) = make_uint2(wv[0], wv[1]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B_g visible to the tensor core
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive_local(&bfull[g]);
        }
        // ---- epilogue of group g: row `row`, lanes 4 half .. 4 half + 3
        OZ_MARK(2);  // compute: layer 0
        mbar_wait_parity_cta(&dfull[g], (uint32_t)(it & 1));
        __syncwarp();  // reconverge after the spin loop: tcgen05.ld below is .sync.aligned
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        OZ_MARK(3);  // compute: waiting for the MMAs
        {
          uint32_t d[S][4];
          const uint32_t tl = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(g * NG + half * 4);
#pragma unroll
          for (int t = 0; t < S; ++t) oz_ld4(tl + (uint32_t)(t * OZP_G), d[t]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          // each lane's scale 2^-G, recomputed from x0 exactly as layer 0 did
          // (no cross-thread handoff between the layer-0 and epilogue threads)
          double h[4], sq[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) sq[q] = rscale * pow2(-gexp[g * OZP_G + half * 4 + q]);  // 2^(8(S-1) - F_r - G)
          long long hi[4], lo[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) hi[q] = lo[q] = 0;
#pragma unroll
          for (int t = 0; t < S; ++t)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const long long v = (long long)(int)d[t][q];
              if (t < S - 3) {
                hi[q] = hi[q] * 256 + v;
              } else {
                lo[q] = lo[q] * 256 + v;
              }
            }
#pragma unroll
          for (int q = 0; q < 4; ++q) h[q] = fma(i51_to_double(hi[q]), 16777216.0, i51_to_double(lo[q])) * sq[q];
          if (rbad) {  // non-finite weight in this row: fp64 dot product, layer 0 recomputed
            const double* xg = x0 + g * 4 * OZP_G;
            for (int q = 0; q < 4; ++q) {
              const int e = half * 4 + q;
              double z = 0.0;
              for (int k = 0; k < W1; ++k) {
                double a = b0[k];
                for (int kk = 0; kk < 4; ++kk) a = fma(W0[kk * W1p + k], xg[kk * OZP_G + e], a);
                z = fma(w1(k), fmax(a, 0.0), z);
              }
              h[q] = z;
            }
          }
          uint32_t bad = 0u;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double zz = h[q] + b1r;
            h[q] = zz > 0.0 ? zz : 0.0;  // ReLU (NaN -> 0, as cwiseMax)
            if (h[q] == INFINITY) bad |= 1u << (half * 4 + q);
          }
          if (__any_sync(0xffffffffu, bad != 0u)) {  // (rare: an infinite layer-1 activation)
            bad = __reduce_or_sync(0xffffffffu, bad);
            if (lane < OZP_G && ((bad >> lane) & 1u)) bad1[g * OZP_G + lane] = (uint32_t)it + 1u;
          }
          // output layer: v[q] = w2[row][o] h[q] summed over the warp's 32 rows by a
          // reduce-scatter (lane bits 4, 3 select the lane q it ends on)
          const int b4 = (lane >> 4) & 1, b3 = (lane >> 3) & 1;
#pragma unroll
          for (int o = 0; o < OZ_MAXO; ++o) {
            if (o >= O) break;
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = w2r[o] * h[q];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const double send = b4 ? v[i] : v[i + 2];
              const double keep = b4 ? v[i + 2] : v[i];
              v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
            {
              const double send = b3 ? v[0] : v[1];
              const double keep = b3 ? v[1] : v[0];
              v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 4);
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            if ((lane & 7) == 0) red[((g * 4 + quad) * O + o) * OZP_G + half * 4 + b4 * 2 + b3] = v[0];
          }
        }
        OZ_MARK(4);  // compute: epilogue
        named_sync_n(1, 32 * OZP_CW);  // red / stamps of group g complete
        // partial outputs (fixed quadrant order) + each lane's first non-finite
        // layer -> every CTA of the cluster
        if (tid < OE1g) {
          const int oe = tid;
          const double* rg4 = red + g * 4 * OEg;
          double v;
          if (oe < OEg) {
            v = ((rg4[oe] + rg4[OEg + oe]) + rg4[2 * OEg + oe]) + rg4[3 * OEg + oe];
          } else {
            const int e = oe - OEg;
            int bl = 3;
            if (bad1[g * OZP_G + e] == (uint32_t)it + 1u) bl = 1;
            if (bad0[g * OZP_G + e] == (uint32_t)it + 1u) bl = 0;
            v = (double)bl;
          }
          double* pg = pout + (size_t)(g * 2 + (it & 1)) * C * OE1g;
          if constexpr (C > 1) {
            const uint32_t la = smem_u32(pg + crank * OE1g + oe), lb = smem_u32(&xbar[2 * g + (it & 1)]);
#pragma unroll
            for (int c = 0; c < C; ++c) st_async(map_cluster(la, (uint32_t)c), v, map_cluster(lb, (uint32_t)c));
          } else {
            pg[oe] = v;
          }
        }
        if constexpr (C == 1) {
          named_sync_n(1, 32 * OZP_CW);
          if (tid == 0) mbar_arrive_local(&xbar[2 * g + (it & 1)]);
        }
      }
    }
  }
#ifdef EVB_TC_PROFILE
  if (tid == 0) {
    for (int i = 0; i < 6; ++i) atomicAdd(&g_oz_prof[i], prof[i]);
    atomicAdd(&g_oz_prof[8], 1ull);
  }
  if (tid == 32 * OZP_CW) {
    atomicAdd(&g_oz_prof[6], prof[6]);
    atomicAdd(&g_oz_prof[7], prof[7]);
    for (int i = 11; i < 15; ++i) atomicAdd(&g_oz_prof[i], prof[i]);
  }
  if (tid == 32 * (OZP_CW + 2)) {
    atomicAdd(&g_oz_prof[9], prof[9]);
    atomicAdd(&g_oz_prof[10], prof[10]);
  }
#endif
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == OZP_CW + 2) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(OZ_TMEM_COLS));
  }
  if constexpr (C > 1) cluster_sync_all();
}


// ---------------------------------------------------------------------------
// Pre-split layer-1 weights (materialised ask): one parallel pass over every
// (agent, CTA, row) computes the row's fixed-point exponent and its S byte
// slices in the layout the team's prologue stores to TMEM, so the prologue is
// a coalesced 16-byte-load + tcgen05.st loop instead of 2 x 256 parameter
// fetches and int64 slicing per row.  Block of one (agent, CTA):
//   [S][W1p/32][128 rows][8 words] slice bytes (word u = k 4u..4u+3 of the
//   32-wide chunk, low byte first), then [128] int32 meta = (F_r & 0xFFFF) |
//   (row holds a non-finite weight) << 16.
long long oz_block_bytes(const TcPlanOut& po) {
  OzPlan p;
  std::memcpy(&p, &po, sizeof p);
  return (long long)p.S * p.W1p * OZ_M + OZ_M * 4;
}

template <int S>
__global__ void k_oz_split(const double* __restrict__ cand, long long d, long long w_off1, int W1, int W2, int W1p,
                           int C, long long total, unsigned char* __restrict__ blocks, long long block_bytes) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int row = (int)(idx % OZ_M);
  const long long ac = idx / OZ_M;  // agent * C + crank
  const int crank = (int)(ac % C);
  const long long agent = ac / C;
  const int r = crank * OZ_M + row;
  const double* wr = cand + agent * d + w_off1 + r;  // weight (r, k) at wr[k * W2]
  const bool ok = r < W2;
  double rm = 0.0;
  bool fin = true;
  for (int k = 0; k < W1 && ok; ++k) {
    const double w = wr[(long long)k * W2];
    rm = fmax(rm, fin_abs(w));
    fin = fin && isfinite(w);
  }
  const int Fr = 8 * S - 1 - bound_exp(rm);
  const double wscale = ldexp(1.0, Fr);
  unsigned char* blk = blocks + ac * block_bytes;
  for (int c = 0; c < W1p / 32; ++c) {
    double w[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int k = c * 32 + q;
      w[q] = (ok && k < W1) ? wr[(long long)k * W2] : 0.0;
    }
    uint32_t sl[S][8];
    oz_slice32<S>(w, wscale, sl);
#pragma unroll
    for (int i = 0; i < S; ++i) {
      uint4* dst = reinterpret_cast<uint4*>(blk + (((size_t)i * (W1p / 32) + c) * OZ_M + row) * 32);
      dst[0] = make_uint4(sl[i][0], sl[i][1], sl[i][2], sl[i][3]);
      dst[1] = make_uint4(sl[i][4], sl[i][5], sl[i][6], sl[i][7]);
    }
  }
  reinterpret_cast<int*>(blk + (size_t)S * W1p * OZ_M)[row] = (Fr & 0xFFFF) | ((ok && !fin) ? (1 << 16) : 0);
}

// The OpenES ask fused with the pre-split, from kept noise rows: a block owns
// noise row nr, one CTA's 16-row tile of layer 1, and both agents using the row
// (nr, and nr + base negated when mirrored).  Thread group h holds the k-range
// [16h, 16h + 16) of every row of the tile: the noise and the mean are read
// once, each agent's weights w = sigma (+-eps) + mean are formed in registers
// (the ask's arithmetic), and the row maximum, exponent and byte slices follow
// as in k_oz_split -- no fp64 layer-1 candidate matrix is written or re-read.
// Rows holding a non-finite weight (a diverged mean) also get their fp64
// values in the candidate matrix: only those are read back by the team.
constexpr int OZ_AS_ROWS = 16;  // rows per block: 16 x 16 half-chunks = 256 threads, two blocks per SM
template <int S>
__global__ void __launch_bounds__(256, 2) k_oz_ask_split(const ParamDesc P, long long d, long long w_off1, int W1,
                                                      int W2, int W1p, int C, int a0, int a1, long long r0,
                                                      const double* __restrict__ eps, double* __restrict__ cand,
                                                      unsigned char* __restrict__ blocks, long long block_bytes) {
  __shared__ double smax[16][OZ_AS_ROWS];
  __shared__ int sfin[16][OZ_AS_ROWS];
  constexpr int TPB = OZ_M / OZ_AS_ROWS;
  const int lane = threadIdx.x % OZ_AS_ROWS, h = threadIdx.x / OZ_AS_ROWS;
  const int tile = (int)(blockIdx.x % TPB);
  const long long rc = blockIdx.x / TPB;
  const int crank = (int)(rc % C);
  const long long nr = r0 + rc / C;  // noise row
  const int row = tile * OZ_AS_ROWS + lane, r = crank * OZ_M + row;
  const bool ok = r < W2;
  const int nh = W1p / 16;  // k half-chunks in use
  double e[16];  // the mean is re-read per side (L1): fewer registers, more resident blocks
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int k = h * 16 + q;
    const bool v = h < nh && ok && k < W1;
    e[q] = v ? eps[nr * d + w_off1 + (long long)k * W2 + r] : 0.0;
  }
  for (int side = 0; side < 2; ++side) {
    const long long a = side == 0 ? nr : (P.mirrored ? nr + P.base : -1);
    if (a < a0 || a >= a1) continue;  // uniform over the block
    double w[16];
    double rm = 0.0;
    bool fin = true;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int k = h * 16 + q;
      const bool v = h < nh && ok && k < W1;
      w[q] = v ? dadd(dmul(P.sigma, side ? -e[q] : e[q]), P.mean[w_off1 + (long long)k * W2 + r])
               : 0.0;  // (sigma * eps) + mean
      rm = fmax(rm, fin_abs(w[q]));
      fin = fin && isfinite(w[q]);
    }
    __syncthreads();  // the previous side's reduction was read
    smax[h][lane] = rm;
    sfin[h][lane] = fin ? 1 : 0;
    __syncthreads();
    for (int j = 0; j < nh; ++j) {
      rm = fmax(rm, smax[j][lane]);
      fin = fin && sfin[j][lane] != 0;
    }
    const int Fr = 8 * S - 1 - bound_exp(rm);
    unsigned char* blk = blocks + ((a - a0) * C + crank) * block_bytes;
    if (h < nh) {
      uint32_t sl[S][4];
      oz_slice16<S>(w, ldexp(1.0, Fr), sl);
#pragma unroll
      for (int i = 0; i < S; ++i)
        *reinterpret_cast<uint4*>(blk + (((size_t)i * (W1p / 32) + (h >> 1)) * OZ_M + row) * 32 + (h & 1) * 16) =
            make_uint4(sl[i][0], sl[i][1], sl[i][2], sl[i][3]);
      if (!fin && ok) {  // the team computes this row in fp64 from the candidate matrix
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int k = h * 16 + q;
          if (k < W1) cand[(a - a0) * d + w_off1 + (long long)k * W2 + r] = w[q];
        }
      }
    }
    if (h == 0)
      reinterpret_cast<int*>(blk + (size_t)S * W1p * OZ_M)[row] = (Fr & 0xFFFF) | ((ok && !fin) ? (1 << 16) : 0);
  }
}

// The other parameters (outside layer 1) of agents [a0, a1) from the kept
// noise rows, as k_cand_from_eps.
__global__ void k_oz_ask_rest(const ParamDesc P, long long d, long long w_off1, long long n_w1, int a0, int a1,
                              long long r0, long long rows, const double* __restrict__ eps, double* __restrict__ cand) {
  const long long rest = d - n_w1;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= rows * rest) return;
  const long long nr = r0 + i / rest, j = i % rest;
  const long long p = j < w_off1 ? j : j + n_w1;
  const double e = eps[nr * d + p], mp = P.mean[p];
  for (int side = 0; side < 2; ++side) {
    const long long a = side == 0 ? nr : (P.mirrored ? nr + P.base : -1);
    if (a < a0 || a >= a1) continue;
    cand[(a - a0) * d + p] = dadd(dmul(P.sigma, side ? -e : e), mp);
  }
}

cudaError_t run_oz_ask_split(const ParamDesc& par, const NetDesc& net, const TcPlanOut& po, int a0, int a1,
                             const double* eps, long long eps_row0, double* cand, unsigned char* blocks,
                             cudaStream_t stream) {
  OzPlan p;
  std::memcpy(&p, &po, sizeof p);
  if (par.src != SRC_OPENES || p.W1p > 256 || p.W1p % 16) return cudaErrorInvalidValue;
  if (a1 <= a0) return cudaSuccess;
  // noise rows the agents use (agent a < base: row a; a >= base: row a - base)
  long long r0 = a0, r1 = a1;
  if (par.mirrored) {
    const long long base = par.base;
    r0 = LLONG_MAX;
    r1 = LLONG_MIN;
    if (a0 < base) {
      r0 = std::min<long long>(r0, a0);
      r1 = std::max<long long>(r1, std::min<long long>(a1, base));
    }
    if (a1 > base) {
      r0 = std::min<long long>(r0, std::max<long long>(a0, base) - base);
      r1 = std::max<long long>(r1, a1 - base);
    }
  }
  if (r0 < eps_row0) return cudaErrorInvalidValue;
  const long long rows = r1 - r0;
  // the kernels index eps by the global row: address of (virtual) row 0
  // (integer arithmetic: only rows >= eps_row0 are ever read)
  eps = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(eps) -
                                        (uintptr_t)(eps_row0 * net.d) * sizeof(double));
  const long long n_w1 = (long long)p.W1 * p.W2;
  const long long bb = oz_block_bytes(po);
  k_oz_ask_rest<<<(unsigned)((rows * (net.d - n_w1) + 255) / 256), 256, 0, stream>>>(
      par, net.d, net.w_off[1], n_w1, a0, a1, r0, rows, eps, cand);
  const unsigned grid = (unsigned)(rows * p.C * (OZ_M / OZ_AS_ROWS));
#ifdef EVB_OZ_S5
  if (p.S == 5) {
    k_oz_ask_split<5><<<grid, 16 * OZ_AS_ROWS, 0, stream>>>(par, net.d, net.w_off[1], p.W1, p.W2, p.W1p, p.C, a0,
                                                            a1, r0, eps, cand, blocks, bb);
    return cudaGetLastError();
  }
#endif
  k_oz_ask_split<6><<<grid, 16 * OZ_AS_ROWS, 0, stream>>>(par, net.d, net.w_off[1], p.W1, p.W2, p.W1p, p.C, a0,
                                                          a1, r0, eps, cand, blocks, bb);
  return cudaGetLastError();
}

cudaError_t run_oz_split(const double* cand, const NetDesc& net, const TcPlanOut& po, int n_agents,
                         unsigned char* blocks, cudaStream_t stream) {
  OzPlan p;
  std::memcpy(&p, &po, sizeof p);
  const long long total = (long long)n_agents * p.C * OZ_M;
  if (total <= 0) return cudaSuccess;
  const long long bb = oz_block_bytes(po);
  const unsigned grid = (unsigned)((total + 127) / 128);
#ifdef EVB_OZ_S5
  if (p.S == 5) {
    k_oz_split<5><<<grid, 128, 0, stream>>>(cand, net.d, net.w_off[1], p.W1, p.W2, p.W1p, p.C, total, blocks, bb);
    return cudaGetLastError();
  }
#endif
  k_oz_split<6><<<grid, 128, 0, stream>>>(cand, net.d, net.w_off[1], p.W1, p.W2, p.W1p, p.C, total, blocks, bb);
  return cudaGetLastError();
}

static int al(int x, int a) { return (x + a - 1) / a * a; }

// S = 6 byte slices; a build with -DEVB_OZ_S5 also has S = 5 instances,
// selected by EVORL_OZ_SLICES=5 (measurements: ~1e-9 instead of ~1e-13 relative
// policy error, 40 instead of 48 MMAs per step)
static int oz_slices() {
#ifdef EVB_OZ_S5
  const char* v = getenv("EVORL_OZ_SLICES");
  if (v && v[0] == '5') return 5;
#endif
  return 6;
}

bool plan_rollout_oz(const NetDesc& net, int obs_dim, int e, TcPlanOut* out) {
  if (net.nlayers != 3 || obs_dim > 4 || e < 5) return false;  // 16-lane teams, obs -> W1 -> W2 -> O
  const int W1 = net.dims[1], W2 = net.dims[2], O = net.dims[3];
  if (net.dims[0] > 4 || O > OZ_MAXO) return false;
  const int S = oz_slices();
  const int W1p = (W1 + 31) / 32 * 32;
  if (S * (W1p / 4) + 2 * OZP_G * (S + 1) > OZ_TMEM_COLS) return false;  // A slices + 2 accumulators in TMEM
  int C = 1;
  while (C * OZ_M < W2) C *= 2;
  if (C > 8) return false;
  OzPlan p{};
  p.C = C;
  p.S = S;
  p.W1 = W1;
  p.W1p = W1p;
  p.W2 = W2;
  int off = 0;
  // rollout_ozp_kernel layout: per-group B buffers, x0, red, pout
  p.off_B = off;
  off = al(off + 2 * OZP_G * (S + 1) * W1p, 1024);
  p.off_W0 = off;
  off = al(off + 4 * W1p * 8, 16);
  p.off_b0 = off;
  off = al(off + W1p * 8, 16);
  p.off_mk = off;
  off = al(off + 5 * 8, 16);
  p.off_x0 = off;
  off = al(off + 2 * 4 * OZP_G * 8, 16);
  p.off_red = off;
  off = al(off + 2 * 4 * O * OZP_G * 8, 16);
  p.off_pout = off;
  off = al(off + 2 * 2 * C * (O + 1) * OZP_G * 8, 16);
  p.off_mask = off;
  off = al(off + 52 * 4, 16);  // stamps bad0[2][8], bad1[2][8], alive[2], gdone[2], gexp[2][8]
  p.off_bar = off;
  off = al(off + 8 * 10, 16);  // x0full[2], bfull[2], dfull[2], xbar[2][2]
  p.off_tslot = off;
  off = al(off + 16, 16);
  p.off_rmax = off;
  off = al(off + 2 * OZ_M * 8, 16);
  p.used = off;
  p.bytes = std::max(off, OZ_MIN_SMEM);
  if (p.bytes > 227 * 1024) return false;

  static_assert(sizeof(OzPlan) <= sizeof(TcPlanOut), "plan storage");
  std::memcpy(out, &p, sizeof p);
  return true;
}

template <int S, int C>
static cudaError_t launch_oz_c(const RolloutArgs& a, const OzPlan& p, cudaStream_t stream) {
  auto kern = rollout_ozp_kernel<S, C>;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.n_agents * a.groups * C));
  cfg.blockDim = dim3(OZP_THREADS);
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

template <int S>
static cudaError_t launch_oz_s(const RolloutArgs& a, const OzPlan& p, cudaStream_t stream) {
  switch (p.C) {
    case 1: return launch_oz_c<S, 1>(a, p, stream);
    case 2: return launch_oz_c<S, 2>(a, p, stream);
    case 4: return launch_oz_c<S, 4>(a, p, stream);
    case 8: return launch_oz_c<S, 8>(a, p, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_rollout_oz(const RolloutArgs& a, const TcPlanOut& po, cudaStream_t stream) {
  if (a.n_agents <= 0) return cudaSuccess;
  if (a.par.src != SRC_EXPLICIT) return cudaErrorInvalidValue;  // oz teams read materialised candidates
  OzPlan p;
  std::memcpy(&p, &po, sizeof p);
#ifdef EVB_OZ_S5
  if (p.S == 5) return launch_oz_s<5>(a, p, stream);
#endif
  return p.S == 6 ? launch_oz_s<6>(a, p, stream) : cudaErrorInvalidValue;
}

#ifdef EVB_TC_PROFILE
extern "C" int evorl_debug_oz_profile(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, g_oz_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 6;
  static const unsigned long long zero[16] = {};
  return cudaMemcpyToSymbol(g_oz_prof, zero, sizeof zero) == cudaSuccess ? 0 : 6;
}
#endif

}  // namespace evorl_b200
