// rollout.cu -- the fused population rollout.
//
// Replaces, for every lane of the m x e grid, the reference's per-lane loop
// (proj/src/rollout.cpp:94-174: normalize -> forward -> draw_action ->
// batched_step -> return accumulation) and the lane scheduling of
// batched_rollout (proj/src/rollout.cpp:176-214).
//
// Design (B200):
//  * One TEAM per (agent, group of ET lanes).  A team is a thread-block
//    cluster of C CTAs; CTA c owns a row slice of every hidden layer.  The
//    agent's weights are materialised ONCE into shared memory (regenerated
//    from the ask key for OpenES/ARS/CEM -- the perturbation is never stored
//    in HBM) and stay resident for the whole horizon.
//  * Per env-step each CTA computes its slice of a hidden layer for all ET
//    lanes as a small register-tiled GEMM (TR rows x ET lanes per thread,
//    k-split across warps), then scatters the slice to every CTA of the
//    cluster through DSMEM (st.shared::cluster) and cluster-barriers.  The
//    output layer is reduced across the cluster in a fixed order, so every
//    CTA holds bit-identical actions and steps the (replicated, fp64) env
//    state identically -- no broadcast is needed and control flow stays
//    uniform across the cluster.
//  * Env dynamics, returns and RunningStats are fp64 in the reference's
//    operation order (env.cuh).  The policy GEMM runs in T = double (parity
//    mode) or float (throughput mode).
#include <algorithm>
#include <climits>
#include <type_traits>
#include <cstdio>

#include "rollout.cuh"

namespace evorl_b200 {

#ifdef EVB_TC_PROFILE
// Phase cycle counters of the cluster team (profiling build only)
__device__ unsigned long long g_rk_prof[16];
#define RK_MARK(i)                                \
  do {                                            \
    const long long t_ = clock64();               \
    rk_prof[i] += (unsigned long long)(t_ - rk_prev); \
    rk_prev = t_;                                 \
  } while (0)
#else
#define RK_MARK(i) \
  do {             \
  } while (0)
#endif

template <typename T>
EVB_DEV T to_T(double v);
template <>
EVB_DEV double to_T<double>(double v) {
  return v;
}
template <>
EVB_DEV float to_T<float>(double v) {
  return __double2float_rn(v);
}

// candidate row base for the global-weights plan (materialised ask)
template <typename T>
EVB_DEV const T* gparams(const ParamDesc& P);
template <>
EVB_DEV const double* gparams<double>(const ParamDesc& P) {
  return P.params;
}
template <>
EVB_DEV const float* gparams<float>(const ParamDesc& P) {
  return P.params_f32;
}


__global__ void k_materialize(const ParamDesc P, long long d, int a0, int a1, double* out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)(a1 - a0) * d;
  if (idx >= n) return;
  const int al = (int)(idx / d);
  out[idx] = param_value(P, d, al, a0 + al, idx % d);
}
__global__ void k_materialize_f32(const ParamDesc P, long long d, int a0, int a1, float* out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)(a1 - a0) * d;
  if (idx >= n) return;
  const int al = (int)(idx / d);
  out[idx] = __double2float_rn(param_value(P, d, al, a0 + al, idx % d));
}

// OpenES (proj/src/ec.cpp:87-94): noise entry t = row * d + p of the sampled
// rows [r0, r1) is normal #t of the ask stream, i.e. the cos (t even) or sin
// (t odd) half of Box-Muller block t >> 1; thread b computes block b once and
// writes both entries to every agent using them (row, and row + base when
// mirrored, negated) -- the same value param_value regenerates.
// eps_out (optional): the noise entries themselves, eps_out[t], kept for the
// tell of the same generation (run_openes_tell reads them instead of
// regenerating the Box-Muller pairs).
template <typename T>
__global__ void k_materialize_openes(const ParamDesc P, long long d, int a0, int a1, long long t0, long long t1,
                                     T* out, double* eps_out, long long e0) {
  const long long b = (t0 >> 1) + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (2 * b >= t1) return;
  double c, sn;
  normal_pair(P.ask_key, (uint64_t)b, c, sn);
  // (row, p) of entry 2b, one division per pair (32-bit when the stream
  // indices fit: a 64-bit division is a long software sequence)
  long long row2b, p2b;
  if (t1 <= 0xFFFFFFFFll && d <= 0xFFFFFFFFll) {
    const uint32_t q = (uint32_t)(2 * b) / (uint32_t)d;
    row2b = q;
    p2b = 2 * b - (long long)q * d;
  } else {
    row2b = (2 * b) / d;
    p2b = 2 * b - row2b * d;
  }
  if (eps_out) {  // entry t at eps_out[t - e0] (the buffer's first row need not be row 0)
    if (2 * b >= t0) eps_out[2 * b - e0] = c;
    if (2 * b + 1 < t1) eps_out[2 * b + 1 - e0] = sn;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const long long t = 2 * b + h;
    if (t < t0 || t >= t1) continue;
    long long row = row2b, p = p2b + h;
    if (p == d) {  // entry 2b + 1 starts the next row
      row += 1;
      p = 0;
    }
    const double eps = h ? sn : c;
    const int ag[2] = {(int)row, P.mirrored ? (int)row + P.base : -1};
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int a = ag[m];
      if (a < a0 || a >= a1) continue;
      const double v = dadd(dmul(P.sigma, m ? -eps : eps), P.mean[p]);
      if constexpr (sizeof(T) == 4) {
        out[(long long)(a - a0) * d + p] = __double2float_rn(v);
      } else {
        out[(long long)(a - a0) * d + p] = v;
      }
    }
  }
}

// sampled noise rows [r0, r1) used by agents [a0, a1) (OpenES: agent a < base
// uses row a, a >= base row a - base when mirrored)
static void openes_rows(const ParamDesc& par, int a0, int a1, long long& r0, long long& r1) {
  r0 = a0;
  r1 = a1;
  if (!par.mirrored) return;
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

template <typename T>
static cudaError_t materialize(const ParamDesc& par, long long d, int a0, int a1, T* out, cudaStream_t stream,
                               double* eps_out = nullptr, long long eps_row0 = 0) {
  const long long n = (long long)(a1 - a0) * d;
  if (n <= 0) return cudaSuccess;
  if (par.src == SRC_OPENES) {
    long long r0, r1;
    openes_rows(par, a0, a1, r0, r1);
    const long long t0 = r0 * d, t1 = r1 * d;
    const long long blocks = ((t1 + 1) >> 1) - (t0 >> 1);
    if (eps_out && r0 < eps_row0) return cudaErrorInvalidValue;
    k_materialize_openes<T><<<(unsigned)((blocks + 255) / 256), 256, 0, stream>>>(par, d, a0, a1, t0, t1, out,
                                                                                     eps_out, eps_row0 * d);
    return cudaGetLastError();
  }
  if constexpr (sizeof(T) == 4) {
    k_materialize_f32<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(par, d, a0, a1, out);
  } else {
    k_materialize<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(par, d, a0, a1, out);
  }
  return cudaGetLastError();
}

cudaError_t run_materialize_f32(const ParamDesc& par, long long d, int a0, int a1, float* out,
                                cudaStream_t stream, double* eps_out, long long eps_row0) {
  if (eps_out && par.src != SRC_OPENES) return cudaErrorInvalidValue;
  return materialize(par, d, a0, a1, out, stream, eps_out, eps_row0);
}
cudaError_t run_materialize(const ParamDesc& par, long long d, int a0, int a1, double* out,
                            cudaStream_t stream, double* eps_out, long long eps_row0) {
  if (eps_out && par.src != SRC_OPENES) return cudaErrorInvalidValue;
  return materialize(par, d, a0, a1, out, stream, eps_out, eps_row0);
}

// ------------------------------------------------ OpenES noise kept ahead
// Normals [0, n) of the ask stream `key` into eps (eps[t] = normal #t), by a
// persistent grid of one small block per SM: launched beside a resident
// rollout (one team CTA per SM leaves room for exactly one such block), it
// fills the next generation's noise rows while the current one rolls out.
constexpr int NOISE_T = 128;
__global__ void __launch_bounds__(NOISE_T) k_noise_rows(DKey key, long long t0, long long t1,
                                                        double* __restrict__ eps) {
  const long long b0 = t0 >> 1, pairs = ((t1 + 1) >> 1) - b0;
  const long long stride = (long long)gridDim.x * NOISE_T;
  for (long long i = blockIdx.x * (long long)NOISE_T + threadIdx.x; i < pairs; i += stride) {
    const long long b = b0 + i;
    double c, sn;
    normal_pair(key, (uint64_t)b, c, sn);
    if (2 * b >= t0) eps[2 * b - t0] = c;
    if (2 * b + 1 < t1) eps[2 * b + 1 - t0] = sn;
  }
}
cudaError_t run_noise_rows(DKey key, long long t0, long long n, double* eps, int blocks, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  k_noise_rows<<<(unsigned)std::max(1, blocks), NOISE_T, 0, stream>>>(key, t0, t0 + n, eps);
  return cudaGetLastError();
}

// The noise a coordinate-sharded tell reads: entries (row, p) of rows
// [0, rows) and columns [p0, p1) into out[row (p1 - p0) + p - p0].  Thread
// (row, j) computes Box-Muller pair j of the row's column range (pairs are
// aligned to the stream, so the range's end pairs are half used).
__global__ void __launch_bounds__(NOISE_T) k_noise_cols(DKey key, long long d, long long p0, long long p1,
                                                        long long rows, double* __restrict__ out) {
  const long long span = p1 - p0, per_row = span / 2 + 2;
  const long long stride = (long long)gridDim.x * NOISE_T;
  for (long long i = blockIdx.x * (long long)NOISE_T + threadIdx.x; i < rows * per_row; i += stride) {
    const long long row = i / per_row, j = i - row * per_row;
    const long long t0 = row * d + p0, t1 = row * d + p1;
    const long long b = (t0 >> 1) + j;
    if (2 * b >= t1) continue;
    double c, sn;
    normal_pair(key, (uint64_t)b, c, sn);
    double* o = out + row * span;
    if (2 * b >= t0) o[2 * b - t0] = c;
    if (2 * b + 1 < t1) o[2 * b + 1 - t0] = sn;
  }
}
cudaError_t run_noise_cols(DKey key, long long d, long long p0, long long p1, long long rows, double* out,
                           int blocks, cudaStream_t stream) {
  if (rows <= 0 || p1 <= p0) return cudaSuccess;
  k_noise_cols<<<(unsigned)std::max(1, blocks), NOISE_T, 0, stream>>>(key, d, p0, p1, rows, out);
  return cudaGetLastError();
}

// The OpenES ask from kept noise rows: entry t = row * d + p of the rows
// [r0, r1) the agents [a0, a1) use gives candidate p of agent row (and of
// row + base, negated, when mirrored) -- the values k_materialize_openes
// computes, without regenerating the normals.
template <typename T>
__global__ void k_cand_from_eps(const ParamDesc P, long long d, int a0, int a1, long long t0, long long t1,
                                const double* __restrict__ eps, long long e0, T* __restrict__ out) {
  const long long t = t0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= t1) return;
  long long row, p;
  if (t1 <= 0xFFFFFFFFll && d <= 0xFFFFFFFFll) {
    const uint32_t q = (uint32_t)t / (uint32_t)d;
    row = q;
    p = t - (long long)q * d;
  } else {
    row = t / d;
    p = t - row * d;
  }
  const double e = eps[t - e0];
  const double m = P.mean[p];
  const int ag[2] = {(int)row, P.mirrored ? (int)row + P.base : -1};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int a = ag[k];
    if (a < a0 || a >= a1) continue;
    const double v = dadd(dmul(P.sigma, k ? -e : e), m);
    if constexpr (sizeof(T) == 4) {
      out[(long long)(a - a0) * d + p] = __double2float_rn(v);
    } else {
      out[(long long)(a - a0) * d + p] = v;
    }
  }
}
template <typename T>
static cudaError_t cand_from_eps(const ParamDesc& par, long long d, int a0, int a1, const double* eps,
                                 long long eps_row0, T* out, cudaStream_t stream) {
  if (par.src != SRC_OPENES) return cudaErrorInvalidValue;
  if (a1 <= a0) return cudaSuccess;
  long long r0, r1;
  openes_rows(par, a0, a1, r0, r1);
  if (r0 < eps_row0) return cudaErrorInvalidValue;
  const long long t0 = r0 * d, t1 = r1 * d;
  k_cand_from_eps<T><<<(unsigned)((t1 - t0 + 255) / 256), 256, 0, stream>>>(par, d, a0, a1, t0, t1, eps,
                                                                             eps_row0 * d, out);
  return cudaGetLastError();
}
cudaError_t run_cand_from_eps(const ParamDesc& par, long long d, int a0, int a1, const double* eps,
                              long long eps_row0, double* out, cudaStream_t stream) {
  return cand_from_eps(par, d, a0, a1, eps, eps_row0, out, stream);
}
cudaError_t run_cand_from_eps_f32(const ParamDesc& par, long long d, int a0, int a1, const double* eps,
                                  long long eps_row0, float* out, cudaStream_t stream) {
  return cand_from_eps(par, d, a0, a1, eps, eps_row0, out, stream);
}
void openes_row_range(const ParamDesc& par, int a0, int a1, long long* r0, long long* r1) {
  openes_rows(par, a0, a1, *r0, *r1);
}

template <typename T, int N>
struct VecLoad {
  EVB_DEV static void load(const T* __restrict__ src, T* dst) {
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = src[i];
  }
};
// 16-byte vector loads from shared memory.
template <int N>
struct VecLoad<double, N> {
  EVB_DEV static void load(const double* __restrict__ src, double* dst) {
    if constexpr (N % 2 == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(src + i);
        dst[i] = v.x;
        dst[i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) dst[i] = src[i];
    }
  }
};
template <int N>
struct VecLoad<float, N> {
  EVB_DEV static void load(const float* __restrict__ src, float* dst) {
    if constexpr (N % 4 == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(src + i);
        dst[i] = v.x;
        dst[i + 1] = v.y;
        dst[i + 2] = v.z;
        dst[i + 3] = v.w;
      }
    } else if constexpr (N % 2 == 0) {
#pragma unroll
      for (int i = 0; i < N; i += 2) {
        const float2 v = *reinterpret_cast<const float2*>(src + i);
        dst[i] = v.x;
        dst[i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) dst[i] = src[i];
    }
  }
};

// Partial GEMM of one hidden-layer slice: part[ks][r][e] = sum_{k in chunk ks}
// W[k][r] * x[k][e].  W is k-major with RSP padded rows (rows contiguous, so a
// warp reads 32*TR consecutive weights); x[k][0..ET) is warp-uniform (broadcast).
template <typename T, int TR, int ET>
EVB_DEV void hidden_partial(const T* __restrict__ Ws, int WS, int RSP, int K, int KS,
                            const T* __restrict__ x, T* __restrict__ part, int tid) {
  const int nrg = RSP / TR;
  const int kc = (K + KS - 1) / KS;
  for (int w = tid; w < nrg * KS; w += ROLLOUT_THREADS) {
    const int rg = w % nrg, ks = w / nrg;
    const int k0 = ks * kc;
    const int k1 = min(K, k0 + kc);
    T acc[TR][ET];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int e = 0; e < ET; ++e) acc[i][e] = T(0);
    const T* wp = Ws + rg * TR;
#pragma unroll 2
    for (int k = k0; k < k1; ++k) {
      T wv[TR], xv[ET];
      VecLoad<T, TR>::load(wp + (size_t)k * WS, wv);
      VecLoad<T, ET>::load(x + (size_t)k * ET, xv);
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int e = 0; e < ET; ++e) acc[i][e] = fma(wv[i], xv[e], acc[i][e]);
    }
    // rows of `part` are XOR-swizzled (psw) so that a warp's stores of
    // element e of 32 consecutive row groups hit distinct banks
    T* pp = part + ((size_t)ks * RSP + rg * TR) * ET;
    const int sw = ET > 1 ? (rg & (ET - 1)) : 0;
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int e = 0; e < ET; ++e) pp[i * ET + (e ^ sw)] = acc[i][e];
  }
}

// physical column of (row r, lane e) in the swizzled partial buffer
template <int TR, int ET>
EVB_DEV int psw(int r, int e) {
  return ET > 1 ? (e ^ ((r / TR) & (ET - 1))) : e;
}

// D(8x8) += A(8x4) * B(4x8), fp64 tensor cores.  Fragments (PTX ISA,
// mma.m8n8k4 .f64): a = A[lane>>2][lane&3], b = B[lane&3][lane>>2],
// d = {D[lane>>2][2(lane&3)], D[lane>>2][2(lane&3)+1]}.
EVB_DEV void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Hidden layer on the FP64 tensor cores with a direct epilogue (ET = 16
// lanes): warp tile = 8 rows x 16 lanes over the whole K (no k-split, no
// partial buffer); two accumulator chains per n-tile (even/odd k-steps) hide
// the DMMA latency; bias + ReLU + store (local, or DSMEM scatter to all C CTAs)
// straight from the accumulator fragments.  Activation rows are XS = 20
// doubles apart so the 4 k-rows of a B fragment fall in distinct bank groups.
template <int C>
EVB_DEV uint32_t hidden_dmma_direct(const double* __restrict__ Ws, int WS, int RSv, int K,
                                    const double* __restrict__ x, int XS, const double* __restrict__ bs,
                                    double* hb, int hrow0, bool scatter, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  uint32_t bad = 0u;
  const int ngroups = (RSv + 7) / 8;
  for (int mg = warp; mg < ngroups; mg += ROLLOUT_THREADS / 32) {
    double acc[2][2][2];  // [chain][n-tile][2]
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) acc[c2][nt][0] = acc[c2][nt][1] = 0.0;
    const int row = mg * 8 + g;
    const double* wb = Ws + row;
    int k = 0;
    for (; k + 8 <= K; k += 8) {
#pragma unroll
      for (int c2 = 0; c2 < 2; ++c2) {
        const int kk = k + 4 * c2 + t;
        const double a = wb[(size_t)kk * WS];
        const double b0 = x[(size_t)kk * XS + g], b1 = x[(size_t)kk * XS + 8 + g];
        dmma(acc[c2][0][0], acc[c2][0][1], a, b0);
        dmma(acc[c2][1][0], acc[c2][1][1], a, b1);
      }
    }
    for (; k < K; k += 4) {  // tail (K not a multiple of 8)
      const int kk = k + t;
      const bool in = kk < K;
      const double a = in ? wb[(size_t)kk * WS] : 0.0;
      const double b0 = in ? x[(size_t)kk * XS + g] : 0.0, b1 = in ? x[(size_t)kk * XS + 8 + g] : 0.0;
      dmma(acc[0][0][0], acc[0][0][1], a, b0);
      dmma(acc[0][1][0], acc[0][1][1], a, b1);
    }
    if (row < RSv) {
      const double b = bs[row];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        double h2[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const double z = (acc[0][nt][i] + acc[1][nt][i]) + b;
          const double h = z > 0.0 ? z : 0.0;  // ReLU (NaN -> 0, as cwiseMax)
          if (h == INFINITY) bad |= 1u << (nt * 8 + 2 * t + i);
          h2[i] = h;
        }
        double* dst = hb + (size_t)(hrow0 + row) * XS + nt * 8 + 2 * t;
        if (!scatter) {
          *reinterpret_cast<double2*>(dst) = make_double2(h2[0], h2[1]);
        } else {
          const uint32_t la = smem_u32(dst);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const uint32_t ra = map_cluster(la, (uint32_t)c);
            asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(ra), "d"(h2[0]), "d"(h2[1])
                         : "memory");
          }
        }
      }
    }
  }
  return bad;
}


// GW: global-weights plan (compile-time, so the SMEM-resident instances keep
// provably-shared weight pointers -- LDS, not generic loads -- in the hot loop)
// TRN: write SampleBatch rows (transition collection) -- compile-time, so the
// generation kernels carry none of it
template <typename T, int TR, int ET, int C, bool MMA, bool GW, bool TRN>
__global__ void __launch_bounds__(ROLLOUT_THREADS, 1) rollout_kernel(const __grid_constant__ RolloutArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemPlan& S = A.plan;
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int tid = threadIdx.x;
  const int crank = C > 1 ? (int)cluster_ctarank() : 0;
  const int team = blockIdx.x / C;
  const int agent_local = team / A.groups;
  const int group = team % A.groups;
  const int agent = A.agent_offset + agent_local;
  const int L = N.nlayers;
  const int nh = L - 1;
  const int O = N.dims[L];

  // ------------------------------------------------------------ prologue
  // Weight rows owned by this CTA: a slice of each hidden layer, or the whole
  // layer when it is replicated (cheap K <= 8 input layers: computing them in
  // every CTA avoids one DSMEM scatter + cluster barrier per step).
  for (int i = tid; i < S.bytes / 4; i += ROLLOUT_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  // global-weights plan: this agent's materialised candidate row (HBM / L2)
  const T* gp = GW ? gparams<T>(A.par) + (long long)agent_local * N.d : nullptr;
  for (int l = 0; l < nh && !GW; ++l) {
    const int K = N.dims[l], W = N.dims[l + 1];
    const int RS = S.RS[l], r0 = S.REP[l] ? 0 : crank * RS;
    const int RSv = max(0, min(RS, W - r0));
    T* Ws = reinterpret_cast<T*>(smem + S.off_w[l]);
    T* bs = reinterpret_cast<T*>(smem + S.off_b[l]);
    for (int i = tid; i < K * RSv; i += ROLLOUT_THREADS) {
      const int k = i / RSv, r = i % RSv;
      Ws[(size_t)k * S.WS[l] + r] =
          to_T<T>(param_value(A.par, N.d, agent_local, agent, N.w_off[l] + (long long)k * W + r0 + r));
    }
    for (int r = tid; r < RSv; r += ROLLOUT_THREADS)
      bs[r] = to_T<T>(param_value(A.par, N.d, agent_local, agent, N.b_off[l] + r0 + r));
  }
  // Output layer: the rows of its input owned by this CTA (the last hidden
  // slice, or the whole observation for a linear policy).
  const int Kout = N.dims[L - 1];
  const int KRS = nh > 0 ? S.RS[nh - 1] : Kout;
  const int KRP = nh > 0 ? S.RSP[nh - 1] : Kout;
  const int k0out = nh > 0 ? crank * KRS : 0;
  const int KRv = max(0, min(KRS, Kout - k0out));
  if (!GW) {
    T* Wo = reinterpret_cast<T*>(smem + S.off_wout);
    T* bo = reinterpret_cast<T*>(smem + S.off_bout);
    for (int i = tid; i < KRv * O; i += ROLLOUT_THREADS) {
      const int k = i / O, o = i % O;
      Wo[i] = to_T<T>(
          param_value(A.par, N.d, agent_local, agent, N.w_off[L - 1] + (long long)(k0out + k) * O + o));
    }
    for (int o = tid; o < O; o += ROLLOUT_THREADS)
      bo[o] = to_T<T>(param_value(A.par, N.d, agent_local, agent, N.b_off[L - 1] + o));
  }

  // output-exchange mbarriers (double-buffered by step parity): every CTA of
  // the cluster st.async's its partial outputs into every CTA's pout, and the
  // env threads wait for the bytes (no cluster barrier per step)
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + S.off_bar);
  if (C > 1 && tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if constexpr (C > 1) cluster_sync_all();  // peers' prologues (SMEM zeroing, barriers) done

  // ------------------------------------------------------------ lane state
  const int j = group * ET + tid;  // lane index within the agent
  const bool is_env = tid < ET;
  const bool valid = is_env && j < A.e;
  const int per = A.count / A.e, rem = A.count % A.e;
  const int eps_this = valid ? per + (j < rem ? 1 : 0) : 0;
  const int slot0 = valid ? j * per + min(j, rem) : 0;
  LaneEnv s{};
  double ep_ret = 0.0, wc = 0.0;
  double wmean[4] = {0, 0, 0, 0}, wm2[4] = {0, 0, 0, 0};
  int ep_len = 0, eps_done = 0;
  long long steps = 0;
  uint32_t myfault = 0, myfault_layer = 0;
  if (valid) {
    const DKey lane_key = fold_in(fold_in(A.rollout_key, (uint64_t)agent), (uint64_t)j);
    env_reset(E, fold_in(lane_key, 0), s);  // proj/src/rollout.cpp:104
  }
  const NormParams nrm = load_norm(A.norm);

  T* x0 = reinterpret_cast<T*>(smem + S.off_x0);
  T* part = reinterpret_cast<T*>(smem + S.off_part);
  T* pout_base = reinterpret_cast<T*>(smem + S.off_pout);
  uint32_t* mask = reinterpret_cast<uint32_t*>(smem + S.off_mask);
  // output layer: flat p = w_off + k * O + o (column-major O x K), the same
  // k-major indexing as the SMEM copy
  const T* Wo = GW ? gp + N.w_off[L - 1] + (long long)k0out * O : reinterpret_cast<const T*>(smem + S.off_wout);
  const T* bo = GW ? gp + N.b_off[L - 1] : reinterpret_cast<const T*>(smem + S.off_bout);
  const int OE = O * ET;
  const int OE1 = (O + 1) * ET;  // + one row carrying each lane's first non-finite layer

  // observation -> (RunningStats) -> normalisation, written into x0 for the
  // next forward pass (proj/src/rollout.cpp:124-126)
  double sin_th = 0.0;  // sin of the current pendulum angle (reused by env_step)
  double cur_raw[4] = {0, 0, 0, 0};  // raw observation of the current state (transitions)
  auto observe_into_x0 = [&](bool act) {
    double raw[4];
    observe(E, s, raw);
    sin_th = raw[1];
    if constexpr (TRN)
      for (int i = 0; i < 4; ++i) cur_raw[i] = raw[i];
    if (act && A.track_stats) {  // WelfordStats::add, proj/src/obs_norm.cpp:7-18
      if (wc == 0.0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // registers, not local memory
          if (i >= E.obs_dim) break;
          wmean[i] = raw[i];
          wm2[i] = 0.0;
        }
        wc = 1.0;
      } else {
        wc = dadd(wc, 1.0);
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // registers, not local memory
          if (i >= E.obs_dim) break;
          const double delta = dsub(raw[i], wmean[i]);
          wmean[i] = dadd(wmean[i], ddiv(delta, wc));
          wm2[i] = dadd(wm2[i], dmul(delta, dsub(raw[i], wmean[i])));
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // registers, not local memory
      if (i >= E.obs_dim) break;
      double v = raw[i];
      if (nrm.active) v = ddiv(dsub(v, nrm.mean[i]), nrm.den[i]);
      x0[i * S.XS + tid] = act ? to_T<T>(v) : T(0);
    }
  };
  if (valid && eps_this > 0 && A.max_iters > 0) observe_into_x0(true);
#ifdef EVB_TC_PROFILE
  unsigned long long rk_prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long rk_prev = clock64();
#endif

  for (int it = 0;; ++it) {
    if (tid < MAXL) mask[(it & 1) * MAXL + tid] = 0u;  // last used two steps ago
    const bool active = valid && myfault == 0 && eps_done < eps_this && it < A.max_iters;
    // warp-level vote first: __any_sync waits for all 32 lanes, so the warp
    // reaches the block-wide reduction barrier converged (the env lanes run
    // extra code; a partially arrived warp at BAR.RED is an illegal instruction)
    const bool wact = __any_sync(0xffffffffu, active);
    if (!__syncthreads_or(wact)) break;  // also orders the x0 writes before layer 0
    RK_MARK(0);  // loop-top barrier
    uint32_t* cur_mask = mask + (it & 1) * MAXL;
    if (C > 1 && tid == 0) mbar_arrive_expect_tx(&xbar[it & 1], (uint32_t)(C * OE1 * sizeof(T)));
    // output partials are double-buffered by step parity: with a single
    // cluster barrier per step, a fast CTA may write step t+1's partials
    // while a slow one still reads step t's
    T* pout = pout_base + (it & 1) * C * OE1;

    // hidden layers (proj/src/net.cpp:86-127): z = W x + b, ReLU
    const int XS = S.XS;
    for (int l = 0; l < nh; ++l) {
      const int K = N.dims[l], W = N.dims[l + 1];
      const bool rep = S.REP[l] != 0;
      const int RS = S.RS[l], RSP = S.RSP[l], r0 = rep ? 0 : crank * RS;
      const int RSv = max(0, min(RS, W - r0));
      const T* xin = l == 0 ? x0 : reinterpret_cast<const T*>(smem + S.off_h[l - 1]);
      // weights k-major with row stride WS: the SMEM slice, or (gw) the
      // candidate row itself -- flat p = w_off + k * W + r is k-major, stride W
      const T* Ws = GW ? gp + N.w_off[l] + r0 : reinterpret_cast<const T*>(smem + S.off_w[l]);
      const T* bs = GW ? gp + N.b_off[l] + r0 : reinterpret_cast<const T*>(smem + S.off_b[l]);
      T* hb = reinterpret_cast<T*>(smem + S.off_h[l]);
      const bool last_hidden = l == nh - 1;
      const bool scatter = C > 1 && !rep && !last_hidden;
      if constexpr (MMA) {
        // FP64 tensor cores, direct epilogue (no partial buffer / reduce pass)
        const uint32_t badm = hidden_dmma_direct<C>(
            reinterpret_cast<const double*>(Ws), S.WS[l], RSv, K, reinterpret_cast<const double*>(xin), XS,
            reinterpret_cast<const double*>(bs), reinterpret_cast<double*>(hb), last_hidden ? 0 : r0,
            scatter, tid);
        if (badm) atomicOr(&cur_mask[l], badm);
      } else if (rep) {
        // replicated cheap layer (K <= 8): each thread owns lane e = tid % ET
        // and rows tid/ET + k*(256/ET); no k-split, no partial pass
        const int e = tid % ET, WSl = S.WS[l];
        T xr[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) xr[k] = k < K ? xin[k * XS + e] : T(0);
        uint32_t bad = 0u;
        for (int r = tid / ET; r < W; r += ROLLOUT_THREADS / ET) {
          T z = T(0);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k < K) z = fma(Ws[(size_t)k * WSl + r], xr[k], z);
          z = z + bs[r];
          const T h = z > T(0) ? z : T(0);  // ReLU (NaN -> 0, as cwiseMax)
          if (h == T(INFINITY)) bad = 1u;
          hb[(size_t)r * XS + e] = h;
        }
        if (bad) atomicOr(&cur_mask[l], 1u << e);
      } else {
        hidden_partial<T, TR, ET>(Ws, S.WS[l], RSP, K, S.KS[l], xin, part, tid);
        __syncthreads();
        const int KSl = S.KS[l];
        // k-split reduction + bias + ReLU: each thread owns lane e = tid % ET
        // and rows tid/ET + q*(256/ET), so index math stays out of the loop
        const int e = tid % ET;
        uint32_t bad = 0u;
        for (int r = tid / ET; r < RSv; r += ROLLOUT_THREADS / ET) {
          const int pe = psw<TR, ET>(r, e);
          T z = part[(size_t)r * ET + pe];
          for (int ks = 1; ks < KSl; ++ks) z += part[((size_t)ks * RSP + r) * ET + pe];
          z = z + bs[r];
          const T h = z > T(0) ? z : T(0);  // ReLU (NaN -> 0, as cwiseMax)
          if (h == T(INFINITY)) bad = 1u;
          if (!scatter) {
            hb[(size_t)(last_hidden ? r : r0 + r) * XS + e] = h;
          } else {
            const uint32_t la = smem_u32(hb + (size_t)(r0 + r) * XS + e);
#pragma unroll
            for (int c = 0; c < C; ++c) st_cluster<T>(map_cluster(la, (uint32_t)c), h);
          }
        }
        if (bad) atomicOr(&cur_mask[l], 1u << e);
      }
      if constexpr (C > 1) {
        if (scatter) {
          cluster_sync_all();
        } else {
          __syncthreads();
        }
      } else {
        __syncthreads();
      }
      RK_MARK(1 + (l > 0 ? 1 : 0));  // layer 0 / layers >= 1 (incl. their barrier)
    }

    // output layer partial over this CTA's rows, reduced across the cluster
    // together with each lane's first non-finite layer (NetFault bookkeeping
    // rides on the same DSMEM exchange: no remote loads in the env phase)
    {
      const T* xin = nh > 0 ? reinterpret_cast<const T*>(smem + S.off_h[nh - 1]) : x0;
      auto publish = [&](int oe, T v) {
        if constexpr (C > 1) {
          const uint32_t la = smem_u32(pout + crank * OE1 + oe), lb = smem_u32(&xbar[it & 1]);
#pragma unroll
          for (int c = 0; c < C; ++c)
            st_async(map_cluster(la, (uint32_t)c), v, map_cluster(lb, (uint32_t)c));
        } else {
          pout[oe] = v;
        }
      };
      auto bad_row = [&](int e) {
        int bl = L;
        for (int l = nh - 1; l >= 0; --l)
          if ((cur_mask[l] >> e) & 1u) bl = l;
        return T(bl);
      };
      if constexpr (ET == 1) {
        // one lane: warp o reduces output o over a 32-way k split with
        // shuffles (no partial buffer, no extra barrier)
        const int warp = tid >> 5, lane = tid & 31;
        if (warp < O) {
          const int kc = (KRv + 31) / 32, k0 = lane * kc, k1 = min(KRv, k0 + kc);
          T acc = T(0);
          for (int k = k0; k < k1; ++k) acc = fma(Wo[k * O + warp], xin[(size_t)k * XS], acc);
#pragma unroll
          for (int sh = 16; sh > 0; sh >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, sh);
          if (lane == 0) publish(warp, acc);
        }
        if (tid == (O < ROLLOUT_THREADS / 32 ? O * 32 : 1)) publish(OE, bad_row(0));
      } else {
        const int KSo = S.KS_out;
        const int kc = (KRP + KSo - 1) / KSo;
        for (int w = tid; w < OE * KSo; w += ROLLOUT_THREADS) {
          const int oe = w % OE, ks = w / OE;
          const int o = oe / ET, e = oe % ET;
          const int k0 = ks * kc, k1 = min(KRv, k0 + kc);
          T acc = T(0);
          for (int k = k0; k < k1; ++k) acc = fma(Wo[k * O + o], xin[(size_t)k * XS + e], acc);
          part[w] = acc;
        }
        __syncthreads();
        for (int oe = tid; oe < OE1; oe += ROLLOUT_THREADS) {
          T v;
          if (oe < OE) {
            v = part[oe];
            for (int ks = 1; ks < KSo; ++ks) v += part[ks * OE + oe];
          } else {
            v = bad_row(oe - OE);
          }
          publish(oe, v);
        }
      }
      if constexpr (C > 1) {
        // only the env threads consume the exchanged outputs: wait for all
        // C * OE1 values of this step (the other warps run on to the loop top)
        if (tid < ET) mbar_wait_parity(&xbar[it & 1], (uint32_t)((it >> 1) & 1));
      } else {
        __syncthreads();
      }
    }

    RK_MARK(3);  // output partial + cluster exchange
    // head + env step (proj/src/rollout.cpp:57-90, :131-153), then the next
    // observation (same threads: no extra barrier)
    if (active) {
      double z[8];
      bool nonfinite_out = false;
      int bad_layer = L;
      for (int c = 0; c < C; ++c) bad_layer = min(bad_layer, (int)pout[c * OE1 + OE + tid]);
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        if (o >= O) break;
        T v = pout[o * ET + tid];
        for (int c = 1; c < C; ++c) v += pout[c * OE1 + o * ET + tid];
        v = v + bo[o];
        z[o] = (double)v;
        if (!isfinite(z[o])) nonfinite_out = true;
      }
      if (bad_layer >= L && nonfinite_out) bad_layer = L - 1;
      if (bad_layer < L) {  // NetFault: the lowest layer with a non-finite activation
        myfault = FAULT_NET;
        myfault_layer = (uint32_t)bad_layer;
      } else {
        double action;
        if (N.head == HEAD_CATEGORICAL) {
          int arg = 0;
          double best = z[0];
#pragma unroll
          for (int o = 1; o < 8; ++o)
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
        const uint32_t f =
            env_step(E, s, action, reward, term, trunc, E.id == ENV_PENDULUM ? &sin_th : nullptr);
        if (TRN && !f && crank == 0) {  // one SampleBatch row (rollout.cpp:132-139)
          double nxt[4];
          observe(E, s, nxt);  // final_obs: the successor before any auto-reset
          const long long row = ((long long)agent_local * A.e + j) * A.t_cap + steps;
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // registers, not local memory
            if (i >= E.obs_dim) break;
            A.t_obs[row * E.obs_dim + i] = cur_raw[i];
            A.t_next[row * E.obs_dim + i] = nxt[i];
          }
          A.t_act[row] = action;
          A.t_rew[row] = reward;
          A.t_term[row] = term ? 1 : 0;
          A.t_trunc[row] = trunc ? 1 : 0;
        }
        if (f) {
          myfault = f;
        } else {
          ep_ret = dadd(ep_ret, reward);  // proj/src/rollout.cpp:143
          ep_len += 1;
          steps += 1;
          if (term || trunc) {
            if (crank == 0) {
              const long long slot = (long long)agent_local * A.count + slot0 + eps_done;
              A.ep_returns[slot] = ep_ret;
              if (A.ep_lengths) A.ep_lengths[slot] = ep_len;
            }
            ep_ret = 0.0;
            ep_len = 0;
            eps_done += 1;
            if (eps_done < eps_this) env_reset(E, s.rng, s);  // auto-reset, env.cpp:163-167
          }
        }
      }
      const bool next = myfault == 0 && eps_done < eps_this && it + 1 < A.max_iters;
      observe_into_x0(next);
    }
    RK_MARK(4);  // head + env + observe
  }
#ifdef EVB_TC_PROFILE
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) atomicAdd(&g_rk_prof[i], rk_prof[i]);
    atomicAdd(&g_rk_prof[8], 1ull);
  }
#endif

  if (valid && crank == 0) {
    const long long lane = (long long)agent_local * A.e + j;
    if (A.lane_steps) A.lane_steps[lane] = steps;
    if (A.track_stats && A.lane_stats) {
      double* st = A.lane_stats + lane * 9;
      st[0] = wc;
      for (int i = 0; i < 4; ++i) {
        st[1 + i] = wmean[i];
        st[5 + i] = wm2[i];
      }
    }
    if (myfault) record_fault(A.fault, (uint64_t)((long long)agent * A.e + j), myfault, myfault_layer);
  }
  if constexpr (C > 1) cluster_sync_all();  // no CTA may exit while peers still address its SMEM
}

// ---------------------------------------------------------------------------
// Pipelined fp64 DMMA team (the fp64 parity path of 2-hidden-layer policies
// with ET = 16 lanes, BASELINE config 3).  The plain cluster team runs one
// serial chain per step -- layer 0, the DMMA slice GEMM, the output exchange,
// then the fp64 env on 16 threads -- so the FP64 tensor pipe idles for the
// env / exchange half of every step (one CTA per SM: the weight slice fills
// SMEM).  Here the 16 lanes are two independent groups of 8 and the CTA is
// warp-specialised: 8 compute warps run group A's layers while a 9th (env)
// warp steps group B's environments, then the roles swap, so the env, the
// DSMEM exchange latency and the GEMMs of the other group overlap.
//   compute warps: [x0(g) ready] L0(g) | L1(g) | out-partial(g) -> st.async
//   env warp     : [partials(g) landed] head, env_step, observe -> x0(g)
// Handshakes: named barrier 1+g (env arrives, compute syncs) for x0 / the
// group-alive flag; the output partials ride st.async + mbarrier complete_tx
// (double-buffered by step parity) exactly as in the plain team.  Groups are
// 8 lanes = one n8 tile of mma.m8n8k4, activation rows 8 doubles apart
// (conflict-free fragment loads).  Numerics per lane are the plain team's.
constexpr int PIPE_EW = 4;  // env warps: one per SM sub-partition, so the env's fp64
                             // work does not pile onto one sub-partition's FP64 pipe
constexpr int PIPE_THREADS = ROLLOUT_THREADS + 32 * PIPE_EW;
constexpr int PG = 8;                  // lanes per group
constexpr int PIPE_CHAINS = 4;         // independent DMMA accumulator chains per warp tile
constexpr int PIPE_LPW = PG / PIPE_EW;  // lanes of one group per env warp

EVB_DEV void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
EVB_DEV void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// 8 weight rows x 8 lanes over K; x is [K][8]; returns the D fragment
// (row g, lanes 2t, 2t+1).  Four accumulator chains: a warp owns one n8
// tile, so the chains are its only DMMA latency cover.
EVB_DEV void dmma_tile8(const double* __restrict__ wb, int WS, int K, const double* __restrict__ x, int g,
                        int t, double& d0, double& d1) {
  constexpr int NC = PIPE_CHAINS;
  double acc[NC][2];
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q][0] = acc[q][1] = 0.0;
  int k = 0;
  for (; k + 4 * NC <= K; k += 4 * NC) {
    double a[NC], b[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      a[q] = wb[(size_t)(k + 4 * q + t) * WS];
      b[q] = x[(k + 4 * q + t) * PG + g];
    }
#pragma unroll
    for (int q = 0; q < NC; ++q) dmma(acc[q][0], acc[q][1], a[q], b[q]);
  }
#pragma unroll
  for (int q = 0; q < NC; ++q) {  // remainder: at most NC - 1 full k4 steps + one partial
    const int kk = k + 4 * q + t;
    if (k + 4 * q < K) {
      const bool in = kk < K;
      dmma(acc[q][0], acc[q][1], in ? wb[(size_t)kk * WS] : 0.0, in ? x[kk * PG + g] : 0.0);
    }
  }
#pragma unroll
  for (int w = 1; w < NC; w <<= 1)
#pragma unroll
    for (int q = 0; q < NC; q += 2 * w) {
      acc[q][0] += acc[q + w][0];
      acc[q][1] += acc[q + w][1];
    }
  d0 = acc[0][0];
  d1 = acc[0][1];
}

// bias + ReLU + store of one tile; returns the lanes with an infinite activation
EVB_DEV uint32_t tile8_epilogue(double d0, double d1, int row, int nrows, const double* bs, double* h, int t) {
  if (row >= nrows) return 0u;
  const double b = bs[row];
  const double z0 = d0 + b, z1 = d1 + b;
  const double h0 = z0 > 0.0 ? z0 : 0.0, h1 = z1 > 0.0 ? z1 : 0.0;  // ReLU (NaN -> 0, as cwiseMax)
  *reinterpret_cast<double2*>(h + row * PG + 2 * t) = make_double2(h0, h1);
  return (h0 == INFINITY ? 1u << (2 * t) : 0u) | (h1 == INFINITY ? 2u << (2 * t) : 0u);
}

template <int C>
__global__ void __launch_bounds__(PIPE_THREADS, 1) rollout_pipe_kernel(const __grid_constant__ RolloutArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemPlan& S = A.plan;
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int tid = threadIdx.x;
  const int crank = (int)cluster_ctarank();
  const int team = blockIdx.x / C;
  const int agent_local = team / A.groups;
  const int group = team % A.groups;
  const int agent = A.agent_offset + agent_local;
  const int L = 3, O = N.dims[3];
  const int K0 = N.dims[0], W0 = N.dims[1], W1 = N.dims[2];
  const int RS1 = S.RS[1], r01 = crank * RS1, RSv1 = max(0, min(RS1, W1 - r01));

  // ------------------------------------------------------------ prologue
  for (int i = tid; i < S.bytes / 4; i += PIPE_THREADS) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  {
    double* W0s = reinterpret_cast<double*>(smem + S.off_w[0]);
    double* b0s = reinterpret_cast<double*>(smem + S.off_b[0]);
    for (int i = tid; i < K0 * W0; i += PIPE_THREADS) {
      const int k = i / W0, r = i % W0;
      W0s[k * S.WS[0] + r] = param_value(A.par, N.d, agent_local, agent, N.w_off[0] + (long long)k * W0 + r);
    }
    for (int r = tid; r < W0; r += PIPE_THREADS)
      b0s[r] = param_value(A.par, N.d, agent_local, agent, N.b_off[0] + r);
    double* W1s = reinterpret_cast<double*>(smem + S.off_w[1]);
    double* b1s = reinterpret_cast<double*>(smem + S.off_b[1]);
    for (int i = tid; i < W0 * RSv1; i += PIPE_THREADS) {
      const int k = i / RSv1, r = i % RSv1;
      W1s[(size_t)k * S.WS[1] + r] =
          param_value(A.par, N.d, agent_local, agent, N.w_off[1] + (long long)k * W1 + r01 + r);
    }
    for (int r = tid; r < RSv1; r += PIPE_THREADS)
      b1s[r] = param_value(A.par, N.d, agent_local, agent, N.b_off[1] + r01 + r);
    double* Wo = reinterpret_cast<double*>(smem + S.off_wout);
    double* bo = reinterpret_cast<double*>(smem + S.off_bout);
    for (int i = tid; i < RSv1 * O; i += PIPE_THREADS) {
      const int k = i / O, o = i % O;
      Wo[i] = param_value(A.par, N.d, agent_local, agent, N.w_off[2] + (long long)(r01 + k) * O + o);
    }
    for (int o = tid; o < O; o += PIPE_THREADS) bo[o] = param_value(A.par, N.d, agent_local, agent, N.b_off[2] + o);
  }
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem + S.off_bar);  // [group][parity]
  int* alive_flag = reinterpret_cast<int*>(smem + S.off_bar + 32);  // [group][env warp]
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&xbar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_sync_all();

  double* x0 = reinterpret_cast<double*>(smem + S.off_x0);       // [group][4][8]
  double* pout0 = reinterpret_cast<double*>(smem + S.off_pout);  // [group][parity][C][(O+1)*8]
  uint32_t* mask0 = reinterpret_cast<uint32_t*>(smem + S.off_mask);  // [group][parity][2]
  const int OE = O * PG, OE1 = (O + 1) * PG;
  const uint32_t xbytes = (uint32_t)(C * OE1 * sizeof(double));

#ifdef EVB_TC_PROFILE
  unsigned long long rk_prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long rk_prev = clock64();
#endif
  if (tid < ROLLOUT_THREADS) {
    // ====================================================== compute warps
    const int warp = tid >> 5, lane = tid & 31;
    const int g8 = lane >> 2, t4 = lane & 3;
    const double* W0s = reinterpret_cast<const double*>(smem + S.off_w[0]);
    const double* b0s = reinterpret_cast<const double*>(smem + S.off_b[0]);
    const double* W1s = reinterpret_cast<const double*>(smem + S.off_w[1]);
    const double* b1s = reinterpret_cast<const double*>(smem + S.off_b[1]);
    const double* Wo = reinterpret_cast<const double*>(smem + S.off_wout);
    double* h0 = reinterpret_cast<double*>(smem + S.off_h[0]);
    double* opart = reinterpret_cast<double*>(smem + S.off_part);  // [warp][o][8 lanes]
    int alive = 3;  // bit g: group g still has active lanes
    for (int it = 0;; ++it) {
      const int par = it & 1;
#pragma unroll 1
      for (int gq = 0; gq < 2; ++gq) {
        if (!((alive >> gq) & 1)) continue;
        uint32_t* cm = mask0 + (gq * 2 + par) * 2;
        if (tid < 2) cm[tid] = 0u;  // last read by this group's output pass two steps ago
        RK_MARK(7);
        named_sync(1 + gq, PIPE_THREADS);  // x0(g) of this step + alive flag
        RK_MARK(0);
        int any_alive = 0;
#pragma unroll
        for (int w = 0; w < PIPE_EW; ++w) any_alive |= alive_flag[gq * PIPE_EW + w];
        if (!any_alive) {
          alive &= ~(1 << gq);
          continue;
        }
        const double* xg = x0 + gq * 4 * PG;
        // layer 0 (replicated, K0 <= 4): one DMMA per 8-row tile, the B
        // fragment (this group's observations) shared by all of a warp's tiles
        uint32_t bad = 0u;
        {
          const bool kin = t4 < K0;
          const double xb = kin ? xg[t4 * PG + g8] : 0.0;
          const int nt0 = (W0 + 7) / 8;
          for (int mg0 = warp; mg0 < nt0; mg0 += 4 * (ROLLOUT_THREADS / 32)) {
            double d[4][2];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int mg = mg0 + q * (ROLLOUT_THREADS / 32);
              d[q][0] = d[q][1] = 0.0;
              if (mg < nt0) dmma(d[q][0], d[q][1], kin ? W0s[t4 * S.WS[0] + mg * 8 + g8] : 0.0, xb);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int mg = mg0 + q * (ROLLOUT_THREADS / 32);
              if (mg < nt0) bad |= tile8_epilogue(d[q][0], d[q][1], mg * 8 + g8, W0, b0s, h0, t4);
            }
          }
        }
        if (bad) atomicOr(&cm[0], bad);
        named_sync(3, ROLLOUT_THREADS);
        RK_MARK(1);
        // layer 1: this CTA's RS1-row slice (DMMA over K = W0); the output
        // layer's partial is folded into the epilogue: each warp reduces its
        // tile's rows (shuffles over g) into opart[warp][o][lane]
        bad = 0u;
        for (int mg = warp; mg * 8 < RSv1; mg += ROLLOUT_THREADS / 32) {
          double d0, d1;
          dmma_tile8(W1s + mg * 8 + g8, S.WS[1], W0, h0, g8, t4, d0, d1);
          const int row = mg * 8 + g8;
          double hv0 = 0.0, hv1 = 0.0;
          if (row < RSv1) {
            const double b = b1s[row];
            const double z0 = d0 + b, z1 = d1 + b;
            hv0 = z0 > 0.0 ? z0 : 0.0;  // ReLU (NaN -> 0, as cwiseMax)
            hv1 = z1 > 0.0 ? z1 : 0.0;
            bad |= (hv0 == INFINITY ? 1u << (2 * t4) : 0u) | (hv1 == INFINITY ? 2u << (2 * t4) : 0u);
          }
          for (int o = 0; o < O; ++o) {
            const double w = row < RSv1 ? Wo[row * O + o] : 0.0;
            double c0 = w * hv0, c1 = w * hv1;
#pragma unroll
            for (int sh = 4; sh < 32; sh <<= 1) {
              c0 += __shfl_xor_sync(0xffffffffu, c0, sh);
              c1 += __shfl_xor_sync(0xffffffffu, c1, sh);
            }
            if (g8 == 0) {
              double2* dst = reinterpret_cast<double2*>(opart + (warp * 8 + o) * PG + 2 * t4);
              if (mg == warp) {
                *dst = make_double2(c0, c1);
              } else {
                const double2 v = *dst;
                *dst = make_double2(v.x + c0, v.y + c1);
              }
            }
          }
        }
        if (bad) atomicOr(&cm[1], bad);
        named_sync(3, ROLLOUT_THREADS);
        RK_MARK(2);
        // output partials (sum over warps in order) + the NetFault row,
        // st.async to all C CTAs
        double* pout = pout0 + (gq * 2 + par) * C * OE1;
        const uint32_t lb = smem_u32(&xbar[gq * 2 + par]);
        const int nw1 = min(ROLLOUT_THREADS / 32, (RSv1 + 7) / 8);  // warps that own a tile
        if (tid < OE) {
          double v = 0.0;
          for (int w = 0; w < nw1; ++w) v += opart[w * 8 * PG + tid];
          const uint32_t la = smem_u32(pout + crank * OE1 + tid);
#pragma unroll
          for (int c = 0; c < C; ++c) st_async(map_cluster(la, (uint32_t)c), v, map_cluster(lb, (uint32_t)c));
        } else if (tid < OE1) {
          const int e = tid - OE;
          int bl = L;
          for (int l = 1; l >= 0; --l)
            if ((cm[l] >> e) & 1u) bl = l;
          const uint32_t la = smem_u32(pout + crank * OE1 + tid);
#pragma unroll
          for (int c = 0; c < C; ++c)
            st_async(map_cluster(la, (uint32_t)c), (double)bl, map_cluster(lb, (uint32_t)c));
        }
        RK_MARK(3);
      }
      if (!alive) break;
    }
  } else {
    // ========================================================== env warp
    const int ew = (tid - ROLLOUT_THREADS) >> 5, lane = tid & 31;
    const bool mine = lane < 2 * PIPE_LPW;  // this thread owns a lane of the team
    const int gq_me = mine ? lane / PIPE_LPW : 2, e = ew * PIPE_LPW + lane % PIPE_LPW;
    const int j = group * 16 + gq_me * PG + e;  // lane index within the agent
    const bool valid = mine && j < A.e;
    const int per = A.count / A.e, rem = A.count % A.e;
    const int eps_this = valid ? per + (j < rem ? 1 : 0) : 0;
    const int slot0 = valid ? j * per + min(j, rem) : 0;
    LaneEnv s{};
    double ep_ret = 0.0, wc = 0.0;
    double wmean[4] = {0, 0, 0, 0}, wm2[4] = {0, 0, 0, 0};
    int ep_len = 0, eps_done = 0;
    long long steps = 0;
    uint32_t myfault = 0, myfault_layer = 0;
    if (valid) {
      const DKey lane_key = fold_in(fold_in(A.rollout_key, (uint64_t)agent), (uint64_t)j);
      env_reset(E, fold_in(lane_key, 0), s);  // proj/src/rollout.cpp:104
    }
    const NormParams nrm = load_norm(A.norm);
    const double* bo = reinterpret_cast<const double*>(smem + S.off_bout);
    double sin_th = 0.0;
    auto observe_into_x0 = [&](bool act) {
      double raw[4];
      observe(E, s, raw);
      sin_th = raw[1];
      if (act && A.track_stats) {  // WelfordStats::add, proj/src/obs_norm.cpp:7-18
        if (wc == 0.0) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // registers, not local memory
            if (i >= E.obs_dim) break;
            wmean[i] = raw[i];
            wm2[i] = 0.0;
          }
          wc = 1.0;
        } else {
          wc = dadd(wc, 1.0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // registers, not local memory
            if (i >= E.obs_dim) break;
            const double delta = dsub(raw[i], wmean[i]);
            wmean[i] = dadd(wmean[i], ddiv(delta, wc));
            wm2[i] = dadd(wm2[i], dmul(delta, dsub(raw[i], wmean[i])));
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // registers, not local memory
        if (i >= E.obs_dim) break;
        double v = raw[i];
        if (nrm.active) v = ddiv(dsub(v, nrm.mean[i]), nrm.den[i]);
        x0[(gq_me * 4 + i) * PG + e] = act ? v : 0.0;
      }
    };
    bool act = valid && eps_this > 0 && A.max_iters > 0;
    if (mine) observe_into_x0(act);
    int alive = 0;
#pragma unroll
    for (int gq = 0; gq < 2; ++gq) {
      const bool a = __any_sync(0xffffffffu, act && gq_me == gq);
      if (lane == 0) alive_flag[gq * PIPE_EW + ew] = a ? 1 : 0;
    }
    named_sync(4, 32 * PIPE_EW);
#pragma unroll
    for (int gq = 0; gq < 2; ++gq)
      for (int w = 0; w < PIPE_EW; ++w) alive |= alive_flag[gq * PIPE_EW + w] ? 1 << gq : 0;
    named_arrive(1, PIPE_THREADS);
    named_arrive(2, PIPE_THREADS);
    for (int it = 0; alive; ++it) {
      const int par = it & 1;
#pragma unroll 1
      for (int gq = 0; gq < 2; ++gq) {
        if (!((alive >> gq) & 1)) continue;
        uint64_t* bar = &xbar[gq * 2 + par];
        if (ew == 0 && lane == 0) mbar_arrive_expect_tx(bar, xbytes);
        RK_MARK(6);
        mbar_wait_parity(bar, (uint32_t)((it >> 1) & 1));
        RK_MARK(4);
        const double* pout = pout0 + (gq * 2 + par) * C * OE1;
        if (gq_me == gq && act) {
          // head + env step (proj/src/rollout.cpp:57-90, :131-153)
          double z[8];
          bool nonfinite_out = false;
          int bad_layer = L;
          for (int c = 0; c < C; ++c) bad_layer = min(bad_layer, (int)pout[c * OE1 + OE + e]);
#pragma unroll
          for (int o = 0; o < 8; ++o) {
            if (o >= O) break;
            double v = pout[o * PG + e];
            for (int c = 1; c < C; ++c) v += pout[c * OE1 + o * PG + e];
            z[o] = v + bo[o];
            if (!isfinite(z[o])) nonfinite_out = true;
          }
          if (bad_layer >= L && nonfinite_out) bad_layer = L - 1;
          if (bad_layer < L) {  // NetFault: the lowest layer with a non-finite activation
            myfault = FAULT_NET;
            myfault_layer = (uint32_t)bad_layer;
          } else {
            double action;
            if (N.head == HEAD_CATEGORICAL) {
              int arg = 0;
              double best = z[0];
#pragma unroll
              for (int o = 1; o < 8; ++o)
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
            const uint32_t f =
                env_step(E, s, action, reward, term, trunc, E.id == ENV_PENDULUM ? &sin_th : nullptr);
            if (f) {
              myfault = f;
            } else {
              ep_ret = dadd(ep_ret, reward);  // proj/src/rollout.cpp:143
              ep_len += 1;
              steps += 1;
              if (term || trunc) {
                if (crank == 0) {
                  const long long slot = (long long)agent_local * A.count + slot0 + eps_done;
                  A.ep_returns[slot] = ep_ret;
                  if (A.ep_lengths) A.ep_lengths[slot] = ep_len;
                }
                ep_ret = 0.0;
                ep_len = 0;
                eps_done += 1;
                if (eps_done < eps_this) env_reset(E, s.rng, s);  // auto-reset, env.cpp:163-167
              }
            }
          }
          act = myfault == 0 && eps_done < eps_this && it + 1 < A.max_iters;
          observe_into_x0(act);
        }
        const bool a = __any_sync(0xffffffffu, act && gq_me == gq);
        if (lane == 0) alive_flag[gq * PIPE_EW + ew] = a ? 1 : 0;
        named_sync(4, 32 * PIPE_EW);  // every env warp sees the group's flags
        int any_alive = 0;
#pragma unroll
        for (int w = 0; w < PIPE_EW; ++w) any_alive |= alive_flag[gq * PIPE_EW + w];
        if (!any_alive) alive &= ~(1 << gq);
        named_arrive(1 + gq, PIPE_THREADS);
        RK_MARK(5);
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
  }
#ifdef EVB_TC_PROFILE
  if (tid == 0 || tid == ROLLOUT_THREADS) {  // compute warp 0 / env warp 0
    for (int i = 0; i < 8; ++i) atomicAdd(&g_rk_prof[i], rk_prof[i]);
    if (tid == 0) atomicAdd(&g_rk_prof[8], 1ull);
  }
#endif
  cluster_sync_all();  // no CTA may exit while peers still address its SMEM
}

#ifdef EVB_TC_PROFILE
extern "C" int evorl_debug_rk_profile(unsigned long long* out16) {
  if (cudaMemcpyFromSymbol(out16, g_rk_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 6;
  static const unsigned long long zero[16] = {};
  return cudaMemcpyToSymbol(g_rk_prof, zero, sizeof zero) == cudaSuccess ? 0 : 6;
}
#endif

// ------------------------------------------------------------------ host side
static int align16(int x) { return (x + 15) & ~15; }
static int pow2floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

static bool try_plan(const NetDesc& net, int obs_dim, int ET, int TR, int C, int tsize, SmemPlan* P,
                     bool mma = false, bool gw = false) {
  const int L = net.nlayers, nh = L - 1, O = net.dims[L];
  if (nh == 0 && C > 1) return false;
  if (O > 8 || obs_dim > 4) return false;
  SmemPlan p{};
  p.C = C;
  p.TR = TR;
  p.ET = ET;
  int off = 0;
  size_t part = 0;
  for (int l = 0; l < nh; ++l) {
    const int K = net.dims[l], W = net.dims[l + 1];
    if (W < C) return false;
    // cheap non-final layers (K <= 8: the observation layer) are computed in
    // full by every CTA instead of sliced + exchanged
    const bool rep = C > 1 && K <= 8 && l < nh - 1;
    p.REP[l] = rep ? 1 : 0;
    const int RS = rep ? W : (W + C - 1) / C;
    // DMMA plan: 8-row warp tiles; SIMT: 32*TR-row warp groups
    const int RSP = mma ? (RS + 7) / 8 * 8 : (RS + 32 * TR - 1) / (32 * TR) * (32 * TR);
    const int nrg = RSP / TR;
    int KS = nrg >= ROLLOUT_THREADS ? 1 : pow2floor(ROLLOUT_THREADS / nrg);
    while (KS > 1 && K / KS < 8) KS /= 2;
    int WS = RSP;
    if (mma) {  // DMMA direct epilogue: no k-split; padded rows (bank spread)
      KS = 1;
      WS = RSP + 4;
    }
    if (gw) WS = W;  // the candidate row's own layout
    p.RS[l] = RS;
    p.RSP[l] = RSP;
    p.KS[l] = KS;
    p.WS[l] = WS;
    p.off_w[l] = off;
    if (!gw) off = align16(off + K * WS * tsize);
    p.off_b[l] = off;
    if (!gw) off = align16(off + RSP * tsize);
    if (!mma) part = std::max(part, (size_t)KS * RSP * ET * tsize);
  }
  const int XS = mma ? ET + 4 : ET;
  p.XS = XS;
  const int KRP = nh > 0 ? p.RSP[nh - 1] : net.dims[0];
  p.off_wout = off;
  if (!gw) off = align16(off + KRP * O * tsize);
  p.off_bout = off;
  if (!gw) off = align16(off + O * tsize);
  p.off_x0 = off;
  off = align16(off + 4 * XS * tsize);
  for (int l = 0; l < nh; ++l) {
    p.off_h[l] = off;
    const int rows = (l == nh - 1) ? p.RSP[l] : net.dims[l + 1];
    off = align16(off + rows * XS * tsize);
  }
  int KSo = pow2floor(std::max(1, ROLLOUT_THREADS / (O * ET)));
  while (KSo > 1 && KRP / KSo < 4) KSo /= 2;
  p.KS_out = KSo;
  part = std::max(part, (size_t)KSo * O * ET * tsize);
  p.off_part = off;
  off = align16(off + (int)part);
  p.off_pout = off;
  off = align16(off + 2 * C * (O + 1) * ET * tsize);
  p.off_mask = off;
  off = align16(off + 2 * MAXL * 4);
  p.off_bar = off;  // two mbarriers (output exchange, double-buffered by step)
  off = align16(off + 16);
  p.bytes = off;
  p.mma = mma ? 1 : 0;
  p.gw = gw ? 1 : 0;
  if (off > 227 * 1024) return false;
  *P = p;
  return true;
}

// Pipelined fp64 DMMA team (rollout_pipe_kernel): 2 hidden layers, the
// first replicated (K <= 8), the second sliced over C CTAs; activations in
// 8-lane groups (rows 8 doubles apart).
constexpr int PG_HOST = 8;
static bool try_plan_pipe(const NetDesc& net, int obs_dim, int C, SmemPlan* P) {
  if (net.nlayers != 3) return false;
  const int K0 = net.dims[0], W0 = net.dims[1], W1 = net.dims[2], O = net.dims[3];
  if (K0 > 4 || obs_dim > 4 || O > 8 || W1 < C || W0 < 8) return false;
  SmemPlan p{};
  p.C = C;
  p.TR = 1;
  p.ET = 16;
  p.mma = 1;
  p.pipe = 1;
  p.XS = 8;
  const int RS1 = (W1 + C - 1) / C, RSP1 = (RS1 + 7) / 8 * 8;
  p.REP[0] = 1;
  p.RS[0] = p.RSP[0] = (W0 + 7) / 8 * 8;
  p.WS[0] = p.RSP[0] + 4;
  p.RS[1] = RS1;
  p.RSP[1] = RSP1;
  p.WS[1] = RSP1 + 4;  // 4 k-rows of an A fragment land 8 banks apart
  p.KS[0] = p.KS[1] = 1;
  int off = 0;
  p.off_w[0] = off;
  off = align16(off + K0 * p.WS[0] * 8);
  p.off_b[0] = off;
  off = align16(off + p.RSP[0] * 8);
  p.off_w[1] = off;
  off = align16(off + W0 * p.WS[1] * 8);
  p.off_b[1] = off;
  off = align16(off + RSP1 * 8);
  p.off_wout = off;
  off = align16(off + RSP1 * O * 8);
  p.off_bout = off;
  off = align16(off + O * 8);
  p.off_x0 = off;
  off = align16(off + 2 * 4 * 8 * 8);
  p.off_h[0] = off;
  off = align16(off + p.RSP[0] * 8 * 8);
  p.off_h[1] = off;  // (unused: the output partial is folded into layer 1's epilogue)
  p.off_part = off;
  off = align16(off + 8 * 8 * PG_HOST * 8);
  p.off_pout = off;
  off = align16(off + 2 * 2 * C * (O + 1) * 8 * 8);
  p.off_mask = off;
  off = align16(off + 2 * 2 * 2 * 4);
  p.off_bar = off;  // 4 mbarriers [group][parity] + group-alive flags [group][env warp]
  off = align16(off + 32 + 2 * 8 * 4);
  p.bytes = off;
  if (off > 227 * 1024) return false;
  *P = p;
  return true;
}

// opt-in (EVORL_FP64_PIPE=1): measured slower than the plain DMMA team on
// B200 (profiles/README.md): DMMA and the env's DFMA share the FP64 pipe, and
// 8-lane groups lose the A-fragment reuse of 16-lane tiles
static bool pipe_enabled() {
  const char* v = getenv("EVORL_FP64_PIPE");
  return v && v[0] == '1';
}

bool plan_rollout(const NetDesc& net, int obs_dim, int e, int precision, SmemPlan* plan, bool simple_only) {
  const int ET = e >= 5 ? 16 : (e >= 2 ? 4 : 1);
  plan->trn = 0;
  plan->pipe = 0;
  plan->oz = 0;
  if (precision == 3) {  // EVORL_PREC_OZ: int8-sliced tcgen05 team if the shape fits, else the fp64 team
    if (!simple_only && plan_rollout_oz(net, obs_dim, e, &plan->tcp)) {
      plan->oz = 1;
      plan->tc = 0;
      plan->ET = 16;
      plan->C = plan->tcp.data[0];
      return true;
    }
    precision = 0;
  }
  if (simple_only) {  // TR = 1 SIMT, resident or global-weights
    plan->tc = 0;
    const int ts = precision == 0 ? 8 : 4;
    for (int C : {1, 2, 4, 8})
      if (try_plan(net, obs_dim, ET, 1, C, ts, plan)) return true;
    for (int C : {8, 4, 2, 1})
      if (try_plan(net, obs_dim, ET, 1, C, ts, plan, false, true)) return true;
    return false;
  }
  if (precision == 2) {  // EVORL_PREC_TC: tcgen05 team if the shape fits, else the fp32 team
    if (plan_rollout_tc(net, obs_dim, e, &plan->tcp)) {
      plan->tc = 1;
      plan->ET = 16;
      plan->C = plan->tcp.data[0];
      return true;
    }
    precision = 1;
  }
  plan->tc = 0;
  const int tsize = precision == 0 ? 8 : 4;
  if (precision == 0 && ET == 16 && pipe_enabled())
    for (int C : {2, 4, 8})
      if (try_plan_pipe(net, obs_dim, C, plan)) return true;
  for (int C : {1, 2, 4, 8}) {
    // fp64 with 16 lanes: hidden-layer GEMMs on the FP64 tensor cores
    if (precision == 0 && ET == 16 && try_plan(net, obs_dim, ET, 1, C, tsize, plan, true)) return true;
    if (ET == 16 && try_plan(net, obs_dim, ET, 2, C, tsize, plan)) {
      // TR=2 needs enough row groups x k-splits to occupy the CTA
      bool ok = true;
      for (int l = 0; l < net.nlayers - 1; ++l)
        if ((plan->RSP[l] / 2) * plan->KS[l] < ROLLOUT_THREADS / 2 && net.dims[l] >= 64) ok = false;
      if (ok) return true;
    }
    if (try_plan(net, obs_dim, ET, 1, C, tsize, plan)) return true;
  }
  // too large for SMEM residency: weights streamed from the materialised
  // candidates (HBM / L2), rows split over the largest cluster that fits
  for (int C : {8, 4, 2, 1})
    if (try_plan(net, obs_dim, ET, 1, C, tsize, plan, false, true)) return true;
  return false;
}

template <typename T, int TR, int ET, int C, bool MMA, bool GW = false, bool TRN = false>
static cudaError_t launch_inst(const RolloutArgs& a, cudaStream_t stream) {
  auto kern = rollout_kernel<T, TR, ET, C, MMA, GW, TRN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.n_agents * a.groups * C));
  cfg.blockDim = dim3(ROLLOUT_THREADS);
  cfg.dynamicSmemBytes = (size_t)a.plan.bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int C>
static cudaError_t launch_pipe_inst(const RolloutArgs& a, cudaStream_t stream) {
  auto kern = rollout_pipe_kernel<C>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.n_agents * a.groups * C));
  cfg.blockDim = dim3(PIPE_THREADS);
  cfg.dynamicSmemBytes = (size_t)a.plan.bytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

static cudaError_t launch_pipe(const RolloutArgs& a, cudaStream_t s) {
  switch (a.plan.C) {
    case 2: return launch_pipe_inst<2>(a, s);
    case 4: return launch_pipe_inst<4>(a, s);
    case 8: return launch_pipe_inst<8>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T, int TR, int ET, bool MMA = false, bool GW = false, bool TRN = false>
static cudaError_t launch_c(const RolloutArgs& a, cudaStream_t s) {
  switch (a.plan.C) {
    case 1: return launch_inst<T, TR, ET, 1, MMA, GW, TRN>(a, s);
    case 2: return launch_inst<T, TR, ET, 2, MMA, GW, TRN>(a, s);
    case 4: return launch_inst<T, TR, ET, 4, MMA, GW, TRN>(a, s);
    case 8: return launch_inst<T, TR, ET, 8, MMA, GW, TRN>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <typename T, bool GW>
static cudaError_t launch_trn(const RolloutArgs& a, cudaStream_t s) {
  if (a.plan.ET == 1) return launch_c<T, 1, 1, false, GW, true>(a, s);
  if (a.plan.ET == 4) return launch_c<T, 1, 4, false, GW, true>(a, s);
  return launch_c<T, 1, 16, false, GW, true>(a, s);
}

template <typename T>
static cudaError_t launch_t(const RolloutArgs& a, cudaStream_t s) {
  if (a.plan.trn) return a.plan.gw ? launch_trn<T, true>(a, s) : launch_trn<T, false>(a, s);
  if (a.plan.gw) {  // global-weights plans are SIMT, TR = 1
    if (a.plan.ET == 1) return launch_c<T, 1, 1, false, true>(a, s);
    if (a.plan.ET == 4) return launch_c<T, 1, 4, false, true>(a, s);
    return launch_c<T, 1, 16, false, true>(a, s);
  }
  if (a.plan.ET == 1) return launch_c<T, 1, 1>(a, s);
  if (a.plan.ET == 4) return launch_c<T, 1, 4>(a, s);
  if (a.plan.TR == 2) return launch_c<T, 2, 16>(a, s);
  if constexpr (std::is_same<T, double>::value)
    if (a.plan.mma) return launch_c<double, 1, 16, true>(a, s);
  return launch_c<T, 1, 16>(a, s);
}

cudaError_t launch_rollout(const RolloutArgs& a, int precision, cudaStream_t stream) {
  if (a.n_agents <= 0) return cudaSuccess;
  if (a.plan.tc) return launch_rollout_tc(a, a.plan.tcp, stream);
  if (a.plan.oz) return launch_rollout_oz(a, a.plan.tcp, stream);
  if (a.plan.pipe) return launch_pipe(a, stream);
  return (precision == 0 || precision == 3) ? launch_t<double>(a, stream) : launch_t<float>(a, stream);
}

}  // namespace evorl_b200
