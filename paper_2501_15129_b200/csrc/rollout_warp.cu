// rollout_warp.cu -- the population rollout for small policies: one WARP per
// lane (agent a, env j), many warps per CTA, the agent's whole parameter
// vector resident in that warp's shared-memory slot for the horizon.
//
// Used when a lane-team of 256 threads would idle (e = 1 or 2 lanes per
// agent, widths <= 256; BASELINE configs 1, 2 and 4): each warp runs its
// lane's 200-1000 serial env-steps with only __syncwarp() between layers, and
// a CTA carries 1-8 independent lanes so the SM stays full.  Semantics are
// identical to rollout_kernel (proj/src/rollout.cpp:94-174): lane (a, j) is
// keyed fold_in(fold_in(key, a), j); every lane of the warp evaluates the env
// identically (no broadcast needed); hidden layer rows are spread over the
// lanes; the output dot products are reduced by an xor butterfly, whose result
// is bit-identical in every lane (IEEE addition is commutative).
#include <algorithm>
#include <cstring>

#include "kernels.cuh"

namespace evorl_b200 {

template <typename T>
EVB_DEV T cvt(double v);
template <>
EVB_DEV double cvt<double>(double v) {
  return v;
}
template <>
EVB_DEV float cvt<float>(double v) {
  return __double2float_rn(v);
}

EVB_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
EVB_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Per-warp shared-memory slot: W_l stored k-major ([k][rows], rows padded to
// a multiple of 32), biases, then two activation ping-pong buffers.
struct WarpPlan {
  int wpb;            // warps (lanes) per CTA
  int slot_bytes;     // bytes per warp slot
  int rows_p[MAXL];   // padded rows per layer
  int off_w[MAXL], off_b[MAXL];
  int off_act0, off_act1;
};

template <typename T>
__global__ void __launch_bounds__(256) rollout_warp_kernel(const __grid_constant__ RolloutArgs A,
                                                          const __grid_constant__ WarpPlan P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long lane_global = (long long)blockIdx.x * P.wpb + warp;  // over n_agents * e
  const long long total_lanes = (long long)A.n_agents * A.e;
  if (lane_global >= total_lanes) return;  // whole warp exits together
  const int agent_local = (int)(lane_global / A.e);
  const int j = (int)(lane_global % A.e);
  const int agent = A.agent_offset + agent_local;
  const NetDesc& N = A.net;
  const EnvDesc& E = A.env;
  const int L = N.nlayers, O = N.dims[L];
  unsigned char* slot = smem + (size_t)warp * P.slot_bytes;

  // ---------------- prologue: this agent's parameters -> slot (k-major)
  for (int l = 0; l < L; ++l) {
    const int K = N.dims[l], W = N.dims[l + 1], RP = P.rows_p[l];
    T* Ws = reinterpret_cast<T*>(slot + P.off_w[l]);
    T* bs = reinterpret_cast<T*>(slot + P.off_b[l]);
    for (int i = lane; i < K * RP; i += 32) {
      const int k = i / RP, r = i % RP;
      Ws[i] = r < W ? cvt<T>(A.par.params[(long long)agent_local * N.d + N.w_off[l] + (long long)k * W + r])
                    : T(0);
    }
    for (int r = lane; r < RP; r += 32)
      bs[r] = r < W ? cvt<T>(A.par.params[(long long)agent_local * N.d + N.b_off[l] + r]) : T(0);
  }
  __syncwarp();

  // ---------------- lane state (identical in all 32 lanes)
  const int per = A.count / A.e, rem = A.count % A.e;
  const int eps_this = per + (j < rem ? 1 : 0);
  const int slot0 = j * per + min(j, rem);
  LaneEnv s{};
  const DKey lane_key = fold_in(fold_in(A.rollout_key, (uint64_t)agent), (uint64_t)j);
  env_reset(E, fold_in(lane_key, 0), s);
  const NormParams nrm = load_norm(A.norm);
  double ep_ret = 0.0, wc = 0.0, wmean[4] = {0, 0, 0, 0}, wm2[4] = {0, 0, 0, 0};
  int ep_len = 0, eps_done = 0;
  long long steps = 0;
  uint32_t fault = 0, fault_layer = 0;
  T* const act0 = reinterpret_cast<T*>(slot + P.off_act0);  // ping-pong activations (selected, not
  T* const act1 = reinterpret_cast<T*>(slot + P.off_act1);  // indexed: no local-memory array)

  for (int it = 0; eps_done < eps_this && fault == 0 && it < A.max_iters; ++it) {
    double raw[4];
    observe(E, s, raw);
    if (A.track_stats) {  // WelfordStats::add (proj/src/obs_norm.cpp:7-18)
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
    T x0[4];
    for (int i = 0; i < 4; ++i) {
      double v = i < E.obs_dim ? raw[i] : 0.0;
      if (nrm.active && i < E.obs_dim) v = ddiv(dsub(v, nrm.mean[i]), nrm.den[i]);
      x0[i] = cvt<T>(v);
    }
    // hidden layers: lane owns rows lane, lane+32, ...
    int bad = -1;
    for (int l = 0; l < L - 1; ++l) {
      const int K = N.dims[l], W = N.dims[l + 1], RP = P.rows_p[l];
      const T* Ws = reinterpret_cast<const T*>(slot + P.off_w[l]);
      const T* bs = reinterpret_cast<const T*>(slot + P.off_b[l]);
      const T* xin = (l & 1) ? act0 : act1;
      T* hout = (l & 1) ? act1 : act0;
      bool nonfinite = false;
      for (int r0 = 0; r0 < RP; r0 += 128) {  // up to 4 rows per lane per pass
        T acc[4] = {T(0), T(0), T(0), T(0)};
        const int nr = min(4, (RP - r0) / 32);
        for (int k = 0; k < K; ++k) {
          const T xv = l == 0 ? (k == 0 ? x0[0] : k == 1 ? x0[1] : k == 2 ? x0[2] : x0[3]) : xin[k];
          const T* wr = Ws + (size_t)k * RP + r0 + lane;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nr) acc[q] = fma(wr[q * 32], xv, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = r0 + q * 32 + lane;
          if (q < nr && r < W) {
            const T z = acc[q] + bs[r];
            const T h = z > T(0) ? z : T(0);
            if (!isfinite((double)h)) nonfinite = true;
            hout[r] = h;
          }
        }
      }
      if (__any_sync(0xffffffffu, nonfinite) && bad < 0) bad = l;
      __syncwarp();
    }
    // output layer: lane-partial dot products, butterfly-reduced
    double z[8];
    {
      const int l = L - 1, K = N.dims[l], RP = P.rows_p[l];
      const T* Ws = reinterpret_cast<const T*>(slot + P.off_w[l]);
      const T* bs = reinterpret_cast<const T*>(slot + P.off_b[l]);
      const T* xin = (l & 1) ? act0 : act1;
#pragma unroll
      for (int o = 0; o < 8; ++o) {
        if (o >= O) break;
        T part = T(0);
        // linear policy: K = obs_dim <= 4 lives in registers (lane < K only),
        // selected without a dynamic index (which would put x0 in local memory)
        for (int k = lane; k < K; k += 32) {
          const T xk = L == 1 ? (k == 0 ? x0[0] : k == 1 ? x0[1] : k == 2 ? x0[2] : x0[3]) : xin[k];
          part = fma(Ws[(size_t)k * RP + o], xk, part);
        }
        const T tot = warp_sum(part);
        z[o] = (double)(tot + bs[o]);
      }
    }
    __syncwarp();
    bool nonfinite_out = false;
#pragma unroll
    for (int o = 0; o < 8; ++o)
      if (o < O && !isfinite(z[o])) nonfinite_out = true;
    if (bad < 0 && nonfinite_out) bad = L - 1;
    if (bad >= 0) {
      fault = FAULT_NET;
      fault_layer = (uint32_t)bad;
      break;
    }
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
    const uint32_t f = env_step(E, s, action, reward, term, trunc);
    if (f) {
      fault = f;
      break;
    }
    ep_ret = dadd(ep_ret, reward);
    ep_len += 1;
    steps += 1;
    if (term || trunc) {
      if (lane == 0) {
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
  if (lane == 0) {
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
    if (fault) record_fault(A.fault, (uint64_t)((long long)agent * A.e + j), fault, fault_layer);
  }
}

static int a16(int x) { return (x + 15) & ~15; }

bool plan_rollout_warp(const NetDesc& net, int obs_dim, int e, int precision, WarpPlanOut* out) {
  const int ts = (precision == 0 || precision == 3) ? 8 : 4;
  const int L = net.nlayers;
  if (e > 2 || net.dims[L] > 8 || obs_dim > 4) return false;
  WarpPlan p{};
  int off = 0, maxw = 0;
  for (int l = 0; l < L; ++l) {
    const int W = net.dims[l + 1];
    if (l < L - 1 && W > 256) return false;
    const int RP = l < L - 1 ? (W + 31) / 32 * 32 : W;
    p.rows_p[l] = RP;
    p.off_w[l] = off;
    off = a16(off + net.dims[l] * RP * ts);
    p.off_b[l] = off;
    off = a16(off + RP * ts);
    if (l < L - 1) maxw = std::max(maxw, RP);
  }
  p.off_act0 = off;
  off = a16(off + std::max(maxw, 4) * ts);
  p.off_act1 = off;
  off = a16(off + std::max(maxw, 4) * ts);
  p.slot_bytes = off;
  if (off > 100 * 1024) return false;
  p.wpb = std::max(1, std::min(8, (227 * 1024) / off));
  static_assert(sizeof(WarpPlan) <= sizeof(WarpPlanOut), "plan storage");
  std::memcpy(out, &p, sizeof p);
  return true;
}

cudaError_t launch_rollout_warp(const RolloutArgs& a, const WarpPlanOut& po, int precision,
                                cudaStream_t stream) {
  WarpPlan p;
  std::memcpy(&p, &po, sizeof p);
  const long long lanes = (long long)a.n_agents * a.e;
  if (lanes <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)((lanes + p.wpb - 1) / p.wpb);
  const size_t smem = (size_t)p.wpb * p.slot_bytes;
  if (precision == 0 || precision == 3) {  // EVORL_PREC_OZ: small policies run the fp64 warp team
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(rollout_warp_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      set = true;
    }
    rollout_warp_kernel<double><<<grid, 32 * p.wpb, smem, stream>>>(a, p);
  } else {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(rollout_warp_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      set = true;
    }
    rollout_warp_kernel<float><<<grid, 32 * p.wpb, smem, stream>>>(a, p);
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace evorl_b200
