// kernels.cu -- noise, ranks, fitness reduction, EC tells, observation
// statistics and init for the B200 generation path.  Every kernel cites the
// reference function it restates.
#include <algorithm>
#include <atomic>
#include <cstdio>

#include "kernels.cuh"

namespace evorl_b200 {

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
long long kernel_launch_count() { return g_launches.load(); }

#define EVB_CHECK_LAUNCH() \
  do {                     \
    count_launch();        \
    return cudaGetLastError(); \
  } while (0)

static unsigned blocks_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 2147483647LL) b = 2147483647LL;
  return (unsigned)b;
}

// ----------------------------------------------------------------- noise
__global__ void k_threefry_batch(const uint64_t* keys, const uint64_t* ctrs, uint64_t* out, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  threefry2x64(keys[2 * i], keys[2 * i + 1], ctrs[2 * i], ctrs[2 * i + 1], out[2 * i], out[2 * i + 1]);
}
cudaError_t run_threefry_batch(const uint64_t* keys, const uint64_t* ctrs, uint64_t* out, long long n,
                               cudaStream_t s) {
  k_threefry_batch<<<blocks_for(n, 256), 256, 0, s>>>(keys, ctrs, out, n);
  EVB_CHECK_LAUNCH();
}

__global__ void k_stream_words(DKey key, long long first, long long n, uint64_t* out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = stream_word(key, (uint64_t)(first + i));
}
cudaError_t run_stream_words(DKey key, long long first, long long n, uint64_t* out, cudaStream_t s) {
  k_stream_words<<<blocks_for(n, 256), 256, 0, s>>>(key, first, n, out);
  EVB_CHECK_LAUNCH();
}

// gaussian_matrix (proj/src/ec.cpp:22-28): normal #idx of one stream,
// row-major.  One thread per Box-Muller block (two normals).
__global__ void k_gaussian_matrix(DKey key, long long total, double* out) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (2 * b >= total) return;
  double c, s;
  normal_pair(key, (uint64_t)b, c, s);
  out[2 * b] = c;
  if (2 * b + 1 < total) out[2 * b + 1] = s;
}
cudaError_t run_gaussian_matrix(DKey key, long long rows, long long cols, double* out, cudaStream_t s) {
  const long long total = rows * cols;
  if (total <= 0) return cudaSuccess;
  k_gaussian_matrix<<<blocks_for((total + 1) / 2, 256), 256, 0, s>>>(key, total, out);
  EVB_CHECK_LAUNCH();
}

// ----------------------------------------------------------------- ranks
// Order-preserving u64 image of a double; -0.0 and +0.0 compare equal in the
// reference (operator<), so both map to the image of +0.0.
EVB_DEV uint64_t ordered_key(double x) {
  if (x == 0.0) x = 0.0;
  const uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// Stable rank by counting (std::stable_sort semantics, proj/src/ec.cpp:14-46):
// rank[i] = #{j : key_j < key_i} + #{j < i : key_j == key_i}.  Exact and
// deterministic; one thread per element, keys tiled through shared memory.
__global__ void k_rank(const double* keys, int n, int desc, int* rank) {
  __shared__ uint64_t tile[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t ki = 0;
  if (i < n) {
    ki = ordered_key(keys[i]);
    if (desc) ki = ~ki;
  }
  int r = 0;
  for (int t0 = 0; t0 < n; t0 += 256) {
    const int j = t0 + threadIdx.x;
    if (j < n) {
      uint64_t kj = ordered_key(keys[j]);
      tile[threadIdx.x] = desc ? ~kj : kj;
    }
    __syncthreads();
    const int lim = min(256, n - t0);
    if (i < n) {
      for (int q = 0; q < lim; ++q) {
        const uint64_t kj = tile[q];
        r += (kj < ki) || (kj == ki && (t0 + q) < i);
      }
    }
    __syncthreads();
  }
  if (i < n) rank[i] = r;
}
// Stable LSD radix sort (4-bit digits) of the order-preserving key images in
// one CTA of 1024 threads: thread t owns a contiguous chunk; per pass a
// digit-major / thread-minor histogram is exclusive-scanned, so equal digits
// keep thread order then chunk order (stability, i.e. std::stable_sort's tie
// rule).  Passes whose digit is constant over all keys are skipped.  Output:
// rank[i] = position of i.  Scratch: 2n u64 + 2n int in global memory.
constexpr int RADIX_T = 1024;
__global__ void __launch_bounds__(RADIX_T) k_radix_rank(const double* keys, int n, int desc, uint64_t* kb,
                                                        int* ib, int* rank) {
  __shared__ uint16_t hist[16][RADIX_T];
  __shared__ uint32_t wsum[RADIX_T / 32];
  __shared__ int any_split;
  const int t = threadIdx.x;
  const int chunk = (n + RADIX_T - 1) / RADIX_T;
  const int i0 = min(n, t * chunk), i1 = min(n, i0 + chunk);
  uint64_t* k0 = kb;
  uint64_t* k1 = kb + n;
  int* x0 = ib;
  int* x1 = ib + n;
  for (int i = i0; i < i1; ++i) {
    const uint64_t k = ordered_key(keys[i]);
    k0[i] = desc ? ~k : k;
    x0[i] = i;
  }
  __syncthreads();
  for (int pass = 0; pass < 16; ++pass) {
    const int shift = 4 * pass;
    for (int d = 0; d < 16; ++d) hist[d][t] = 0;
    if (t == 0) any_split = 0;
    __syncthreads();
    for (int i = i0; i < i1; ++i) ++hist[(k0[i] >> shift) & 15][t];
    __syncthreads();
    // skip the pass if one digit holds every key (common for high bits)
    if (t < 16) {
      uint32_t c = 0;
      for (int q = 0; q < RADIX_T; ++q) c += hist[t][q];
      if (c != 0 && c != (uint32_t)n) any_split = 1;
    }
    __syncthreads();
    if (!any_split) continue;
    // exclusive scan of the 16 x 1024 counts in (digit, thread) order:
    // thread t owns linear entries [16t, 16t + 16)
    uint16_t* flat = &hist[0][0];
    uint32_t local = 0;
    for (int q = 0; q < 16; ++q) local += flat[16 * t + q];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((t & 31) >= o) incl += v;
    }
    if ((t & 31) == 31) wsum[t >> 5] = incl;
    __syncthreads();
    if (t < 32) {
      uint32_t w = wsum[t];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
        if (t >= o) w += v;
      }
      wsum[t] = w;  // inclusive over warps
    }
    __syncthreads();
    // exclusive start offset of each owned (digit, thread) entry; the 16x1024
    // offsets (u32: they exceed u16) are published through the idle output
    // key buffer k1 (>= 8192 u64 = 16384 u32 since n >= 8192 on this path)
    uint32_t run = incl - local + ((t >> 5) ? wsum[(t >> 5) - 1] : 0u);
    uint32_t* offs = reinterpret_cast<uint32_t*>(k1);
    for (int q = 0; q < 16; ++q) {
      offs[16 * t + q] = run;
      run += flat[16 * t + q];
    }
    __syncthreads();
    // this thread's column (d, t) lives at linear 1024*d + t
    uint32_t my[16];
    for (int d = 0; d < 16; ++d) my[d] = offs[RADIX_T * d + t];
    __syncthreads();  // k1 is overwritten by the scatter below
    for (int i = i0; i < i1; ++i) {
      const uint64_t k = k0[i];
      const int d = (int)((k >> shift) & 15);
      const uint32_t p = my[d]++;
      k1[p] = k;
      x1[p] = x0[i];
    }
    __syncthreads();
    uint64_t* tk = k0;
    k0 = k1;
    k1 = tk;
    int* tx = x0;
    x0 = x1;
    x1 = tx;
  }
  for (int i = i0; i < i1; ++i) rank[x0[i]] = i;
}

static uint64_t* g_radix_k = nullptr;
static int* g_radix_i = nullptr;
static int g_radix_cap = 0;

cudaError_t run_rank(const double* keys, int n, int desc, int* rank, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n < 8192) {  // O(n^2 / P) counting is faster than 16 serial passes here
    k_rank<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, desc, rank);
    EVB_CHECK_LAUNCH();
  }
  if (n > g_radix_cap) {
    cudaStreamSynchronize(s);
    if (g_radix_k) cudaFree(g_radix_k);
    if (g_radix_i) cudaFree(g_radix_i);
    // k needs 2n u64 (+ the 16 x 1024 u32 offset table in the spare half)
    const size_t kn = std::max<size_t>(2 * (size_t)n, (size_t)n + 16 * RADIX_T / 2 + 1);
    if (cudaMalloc(&g_radix_k, sizeof(uint64_t) * kn) != cudaSuccess) return cudaErrorMemoryAllocation;
    if (cudaMalloc(&g_radix_i, sizeof(int) * 2 * (size_t)n) != cudaSuccess) return cudaErrorMemoryAllocation;
    g_radix_cap = n;
  }
  k_radix_rank<<<1, RADIX_T, 0, s>>>(keys, n, desc, g_radix_k, g_radix_i, rank);
  EVB_CHECK_LAUNCH();
}

// centered_ranks (proj/src/ec.cpp:39-45): rank / (n - 1) - 0.5; n == 1 -> 0.
__global__ void k_shaped(const int* rank, int n, double* shaped) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  shaped[i] = n == 1 ? 0.0 : dsub(ddiv((double)rank[i], (double)(n - 1)), 0.5);
}
cudaError_t run_shaped_from_rank(const int* rank, int n, double* shaped, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_shaped<<<blocks_for(n, 256), 256, 0, s>>>(rank, n, shaped);
  EVB_CHECK_LAUNCH();
}
__global__ void k_order(const int* rank, int n, int* order) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) order[rank[i]] = i;
}
cudaError_t run_order_from_rank(const int* rank, int n, int* order, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_order<<<blocks_for(n, 256), 256, 0, s>>>(rank, n, order);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------------- fitness reduction
// proj/src/workflow_es.cpp:127-135: fitness = (sum of the agent's episode
// returns in lane-major order) / count; env_steps += steps.
__global__ void k_fitness(const double* ep_returns, int count, int n_agents, int agent_offset,
                          double* fitness, const long long* lane_steps, int e,
                          unsigned long long* steps_accum) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_agents) return;
  double sum = 0.0;
  for (int q = 0; q < count; ++q) sum = dadd(sum, ep_returns[(long long)a * count + q]);
  fitness[agent_offset + a] = ddiv(sum, (double)count);
  if (steps_accum) {
    long long st = 0;
    for (int j = 0; j < e; ++j) st += lane_steps[(long long)a * e + j];
    atomicAdd(steps_accum, (unsigned long long)st);
  }
}
cudaError_t run_fitness(const double* ep_returns, int count, int n_agents, int agent_offset,
                        double* fitness, const long long* lane_steps, int e,
                        unsigned long long* steps_accum, cudaStream_t s) {
  if (n_agents <= 0) return cudaSuccess;
  k_fitness<<<blocks_for(n_agents, 128), 128, 0, s>>>(ep_returns, count, n_agents, agent_offset, fitness,
                                                      lane_steps, e, steps_accum);
  EVB_CHECK_LAUNCH();
}

// fitness.mean()/maxCoeff()/minCoeff() (proj/src/workflow_es.cpp:166-168):
// fixed-order block reduction (chunked sequential sums, then a fixed tree).
__global__ void k_metrics(const double* f, int n, double* out) {
  __shared__ double ssum[256], smax[256], smin[256];
  const int t = threadIdx.x;
  const int chunk = (n + 255) / 256;
  double s = 0.0, mx = -INFINITY, mn = INFINITY;
  for (int i = t * chunk; i < min(n, (t + 1) * chunk); ++i) {
    s = dadd(s, f[i]);
    mx = fmax(mx, f[i]);
    mn = fmin(mn, f[i]);
  }
  ssum[t] = s;
  smax[t] = mx;
  smin[t] = mn;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) {
      ssum[t] = dadd(ssum[t], ssum[t + w]);
      smax[t] = fmax(smax[t], smax[t + w]);
      smin[t] = fmin(smin[t], smin[t + w]);
    }
    __syncthreads();
  }
  if (t == 0) {
    out[0] = ddiv(ssum[0], (double)n);
    out[1] = smax[0];
    out[2] = smin[0];
  }
}
cudaError_t run_metrics(const double* f, int n, double* out, cudaStream_t s) {
  k_metrics<<<1, 256, 0, s>>>(f, n, out);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------------------- OpenES tell
// openes_tell (proj/src/ec.cpp:99-109) fused with adam_step
// (proj/src/optim.cpp:7-17).  g_p = sum_i eps_i[p] * shaped_i / (n sigma),
// eps regenerated from the ask key; with block mirroring eps_{i+base} =
// -eps_i, so g_p = sum_{i<base} eps_i[p] (shaped_i - shaped_{i+base}) / (n sigma).
// Each thread owns V consecutive coordinates so one Box-Muller block feeds
// two of them (normal #2b -> cos, #2b+1 -> sin).
constexpr int TELL_V = 8;
constexpr int TELL_T = 128;
// Partial contraction of one row chunk: partial[chunk][p - p0] =
// sum_{i in chunk} eps_i[p] w_i (sequential fma over the chunk's rows).
__global__ void __launch_bounds__(TELL_T) k_openes_tell_partial(const OpenEsTellArgs a, int chunk_rows) {
  __shared__ double wsh[1024];
  const long long pbase = a.p0 + (blockIdx.x * (long long)blockDim.x + threadIdx.x) * TELL_V;
  const int rows = a.mirrored ? a.base : a.n;
  const int r0 = blockIdx.y * chunk_rows, r1 = min(rows, r0 + chunk_rows);
  double acc[TELL_V];
#pragma unroll
  for (int v = 0; v < TELL_V; ++v) acc[v] = 0.0;
  for (int i0 = r0; i0 < r1; i0 += 1024) {
    const int lim = min(1024, r1 - i0);
    __syncthreads();
    for (int q = threadIdx.x; q < lim; q += blockDim.x) {
      const int i = i0 + q;
      wsh[q] = a.mirrored ? dsub(a.shaped[i], a.shaped[i + a.base]) : a.shaped[i];
    }
    __syncthreads();
    if (pbase < a.p1 && a.table != nullptr) {  // noise-table rows (proj/src/ec.cpp:79-86)
      for (int q = 0; q < lim; ++q) {
        const double w = wsh[q];
        const double* row = a.table + a.offsets[i0 + q] + pbase;
#pragma unroll
        for (int v = 0; v < TELL_V; ++v)
          if (pbase + v < a.p1) acc[v] = fma(row[v], w, acc[v]);
      }
    } else if (pbase < a.p1) {
      for (int q = 0; q < lim; ++q) {
        const double w = wsh[q];
        const uint64_t k0 = (uint64_t)((long long)(i0 + q) * a.d + pbase);
        // blocks covering normals [k0, k0 + V) (the two alignments spelled out
        // so every acc index is a compile-time constant: acc stays in registers)
        uint64_t b = k0 >> 1;
        double c, sn;
        if (k0 & 1) {  // first coordinate is the sin half of block b
          normal_pair(a.ask_key, b++, c, sn);
          acc[0] = fma(sn, w, acc[0]);
#pragma unroll
          for (int vv = 1; vv < TELL_V; vv += 2) {
            normal_pair(a.ask_key, b++, c, sn);
            acc[vv] = fma(c, w, acc[vv]);
            if (vv + 1 < TELL_V) acc[vv + 1] = fma(sn, w, acc[vv + 1]);
          }
        } else {
#pragma unroll
          for (int vv = 0; vv < TELL_V; vv += 2) {
            normal_pair(a.ask_key, b++, c, sn);
            acc[vv] = fma(c, w, acc[vv]);
            acc[vv + 1] = fma(sn, w, acc[vv + 1]);
          }
        }
      }
    }
  }
  if (pbase >= a.p1) return;
  const long long span = a.p1 - a.p0;
  double* out = a.partial + (long long)blockIdx.y * span + (pbase - a.p0);
#pragma unroll
  for (int v = 0; v < TELL_V; ++v)
    if (pbase + v < a.p1) out[v] = acc[v];
}

// The same contraction with the noise rows kept by the ask
// (run_materialize's eps_out): one coordinate per thread, so every row is a
// coalesced read.  Each coordinate accumulates the rows of its chunk in the
// same order as k_openes_tell_partial, so the partials are bit-identical.
__global__ void __launch_bounds__(TELL_T) k_openes_tell_rows(const OpenEsTellArgs a, int chunk_rows) {
  __shared__ double wsh[1024];
  const long long p = a.p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int rows = a.mirrored ? a.base : a.n;
  const int r0 = blockIdx.y * chunk_rows, r1 = min(rows, r0 + chunk_rows);
  double acc = 0.0;
  for (int i0 = r0; i0 < r1; i0 += 1024) {
    const int lim = min(1024, r1 - i0);
    __syncthreads();
    for (int q = threadIdx.x; q < lim; q += blockDim.x) {
      const int i = i0 + q;
      wsh[q] = a.mirrored ? dsub(a.shaped[i], a.shaped[i + a.base]) : a.shaped[i];
    }
    __syncthreads();
    if (p < a.p1) {
      const long long ld = a.eps_ld;
      const double* col = a.eps_rows + (long long)i0 * ld + (p - a.eps_p0);
      int q = 0;
      for (; q + 4 <= lim; q += 4) {  // four rows' loads in flight
        const double e0 = __ldcs(col), e1 = __ldcs(col + ld), e2 = __ldcs(col + 2 * ld),
                     e3 = __ldcs(col + 3 * ld);
        acc = fma(e0, wsh[q], acc);
        acc = fma(e1, wsh[q + 1], acc);
        acc = fma(e2, wsh[q + 2], acc);
        acc = fma(e3, wsh[q + 3], acc);
        col += 4 * ld;
      }
      for (; q < lim; ++q, col += ld) acc = fma(__ldcs(col), wsh[q], acc);
    }
  }
  if (p >= a.p1) return;
  a.partial[(long long)blockIdx.y * (a.p1 - a.p0) + (p - a.p0)] = acc;
}

// g_p = sum over chunks (fixed order) / (n sigma), then adam_step.
__global__ void k_openes_adam(const OpenEsTellArgs a, int chunks) {
  const long long p = a.p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= a.p1 || p >= a.d) return;
  const long long span = a.p1 - a.p0;
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) acc = dadd(acc, a.partial[(long long)c * span + (p - a.p0)]);
  const long long t = *a.t_dev + 1;
  double bc1, bc2;
  if (t <= a.adam_bc_len) {
    bc1 = a.adam_bc[2 * (t - 1)];
    bc2 = a.adam_bc[2 * (t - 1) + 1];
  } else {
    bc1 = 1.0 - pow(a.beta1, (double)t);
    bc2 = 1.0 - pow(a.beta2, (double)t);
  }
  const double denom = dmul((double)a.n, a.sigma);
  const double grad = -ddiv(acc, denom);  // Adam descends along -g
  const double m = dadd(dmul(a.beta1, a.m[p]), dmul(a.omb1, grad));
  const double vv = dadd(dmul(a.beta2, a.v[p]), dmul(a.omb2, dmul(grad, grad)));
  double prm = a.mean[p];
  prm = dsub(prm, ddiv(dmul(a.lr, ddiv(m, bc1)), dadd(sqrt(ddiv(vv, bc2)), a.eps)));
  if (a.weight_decay != 0.0) prm = dsub(prm, dmul(a.lrwd, prm));
  a.m[p] = m;
  a.v[p] = vv;
  a.mean[p] = prm;
}

int openes_tell_chunks(int rows, long long d) {
  // fill ~8 resident CTAs of TELL_T threads per SM over 148 SMs, keeping
  // >= 32 rows per chunk so the Box-Muller work dominates the partial traffic.
  // Sized from the FULL dimension d, never from a shard's span: the row-chunk
  // boundaries fix the summation order of g_p, which must not depend on the
  // world size (dist.py: bit-identical results for any sharding).
  const long long coord_threads = (d + TELL_V - 1) / TELL_V;
  const long long want = (148LL * 8 * TELL_T + coord_threads - 1) / std::max(1LL, coord_threads);
  const long long by_rows = std::max(1, rows / 32);
  return (int)std::max(1LL, std::min({want, by_rows, 256LL}));
}

cudaError_t run_openes_tell(const OpenEsTellArgs& a, cudaStream_t s) {
  const long long span = a.p1 - a.p0;
  if (span <= 0) return cudaSuccess;
  const int rows = a.mirrored ? a.base : a.n;
  const int chunks = openes_tell_chunks(rows, a.d);
  const int chunk_rows = (rows + chunks - 1) / chunks;
  if (a.eps_rows && !a.table) {
    dim3 grid((unsigned)((span + TELL_T - 1) / TELL_T), (unsigned)chunks);
    k_openes_tell_rows<<<grid, TELL_T, 0, s>>>(a, chunk_rows);
  } else {
    const long long threads = (span + TELL_V - 1) / TELL_V;
    dim3 grid((unsigned)((threads + TELL_T - 1) / TELL_T), (unsigned)chunks);
    k_openes_tell_partial<<<grid, TELL_T, 0, s>>>(a, chunk_rows);
  }
  k_openes_adam<<<blocks_for(span, 256), 256, 0, s>>>(a, chunks);
  EVB_CHECK_LAUNCH();
}

__global__ void k_inc(long long* t) { *t += 1; }
cudaError_t run_inc_counter(long long* t, cudaStream_t s) {
  k_inc<<<1, 1, 0, s>>>(t);
  EVB_CHECK_LAUNCH();
}

// openes_ask materialised (proj/src/ec.cpp:71-97), for the parity ABI.
__global__ void k_openes_ask(const double* mean, long long d, double sigma, int mirrored, DKey key, int n,
                             double* cand, double* eps) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * d) return;
  const long long i = idx / d, p = idx % d;
  const int base = mirrored ? n / 2 : n;
  long long row = i;
  bool neg = false;
  if (mirrored && i >= base) {
    row = i - base;
    neg = true;
  }
  double e = normal_at(key, (uint64_t)(row * d + p));
  if (neg) e = -e;
  if (eps) eps[idx] = e;
  if (cand) cand[idx] = dadd(dmul(sigma, e), mean[p]);
}
cudaError_t run_openes_ask(const double* mean, long long d, double sigma, int mirrored, DKey key, int n,
                           double* cand, double* eps, cudaStream_t s) {
  k_openes_ask<<<blocks_for((long long)n * d, 256), 256, 0, s>>>(mean, d, sigma, mirrored, key, n, cand, eps);
  EVB_CHECK_LAUNCH();
}

// ---------------------------------------------------------------- ARS
__global__ void k_ars_ask(const double* mean, long long d, double sigma, DKey key, int n, double* deltas,
                          double* cand) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int half = n / 2;
  if (idx >= (long long)half * d) return;
  const long long k = idx / d, p = idx % d;
  const double dl = normal_at(key, (uint64_t)idx);
  if (deltas) deltas[idx] = dl;
  if (cand) {
    const double sd = dmul(sigma, dl);
    cand[(2 * k) * d + p] = dadd(mean[p], sd);
    cand[(2 * k + 1) * d + p] = dsub(mean[p], sd);
  }
}
cudaError_t run_ars_ask(const double* mean, long long d, double sigma, DKey key, int n, double* deltas,
                        double* cand, cudaStream_t s) {
  k_ars_ask<<<blocks_for((long long)(n / 2) * d, 256), 256, 0, s>>>(mean, d, sigma, key, n, deltas, cand);
  EVB_CHECK_LAUNCH();
}

// scores = r_plus.cwiseMax(r_minus) with r_plus = fitness[2k], r_minus =
// fitness[2k+1] (proj/src/workflow_es.cpp:146-151, proj/src/ec.cpp:133)
__global__ void k_ars_scores(const double* f, int half, double* scores) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= half) return;
  const double rp = f[2 * k], rm = f[2 * k + 1];
  scores[k] = rp < rm ? rm : rp;
}
cudaError_t run_ars_scores(const double* f, int half, double* scores, cudaStream_t s) {
  k_ars_scores<<<blocks_for(half, 256), 256, 0, s>>>(f, half, scores);
  EVB_CHECK_LAUNCH();
}

// Elites = the b directions of lowest descending rank; sigma_R = population
// std of the 2b elite rewards [r+_0, r-_0, r+_1, ...] (proj/src/ec.cpp:131-147).
__global__ void k_ars_select(const double* f, const int* rank, int half, int elites, double lr,
                             int* elite_idx, double* elite_diff, ArsSel* sel) {
  const int b = min(elites, half);
  for (int k = threadIdx.x; k < half; k += blockDim.x)
    if (rank[k] < b) elite_idx[rank[k]] = k;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double sum = 0.0;
  for (int k = 0; k < b; ++k) {
    sum = dadd(sum, f[2 * elite_idx[k]]);
    sum = dadd(sum, f[2 * elite_idx[k] + 1]);
  }
  const double mean = ddiv(sum, (double)(2 * b));
  double sq = 0.0;
  for (int k = 0; k < b; ++k) {
    const double a0 = dsub(f[2 * elite_idx[k]], mean), a1 = dsub(f[2 * elite_idx[k] + 1], mean);
    sq = dadd(sq, dmul(a0, a0));
    sq = dadd(sq, dmul(a1, a1));
  }
  const double sigma_r = sqrt(ddiv(sq, (double)(2 * b)));
  for (int k = 0; k < b; ++k) elite_diff[k] = dsub(f[2 * elite_idx[k]], f[2 * elite_idx[k] + 1]);
  sel->b = b;
  sel->sigma_r = sigma_r;
  sel->skipped = sigma_r == 0.0 ? 1 : 0;
  sel->scale = sigma_r == 0.0 ? 0.0 : ddiv(lr, dmul((double)b, sigma_r));
}
cudaError_t run_ars_select(const double* f, const int* rank, int half, int elites, double lr, int* elite_idx,
                           double* elite_diff, ArsSel* sel, cudaStream_t s) {
  k_ars_select<<<1, 256, 0, s>>>(f, rank, half, elites, lr, elite_idx, elite_diff, sel);
  EVB_CHECK_LAUNCH();
}

// mean += scale * sum_k diff_k * delta_{idx_k}  (step accumulated from zero in
// elite order, proj/src/ec.cpp:149-152)
__global__ void k_ars_update(double* mean, long long p0, long long p1, long long d, DKey key,
                             const int* elite_idx, const double* elite_diff, const ArsSel* sel) {
  const long long p = p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= p1 || sel->skipped) return;
  double step = 0.0;
  for (int k = 0; k < sel->b; ++k)
    step = dadd(step, dmul(elite_diff[k], normal_at(key, (uint64_t)((long long)elite_idx[k] * d + p))));
  mean[p] = dadd(mean[p], dmul(sel->scale, step));
}
cudaError_t run_ars_update(double* mean, long long d, long long p0, long long p1, DKey key,
                           const int* elite_idx, const double* elite_diff, const ArsSel* sel,
                           cudaStream_t s) {
  if (p1 <= p0) return cudaSuccess;
  k_ars_update<<<blocks_for(p1 - p0, 256), 256, 0, s>>>(mean, p0, p1, d, key, elite_idx, elite_diff, sel);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------------------- VES / CEM
// ves_tell (proj/src/ec.cpp:177-187): mean = sum_{i<mu} w_i cand_{order_i},
// cand regenerated as (sigma * eps) + mean_old.
__global__ void k_ves_tell(double* mean, long long d, long long p0, long long p1, double sigma,
                           int mirrored, int base, DKey key, const int* order, const double* w, int mu) {
  const long long p = p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const double m0 = mean[p];
  double acc = 0.0;
  for (int i = 0; i < mu; ++i) {
    const int a = order[i];
    long long row = a;
    bool neg = false;
    if (mirrored && a >= base) {
      row = a - base;
      neg = true;
    }
    double e = normal_at(key, (uint64_t)(row * d + p));
    if (neg) e = -e;
    acc = dadd(acc, dmul(w[i], dadd(dmul(sigma, e), m0)));
  }
  mean[p] = acc;
}
cudaError_t run_ves_tell(double* mean, long long d, long long p0, long long p1, double sigma, int mirrored,
                         int base, DKey key, const int* order, const double* w, int mu, cudaStream_t s) {
  if (p1 <= p0) return cudaSuccess;
  k_ves_tell<<<blocks_for(p1 - p0, 256), 256, 0, s>>>(mean, d, p0, p1, sigma, mirrored, base, key, order,
                                                       w, mu);
  EVB_CHECK_LAUNCH();
}

// cem_tell (proj/src/ec.cpp:315-336): elite mean, elite population variance
// plus the decaying floor; candidates regenerated as z * sqrt(var) + mean.
__global__ void k_cem_tell(double* mean, double* var, long long d, long long p0, long long p1, DKey key,
                           const int* order, int h, double floor_) {
  const long long p = p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p >= p1) return;
  const double m0 = mean[p], sd = sqrt(var[p]);
  double mu = 0.0;
  for (int i = 0; i < h; ++i)
    mu = dadd(mu, dadd(dmul(normal_at(key, (uint64_t)((long long)order[i] * d + p)), sd), m0));
  mu = ddiv(mu, (double)h);
  double vs = 0.0;
  for (int i = 0; i < h; ++i) {
    const double x = dsub(dadd(dmul(normal_at(key, (uint64_t)((long long)order[i] * d + p)), sd), m0), mu);
    vs = dadd(vs, dmul(x, x));
  }
  vs = ddiv(vs, (double)h);
  mean[p] = mu;
  var[p] = dadd(vs, floor_);
}
cudaError_t run_cem_tell(double* mean, double* var, long long d, long long p0, long long p1, DKey key,
                         const int* order, int h, double floor_, cudaStream_t s) {
  if (p1 <= p0) return cudaSuccess;
  k_cem_tell<<<blocks_for(p1 - p0, 256), 256, 0, s>>>(mean, var, d, p0, p1, key, order, h, floor_);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------- observation statistics
struct W9 {
  double c, m[4], q[4];
};
// WelfordStats::merge (proj/src/obs_norm.cpp:20-31)
EVB_DEV void welford_merge(W9& w, const W9& o, int dim) {
  if (o.c == 0.0) return;
  if (w.c == 0.0) {
    w = o;
    return;
  }
  const double total = dadd(w.c, o.c);
  const double s = ddiv(dmul(w.c, o.c), total);
  const double f = ddiv(o.c, total);
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // registers, not local memory
    if (i >= dim) break;
    const double delta = dsub(o.m[i], w.m[i]);
    w.q[i] = dadd(w.q[i], dadd(o.q[i], dmul(dmul(delta, delta), s)));
    w.m[i] = dadd(w.m[i], dmul(delta, f));
  }
  w.c = total;
}
EVB_DEV W9 load9(const double* p) {
  W9 w;
  w.c = p[0];
  for (int i = 0; i < 4; ++i) {
    w.m[i] = p[1 + i];
    w.q[i] = p[5 + i];
  }
  return w;
}

// lane-major merge per agent (proj/src/rollout.cpp:195-209)
__global__ void k_agent_stats(const double* lane_stats, int n_agents, int e, int dim, double* agent_stats) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n_agents) return;
  W9 w{};
  for (int j = 0; j < e; ++j) welford_merge(w, load9(lane_stats + ((long long)a * e + j) * 9), dim);
  double* o = agent_stats + (long long)a * 9;
  o[0] = w.c;
  for (int i = 0; i < 4; ++i) {
    o[1 + i] = w.m[i];
    o[5 + i] = w.q[i];
  }
}
cudaError_t run_agent_stats(const double* lane_stats, int n_agents, int e, double* agent_stats,
                            cudaStream_t s) {
  k_agent_stats<<<blocks_for(n_agents, 128), 128, 0, s>>>(lane_stats, n_agents, e, 4, agent_stats);
  EVB_CHECK_LAUNCH();
}

EVB_DEV void norm_params_from(const DevNorm& nm, NormParams& p) {
  p.active = (nm.mode != 0 && nm.count != 0.0) ? 1 : 0;
  p.dim = nm.dim;
  for (int i = 0; i < 4; ++i) {
    p.mean[i] = nm.mean[i];
    const double sd = sqrt(nm.var[i]);
    p.den[i] = sd > 1e-8 ? sd : 1e-8;  // .sqrt().max(1e-8)
  }
}

// Agent merge (proj/src/workflow_es.cpp:136) then rs_update
// (proj/src/obs_norm.cpp:56-68) into the device ObsNormState.  The reference
// merges agents sequentially; Welford merging is exact in real arithmetic but
// not associative in floating point, so this fixed-order tree (each thread
// folds a contiguous run of agents, then a pairwise tree in rank order) differs
// from it only in rounding (~1e-16 rel), is deterministic, and replaces a
// 1024-long serial dependency chain with ~10 levels.
constexpr int RS_THREADS = 256;
__global__ void k_rs_update(const double* agent_stats, int n_agents, DevNorm* norm, NormParams* params) {
  __shared__ W9 tree[RS_THREADS];
  const int t = threadIdx.x;
  const int dim = norm->dim;
  const int chunk = (n_agents + RS_THREADS - 1) / RS_THREADS;
  W9 w{};
  for (int a = t * chunk; a < min(n_agents, (t + 1) * chunk); ++a)
    welford_merge(w, load9(agent_stats + (long long)a * 9), dim);
  tree[t] = w;
  __syncthreads();
  for (int stride = 1; stride < RS_THREADS; stride *= 2) {
    if ((t % (2 * stride)) == 0) welford_merge(tree[t], tree[t + stride], dim);
    __syncthreads();
  }
  if (t != 0) return;
  const W9 batch = tree[0];
  DevNorm nm = *norm;
  if (nm.mode == 2 && batch.c != 0.0) {
    W9 cur{};
    if (nm.count > 0.0) {
      cur.c = nm.count;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // registers, not local memory
        if (i >= dim) break;
        cur.m[i] = nm.mean[i];
        cur.q[i] = dmul(nm.var[i], nm.count);
      }
    }
    welford_merge(cur, batch, dim);
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // registers, not local memory
      if (i >= dim) break;
      nm.mean[i] = cur.m[i];
      nm.var[i] = cur.c == 0.0 ? cur.m[i] : ddiv(cur.q[i], cur.c);
    }
    nm.count = cur.c;
    *norm = nm;
  }
  norm_params_from(nm, *params);
}
cudaError_t run_rs_merge(const double* lane_stats, int n_agents, int e, DevNorm* norm, NormParams* params,
                         double* agent_scratch, cudaStream_t s) {
  cudaError_t err = run_agent_stats(lane_stats, n_agents, e, agent_scratch, s);
  if (err != cudaSuccess) return err;
  k_rs_update<<<1, RS_THREADS, 0, s>>>(agent_scratch, n_agents, norm, params);
  EVB_CHECK_LAUNCH();
}

__global__ void k_norm_params(const DevNorm* norm, NormParams* params) {
  if (threadIdx.x == 0) norm_params_from(*norm, *params);
}
cudaError_t run_norm_params(const DevNorm* norm, NormParams* params, cudaStream_t s) {
  k_norm_params<<<1, 32, 0, s>>>(norm, params);
  EVB_CHECK_LAUNCH();
}

// vbn_fit (proj/src/rollout.cpp:216-224): one lane of n uniform-random steps
// with auto-resets, Welford stats of the raw observations, frozen as VBN.
// Inherently serial (one lane); runs once at init.
__global__ void k_vbn_fit(EnvDesc env, DKey lane_key, int n, DevNorm* norm, NormParams* params) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  LaneEnv s;
  env_reset(env, fold_in(lane_key, 0), s);
  const DKey sk = fold_in(lane_key, 1);
  uint64_t word = 0;
  W9 w{};
  const int dim = env.obs_dim;
  for (int t = 0; t < n; ++t) {
    double raw[4];
    observe(env, s, raw);
    if (w.c == 0.0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // registers, not local memory
        if (i >= dim) break;
        w.m[i] = raw[i];
        w.q[i] = 0.0;
      }
      w.c = 1.0;
    } else {
      w.c = dadd(w.c, 1.0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // registers, not local memory
        if (i >= dim) break;
        const double delta = dsub(raw[i], w.m[i]);
        w.m[i] = dadd(w.m[i], ddiv(delta, w.c));
        w.q[i] = dadd(w.q[i], dmul(delta, dsub(raw[i], w.m[i])));
      }
    }
    double action;
    if (env.discrete) {  // randint(num_actions), proj/src/rng.cpp:89-96
      const uint64_t nn = (uint64_t)env.num_actions;
      const uint64_t m = (~0ull % nn + 1) % nn;
      for (;;) {
        const uint64_t x = stream_word(sk, word++);
        if (m == 0 || x < 0ull - m) {
          action = (double)(x % nn);
          break;
        }
      }
    } else {
      action = uniform_range(env.act_low, env.act_high, word_to_uniform(stream_word(sk, word++)));
    }
    double reward;
    bool term, trunc;
    env_step(env, s, action, reward, term, trunc);
    if (term || trunc) env_reset(env, s.rng, s);
  }
  DevNorm nm{};
  nm.mode = 1;
  nm.dim = dim;
#pragma unroll
  for (int i = 0; i < 4; ++i) {  // registers, not local memory
    if (i >= dim) break;
    nm.mean[i] = w.m[i];
    nm.var[i] = w.c == 0.0 ? w.m[i] : ddiv(w.q[i], w.c);
  }
  nm.count = w.c;
  *norm = nm;
  norm_params_from(nm, *params);
}
cudaError_t run_vbn_fit(const EnvDesc& env, DKey lane_key, int n, DevNorm* norm, NormParams* params,
                        cudaStream_t s) {
  k_vbn_fit<<<1, 32, 0, s>>>(env, lane_key, n, norm, params);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------------------- init params
// init_params (proj/src/net.cpp:52-68): one stream, weight segments in layout
// order, column-major draws; uniform draw #q is stream word #q.
__global__ void k_init_params(NetDesc net, DKey key, double* p, const double* limits) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= net.d) return;
  long long draw = 0;
  for (int l = 0; l < net.nlayers; ++l) {
    const long long nw = (long long)net.dims[l] * net.dims[l + 1];
    if (idx >= net.w_off[l] && idx < net.w_off[l] + nw) {
      const double lim = limits[l];
      p[idx] = uniform_range(-lim, lim, word_to_uniform(stream_word(key, (uint64_t)(draw + idx - net.w_off[l]))));
      return;
    }
    draw += nw;
  }
  p[idx] = 0.0;  // biases
}
cudaError_t run_init_params(const NetDesc& net, DKey key, double* p, cudaStream_t s) {
  double lim[MAXL];
  for (int l = 0; l < net.nlayers; ++l) lim[l] = std::sqrt(6.0 / (net.dims[l] + net.dims[l + 1]));
  double* dlim = nullptr;
  cudaError_t e = cudaMallocAsync(&dlim, sizeof(lim), s);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(dlim, lim, sizeof(lim), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  k_init_params<<<blocks_for(net.d, 256), 256, 0, s>>>(net, key, p, dlim);
  count_launch();
  e = cudaGetLastError();
  cudaFreeAsync(dlim, s);
  return e;
}

// ------------------------------------------------------ env unit (parity)
__global__ void k_env_step_batch(EnvDesc env, long long n, double* phys, int* step_count,
                                 const double* action, double* reward, int* term, int* trunc, int* fault) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  LaneEnv s{};
  s.p0 = phys[4 * i];
  s.p1 = phys[4 * i + 1];
  s.p2 = phys[4 * i + 2];
  s.p3 = phys[4 * i + 3];
  s.step_count = step_count[i];
  double r = 0.0;
  bool te = false, tr = false;
  const uint32_t f = env_step(env, s, action[i], r, te, tr);
  fault[i] = f ? 3 : 0;
  if (f) return;
  phys[4 * i] = s.p0;
  phys[4 * i + 1] = s.p1;
  phys[4 * i + 2] = s.p2;
  phys[4 * i + 3] = s.p3;
  step_count[i] = s.step_count;
  reward[i] = r;
  term[i] = te;
  trunc[i] = tr;
}
cudaError_t run_env_step_batch(const EnvDesc& env, long long n, double* phys, int* step_count,
                               const double* action, double* reward, int* term, int* trunc, int* fault,
                               cudaStream_t s) {
  k_env_step_batch<<<blocks_for(n, 256), 256, 0, s>>>(env, n, phys, step_count, action, reward, term, trunc,
                                                      fault);
  EVB_CHECK_LAUNCH();
}

// eval_params statistics (proj/src/workflow.cpp:114-127): sequential order.
__global__ void k_eval_reduce(const double* r, int n, double* out) {
  if (threadIdx.x != 0) return;
  double sum = 0.0, sq = 0.0;
  for (int i = 0; i < n; ++i) {
    sum = dadd(sum, r[i]);
    sq = dadd(sq, dmul(r[i], r[i]));
  }
  const double m = ddiv(sum, (double)n);
  const double var = dsub(ddiv(sq, (double)n), dmul(m, m));
  out[0] = m;
  out[1] = sqrt(var > 0.0 ? var : 0.0);
}
cudaError_t run_eval_reduce(const double* r, int n, double* out, cudaStream_t s) {
  k_eval_reduce<<<1, 32, 0, s>>>(r, n, out);
  EVB_CHECK_LAUNCH();
}

// ------------------------------------------------------------ fp64 peak
// DFMA-bound kernel: 8 independent chains per thread, 4096 iterations.
__global__ void k_fp64_peak(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * 1e-3 + threadIdx.x * 1e-9;
  const double b = 0.999999, c = 1e-7;
  for (int it = 0; it < 4096; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;
}
double measure_fp64_peak_tflops() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, 8);
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_fp64_peak<<<blocks, threads>>>(d, 1.0);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fp64_peak<<<blocks, threads>>>(d, 1.0 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  count_launch(6);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double flops = 2.0 * 8 * 4096 * (double)blocks * threads;
  return flops / (best * 1e-3) / 1e12;
}

}  // namespace evorl_b200

namespace evorl_b200 {
// ------------------------------------------------------------ DMMA peak
// FP64 tensor-core throughput (mma.sync.m8n8k4.f64): 8 independent
// accumulators per warp, register operands only.
__global__ void k_dmma_peak(double* out, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 0.5 + threadIdx.x * 1e-10;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i * 1e-3;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
double measure_dmma_peak_tflops() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  cudaMalloc(&d, 8);
  const int blocks = sms * 4, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_dmma_peak<<<blocks, threads>>>(d, 1.0);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_dmma_peak<<<blocks, threads>>>(d, 1.0 + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  count_launch(6);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  const double warps = (double)blocks * threads / 32;
  const double flops = 2.0 * 256 * 8 * 2048 * warps;  // 8x8x4 MACs per mma
  return flops / (best * 1e-3) / 1e12;
}
}  // namespace evorl_b200
