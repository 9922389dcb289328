// umma_i8_bench.cu -- correctness + timing of the int8 tcgen05 MMAs behind the
// sliced-fixed-point (Ozaki) layer of the rollout team: M = 128 rows, K = 256
// (8 k-steps of 32), S byte slices, A slice i in TMEM (TS MMA), B = a window
// of a zero-padded slice buffer so that MMA i accumulates A_i . B_{c-i} into
// column block c of ONE accumulator (D_t = sum_{i+j=t} A_i B_j, t < S).
// A_0 is signed (s8), A_i>0 and every B_j unsigned (u8).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_i8_bench tools/umma_i8_bench.cu
//   ./tools/umma_i8_bench
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// kind::i8: D = s32 (c_format 2), A s8 (1) / u8 (0), B u8, K-major both
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t atm, uint64_t bd, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(atm), "l"(bd), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ uint32_t boff(int n, int k, int R) {
  return (uint32_t)((k >> 4) * (R >> 3) * 128 + (n >> 3) * 128 + (n & 7) * 16 + (k & 15));
}

constexpr int M = 128, K = 256, NL = 16;

// A: [S][128][256] bytes (slice, row, k); B: [S][16][256] (slice, lane, k); out: [128][16*S] int32
template <int S>
__global__ void bench(const uint8_t* A, const uint8_t* B, int* out, long long* cyc, int reps) {
  constexpr int R = NL * (2 * S - 1);  // rows of the zero-padded B buffer
  constexpr int N = NL * S;
  constexpr uint32_t LBO = (R / 8) * 128;
  __shared__ __align__(1024) uint8_t Bs[R * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int i = tid; i < R * K / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(Bs)[i] = 0u;
  __syncthreads();
  for (int i = tid; i < S * NL * K; i += blockDim.x) {
    const int j = i / (NL * K), e = (i / K) % NL, k = i % K;
    Bs[boff((S - 1 + j) * NL + e, k, R)] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t colA = 512 - 64 * S;
  // A slices -> TMEM: lane = row, slice i at columns colA + 64 i, 4 k per column (low byte first)
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int i = 0; i < S; ++i)
      for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t v[8];
        for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const uint32_t*>(A + ((size_t)i * M + row) * K + (c0 + q) * 4);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((uint32_t)(warp * 32) << 16) + colA + 64 * i + c0),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    uint32_t phase = 0;
    long long best = 1ll << 60;
    for (int rep = 0; rep < reps; ++rep) {
      const long long t0 = clock64();
      for (int ks = 0; ks < K / 32; ++ks)
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const uint64_t bd = desc(su32(Bs) + (S - 1 - i) * NL / 8 * 128 + ks * 2 * LBO, LBO, 128);
          mma_ts(tmem, tmem + colA + 64 * i + ks * 8, bd, idesc_i8(M, N, i == 0), (ks | i) ? 1u : 0u);
        }
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
          : "memory");
      const long long t1 = clock64();
      mbar_wait(&bar, phase);
      phase ^= 1;
      const long long t2 = clock64();
      if (t2 - t0 < best) {
        best = t2 - t0;
        if (lane == 0) {
          cyc[0] = t1 - t0;
          cyc[1] = t2 - t0;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 16; ++q) out[row * N + c0 + q] = (int)v[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int S>
int run(int reps) {
  constexpr int N = NL * S;
  std::vector<uint8_t> A((size_t)S * M * K), B((size_t)S * NL * K);
  srand(1234 + S);
  for (auto& x : A) x = (uint8_t)(rand() & 0xFF);
  for (auto& x : B) x = (uint8_t)(rand() & 0xFF);
  uint8_t *dA, *dB;
  int* dO;
  long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, sizeof(int) * M * N);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dO, 0, sizeof(int) * M * N);
  bench<S><<<1, 128>>>(dA, dB, dO, dc, reps);
  std::vector<int> O((size_t)M * N);
  long long cyc[2];
  cudaError_t e = cudaMemcpy(O.data(), dO, sizeof(int) * M * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("S=%d: %s\n", S, cudaGetErrorString(e));
    return 1;
  }
  long long bad = 0;
  for (int r = 0; r < M; ++r)
    for (int t = 0; t < S; ++t)
      for (int l = 0; l < NL; ++l) {
        long long acc = 0;
        for (int i = 0; i <= t; ++i) {
          const int j = t - i;
          for (int k = 0; k < K; ++k) {
            const int a = i == 0 ? (int)(int8_t)A[((size_t)i * M + r) * K + k] : (int)A[((size_t)i * M + r) * K + k];
            acc += (long long)a * (int)B[((size_t)j * NL + l) * K + k];
          }
        }
        if (acc != (long long)O[r * N + t * NL + l]) {
          if (bad < 5) printf("  mismatch r=%d t=%d lane=%d: got %d want %lld\n", r, t, l, O[r * N + t * NL + l], acc);
          ++bad;
        }
      }
  printf("S=%d N=%d: %d MMAs (M=128 K=32 i8 TS) issue %lld cyc, complete %lld cyc -> %.1f cyc/MMA; mismatches %lld\n", S,
         N, 8 * S, cyc[0], cyc[1], (double)cyc[1] / (8 * S), bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  cudaFree(dc);
  return bad != 0;
}


// Exact-N variant for 8-lane groups (the pipelined team): MMA i writes D
// columns [8i, 8i + N_i) with N_i = 8(S-i) rounded up to 16 and reads the data
// blocks B_0.. from block 0 (no zero blocks); the rounding spills into column
// block S (ignored).  Checks D_t = sum_{i+j=t} A_i B_j for t < S and times it.
template <int S, int G>
__global__ void bench_exact(const uint8_t* A, const uint8_t* B, int* out, long long* cyc, int reps) {
  constexpr int R = (G * (S + 1) + 7) / 8 * 8;  // data blocks + spill, whole 8-row core groups
  constexpr uint32_t LBO = (R / 8) * 128;
  __shared__ __align__(1024) uint8_t Bs[R * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int i = tid; i < R * K / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(Bs)[i] = 0u;
  __syncthreads();
  for (int i = tid; i < S * G * K; i += blockDim.x) {
    const int j = i / (G * K), e = (i / K) % G, k = i % K;
    Bs[boff(j * G + e, k, R)] = B[(j * NL + e) * K + k];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const uint32_t colA = 512 - 64 * S;
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int i = 0; i < S; ++i)
      for (int c0 = 0; c0 < 64; c0 += 8) {
        uint32_t v[8];
        for (int q = 0; q < 8; ++q) v[q] = *reinterpret_cast<const uint32_t*>(A + ((size_t)i * M + row) * K + (c0 + q) * 4);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + ((uint32_t)(warp * 32) << 16) + colA + 64 * i + c0),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
      }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    uint32_t phase = 0;
    long long best = 1ll << 60;
    for (int rep = 0; rep < reps; ++rep) {
      const long long t0 = clock64();
      for (int ks = 0; ks < K / 32; ++ks)
#pragma unroll
        for (int i = 0; i < S; ++i) {
          const int n = ((G * (S - i)) + 15) / 16 * 16;
          const uint64_t bd = desc(su32(Bs) + ks * 2 * LBO, LBO, 128);
          mma_ts(tmem + G * i, tmem + colA + 64 * i + ks * 8, bd, idesc_i8(M, n, i == 0),
                 (ks > 0 || i > 0) ? 1u : 0u);
        }
      asm volatile(
          "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
          : "memory");
      const long long t1 = clock64();
      mbar_wait(&bar, phase);
      phase ^= 1;
      const long long t2 = clock64();
      if (t2 - t0 < best) {
        best = t2 - t0;
        if (lane == 0) {
          cyc[0] = t1 - t0;
          cyc[1] = t2 - t0;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < (G * S + 7) / 8 * 8; c0 += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 8; ++q)
        if (c0 + q < G * S) out[row * (G * S) + c0 + q] = (int)v[q];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int S, int G>
int run_exact(int reps) {
  constexpr int N = G * S;
  std::vector<uint8_t> A((size_t)S * M * K), B((size_t)S * NL * K);
  srand(77 + S);
  for (auto& x : A) x = (uint8_t)(rand() & 0xFF);
  for (auto& x : B) x = (uint8_t)(rand() & 0xFF);
  uint8_t *dA, *dB;
  int* dO;
  long long* dc;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, sizeof(int) * M * N);
  cudaMalloc(&dc, 16);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  bench_exact<S, G><<<1, 128>>>(dA, dB, dO, dc, reps);
  std::vector<int> O((size_t)M * N);
  long long cyc[2];
  cudaError_t e = cudaMemcpy(O.data(), dO, sizeof(int) * M * N, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 16, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("exact S=%d: %s\n", S, cudaGetErrorString(e));
    return 1;
  }
  long long bad = 0;
  for (int r = 0; r < M; ++r)
    for (int t = 0; t < S; ++t)
      for (int l = 0; l < G; ++l) {
        long long acc = 0;
        for (int i = 0; i <= t; ++i)
          for (int k = 0; k < K; ++k) {
            const int a = i == 0 ? (int)(int8_t)A[((size_t)i * M + r) * K + k] : (int)A[((size_t)i * M + r) * K + k];
            acc += (long long)a * (int)B[((size_t)(t - i) * NL + l) * K + k];
          }
        if (acc != (long long)O[r * N + t * G + l]) {
          if (bad < 5) printf("  mismatch r=%d t=%d lane=%d: got %d want %lld\n", r, t, l, O[r * N + t * G + l], acc);
          ++bad;
        }
      }
  printf("exact-N S=%d (%d-lane group): %d MMAs issue %lld cyc, complete %lld cyc -> %.1f cyc/MMA; mismatches %lld\n", S,
         G, 8 * S, cyc[0], cyc[1], (double)cyc[1] / (8 * S), bad);
  return bad != 0;
}

int main() {
  int rc = 0;
  rc |= run<4>(8);
  rc |= run<5>(8);
  rc |= run<6>(8);
  rc |= run_exact<6, 8>(8);
  rc |= run_exact<6, 4>(8);
  return rc;
}
