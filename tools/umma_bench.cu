// umma_bench.cu -- microbenchmark of small tcgen05.mma shapes on one SM
// (the rollout team's layer-1 MMAs: M = 128, K = 16, N = 16 / 32, A from
// shared memory (SS) or tensor memory (TS)), dependent accumulator chain vs
// independent accumulators.  Operand contents are irrelevant (zeros).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/umma_bench tools/umma_bench.cu
//   /tmp/umma_bench
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout = 0) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}
constexpr uint32_t idesc(int M, int N) { return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24); }

template <int N, bool TS>
__device__ __forceinline__ void mma(uint32_t d, uint32_t atm, uint64_t ad, uint64_t bd, uint32_t acc) {
  if constexpr (TS)
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(atm), "l"(bd), "n"(idesc(128, N)), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(ad), "l"(bd), "n"(idesc(128, N)), "r"(acc));
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}

// NMMA MMAs, rotating over NACC accumulators of N columns each
template <int N, bool TS, int NACC, bool SW128 = false>
__global__ void bench(long long* out, int nmma) {
  __shared__ __align__(1024) unsigned char A[128 * 16 * 2 * 4];  // 4 k-steps of A (16 KB)
  __shared__ __align__(1024) unsigned char B[256 * 16 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < (int)sizeof(A) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0;
  for (int i = threadIdx.x; i < (int)sizeof(B) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(B)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 0) {
    uint32_t phase = 0;
    long long best = 1ll << 60;
    for (int rep = 0; rep < 4; ++rep) {
      const long long t0 = clock64();
      for (int i = 0; i < nmma; ++i) {
        const int k = i & 3;
        // SW128: 128-byte swizzle atoms (8 rows x 64 halves, 1024 B), the k-step
        // advances the start address 32 B inside the atom
        const uint64_t ad = SW128 ? desc(su32(A) + k * 32, 16, 1024, 2) : desc(su32(A) + k * 2 * 2048, 2048, 128);
        const uint64_t bd = desc(su32(B), (N / 8) * 128, 128);
        const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
        mma<N, TS>(d, tmem + 256 + k * 8, ad, bd, i >= NACC ? 1u : 0u);
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
        if (threadIdx.x == 0) {
          out[0] = t1 - t0;
          out[1] = t2 - t0;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool TS, int NACC, bool SW128 = false>
void run(const char* name, long long* d, int nmma) {
  bench<N, TS, NACC, SW128><<<1, 128>>>(d, nmma);
  long long h[2];
  cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    return;
  }
  printf("%-28s nmma=%4d  issue %6lld cyc  complete %6lld cyc  -> %6.1f cyc/MMA\n", name, nmma, h[0], h[1],
         (double)h[1] / nmma);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16 * sizeof(long long));
  for (int n : {16, 64}) {
    run<16, false, 1, true>("SS SW128 N=16 1 acc", d, n);
    run<32, false, 1, true>("SS SW128 N=32 1 acc", d, n);
    run<256, false, 1, true>("SS SW128 N=256 1 acc", d, n);
  }
  for (int n : {1, 2, 4, 16, 64}) {
    run<16, false, 1>("SS N=16 1 acc", d, n);
    run<32, false, 1>("SS N=32 1 acc", d, n);
    run<32, true, 1>("TS N=32 1 acc", d, n);
    run<16, true, 1>("TS N=16 1 acc", d, n);
    run<32, true, 4>("TS N=32 4 acc", d, n);
    run<16, false, 4>("SS N=16 4 acc", d, n);
    run<64, true, 1>("TS N=64 1 acc", d, n);
    run<128, true, 1>("TS N=128 1 acc", d, n);
    run<256, false, 1>("SS N=256 1 acc", d, n);
  }
  return 0;
}
