// Hand-off latency of a CTA-local mbarrier between warps (one B200 SM):
// producer warps write shared memory, optionally fence the async proxy, and
// arrive; a consumer warp waits (try_wait loop or test_wait spin).  Prints the
// average cycles from the last producer's pre-arrive timestamp to the
// consumer's wake-up.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mbar_latency tools/mbar_latency.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int PRODUCERS, int FENCE, int SPIN>
__global__ void k_handoff(unsigned long long* out, int iters) {
  __shared__ __align__(16) unsigned char buf[PRODUCERS * 32 * 64];
  __shared__ uint64_t bar;
  __shared__ unsigned long long t_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(PRODUCERS));
    t_last = 0;
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (warp < PRODUCERS) {
      // some shared stores (a producer's share of an operand)
      uint2* p = reinterpret_cast<uint2*>(buf + (warp * 32 + lane) * 64);
#pragma unroll
      for (int j = 0; j < 8; ++j) p[j] = make_uint2(it + j, lane);
      if (FENCE == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        atomicMax(&t_last, (unsigned long long)clock64());
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar)) : "memory");
      }
    } else if (warp == PRODUCERS) {
      uint32_t ok = 0;
      while (!ok) {
        if (SPIN)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)(it & 1)) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
                       "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bar)), "r"((uint32_t)(it & 1)) : "memory");
      }
      __syncwarp();
      if (FENCE == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // consumer-side fence
      const unsigned long long t = clock64();
      if (it > 10) acc += t - t_last;
    }
    __syncthreads();
  }
  if (warp == PRODUCERS && lane == 0) out[0] = acc / (iters - 11);
}

template <int P, int F, int S>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  k_handoff<P, F, S><<<1, 32 * (P + 1)>>>(d, 2000);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-48s %llu cycles\n", name, h);
  cudaFree(d);
}

int main() {
  run<1, 0, 0>("1 producer, no fence, try_wait");
  run<1, 0, 1>("1 producer, no fence, test_wait spin");
  run<1, 1, 0>("1 producer, proxy fence, try_wait");
  run<1, 1, 1>("1 producer, proxy fence, test_wait spin");
  run<8, 0, 0>("8 producers, no fence, try_wait");
  run<8, 1, 0>("8 producers, proxy fence, try_wait");
  run<8, 1, 1>("8 producers, proxy fence, test_wait spin");
  run<8, 2, 0>("8 producers, consumer-side proxy fence, try_wait");
  run<8, 2, 1>("8 producers, consumer-side proxy fence, spin");
  return 0;
}
