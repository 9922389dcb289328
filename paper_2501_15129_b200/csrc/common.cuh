// common.cuh -- device primitives shared by every kernel of the B200 ES
// generation path (sm_100a).
//
//  * Threefry2x64-20 exactly as proj/src/rng.cpp:18-34 (bit-exact u64 words).
//  * Counter-addressed stream draws: word #w of RandomStream(K) is
//    threefry(K, (1, w>>1))[w&1]; normal #k is Box-Muller on block k>>1,
//    cos for even k and sin for odd k (proj/src/rng.cpp:54-87).  This is what
//    lets every kernel regenerate noise from (key, row, column) instead of
//    storing it.
//  * Exact-order fp64 helpers (__dmul_rn/__dadd_rn are never contracted into
//    FMA) for the places where the reference evaluates a*b+c as two rounded
//    operations (the reference Release build has no FMA, proj/CMakeLists.txt).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace evorl_b200 {

struct DKey {
  uint64_t hi, lo;
};

#define EVB_DEV __device__ __forceinline__
#define EVB_HD __host__ __device__ __forceinline__

// ------------------------------------------------------------------ exact fp64
EVB_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
EVB_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
EVB_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
EVB_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// ------------------------------------------------------------------ threefry
EVB_HD uint64_t rotl64(uint64_t x, int r) { return (x << r) | (x >> (64 - r)); }

// proj/src/rng.cpp:18-34 (rotations {16,42,12,31,16,32,24,21}, parity
// 0x1BD11BDAA9FC1A22, key injection every 4 rounds).  Fully unrolled.
EVB_HD void threefry2x64(uint64_t k0, uint64_t k1, uint64_t c0, uint64_t c1, uint64_t& o0,
                         uint64_t& o1) {
  const uint64_t k2 = 0x1BD11BDAA9FC1A22ull ^ k0 ^ k1;
  uint64_t x0 = c0 + k0, x1 = c1 + k1;
#define EVB_R(rot)   \
  x0 += x1;          \
  x1 = rotl64(x1, rot); \
  x1 ^= x0;
  EVB_R(16) EVB_R(42) EVB_R(12) EVB_R(31) x0 += k1; x1 += k2 + 1;
  EVB_R(16) EVB_R(32) EVB_R(24) EVB_R(21) x0 += k2; x1 += k0 + 2;
  EVB_R(16) EVB_R(42) EVB_R(12) EVB_R(31) x0 += k0; x1 += k1 + 3;
  EVB_R(16) EVB_R(32) EVB_R(24) EVB_R(21) x0 += k1; x1 += k2 + 4;
  EVB_R(16) EVB_R(42) EVB_R(12) EVB_R(31) x0 += k2; x1 += k0 + 5;
#undef EVB_R
  o0 = x0;
  o1 = x1;
}

// proj/src/rng.cpp:43-46
EVB_HD DKey fold_in(DKey k, uint64_t i) {
  DKey r;
  threefry2x64(k.hi, k.lo, 0, i, r.hi, r.lo);
  return r;
}

// Word #w of RandomStream(k) (proj/src/rng.cpp:54-63).
EVB_HD uint64_t stream_word(DKey k, uint64_t w) {
  uint64_t o0, o1;
  threefry2x64(k.hi, k.lo, 1, w >> 1, o0, o1);
  return (w & 1) ? o1 : o0;
}

// proj/src/rng.cpp:65-68
EVB_DEV double word_to_uniform(uint64_t w) { return (double)(w >> 11) * 0x1.0p-53; }
// proj/src/rng.cpp:70-72: lo + (hi - lo) * u
EVB_DEV double uniform_range(double lo, double hi, double u) { return dadd(lo, dmul(hi - lo, u)); }

// exact u64 -> double for x < 2^52: x lands in the mantissa of 2^52 + x
EVB_DEV double u52_to_double(uint64_t x) {
  return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0;
}

// Box-Muller pair of block b (proj/src/rng.cpp:74-87): normal #2b = c, #2b+1 = s.
EVB_DEV void normal_pair(DKey k, uint64_t b, double& c, double& s) {
  uint64_t w0, w1;
  threefry2x64(k.hi, k.lo, 1, b, w0, w1);
  // u1 = ((w0 >> 11) + 1) 2^-53, u2 = (w1 >> 11) 2^-53, converted exactly
  // without the conversion pipe: the top 52 bits land in a mantissa, the last
  // bit and the +1 are exact fp64 adds (every intermediate is an integer < 2^53)
  const double u1 =
      dadd(dadd(dmul(u52_to_double(w0 >> 12), 2.0), ((w0 >> 11) & 1) ? 1.0 : 0.0), 1.0) * 0x1.0p-53;
  const double u2 = dadd(dmul(u52_to_double(w1 >> 12), 2.0), ((w1 >> 11) & 1) ? 1.0 : 0.0) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586 * u2;  // 2.0 * M_PI * u2
  double sa, ca;
  sincos(a, &sa, &ca);
  c = r * ca;
  s = r * sa;
}

// Normal #idx of RandomStream(k).
EVB_DEV double normal_at(DKey k, uint64_t idx) {
  double c, s;
  normal_pair(k, idx >> 1, c, s);
  return (idx & 1) ? s : c;
}

// ----------------------------------------------------------- cluster / DSMEM
EVB_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

EVB_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// Map a local shared-memory address to the same offset in CTA `rank` of the
// cluster (shared::cluster window).
EVB_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

EVB_DEV uint32_t map_cluster(uint32_t local_saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_saddr), "r"(rank));
  return r;
}

EVB_DEV void st_cluster_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
EVB_DEV void st_cluster_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
template <typename T>
EVB_DEV void st_cluster(uint32_t addr, T v);
template <>
EVB_DEV void st_cluster<double>(uint32_t addr, double v) {
  st_cluster_f64(addr, v);
}
template <>
EVB_DEV void st_cluster<float>(uint32_t addr, float v) {
  st_cluster_f32(addr, v);
}
template <>
EVB_DEV void st_cluster<uint32_t>(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// st.async: asynchronous store into a cluster CTA's shared memory whose
// completion is counted (bytes) by that CTA's mbarrier -- no fence on the
// sender; the receiver's mbarrier wait makes the data visible.
EVB_DEV void st_async(uint32_t addr, double v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(addr), "d"(v),
               "r"(bar)
               : "memory");
}
EVB_DEV void st_async(uint32_t addr, float v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr),
               "r"(__float_as_uint(v)), "r"(bar)
               : "memory");
}
// Arm a local mbarrier for this phase: one arrival + the bytes peers will send.
EVB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// ---------------------------------------------------------------- mbarrier
EVB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// Arrive (release, cluster scope) on the same-offset mbarrier of CTA `rank`.
EVB_DEV void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  const uint32_t ra = map_cluster(smem_u32(bar), rank);
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
// Arrive (release, CTA scope) on a local mbarrier.
EVB_DEV void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Wait (acquire, CTA / cluster scope) for the phase with the given parity.
// The spin loop is C++ around a single try_wait: a branch hidden inside an asm
// block is invisible to the compiler, which then assumes the warp reconverged
// after it -- lanes leaving the spin at different times stay diverged into the
// following warp-synchronous code (a block-wide BAR.RED reached by half a warp
// was an illegal instruction on B200).
EVB_DEV bool mbar_try_wait_parity_cta(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
EVB_DEV bool mbar_try_wait_parity_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
EVB_DEV void mbar_wait_parity_cta(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_parity_cta(bar, parity)) {
  }
}
EVB_DEV void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_parity_cluster(bar, parity)) {
  }
}

// ------------------------------------------------------------------- errors
// Device error word: lowest failing lane wins (proj/src/thread_pool.cpp:49-51).
// Encoding: (lane << 8) | (kind << 4) | layer; kind 1..3 = EnvFault variants,
// kind 4 = NetFault, kind 5 = tcgen05 operand range (EVORL_PREC_TC only).  0xFFFF... = no error.
enum : uint32_t {
  FAULT_ENV_STATE = 1,
  FAULT_ENV_ACTION = 2,
  FAULT_ENV_SUCCESSOR = 3,
  FAULT_NET = 4,
  FAULT_TC_RANGE = 5,  // EVORL_PREC_TC: a finite activation beyond the fp16 split's range
};
EVB_DEV void record_fault(unsigned long long* word, uint64_t lane, uint32_t kind, uint32_t layer) {
  const unsigned long long code = (lane << 8) | ((uint64_t)kind << 4) | (layer & 15u);
  atomicMin(word, code);
}

}  // namespace evorl_b200
