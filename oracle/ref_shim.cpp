// ref_shim.cpp -- TEST INFRASTRUCTURE.  A C-ABI shim over the reference's own
// RNG (proj/src/rng.cpp, compiled unchanged from /root/reference by
// oracle/Makefile into oracle/_ref/libevorl_ref.so).  Used only by tests to
// pin the oracle's Threefry/stream restatement bit-for-bit against the
// reference implementation.  The rest of the reference path needs Eigen3,
// which is not installed (proj/CMakeLists.txt:12), so it is not built.
#include <cstdint>

#include "evorl/rng.hpp"

extern "C" {

void ref_threefry2x64(const uint64_t key[2], const uint64_t ctr[2], uint64_t out[2]) {
  const auto o = evorl::threefry2x64({key[0], key[1]}, {ctr[0], ctr[1]});
  out[0] = o[0];
  out[1] = o[1];
}

void ref_key_from_seed(uint64_t seed, uint64_t out[2]) {
  const auto k = evorl::key_from_seed(seed);
  out[0] = k.hi;
  out[1] = k.lo;
}

void ref_fold_in(const uint64_t key[2], uint64_t index, uint64_t out[2]) {
  const auto k = evorl::fold_in({key[0], key[1]}, index);
  out[0] = k.hi;
  out[1] = k.lo;
}

// kind: 0 next_u64 (as double bits), 1 uniform, 2 normal, 3 randint(arg)
void ref_stream_draw(const uint64_t key[2], int kind, uint64_t arg, int64_t n, void* out) {
  evorl::RandomStream s({key[0], key[1]});
  for (int64_t i = 0; i < n; ++i) {
    switch (kind) {
      case 0: static_cast<uint64_t*>(out)[i] = s.next_u64(); break;
      case 1: static_cast<double*>(out)[i] = s.uniform(); break;
      case 2: static_cast<double*>(out)[i] = s.normal(); break;
      default: static_cast<uint64_t*>(out)[i] = s.randint(arg); break;
    }
  }
}

}  // extern "C"
