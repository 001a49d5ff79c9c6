// numpy's PCG64 bit generator (128-bit LCG, XSL-RR 128/64 output), host and device.
// Shared by the parity normals (npzig.cu) and the k-means++ seeding (kmeans.cu).
#pragma once
#include <cstdint>

namespace csc {

using u128 = unsigned __int128;

__host__ __device__ inline u128 make128(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__host__ __device__ inline u128 pcg_mult() { return make128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull); }

// state after `delta` LCG steps
__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

// step then output (numpy's pcg64 next_uint64)
__host__ __device__ inline uint64_t pcg_next(u128& state, u128 inc) {
  state = state * pcg_mult() + inc;
  const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  const uint64_t x = hi ^ lo;
  const unsigned r = (unsigned)(hi >> 58);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// numpy's next_double: 53 high bits of one raw
__host__ __device__ inline double pcg_next_double(u128& state, u128 inc) {
  return (double)(pcg_next(state, inc) >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace csc
