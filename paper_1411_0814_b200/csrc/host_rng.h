// host_rng.h -- the reference's counter-based splitmix64 streams on the host
// (include/rsm/rng.hpp:12-57 of /root/reference/proj): Rng(seed, tag, index),
// next_u64, next_unit, next_normal (Box-Muller with the C library's
// log/cos, as the reference). Stream tags (rng.hpp:62-67): FACTOR_A=1,
// FACTOR_B=2, NOISE=3, MASK=4, TRIAL=5, ALS_INIT=6; this library adds
// TRACK_POINT=16, TRACK_CAMERA=17, TRACK_WINDOW=18, TRACK_NOISE=19 for the
// structured-missingness (config 5) generator.
#pragma once

#include <cmath>
#include <cstdint>

namespace rsmh {

inline uint64_t mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

struct Rng {
  uint64_t s;
  Rng(uint64_t seed, uint64_t tag, uint64_t index) {
    s = mix(seed + 0x9e3779b97f4a7c15ull * tag);
    s = mix(s + 0xbf58476d1ce4e5b9ull * index);
  }
  uint64_t next_u64() {
    s += 0x9e3779b97f4a7c15ull;
    return mix(s);
  }
  double next_unit() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
  uint64_t next_below(uint64_t bound) {  // rejection, rng.hpp:30-36
    const uint64_t limit = bound * (UINT64_MAX / bound);
    for (;;) {
      const uint64_t v = next_u64();
      if (v < limit) return v % bound;
    }
  }
  double next_normal() {
    const double u1 = next_unit();
    const double u2 = next_unit();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
};

namespace stream {
constexpr uint64_t ALS_INIT = 6;
constexpr uint64_t TRACK_POINT = 16, TRACK_CAMERA = 17, TRACK_WINDOW = 18, TRACK_NOISE = 19;
}  // namespace stream

}  // namespace rsmh
