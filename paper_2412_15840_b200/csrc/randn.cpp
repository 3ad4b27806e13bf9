// Harness utility (not on the solve path): seeded standard normals for the synthetic BASELINE
// inputs ("generator v1"). Counter-based, so any slice can be generated
// independently and in parallel: value pair m of (seed, stream) comes from two splitmix64
// outputs at counters 2m and 2m+1, mapped to u1 in (0, 1] and u2 in [0, 1) with 53 bits each,
// then Box–Muller: out[2m] = r cos(2 pi u2), out[2m+1] = r sin(2 pi u2), r = sqrt(-2 ln u1).
#include <cmath>
#include <cstdint>

#include "schur.h"

namespace nds {

namespace {

inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline uint64_t counter_bits(uint64_t key, uint64_t ctr) { return mix64(key + (ctr + 1) * 0x9e3779b97f4a7c15ULL); }

}  // namespace

void randn_host(uint64_t seed, uint64_t stream, int64_t count, double* out) {
  const uint64_t key = mix64(mix64(seed) ^ (stream * 0xd1342543de82ef95ULL + 0x632be59bd9b4e019ULL));
  const int64_t pairs = (count + 1) / 2;
  const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
  for (int64_t m = 0; m < pairs; ++m) {
    const uint64_t b1 = counter_bits(key, 2 * (uint64_t)m);
    const uint64_t b2 = counter_bits(key, 2 * (uint64_t)m + 1);
    const double u1 = (double)((b1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(b2 >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = two_pi * u2;
    out[2 * m] = r * std::cos(th);
    if (2 * m + 1 < count) out[2 * m + 1] = r * std::sin(th);
  }
}

}  // namespace nds
