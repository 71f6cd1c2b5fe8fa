// Pin helper for the oracle's Philox4x32-10: evaluates cuRAND's library
// routine curand_Philox4x32_10 (/usr/local/cuda/include/curand_philox4x32_x.h)
// on the HOST for each "c0 c1 c2 c3 k0 k1" line of stdin.  Test-only.
#include <cstdio>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = {c0, c1, c2, c3};
    uint2 k = {k0, k1};
    uint4 r = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
  return 0;
}
