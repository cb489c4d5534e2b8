// Host build of NVIDIA's curand_Philox4x32_10 (curand_philox4x32_x.h) to pin
// oracle/philox.py -- test infrastructure (oracle/build_ref.sh builds it into
// oracle/_ref/philox_curand_check). Prints "c0 c1 c2 c3 k0 k1 -> o0 o1 o2 o3".
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char** argv) {
  unsigned s = 12345u;
  for (int t = 0; t < 64; ++t) {
    unsigned v[6];
    for (int j = 0; j < 6; ++j) { s = s * 1664525u + 1013904223u; v[j] = s ^ (s >> 13); }
    uint4 c = make_uint4(v[0], v[1], v[2], v[3]);
    uint2 k = make_uint2(v[4], v[5]);
    uint4 o = curand_Philox4x32_10(c, k);
    printf("%08x %08x %08x %08x %08x %08x %08x %08x %08x %08x\n", c.x, c.y, c.z, c.w, k.x, k.y,
           o.x, o.y, o.z, o.w);
  }
  return 0;
}
