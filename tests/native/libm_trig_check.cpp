// Host check of csrc/hrg_libm_trig.cuh against the host libm's sin/cos.
// Usage: libm_trig_check N SEED  -> prints "mismatches <count> checked <count>"
// Inputs: N seeded uniform angles in [0, 2pi) drawn the way the sampler
// draws them (2pi * u53 / 2^53), N arbitrary doubles in [0, 2pi) by bit
// pattern, every branch boundary +-64 ulps, and k/128 +-64 ulps for every
// table entry (the table path's rounding-sensitive points).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "../../paper_1501_03545_b200/csrc/hrg_libm_trig.cuh"

static uint64_t sm64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double from_bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t to_bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

static long long bad = 0, checked = 0;
static volatile double sink;
static void check(double x) {
  const double s0 = sin(x), c0 = cos(x);
  const double s1 = hrg::libm::sin(x), c1 = hrg::libm::cos(x);
  ++checked;
  if (to_bits(s0) != to_bits(s1) || to_bits(c0) != to_bits(c1)) {
    if (bad < 10) printf("x=%a sin %a vs %a cos %a vs %a\n", x, s0, s1, c0, c1);
    ++bad;
  }
}
static void around(double x, int w) {
  const uint64_t b = to_bits(x);
  for (int d = -w; d <= w; ++d) {
    const double y = from_bits(b + d);
    if (y >= 0.0 && y < 6.283185307179586) check(y);
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 1000000;
  uint64_t s = argc > 2 ? strtoull(argv[2], 0, 10) : 1;
  const double two_pi = 6.283185307179586;
  for (long long i = 0; i < n; ++i) check(two_pi * ((double)(sm64(s) >> 11) * 0x1.0p-53));
  const uint64_t top = to_bits(two_pi);
  for (long long i = 0; i < n; ++i) check(from_bits(sm64(s) % top));
  const double edges[] = {0.0, 0x1.0p-27, 0x1.0p-26, 0x1.020c49ba5e354p-3, 0.85546875,
                          2.426265, from_bits(0x400368fd00000000ull), 1.5707963267948966,
                          3.141592653589793, 4.71238898038469, 0.7853981633974483,
                          2.356194490192345, 3.9269908169872414, 5.497787143782138,
                          6.283185307179586};
  for (double e : edges) around(e, 64);
  for (int k = 0; k < 110; ++k) {
    around(k / 128.0, 64);
    around(k / 128.0 + 1.0 / 256.0, 64);
    around(1.5707963267948966 - k / 128.0, 64);
    around(1.5707963267948966 + k / 128.0, 64);
  }
  printf("mismatches %lld checked %lld\n", bad, checked);
  return bad != 0;
}
