// hrg_libm_trig.cuh -- sin/cos bit-identical to the reference's.
//
// hrgen evaluates p_x = r*cos(phi), p_y = r*sin(phi) and c_x, c_y with numpy
// (quadtree.py:474-475, 516-517), and numpy's float64 cos/sin on this image
// are glibc's libm.  The edge predicate (quadtree.py:611-613) is badly
// conditioned near the rim of the disk -- at config 2 one ulp of cos(phi)
// moves a pair whose hyperbolic distance is 3e-5 (relative) away from R --
// so an edge set identical to hrgen's needs glibc's sin/cos, not a correctly
// rounded one.
//
// Third-party dependency: glibc 2.39 (Ubuntu GLIBC 2.39-0ubuntu8.5), libm's
// dbl-64 sin/cos as built for x86-64 with FMA (the __sin_fma / __cos_fma
// ifunc variants, selected on every CPU with FMA + AVX2).  Its published
// algorithm (IBM Accurate Mathematical Library, s_sin.c) is restated below
// for finite |x| < 105414350, the range of every angle here:
//
//   |x| < 2^-26 (sin) / 2^-27 (cos)  sin x = x, cos x = 1
//   |x| < 0.85546875                 table + polynomial around k/128
//   |x| < 2.426265                   pi/2 - |x| as a double-double, then
//                                    the table path of the other function
//   otherwise                        Cody-Waite reduction by pi/2 with a
//                                    4-part pi/2 to a double-double (a, da)
//
// The table path takes k = round(128 |x|) (by adding 1.5*2^45), the
// table's double-double sin/cos of k/128 (hrg_libm_table.inc), and short
// polynomials in the remainder; |reduced argument| < 0.126 uses a Taylor
// polynomial instead.  The operation order and every fused multiply-add are
// those of the compiled x86-64 variant (read off its machine code: gcc
// contracts a*b+c there), so the result is the same double for every input.
// tests/test_libm_trig.py compiles this header for the host and compares it
// with the host's sin/cos; tests/test_gpu_parity.py does the same for the
// device.
#pragma once
#include <stdint.h>
#include <cmath>
#include <cstring>

#if defined(__CUDACC__)
#define HRG_HD __host__ __device__ __forceinline__
#else
#define HRG_HD inline
#endif

namespace hrg {
namespace libm {

#if defined(__CUDACC__)
__device__ const double kTabDev[4 * 110] = {
#include "hrg_libm_table.inc"
};
#endif
static const double kTabHost[4 * 110] = {
#include "hrg_libm_table.inc"
};

// Every operation rounded on its own, fused only where glibc's code fuses.
// (Host builds: -ffp-contract=off keeps mul/add unfused.)
#ifdef __CUDA_ARCH__
HRG_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
HRG_HD double mul(double a, double b) { return __dmul_rn(a, b); }
HRG_HD double add(double a, double b) { return __dadd_rn(a, b); }
HRG_HD double sub(double a, double b) { return __dsub_rn(a, b); }
HRG_HD uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
HRG_HD double tab(int i) { return __ldg(kTabDev + i); }
#else
HRG_HD double fma_(double a, double b, double c) { return std::fma(a, b, c); }
HRG_HD double mul(double a, double b) { return a * b; }
HRG_HD double add(double a, double b) { return a + b; }
HRG_HD double sub(double a, double b) { return a - b; }
HRG_HD uint64_t bits(double x) { uint64_t u; std::memcpy(&u, &x, 8); return u; }
HRG_HD double tab(int i) { return kTabHost[i]; }
#endif

// polynomial coefficients of the table path and the Taylor path
constexpr double kSn3 = -0x1.5555555555515p-3, kSn5 = 0x1.11110e829872fp-7;
constexpr double kCs2 = 0x1.0p-1, kCs4 = -0x1.5555555555535p-5, kCs6 = 0x1.6c16bedd9e239p-10;
constexpr double kS1 = -0x1.5555555555555p-3, kS2 = 0x1.1111111110ecep-7,
                 kS3 = -0x1.a01a019db08b8p-13, kS4 = 0x1.71de27b9a7ed9p-19,
                 kS5 = -0x1.addffc2fcdf59p-26;
constexpr double kBig = 0x1.8p45;          // |x| + kBig: k/128 in the low word
constexpr double kHp0 = 0x1.921fb54442d18p0, kHp1 = 0x1.1a62633145c07p-54;  // pi/2 = hp0 + hp1
constexpr double kHpInv = 0x1.45f306dc9c883p-1, kToInt = 0x1.8p52;           // 2/pi, 1.5*2^52
constexpr double kMp1 = 0x1.921fb58p0, kMp2 = -0x1.dde973cp-27;              // pi/2, 4 parts
constexpr double kPp3 = -0x1.cb3b398p-55, kPp4 = -0x1.d747f23e32ed7p-83;
constexpr double kTaylorMax = 0x1.020c49ba5e354p-3;  // 0.126

HRG_HD double copysign_(double m, double s) {
  return s < 0.0 || (s == 0.0 && (bits(s) >> 63)) ? -fabs(m) : fabs(m);
}

// a + da (da tiny): a + (da + a^3 P(a^2) - a^2 da/2) with P of degree 4.
HRG_HD double taylor_sin(double a, double da) {
  const double xx = mul(a, a);
  double p = fma_(xx, kS5, kS4);
  p = fma_(xx, p, kS3);
  p = fma_(xx, p, kS2);
  p = fma_(xx, p, kS1);
  const double q = fma_(p, a, -mul(da, 0.5));
  return add(a, fma_(xx, q, da));
}

// sin(a + da) from the table around k/128 (|a| >= 0.126).
HRG_HD double table_sin(double a, double da) {
  const double ax = fabs(a);
  const double d = a <= 0.0 ? -da : da;
  const double u = add(ax, kBig);
  const int k = (int)(uint32_t)bits(u);
  const double x = sub(ax, sub(u, kBig));
  const double xx = mul(x, x);
  const double s = add(x, fma_(mul(x, xx), fma_(xx, kSn5, kSn3), d));
  const double c = fma_(x, d, mul(xx, fma_(xx, fma_(xx, kCs6, kCs4), kCs2)));
  const double sn = tab(4 * k), ssn = tab(4 * k + 1), cs = tab(4 * k + 2), ccs = tab(4 * k + 3);
  const double cor = fma_(s, cs, fma_(-c, sn, fma_(s, ccs, ssn)));
  return copysign_(add(sn, cor), a);
}

HRG_HD double do_sin(double a, double da) {
  return fabs(a) < kTaylorMax ? taylor_sin(a, da) : table_sin(a, da);
}

// cos(a + da) from the table around k/128.
HRG_HD double do_cos(double a, double da) {
  const double ax = fabs(a);
  const double d = a < 0.0 ? -da : da;
  const double u = add(ax, kBig);
  const int k = (int)(uint32_t)bits(u);
  const double x = add(sub(ax, sub(u, kBig)), d);
  const double xx = mul(x, x);
  const double s = fma_(mul(x, xx), fma_(xx, kSn5, kSn3), x);
  const double c = mul(xx, fma_(xx, fma_(xx, kCs6, kCs4), kCs2));
  const double sn = tab(4 * k), ssn = tab(4 * k + 1), cs = tab(4 * k + 2), ccs = tab(4 * k + 3);
  const double cor = fma_(-s, sn, fma_(-c, cs, fma_(-s, ssn, ccs)));
  return add(cs, cor);
}

// x = n*pi/2 + (a + da), n mod 4 returned.
HRG_HD int reduce(double x, double& a, double& da) {
  const double t = fma_(x, kHpInv, kToInt);
  const double xn = sub(t, kToInt);
  const int n = (int)(bits(t) & 3);
  double y = fma_(-xn, kMp1, x);
  y = fma_(-xn, kMp2, y);
  const double t2 = fma_(-xn, kPp3, y);
  const double db = fma_(-kPp3, xn, sub(y, t2));
  const double b = fma_(-xn, kPp4, t2);
  da = add(db, fma_(-xn, kPp4, sub(t2, b)));
  a = b;
  return n;
}

HRG_HD uint32_t hiword(double x) { return (uint32_t)(bits(x) >> 32) & 0x7fffffffu; }

// glibc sin for finite |x| < 105414350.
HRG_HD double sin(double x) {
  const uint32_t k = hiword(x);
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(x, 0.0);
  if (k < 0x400368fdu) return copysign_(do_cos(sub(kHp0, fabs(x)), kHp1), x);
  double a, da;
  const int n = reduce(x, a, da);
  const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
  return (n & 2) ? -r : r;
}

// glibc cos for finite |x| < 105414350.
HRG_HD double cos(double x) {
  const uint32_t k = hiword(x);
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(x, 0.0);
  if (k < 0x400368fdu) {
    const double y = sub(kHp0, fabs(x));
    const double a = add(y, kHp1);
    return do_sin(a, add(sub(y, a), kHp1));
  }
  double a, da;
  const int n = reduce(x, a, da);
  const double r = (n & 1) ? do_sin(a, da) : do_cos(a, da);
  return ((n + 1) & 2) ? -r : r;
}

}  // namespace libm
}  // namespace hrg
