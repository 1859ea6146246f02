// hrg_math.cuh -- device arithmetic helpers for the hyperbolic range query.
//
//  * Philox4x32-10 counter-based RNG (one counter per vertex, so sampling is
//    embarrassingly parallel and independent of launch geometry).
//  * double-double (dd) arithmetic and a correctly rounded sin/cos for
//    angles in [0, 2*pi).  The reference computes p_x = r*cos(phi) with
//    numpy/libm (hrgen quadtree.py:474, 516); a correctly rounded value is
//    the one well-defined target a GPU can hit, and it agrees with glibc's
//    on >99.8% of inputs (tests/test_oracle.py measures the remainder).
//  * The reference predicate (quadtree.py:611-613) and circle transform
//    (geometry.py:149-157) with every multiply/add rounded separately:
//    numpy never contracts a*b+c into an FMA, so neither may we.  All fp64
//    arithmetic that feeds a decision uses __dmul_rn/__dadd_rn/__dsub_rn/
//    __ddiv_rn/__dsqrt_rn explicitly.
#pragma once
#include <stdint.h>

namespace hrg {

// ---------------------------------------------------------------- Philox
__host__ __device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
#else
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
}

// ---------------------------------------------------------------- dd
struct dd { double hi, lo; };

__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
  double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {  // accurate (IEEE-style) dd addition
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = __dadd_rn(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = __dadd_rn(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_add_d(dd a, double b) {
  dd s = two_sum(a.hi, b);
  s.lo = __dadd_rn(s.lo, a.lo);
  return fast_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  double p = __dmul_rn(a.hi, b.hi);
  double e = fma(a.hi, b.hi, -p);  // exact product error
  e = __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
  return fast_two_sum(p, e);
}

// (-1)^k/(2k+1)! and (-1)^k/(2k)!, k = 0..13, split hi+lo (exact rationals).
__device__ __constant__ double kSinC[14][2] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {-0x1.5555555555555p-3, -0x1.5555555555555p-57},
    {0x1.1111111111111p-7, 0x1.1111111111111p-63},
    {-0x1.a01a01a01a01ap-13, -0x1.a01a01a01a01ap-73},
    {0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73},
    {-0x1.ae64567f544e4p-26, 0x1.c062e06d1f209p-80},
    {0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87},
    {-0x1.ae7f3e733b81fp-41, -0x1.1d8656b0ee8cbp-97},
    {0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103},
    {-0x1.2f49b46814157p-57, -0x1.2650f61dbdcb4p-112},
    {0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120},
    {-0x1.761b41316381ap-75, 0x1.3423c7d91404fp-130},
    {0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139},
    {-0x1.d1ab1c2dccea3p-94, -0x1.054d0c78aea14p-149}};
__device__ __constant__ double kCosC[14][2] = {
    {0x1.0000000000000p+0, 0x0.0p+0},
    {-0x1.0000000000000p-1, 0x0.0p+0},
    {0x1.5555555555555p-5, 0x1.5555555555555p-59},
    {-0x1.6c16c16c16c17p-10, 0x1.f49f49f49f49fp-65},
    {0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76},
    {-0x1.27e4fb7789f5cp-22, -0x1.cbbc05b4fa99ap-76},
    {0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83},
    {-0x1.93974a8c07c9dp-37, -0x1.05d6f8a2efd1fp-92},
    {0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101},
    {-0x1.6827863b97d97p-53, -0x1.eec01221a8b0bp-107},
    {0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120},
    {-0x1.0ce396db7f853p-70, 0x1.aebcdbd20331cp-124},
    {0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135},
    {-0x1.88e85fc6a4e5ap-89, 0x1.71c37ebd16540p-143}};

// Horner in dd over coefficient table C for s2 = r^2; terms k >= 8 are
// smaller than 2^-50 relative and are accumulated in plain double.
template <bool kSin>
__device__ __forceinline__ dd poly_dd(dd s2) {
#define HRG_C(k, i) (kSin ? kSinC[k][i] : kCosC[k][i])
  double t = HRG_C(13, 0);
#pragma unroll
  for (int k = 12; k >= 8; --k) t = fma(s2.hi, t, HRG_C(k, 0));
  dd p = {t, 0.0};
#pragma unroll
  for (int k = 7; k >= 0; --k) p = dd_add(dd{HRG_C(k, 0), HRG_C(k, 1)}, dd_mul(s2, p));
#undef HRG_C
  return p;
}

// Correctly rounded sin/cos of x in [0, 2*pi) (to within ~2^-100 relative
// before the final rounding, i.e. correctly rounded except on inputs within
// 2^-100 of a rounding midpoint).
__device__ __forceinline__ void sincos_cr(double x, double* s_out, double* c_out) {
  const double P1 = 0x1.921fb54400000p+0;   // pi/2 = P1+P2+P3+P4, P1..P3 33-bit
  const double P2 = 0x1.0b4611a600000p-34;
  const double P3 = 0x1.3198a2e000000p-69;
  const double P4 = 0x1.b839a252049c1p-104;
  double kd = rint(__dmul_rn(x, 0x1.45f306dc9c883p-1));  // x * 2/pi
  int k = (int)kd;
  // r = x - k*pi/2: k*P1, k*P2, k*P3 are exact (k < 8)
  dd r = {__dsub_rn(x, __dmul_rn(kd, P1)), 0.0};
  r = dd_add_d(r, -__dmul_rn(kd, P2));
  r = dd_add_d(r, -__dmul_rn(kd, P3));
  r = dd_add_d(r, -__dmul_rn(kd, P4));
  dd s2 = dd_mul(r, r);
  dd sp = dd_mul(r, poly_dd<true>(s2));
  dd cp = poly_dd<false>(s2);
  double sr = __dadd_rn(sp.hi, sp.lo), cr = __dadd_rn(cp.hi, cp.lo);
  switch (k & 3) {
    case 0: *s_out = sr; *c_out = cr; break;
    case 1: *s_out = cr; *c_out = -sr; break;
    case 2: *s_out = -sr; *c_out = -cr; break;
    default: *s_out = -cr; *c_out = sr; break;
  }
}

// ----------------------------------------- fast path with a rounding test
// sin/cos of a = i/128, i in [-kScHalf, kScHalf], as double-doubles (hi, lo)
// to ~2^-100, filled once per device by k_sincos_table from the same
// double-double Taylor series as sincos_cr.
constexpr int kScHalf = 101;                // 101/128 > pi/4 + the reduction's slack
__device__ double4 g_sctab[2 * kScHalf + 1];  // (sin hi, sin lo, cos hi, cos lo)

__global__ void k_sincos_table() {
  const int i = threadIdx.x;
  if (i > 2 * kScHalf) return;
  const dd a = {(double)(i - kScHalf) * 0x1.0p-7, 0.0};
  const dd s2 = dd_mul(a, a);
  const dd sp = dd_mul(a, poly_dd<true>(s2));
  const dd cp = poly_dd<false>(s2);
  g_sctab[i] = make_double4(sp.hi, sp.lo, cp.hi, cp.lo);
}

// y = fl(v) for v = y + e (+- err), i.e. is y correctly rounded?  The
// rounding interval of y is [y - dn/2, y + up/2] (dn != up at powers of 2).
__device__ __forceinline__ bool rounds_to(double y, double e, double err) {
  const double a = fabs(y);
  if (!(a > 0.0)) return false;
  const long long b = __double_as_longlong(a);
  const double gap_up = __dsub_rn(__longlong_as_double(b + 1), a);  // above |y|
  const double gap_dn = __dsub_rn(a, __longlong_as_double(b - 1));  // below |y|
  const double up = y > 0.0 ? gap_up : gap_dn, dn = y > 0.0 ? gap_dn : gap_up;
  return __dadd_rn(e, err) < __dmul_rn(0.5, up) && __dsub_rn(e, err) > __dmul_rn(-0.5, dn);
}

// sin/cos of x in [0, 2pi), correctly rounded.  Fast path: table value at
// a = i/128 nearest to the reduced argument r, and the short series in
// t = r - a (|t| <= 2^-8): sin r = S + C t + [S (cos t - 1) + C (sin t - t)],
// cos r = C - S t + [C (cos t - 1) - S (sin t - t)], with the leading product
// exact (fma) and the bracket (< 2^-16) in double.  Error of the bracket:
// ten roundings of at most its magnitude A <= (|S| + |t|) t^2 / 2 (+ ulp-level
// terms) give <= 2^-49.7 A, the omitted products (S_lo (cos t - 1), C_lo (sin
// t - t)), the series' own roundings and truncations add < 2^-51 (|S| + |t|)
// t^2, the table and the reduction < 2^-99: bounded by 2^-48 (|S| + |t|) t^2
// + 2^-96 (C for S in the cosine).  A value whose rounding that error could
// change (a few in 10^4) is recomputed by sincos_cr.
__device__ __forceinline__ bool sincos_crf(double x, double* s_out, double* c_out) {
  const double P1 = 0x1.921fb54400000p+0;
  const double P2 = 0x1.0b4611a600000p-34;
  const double P3 = 0x1.3198a2e000000p-69;
  const double P4 = 0x1.b839a252049c1p-104;
  const double kd = rint(__dmul_rn(x, 0x1.45f306dc9c883p-1));
  const int k = (int)kd;
  dd r = {__dsub_rn(x, __dmul_rn(kd, P1)), 0.0};
  r = dd_add_d(r, -__dmul_rn(kd, P2));
  r = dd_add_d(r, -__dmul_rn(kd, P3));
  r = dd_add_d(r, -__dmul_rn(kd, P4));
  const double fi = rint(__dmul_rn(r.hi, 128.0));
  const int i = max(-kScHalf, min(kScHalf, (int)fi));
  const double th = __dsub_rn(r.hi, __dmul_rn((double)i, 0x1.0p-7));  // exact (Sterbenz)
  const double tl = r.lo;                                               // t = th + tl
  const double4 T = g_sctab[i + kScHalf];
  const double Sh = T.x, Sl = T.y, Ch = T.z, Cl = T.w;
  // t^2 = t2 + t2e exactly for th; cross term 2 th tl
  const double t2 = __dmul_rn(th, th);
  const double t2e = fma(th, th, -t2);
  const double txl = __dmul_rn(th, tl);
  // cos t - 1 = -t^2/2 + t^4/24 - t^6/720  (t^8 term < 2^-71)
  const double c4 = __dmul_rn(t2, __dsub_rn(1.0 / 24.0, __dmul_rn(t2, 1.0 / 720.0)));
  const double cm1 = __dadd_rn(__dmul_rn(-0.5, t2),
                               __dsub_rn(__dmul_rn(t2, c4), __dadd_rn(__dmul_rn(0.5, t2e), txl)));
  // sin t - t = -t^3/6 + t^5/120 - t^7/5040  (t^9 term < 2^-80); d/dt: -t^2/2 tl
  const double t3 = __dmul_rn(t2, th);
  const double sp5 = __dmul_rn(t2, __dsub_rn(1.0 / 120.0, __dmul_rn(t2, 1.0 / 5040.0)));
  const double sm = __dsub_rn(__dmul_rn(t3, __dsub_rn(sp5, 1.0 / 6.0)), __dmul_rn(0.5, __dmul_rn(t2, tl)));
  // sin r
  const double Ph = __dmul_rn(Ch, th), Pl = fma(Ch, th, -Ph);
  const dd M = two_sum(Sh, Ph);
  double sm_s = __dadd_rn(__dmul_rn(Cl, th), __dmul_rn(Ch, tl));
  sm_s = __dadd_rn(sm_s, Pl);
  sm_s = __dadd_rn(sm_s, Sl);
  sm_s = __dadd_rn(sm_s, __dmul_rn(Ch, sm));
  sm_s = __dadd_rn(sm_s, __dmul_rn(Sh, cm1));
  sm_s = __dadd_rn(sm_s, M.lo);
  const dd Ys = two_sum(M.hi, sm_s);
  // cos r
  const double Qh = __dmul_rn(Sh, th), Ql = fma(Sh, th, -Qh);
  const dd N = two_sum(Ch, -Qh);
  double sm_c = __dsub_rn(-__dmul_rn(Sl, th), __dmul_rn(Sh, tl));
  sm_c = __dsub_rn(sm_c, Ql);
  sm_c = __dadd_rn(sm_c, Cl);
  sm_c = __dsub_rn(sm_c, __dmul_rn(Sh, sm));
  sm_c = __dadd_rn(sm_c, __dmul_rn(Ch, cm1));
  sm_c = __dadd_rn(sm_c, N.lo);
  const dd Yc = two_sum(N.hi, sm_c);
  double sr = Ys.hi, cr = Yc.hi;
  const double at = fabs(th);
  const double es = __dadd_rn(__dmul_rn(0x1.0p-48, __dmul_rn(t2, __dadd_rn(at, fabs(Sh)))), 0x1.0p-96);
  const double ec = __dadd_rn(__dmul_rn(0x1.0p-48, __dmul_rn(t2, __dadd_rn(at, fabs(Ch)))), 0x1.0p-96);
  if (!(rounds_to(Ys.hi, Ys.lo, es) && rounds_to(Yc.hi, Yc.lo, ec))) {
    sincos_cr(x, s_out, c_out);
    return false;
  }
  switch (k & 3) {
    case 0: *s_out = sr; *c_out = cr; break;
    case 1: *s_out = cr; *c_out = -sr; break;
    case 2: *s_out = -sr; *c_out = -cr; break;
    default: *s_out = -cr; *c_out = sr; break;
  }
  return true;
}

// ------------------------------------------------- reference arithmetic
// hrgen geometry.py:149-157, literally: b=(1-rh)(1+rh); denom=a*b+2;
// center_r=2*rh/denom; disc=center_r^2-(2*rh^2-a*b)/denom; rad=sqrt(disc).
__device__ __forceinline__ void circle_params(double rh, double a, double* cr, double* rad) {
  double b = __dmul_rn(__dsub_rn(1.0, rh), __dadd_rn(1.0, rh));
  double ab = __dmul_rn(a, b);
  double denom = __dadd_rn(ab, 2.0);
  double c = __ddiv_rn(__dmul_rn(2.0, rh), denom);
  double disc = __dsub_rn(__dmul_rn(c, c),
                          __ddiv_rn(__dsub_rn(__dmul_rn(2.0, __dmul_rn(rh, rh)), ab), denom));
  *cr = c;
  *rad = __dsqrt_rn(disc);
}

// hrgen quadtree.py:611-613: dx = p_x - c_x; dy = p_y - c_y; dx*dx+dy*dy < rad_sq
__device__ __forceinline__ bool ref_pred(double px, double py, double cx, double cy, double rsq) {
  double dx = __dsub_rn(px, cx), dy = __dsub_rn(py, cy);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) < rsq;
}

}  // namespace hrg
