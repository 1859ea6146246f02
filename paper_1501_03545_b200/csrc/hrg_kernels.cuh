// hrg_kernels.cuh -- sm_100a kernels of the random-hyperbolic-graph generator.
//
// Pipeline (one CUDA stream, see hrg_api.cu):
//   k_sample        Philox4x32-10 -> (phi, r_native, r_poincare) per vertex, plus a
//                   59-bit sort key (radial band << 53 | angular fixed point q).
//   cub radix sort  keys -> permutation into (band, angle) order.
//   k_gather        SoA fp64 point/circle records in sorted order: p_x, p_y (the
//                   point), c_x, c_y, rad^2 (its query circle), correctly rounded
//                   sin/cos, hrgen's circle transform (geometry.py:141-157).
//   k_band_setup / k_band_minmax / k_dir_fill / k_dir_tail
//                   per band: position range, min hyperbolic radius, max Poincare
//                   radius, and an angular directory (bucket -> first position).
//   k_query<COUNT>  one warp per query vertex: lane j computes the angular window of
//                   band j, the warp flattens the <=2 position segments per band,
//                   tests 32 candidates per step with the reference predicate and
//                   counts hits.
//   cub scan        degrees -> CSR row pointers.
//   k_query<WRITE>  same traversal, ballot-compacted ordered writes into the CSR.
//
// Replaces hrgen quadtree.py (build 303-340, pack 399-495, query_many 499-631)
// and generator.py:190-225.
#pragma once
#include <stdint.h>
#include "hrg_math.cuh"

namespace hrg {

constexpr int kMaxBands = 32;     // one warp lane per radial band
constexpr int kQBits = 53;
constexpr uint64_t kQMask = (1ull << kQBits) - 1;
constexpr double kTwoPi = 6.283185307179586;  // == 2.0 * math.pi (geometry.py:19)

struct Band {
  int32_t start, end;      // sorted positions of the band
  int32_t qstart, qend;    // query positions (this shard's angular sector)
  int64_t dir_base;        // offset of the band's directory in dir[]
  int32_t shift;           // bucket(q) = q >> shift
  int32_t nb;              // buckets (power of two); directory has nb + 1 entries
  float rmin;              // min hyperbolic radius 2*atanh(r_poincare) in band (rounded down)
  float bmin;              // min (1-r)(1+r) in band (rounded down)
  float sinh_rmin;
  float pad_;
};

struct BandSpec {          // band(rp) = #{ j in [1, L) : thr[j] <= rp }
  double thr[kMaxBands];
  int L;
};

__device__ __forceinline__ int band_of(const BandSpec& S, double rp) {
  int b = 0;
#pragma unroll 4
  for (int j = 1; j < S.L; ++j) b += (S.thr[j] <= rp);
  return b;
}

// Angular fixed point: monotone in phi, identical expression everywhere.
__device__ __forceinline__ uint64_t qkey(double x, double C) {
  double t = floor(__dmul_rn(x, C));
  if (!(t >= 0.0)) t = 0.0;
  uint64_t q = (uint64_t)t;
  return q > kQMask ? kQMask : q;
}

struct SampleParams {
  uint64_t seed;
  double two_over_alpha, sinh_half, r_cap, rp_cap;
  double C;  // 2^53 / (2 pi)
};

// hrgen generator.py:160-179 with a counter-based stream: vertex i draws its
// angle from the first and its radius from the second 53-bit uniform of
// Philox4x32-10(counter = i, key = seed).
__global__ void __launch_bounds__(256) k_sample(int64_t n, SampleParams P, BandSpec S,
                                                double* __restrict__ phi, double* __restrict__ rn,
                                                double* __restrict__ rp,
                                                uint64_t* __restrict__ keys,
                                                int32_t* __restrict__ vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0u};
  philox4x32_10(c, (uint32_t)P.seed, (uint32_t)(P.seed >> 32));
  uint64_t a = (((uint64_t)c[1] << 32) | c[0]) >> 11;
  uint64_t b = (((uint64_t)c[3] << 32) | c[2]) >> 11;
  double u1 = (double)a * 0x1.0p-53, u2 = (double)b * 0x1.0p-53;
  double ph = __dmul_rn(kTwoPi, u1);                                   // :170
  double r = __dmul_rn(P.two_over_alpha, asinh(__dmul_rn(__dsqrt_rn(u2), P.sinh_half)));
  r = fmin(r, P.r_cap);                                                // :174
  double p = fmin(tanh(__dmul_rn(r, 0.5)), P.rp_cap);                 // :175-178
  phi[i] = ph; rn[i] = r; rp[i] = p;
  keys[i] = ((uint64_t)band_of(S, p) << kQBits) | qkey(ph, P.C);
  vals[i] = (int32_t)i;
}

// Keys for caller-supplied coordinates; flags points outside the tree region
// (hrgen quadtree.py:293-299 raises OutOfBoundsError for those).
__global__ void __launch_bounds__(256) k_keys_from_coords(int64_t n, const double* __restrict__ phi,
                                                          const double* __restrict__ rp,
                                                          double max_r, double C, BandSpec S,
                                                          double* __restrict__ rn,
                                                          uint64_t* __restrict__ keys,
                                                          int32_t* __restrict__ vals,
                                                          int* __restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ph = phi[i], p = rp[i];
  if (!(ph >= 0.0 && ph < kTwoPi && p >= 0.0 && p < max_r)) { atomicOr(bad, 1); p = 0.0; ph = 0.0; }
  rn[i] = 2.0 * atanh(p);  // geometry.py:121 to_native_radius
  keys[i] = ((uint64_t)band_of(S, p) << kQBits) | qkey(ph, C);
  vals[i] = (int32_t)i;
}

struct SoA {
  double *phi, *px, *py, *cx, *cy, *rsq;
  float *rf, *bf;
};

// Gather into (band, angle) order and precompute every per-point quantity the
// query needs.  p_x/p_y: quadtree.py:474-475; c_x/c_y/rad^2: quadtree.py:516-518
// with center_r/rad from geometry.py:141-157.
__global__ void __launch_bounds__(256) k_gather(int64_t n, const int32_t* __restrict__ perm,
                                                const double* __restrict__ phi,
                                                const double* __restrict__ rp,
                                                const double* __restrict__ rn, double a, SoA s,
                                                double* __restrict__ s_rp,
                                                double* __restrict__ s_rn) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  int32_t i = perm[p];
  double ph = phi[i], r = rp[i];
  double sn, cs;
  sincos_cr(ph, &sn, &cs);
  double cr, rad;
  circle_params(r, a, &cr, &rad);
  s.phi[p] = ph;
  s.px[p] = __dmul_rn(r, cs);
  s.py[p] = __dmul_rn(r, sn);
  s.cx[p] = __dmul_rn(cr, cs);
  s.cy[p] = __dmul_rn(cr, sn);
  s.rsq[p] = __dmul_rn(rad, rad);
  // hyperbolic radius of the stored Poincare point and (1-r)(1+r), both
  // rounded down: only used to size conservative angular windows.
  double one_m = 1.0 - r;
  double re = log1p(2.0 * r / one_m);  // 2*atanh(r)
  s.rf[p] = __double2float_rd(re);
  s.bf[p] = __double2float_rd(one_m * (1.0 + r));
  if (s_rp) s_rp[p] = r;
  if (s_rn) s_rn[p] = rn[i];
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t key) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One block: band position ranges, shard query ranges, directory sizing.
__global__ void k_band_setup(const uint64_t* __restrict__ keys, int64_t n, int L,
                             uint64_t qsec_lo, uint64_t qsec_hi, Band* __restrict__ bands,
                             int64_t* __restrict__ dir_total) {
  __shared__ int64_t st[kMaxBands + 1];
  int j = threadIdx.x;
  if (j <= L) st[j] = lower_bound_u64(keys, n, (uint64_t)j << kQBits);
  __syncthreads();
  if (j < L) {
    Band B;
    B.start = (int32_t)st[j];
    B.end = (int32_t)st[j + 1];
    uint64_t base = (uint64_t)j << kQBits;
    B.qstart = (int32_t)lower_bound_u64(keys, n, base | qsec_lo);
    B.qend = qsec_hi > kQMask ? B.end : (int32_t)lower_bound_u64(keys, n, base | qsec_hi);
    int64_t cnt = B.end - B.start;
    int lg = 0;
    while ((1ll << lg) < cnt) ++lg;       // nb = next pow2 >= cnt (>= 1)
    B.nb = 1 << lg;
    B.shift = kQBits - lg;
    B.rmin = __int_as_float(0x7f800000);
    B.bmin = __int_as_float(0x7f800000);
    B.sinh_rmin = 0.f;
    B.pad_ = 0.f;
    B.dir_base = 0;
    bands[j] = B;
  }
  __syncthreads();
  if (j == 0) {
    int64_t off = 0;
    for (int b = 0; b < L; ++b) { bands[b].dir_base = off; off += bands[b].nb + 1; }
    *dir_total = off;
  }
}

// Per-band min radius / min (1-r)(1+r): warp-aggregated atomicMin on the bit
// patterns of positive floats (order-preserving, so deterministic).
__global__ void __launch_bounds__(256) k_band_minmax(int64_t n, const uint64_t* __restrict__ keys,
                                                     const float* __restrict__ rf,
                                                     const float* __restrict__ bf,
                                                     Band* __restrict__ bands) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int lane = threadIdx.x & 31;
  bool ok = p < n;
  int band = ok ? (int)(keys[p] >> kQBits) : -1;
  int r = ok ? __float_as_int(rf[p]) : 0x7f800000;
  int b = ok ? __float_as_int(bf[p]) : 0x7f800000;
  // lanes of one band are contiguous (sorted keys): reduce per group, one
  // atomic per group leader
  unsigned same = __match_any_sync(0xffffffffu, band);
  r = (int)__reduce_min_sync(same, (unsigned)r);
  b = (int)__reduce_min_sync(same, (unsigned)b);
  if (ok && lane == __ffs(same) - 1) {
    atomicMin((int*)&bands[band].rmin, r);
    atomicMin((int*)&bands[band].bmin, b);
  }
}

__global__ void k_band_finish(Band* bands, int L) {
  int j = threadIdx.x;
  if (j < L) bands[j].sinh_rmin = sinhf(bands[j].rmin);
}

// dir[base + k] = first position of the band whose bucket >= k.
__global__ void __launch_bounds__(256) k_dir_fill(int64_t n, const uint64_t* __restrict__ keys,
                                                  const Band* __restrict__ bands,
                                                  int32_t* __restrict__ dir) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint64_t key = keys[p];
  int j = (int)(key >> kQBits);
  Band B = bands[j];
  int64_t b = (int64_t)((key & kQMask) >> B.shift);
  int64_t bprev = -1;
  if (p > B.start) bprev = (int64_t)((keys[p - 1] & kQMask) >> B.shift);
  for (int64_t k = bprev + 1; k <= b; ++k) dir[B.dir_base + k] = (int32_t)p;
}

__global__ void k_dir_tail(const uint64_t* __restrict__ keys, const Band* __restrict__ bands,
                           int32_t* __restrict__ dir) {
  Band B = bands[blockIdx.x];
  int64_t last = -1;
  if (B.end > B.start) last = (int64_t)((keys[B.end - 1] & kQMask) >> B.shift);
  for (int64_t k = last + 1 + threadIdx.x; k <= B.nb; k += blockDim.x)
    dir[B.dir_base + k] = B.end;
}

struct QueryArgs {
  SoA s;
  const int32_t* id;       // sorted position -> vertex id (sample order)
  const Band* bands;
  const int32_t* dir;
  int L;
  double C;                // 2^53 / (2 pi)
  float R_pad;             // R rounded up + fp32 slack
  float a_f;               // cosh R - 1
  float E_over_tanh;       // fp64 decision-noise constant / tanh(R)
  int32_t* deg;            // COUNT: row length per vertex id
  const int64_t* rowptr;   // WRITE: row offsets per vertex id
  int32_t* out;            // WRITE: CSR indices
  unsigned long long* cand;  // COUNT: pair tests (stats)
};

__device__ __forceinline__ int32_t dir_lookup(const int32_t* dir, int64_t base, int shift,
                                              double x, double C, int hi) {
  uint64_t q = qkey(x, C);
  return __ldg(dir + base + (int64_t)(q >> shift) + hi);
}

// One warp per query vertex v.
//  Lane j (< L) sizes band j's angular window for v: every w in the band with
//  hyperbolic distance below R + eta lies within it, eta bounding the fp64
//  decision noise of the reference predicate for this (v, band) pair, so no
//  pair that either orientation of the predicate accepts can fall outside.
//  The warp then walks the concatenated candidate segments 32 at a time.
//  Edge {v,w} is decided by the circle of the smaller vertex id, exactly as
//  hrgen (generator.py:182-187) queries from v and keeps ids > v.
template <bool kWrite, bool kSampleIds>
__global__ void __launch_bounds__(256) k_query(QueryArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned FULL = 0xffffffffu;

  // per-lane band constants, resident for the whole kernel
  Band B;
  int64_t qoff_lane = INT64_MAX;
  int64_t total_q = 0;   // queries of this shard = sum of the bands' query ranges
  for (int j = 0; j < A.L; ++j) {
    Band t = A.bands[j];
    if (j == lane) { B = t; qoff_lane = total_q; }
    total_q += t.qend - t.qstart;
  }
  if (lane >= A.L) { B = A.bands[0]; B.start = B.end = 0; }
  unsigned long long cand_local = 0;

  for (int64_t t = warp; t < total_q; t += nwarps) {
    unsigned below = __ballot_sync(FULL, qoff_lane <= t);
    int jq = 31 - __clz(below);
    int64_t q0 = __shfl_sync(FULL, qoff_lane, jq);
    int32_t qs = __shfl_sync(FULL, B.qstart, jq);
    int32_t v = qs + (int32_t)(t - q0);

    const double phi_v = A.s.phi[v];
    const double px_v = A.s.px[v], py_v = A.s.py[v];
    const double cx_v = A.s.cx[v], cy_v = A.s.cy[v], rsq_v = A.s.rsq[v];
    const float rv = A.s.rf[v], bv = A.s.bf[v];
    const int32_t idv = kSampleIds ? A.id[v] : v;

    // ---- band windows (lane j <-> band j)
    int32_t sA = 0, eA = 0, sB = 0, eB = 0;
    if (lane < A.L && B.end > B.start) {
      float bmn = fminf(bv, B.bmin);
      float eta = A.E_over_tanh * (1.0f / bmn + 2.0f / (A.a_f * bv * B.bmin));
      float Rp = A.R_pad + fminf(eta, 64.0f);
      bool whole = rv + B.rmin <= Rp;
      double dlt = 0.0;
      if (!whole) {
        float chR = coshf(Rp);
        float num = (chR - coshf(rv - B.rmin)) + chR * 2e-6f;
        float s2 = num / (2.0f * sinhf(rv) * B.sinh_rmin);
        if (!(s2 < 1.0f)) {
          whole = true;
        } else {
          dlt = (double)(2.0f * asinf(sqrtf(fmaxf(s2, 0.0f)))) * (1.0 + 4e-3) + 1e-14;
          if (dlt >= 3.141592653589793) whole = true;
        }
      }
      if (whole) {
        sA = B.start; eA = B.end;
      } else {
        double lo = phi_v - dlt, hi = phi_v + dlt;
        if (lo < 0.0) {
          sA = B.start; eA = dir_lookup(A.dir, B.dir_base, B.shift, hi, A.C, 1);
          sB = dir_lookup(A.dir, B.dir_base, B.shift, lo + kTwoPi, A.C, 0); eB = B.end;
        } else if (hi >= kTwoPi) {
          sA = B.start; eA = dir_lookup(A.dir, B.dir_base, B.shift, hi - kTwoPi, A.C, 1);
          sB = dir_lookup(A.dir, B.dir_base, B.shift, lo, A.C, 0); eB = B.end;
        } else {
          sA = dir_lookup(A.dir, B.dir_base, B.shift, lo, A.C, 0);
          eA = dir_lookup(A.dir, B.dir_base, B.shift, hi, A.C, 1);
        }
        if (sB < eB && sB < eA) { sA = B.start; eA = B.end; sB = eB = 0; }
      }
    }
    const int32_t lenA = eA - sA;
    const int32_t cnt = lenA + (eB - sB);
    int32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t total = __shfl_sync(FULL, incl, 31);
    const int32_t excl = incl - cnt;
    cand_local += (unsigned long long)total;

    int64_t row = 0;
    if (kWrite) row = A.rowptr[idv];
    int32_t hits = 0;
    for (int32_t base = 0; base < total; base += 32) {
      int32_t i = base + lane;
      int o = 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        int32_t ex = __shfl_sync(FULL, excl, o + s);
        if (ex <= i) o += s;
      }
      int32_t tt = i - __shfl_sync(FULL, excl, o);
      int32_t la = __shfl_sync(FULL, lenA, o);
      int32_t sa = __shfl_sync(FULL, sA, o);
      int32_t sb = __shfl_sync(FULL, sB, o);
      int32_t w = tt < la ? sa + tt : sb + (tt - la);
      bool hit = false;
      int32_t idw = w;
      if (i < total && w != v) {
        if (kSampleIds) idw = A.id[w];
        if (idw < idv) {  // edge decided by w's circle (pred(w -> v))
          hit = ref_pred(px_v, py_v, A.s.cx[w], A.s.cy[w], A.s.rsq[w]);
        } else {          // by v's circle (pred(v -> w))
          hit = ref_pred(A.s.px[w], A.s.py[w], cx_v, cy_v, rsq_v);
        }
      }
      unsigned bal = __ballot_sync(FULL, hit);
      if (kWrite && hit) A.out[row + hits + __popc(bal & ((1u << lane) - 1u))] = idw;
      hits += __popc(bal);
    }
    if (!kWrite && lane == 0) A.deg[idv] = hits;
  }
  if (!kWrite && A.cand) {
    if (lane == 0) atomicAdd(A.cand, cand_local);
  }
}

// Sector bookkeeping for sample-order rows of other shards: nothing to do --
// deg[] is cleared before the count pass, so foreign rows stay empty.

__global__ void __launch_bounds__(256) k_sincos(int64_t n, const double* __restrict__ x,
                                                double* __restrict__ s, double* __restrict__ c) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) sincos_cr(x[i], s + i, c + i);
}

__global__ void __launch_bounds__(256) k_widen(int64_t n, const int32_t* __restrict__ in,
                                               int64_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace hrg
