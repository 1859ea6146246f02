// hrg_kernels.cuh -- sm_100a kernels of the random-hyperbolic-graph generator.
//
// Pipeline (one CUDA stream, see hrg_api.cu):
//   k_sample        Philox4x32-10 -> (phi, r_native, r_poincare) per vertex, plus a
//                   59-bit sort key (radial band << 53 | angular fixed point q).
//   cub radix sort  keys -> permutation into (band, angle) order.
//   k_gather        48-byte fp64 candidate records in sorted order: p_x, p_y (the
//                   point), c_x, c_y, rad^2 (its query circle), id; correctly
//                   rounded sin/cos, hrgen's circle transform (geometry.py:141-157).
//   k_band_setup / k_band_minmax / k_dir_fill / k_dir_tail
//                   per band: position range, min hyperbolic radius, max Poincare
//                   radius, and an angular directory (bucket -> first position).
//   k_plan          per query: angular window of every band -> candidate count;
//                   queries above kLightMax candidates are split into kChunk chunks.
//   k_light<COUNT>  one thread per light query: bands in order, candidates in
//                   position order, reference predicate, count hits.
//   k_heavy<COUNT>  one warp per heavy chunk (hubs): lane j owns band j's window,
//                   the warp walks the flattened segments 32 candidates at a time.
//   cub scan        degrees -> CSR row pointers (+ per-chunk offsets of hubs).
//   k_light/k_heavy<WRITE>  same traversals, writing the rows in order.
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

// Candidate record: everything one pair test needs about a vertex w, in one
// 48-byte line fragment: its point (p_x, p_y) for pred(v -> w), its circle
// (c_x, c_y, rad^2) for pred(w -> v), and its vertex id.
struct __align__(16) Rec {
  double px, py, cx, cy, rsq;
  int32_t id;
  float pad;
};

struct QRec {          // query-side extras, per sorted position
  double* phi;
  float* rf;           // hyperbolic radius 2*atanh(r) (rounded down)
  float* bf;           // (1-r)(1+r) (rounded down)
};

// Gather into (band, angle) order and precompute every per-point quantity the
// query needs.  p_x/p_y: quadtree.py:474-475; c_x/c_y/rad^2: quadtree.py:516-518
// with center_r/rad from geometry.py:141-157.
__global__ void __launch_bounds__(256) k_gather(int64_t n, const int32_t* __restrict__ perm,
                                                const double* __restrict__ phi,
                                                const double* __restrict__ rp,
                                                const double* __restrict__ rn, double a,
                                                Rec* __restrict__ rec, QRec q,
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
  Rec R;
  R.px = __dmul_rn(r, cs);
  R.py = __dmul_rn(r, sn);
  R.cx = __dmul_rn(cr, cs);
  R.cy = __dmul_rn(cr, sn);
  R.rsq = __dmul_rn(rad, rad);
  R.id = i;
  R.pad = 0.f;
  rec[p] = R;
  q.phi[p] = ph;
  // hyperbolic radius of the stored Poincare point and (1-r)(1+r), both
  // rounded down: only used to size conservative angular windows.
  double one_m = 1.0 - r;
  double re = log1p(2.0 * r / one_m);  // 2*atanh(r)
  q.rf[p] = __double2float_rd(re);
  q.bf[p] = __double2float_rd(one_m * (1.0 + r));
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

constexpr int kLightMax = 256;     // queries with more candidates take the heavy path
constexpr int kSegCap = 24;        // non-empty band segments a light query may hold
constexpr int kChunk = 2048;       // heavy-path work item: candidates of one query

struct QueryArgs {
  const Rec* rec;
  QRec q;
  const Band* bands;
  const int32_t* dir;
  const uint64_t* keys;      // sorted (band << 53 | angular key)
  int L;
  double C;                  // 2^53 / (2 pi)
  float R_pad;               // R rounded up + fp32 slack
  float a_f;                 // cosh R - 1
  float E_over_tanh;         // fp64 decision-noise constant / tanh(R)
  // staging: every query's hits land in a private slice sized by its candidates
  int32_t* stage;
  int64_t stage_cap;
  unsigned long long* bump;  // staging allocator
  int64_t* stage_off;        // per sorted position
  int* overflow;
  // heavy queries (hubs), deferred by the light pass
  int32_t* heavy_v;          // entry -> sorted position
  int32_t* heavy_c;          // entry -> candidates
  unsigned* heavy_n;
  int32_t* heavy_of;         // sorted position -> entry, or -1
  const int64_t* chunk_start;// entry -> first chunk (exclusive scan, H + 1)
  int64_t total_chunks;
  int32_t* chunk_hits;
  int32_t* deg;              // row length per vertex id
  unsigned long long* cand_total;
};

struct QView {
  double phi;
  float rv, bv, sinh_rv;
};

// drop leading positions whose angular key is below ql / trailing ones above qh
__device__ __forceinline__ void trim_lo(const uint64_t* keys, int32_t& s, int32_t e, uint64_t ql) {
  while (s < e && (__ldg(keys + s) & kQMask) < ql) ++s;
}
__device__ __forceinline__ void trim_hi(const uint64_t* keys, int32_t s, int32_t& e, uint64_t qh) {
  while (e > s && (__ldg(keys + e - 1) & kQMask) > qh) --e;
}

// Angular window of band B for query q, as <= 2 sorted-position segments
// [sA, eA) then [sB, eB).  Every w of the band whose hyperbolic distance to q
// is below R + eta lies inside, where eta bounds the fp64 decision noise of
// the reference predicate for this (q, band) pair in either orientation
// (DESIGN.md "window padding"), so no pair the predicate accepts is missed.
__device__ __forceinline__ void band_window(const QueryArgs& A, const Band& B, const QView& q,
                                            int32_t& sA, int32_t& eA, int32_t& sB,
                                            int32_t& eB) {
  sA = eA = sB = eB = 0;
  if (B.end <= B.start) return;
  float bmn = fminf(q.bv, B.bmin);
  float eta = A.E_over_tanh * (1.0f / bmn + 2.0f / (A.a_f * q.bv * B.bmin));
  float Rp = A.R_pad + fminf(eta, 64.0f);
  bool whole = q.rv + B.rmin <= Rp;
  double dlt = 0.0;
  if (!whole) {
    float chR = coshf(Rp);
    float num = (chR - coshf(q.rv - B.rmin)) + chR * 2e-6f;
    float s2 = num / (2.0f * q.sinh_rv * B.sinh_rmin);
    if (!(s2 < 1.0f)) {
      whole = true;
    } else {
      dlt = (double)(2.0f * asinf(sqrtf(fmaxf(s2, 0.0f)))) * (1.0 + 4e-3) + 1e-14;
      if (dlt >= 3.141592653589793) whole = true;
    }
  }
  if (whole) { sA = B.start; eA = B.end; return; }
  double lo = q.phi - dlt, hi = q.phi + dlt;
  const int32_t* d = A.dir + B.dir_base;
  // the directory resolves a window to whole buckets; the sorted angular keys
  // then trim the two boundary buckets exactly (keys are monotone in phi)
  if (lo < 0.0) {
    const uint64_t qh = qkey(hi, A.C), ql = qkey(lo + kTwoPi, A.C);
    sA = B.start; eA = __ldg(d + (qh >> B.shift) + 1);
    sB = __ldg(d + (ql >> B.shift)); eB = B.end;
    trim_hi(A.keys, sA, eA, qh);
    trim_lo(A.keys, sB, eB, ql);
  } else if (hi >= kTwoPi) {
    const uint64_t qh = qkey(hi - kTwoPi, A.C), ql = qkey(lo, A.C);
    sA = B.start; eA = __ldg(d + (qh >> B.shift) + 1);
    sB = __ldg(d + (ql >> B.shift)); eB = B.end;
    trim_hi(A.keys, sA, eA, qh);
    trim_lo(A.keys, sB, eB, ql);
  } else {
    const uint64_t ql = qkey(lo, A.C), qh = qkey(hi, A.C);
    sA = __ldg(d + (ql >> B.shift));
    eA = __ldg(d + (qh >> B.shift) + 1);
    trim_lo(A.keys, sA, eA, ql);
    trim_hi(A.keys, sA, eA, qh);
  }
  if (sB < eB && sB < eA) { sA = B.start; eA = B.end; sB = eB = 0; }
}

__device__ __forceinline__ Rec load_rec(const Rec* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  Rec r;
  r.px = a.x; r.py = a.y; r.cx = b.x; r.cy = b.y; r.rsq = c.x;
  r.id = (int32_t)(__double_as_longlong(c.y) & 0xffffffffll);
  r.pad = 0.f;
  return r;
}

struct QFull {
  QView v;
  double px, py, cx, cy, rsq;
  int32_t pos, idv;
};

template <bool kSampleIds>
__device__ __forceinline__ QFull load_query(const QueryArgs& A, int32_t v) {
  QFull f;
  Rec r = load_rec(A.rec + v);
  f.px = r.px; f.py = r.py; f.cx = r.cx; f.cy = r.cy; f.rsq = r.rsq;
  f.pos = v;
  f.idv = kSampleIds ? r.id : v;
  f.v.phi = A.q.phi[v];
  f.v.rv = A.q.rf[v];
  f.v.bv = A.q.bf[v];
  f.v.sinh_rv = sinhf(f.v.rv);
  return f;
}

// Edge {v, w} is decided by the circle of the smaller vertex id, exactly as
// hrgen queries from v and keeps ids > v (generator.py:182-187).
template <bool kSampleIds>
__device__ __forceinline__ bool pair_test(const QFull& f, const Rec& r, int32_t w, int32_t* idw) {
  int32_t id = kSampleIds ? r.id : w;
  *idw = id;
  if (w == f.pos) return false;
  if (id < f.idv) return ref_pred(f.px, f.py, r.cx, r.cy, r.rsq);  // pred(w -> v)
  return ref_pred(r.px, r.py, f.cx, f.cy, f.rsq);                  // pred(v -> w)
}

// Shard query enumeration: flat index t over the bands' [qstart, qend).
struct QMap {
  int64_t off[kMaxBands + 1];
  int32_t qs[kMaxBands];
};

__device__ __forceinline__ void load_qmap(const QueryArgs& A, QMap& m, Band* sb) {
  if (threadIdx.x < A.L) sb[threadIdx.x] = A.bands[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int j = 0; j < A.L; ++j) {
      m.off[j] = acc;
      m.qs[j] = sb[j].qstart;
      acc += sb[j].qend - sb[j].qstart;
    }
    m.off[A.L] = acc;
  }
  __syncthreads();
}

__device__ __forceinline__ int32_t qmap_pos(const QMap& m, int L, int64_t t) {
  int lo = 0, hi = L;  // largest j with off[j] <= t
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (m.off[mid] <= t) lo = mid; else hi = mid;
  }
  return m.qs[lo] + (int32_t)(t - m.off[lo]);
}

// Light pass: one thread per query.  Windows of all bands first (non-empty
// segments go to a per-thread list in shared memory), then one flat loop
// over the query's candidates in (band, angle) order; hits go to the
// query's staging slice.  Queries with more than kLightMax candidates or
// kSegCap segments are deferred to the heavy pass.
constexpr int kLightThreads = 128;

template <bool kSampleIds>
__global__ void __launch_bounds__(kLightThreads) k_light(QueryArgs A) {
  __shared__ Band sb[kMaxBands];
  __shared__ QMap qm;
  __shared__ int2 segs[kSegCap][kLightThreads];
  load_qmap(A, qm, sb);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int64_t total_q = qm.off[A.L];
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long cand_local = 0;
  for (int64_t tile = wid * 32; tile < total_q; tile += nw * 32) {
    const int64_t t = tile + lane;
    const bool active = t < total_q;
    const int32_t v = active ? qmap_pos(qm, A.L, t) : 0;
    QFull f = load_query<kSampleIds>(A, v);
    int nseg = 0;
    int32_t c = 0;
    bool ovf = false;
    if (active) {
      for (int j = 0; j < A.L; ++j) {
        int32_t sA, eA, sB, eB;
        band_window(A, sb[j], f.v, sA, eA, sB, eB);
        if (eA > sA) {
          if (nseg < kSegCap) segs[nseg++][tid] = make_int2(sA, eA - sA); else ovf = true;
          c += eA - sA;
        }
        if (eB > sB) {
          if (nseg < kSegCap) segs[nseg++][tid] = make_int2(sB, eB - sB); else ovf = true;
          c += eB - sB;
        }
      }
    }
    cand_local += (unsigned long long)c;
    const bool heavy = active && (c > kLightMax || ovf);
    // staging slices: warp-aggregated allocation for light queries
    int32_t want = (active && !heavy) ? c : 0;
    int32_t incl = want;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    unsigned long long base = 0;
    if (lane == 31 && incl > 0) base = atomicAdd(A.bump, (unsigned long long)incl);
    base = __shfl_sync(FULL, base, 31);
    if (!active) continue;
    if (heavy) {
      unsigned long long hoff = atomicAdd(A.bump, (unsigned long long)c);
      unsigned e = atomicAdd(A.heavy_n, 1u);
      A.heavy_v[e] = v;
      A.heavy_c[e] = c;
      A.heavy_of[v] = (int32_t)e;
      A.stage_off[v] = (int64_t)hoff;
      continue;
    }
    const int64_t off = (int64_t)base + incl - want;
    A.heavy_of[v] = -1;
    A.stage_off[v] = off;
    if (off + c > A.stage_cap) { atomicOr(A.overflow, 1); A.deg[f.idv] = 0; continue; }
    int32_t* out = A.stage + off;
    int32_t hits = 0;
    int k = 0;
    int2 sg = make_int2(0, 0);
    if (nseg > 0) sg = segs[0][tid];
    for (int32_t i = 0; i < c; ++i) {
      while (sg.y == 0) sg = segs[++k][tid];
      const int32_t w = sg.x;
      sg.x++; sg.y--;
      int32_t idw;
      if (pair_test<kSampleIds>(f, load_rec(A.rec + w), w, &idw)) out[hits++] = idw;
    }
    A.deg[f.idv] = hits;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand_local += __shfl_xor_sync(FULL, cand_local, o);
  if (lane == 0 && cand_local) atomicAdd(A.cand_total, cand_local);
}

__global__ void k_heavy_chunks(const int32_t* __restrict__ heavy_c, int64_t H,
                               int32_t* __restrict__ nchunks) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < H) nchunks[e] = (heavy_c[e] + kChunk - 1) / kChunk;
}

// Heavy pass: one warp per chunk of kChunk candidates of one deferred query;
// lanes own bands for the window phase, then stride the chunk 32 candidates
// at a time (4 batches in flight) with ballot-ordered writes into the
// chunk's slot of the query's staging slice.
template <bool kSampleIds>
__global__ void __launch_bounds__(256) k_heavy(QueryArgs A, int64_t H) {
  __shared__ Band sb[kMaxBands];
  if (threadIdx.x < A.L) sb[threadIdx.x] = A.bands[threadIdx.x];
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < A.total_chunks; c += nwarps) {
    int64_t lo = 0, hi = H;  // entry: largest e with chunk_start[e] <= c
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (A.chunk_start[mid] <= c) lo = mid; else hi = mid;
    }
    const int64_t e = lo;
    const int32_t v = A.heavy_v[e];
    const int64_t local = c - A.chunk_start[e];
    QFull f = load_query<kSampleIds>(A, v);
    int32_t sA = 0, eA = 0, sB = 0, eB = 0;
    if (lane < A.L) band_window(A, sb[lane], f.v, sA, eA, sB, eB);
    const int32_t lenA = eA - sA, cnt = lenA + (eB - sB);
    int32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int32_t total = __shfl_sync(FULL, incl, 31);
    const int32_t excl = incl - cnt;
    const int32_t beg = (int32_t)(local * kChunk);
    const int32_t end = min(total, beg + kChunk);
    const int64_t slot = A.stage_off[v] + local * kChunk;
    int32_t* out = A.stage + slot;
    const bool fits = slot + (end - beg) <= A.stage_cap;
    int32_t hits = 0;
    for (int32_t base = beg; base < end; base += 128) {
      int32_t wv[4];
      bool ok[4];
      Rec r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int32_t i = base + 32 * u + lane;
        int o = 0;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
          int32_t ex = __shfl_sync(FULL, excl, o + s);
          if (ex <= i) o += s;
        }
        int32_t tt = i - __shfl_sync(FULL, excl, o);
        int32_t la = __shfl_sync(FULL, lenA, o);
        int32_t sa = __shfl_sync(FULL, sA, o);
        int32_t sbb = __shfl_sync(FULL, sB, o);
        wv[u] = tt < la ? sa + tt : sbb + (tt - la);
        ok[u] = i < end;
        if (ok[u]) r[u] = load_rec(A.rec + wv[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int32_t idw = 0;
        bool hit = ok[u] && pair_test<kSampleIds>(f, r[u], wv[u], &idw);
        unsigned bal = __ballot_sync(FULL, hit);
        if (hit && fits) out[hits + __popc(bal & ((1u << lane) - 1u))] = idw;
        hits += __popc(bal);
      }
    }
    if (lane == 0) {
      if (!fits) atomicOr(A.overflow, 1);
      A.chunk_hits[c] = hits;
      atomicAdd(&A.deg[f.idv], hits);
    }
  }
}

// Warp-wide bitonic sort of 32*E keys held E per lane (element index
// e = lane*E + t), ascending.
template <int E>
__device__ __forceinline__ void warp_bitonic(int32_t (&x)[E], int lane) {
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
        const int lj = j / E;
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int e = lane * E + t;
          int32_t y = __shfl_xor_sync(0xffffffffu, x[t], lj);
          const bool up = (e & k) == 0;
          const bool lower = (e & j) == 0;
          // keep min if (lower == up) else max
          x[t] = (lower == up) ? min(x[t], y) : max(x[t], y);
        }
      } else {
#pragma unroll
        for (int t = 0; t < E; ++t) {
          const int t2 = t ^ j;
          if (t2 > t) {
            const int e = lane * E + t;
            const bool up = (e & k) == 0;
            int32_t a = x[t], b = x[t2];
            x[t] = up ? min(a, b) : max(a, b);
            x[t2] = up ? max(a, b) : min(a, b);
          }
        }
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void copy_sorted_row(const int32_t* __restrict__ src,
                                                int32_t* __restrict__ dst, int32_t len,
                                                int lane) {
  int32_t x[E];
#pragma unroll
  for (int t = 0; t < E; ++t) {
    const int e = lane * E + t;
    x[t] = e < len ? __ldg(src + e) : INT32_MAX;
  }
  warp_bitonic<E>(x, lane);
#pragma unroll
  for (int t = 0; t < E; ++t) {
    const int e = lane * E + t;
    if (e < len) dst[e] = x[t];
  }
}

// Compaction of light rows: a warp owns 32 consecutive queries and moves
// their rows, one row at a time 32 lanes wide, from the staging slices to
// the CSR slots rowptr[id].  With sample-order ids the row is sorted on the
// way through (registers + shuffles), which is the order hrgen's Graph keeps.
template <bool kSampleIds>
__global__ void __launch_bounds__(256) k_compact_light(QueryArgs A,
                                                       const int64_t* __restrict__ rowptr,
                                                       int32_t* __restrict__ idx) {
  __shared__ Band sb[kMaxBands];
  __shared__ QMap qm;
  load_qmap(A, qm, sb);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t total_q = qm.off[A.L];
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t tile = wid * 32; tile < total_q; tile += nw * 32) {
    const int64_t t = tile + lane;
    const bool active = t < total_q;
    const int32_t v = active ? qmap_pos(qm, A.L, t) : 0;
    const int32_t idv = kSampleIds ? (int32_t)(__double_as_longlong(__ldg(
                                         reinterpret_cast<const double*>(A.rec + v) + 5)) &
                                     0xffffffffll)
                                   : v;
    const bool light = active && A.heavy_of[v] < 0;
    const int64_t dst = light ? rowptr[idv] : 0;
    const int32_t len = light ? (int32_t)(rowptr[idv + 1] - dst) : 0;
    const int64_t src = light ? A.stage_off[v] : 0;
    unsigned todo = __ballot_sync(FULL, len > 0);
    while (todo) {
      const int l = __ffs(todo) - 1;
      todo &= todo - 1;
      const int64_t d = __shfl_sync(FULL, dst, l);
      const int32_t ln = __shfl_sync(FULL, len, l);
      const int64_t s0 = __shfl_sync(FULL, src, l);
      const int32_t* in = A.stage + s0;
      int32_t* out = idx + d;
      if (!kSampleIds) {
        int32_t x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = lane + 32 * u;
          x[u] = k < ln ? __ldg(in + k) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = lane + 32 * u;
          if (k < ln) out[k] = x[u];
        }
      } else if (ln <= 32) {
        copy_sorted_row<1>(in, out, ln, lane);
      } else if (ln <= 64) {
        copy_sorted_row<2>(in, out, ln, lane);
      } else if (ln <= 128) {
        copy_sorted_row<4>(in, out, ln, lane);
      } else {
        copy_sorted_row<8>(in, out, ln, lane);
      }
    }
  }
}

// Compaction of heavy rows: one warp per chunk; the chunk's hits go to
// rowptr[id] + (hits of the row's earlier chunks).
__global__ void __launch_bounds__(256) k_compact_heavy(QueryArgs A, int64_t H,
                                                       const int64_t* __restrict__ chunk_off,
                                                       const int64_t* __restrict__ rowptr,
                                                       int32_t* __restrict__ idx,
                                                       bool sample_ids) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < A.total_chunks; c += nwarps) {
    int64_t lo = 0, hi = H;
    while (hi - lo > 1) {
      int64_t mid = (lo + hi) >> 1;
      if (A.chunk_start[mid] <= c) lo = mid; else hi = mid;
    }
    const int64_t e = lo;
    const int32_t v = A.heavy_v[e];
    const int32_t idv = sample_ids ? (int32_t)(__double_as_longlong(__ldg(
                                         reinterpret_cast<const double*>(A.rec + v) + 5)) &
                                     0xffffffffll)
                                   : v;
    const int64_t c0 = A.chunk_start[e];
    const int64_t d = rowptr[idv] + (chunk_off[c] - chunk_off[c0]);
    const int32_t h = A.chunk_hits[c];
    const int32_t* in = A.stage + A.stage_off[v] + (c - c0) * kChunk;
    for (int32_t k0 = 0; k0 < h; k0 += 256) {
      int32_t x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + lane + 32 * u;
        x[u] = k < h ? __ldg(in + k) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + lane + 32 * u;
        if (k < h) idx[d + k] = x[u];
      }
    }
  }
}

// begin/end offsets of the heavy rows (sample-order ids: these rows still
// need sorting after the chunk-parallel copy)
__global__ void k_heavy_segments(QueryArgs A, int64_t H, const int64_t* __restrict__ rowptr,
                                 int64_t* __restrict__ seg_begin, int64_t* __restrict__ seg_end) {
  int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= H) return;
  const int32_t v = A.heavy_v[e];
  const int32_t idv = (int32_t)(__double_as_longlong(
                                    __ldg(reinterpret_cast<const double*>(A.rec + v) + 5)) &
                                0xffffffffll);
  seg_begin[e] = rowptr[idv];
  seg_end[e] = rowptr[idv + 1];
}

__global__ void __launch_bounds__(256) k_copy_segments(const int32_t* __restrict__ from,
                                                       int32_t* __restrict__ to,
                                                       const int64_t* __restrict__ b,
                                                       const int64_t* __restrict__ e,
                                                       int64_t H) {
  for (int64_t s = blockIdx.x; s < H; s += gridDim.x)
    for (int64_t k = b[s] + threadIdx.x; k < e[s]; k += blockDim.x) to[k] = from[k];
}

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
