// hrg_kernels.cuh -- sm_100a kernels of the random-hyperbolic-graph generator.
//
// Pipeline (the context's stream; the row-sort classes on two side streams;
// see hrg_api.cu and DESIGN.md):
//   k_sample         Philox4x32-10 -> packed (phi, r_p), 32-bit sort key
//                    (radial band << 27 | top 27 bits of the angle), id.
//                    Sharded runs: k_shard_keys / k_shard_select /
//                    k_shard_points keep only the points the sector can reach.
//   cub radix sort   keys -> permutation into (band, angle) order.
//   k_gather         fp64 records in sorted order: the 16-byte point (p_x, p_y)
//                    every pair test reads, and the 32-byte query circle
//                    (c_x, c_y, rad^2) of the query side and the rare
//                    other-orientation test; glibc's sin/cos bit for bit,
//                    hrgen's circle transform (geometry.py:141-157); per-band
//                    innermost radius; 1/D per point (the test's margin).
//   k_band_setup / k_dir_fill / k_dir_gaps / k_dir_tail / k_window_table /
//   k_tile_table     per band: position and sector ranges, an angular
//                    directory (bucket -> first position); per query-radius row
//                    and band: the angular half-width of a conservative window;
//                    query tiles (32 consecutive positions of one band; the
//                    outer bands' tiles interleaved by angle).
//   k_light          a warp per tile: per-band union windows; small unions
//                    tested as a dense block (lane = query), the other bands
//                    resolved per query (integer windows), segments flattened,
//                    a lane-strided walk over the candidates; the reference
//                    predicate in one orientation (the other inside the
//                    rounding margin), hits compacted into staging; queries
//                    with too many candidates or segments are deferred.
//   k_heavy          a warp per 2048-candidate chunk of a deferred query (hubs).
//   cub scan         degrees -> CSR row pointers (+ per-chunk offsets of hubs).
//   k_compact_light / k_compact_heavy   staging -> CSR rows; rows of <= 64 ids
//                    sorted in registers on the way.
//   k_sort_warp / k_sort_rows / k_giant_*   longer rows sorted by length class.
//
// Replaces hrgen quadtree.py (build 303-340, pack 399-495, query_many 499-631)
// and generator.py:190-225.
#pragma once
#include <stdint.h>
#include <utility>
#include "hrg_math.cuh"
#include "hrg_libm_trig.cuh"

namespace hrg {

// tuning knobs (-D overrides for experiments)
#ifndef HRG_WALK_UNROLL
#define HRG_WALK_UNROLL 2
#endif
#ifndef HRG_BAND_GROUP
#define HRG_BAND_GROUP 1
#endif
#ifndef HRG_SMALL_SLOTS
#define HRG_SMALL_SLOTS 64
#endif
#ifndef HRG_TRIM_UNION
#define HRG_TRIM_UNION 1
#endif
#ifndef HRG_DIR_EXTRA
#define HRG_DIR_EXTRA 1
#endif
#ifndef HRG_UNION_SMALL
#define HRG_UNION_SMALL 2
#endif
#ifndef HRG_DENSE_MAX
#define HRG_DENSE_MAX 8
#endif
#ifndef HRG_DENSE_BIG
#define HRG_DENSE_BIG 48
#endif
#ifndef HRG_DENSE_RATIO
#define HRG_DENSE_RATIO 0.25f
#endif
#ifndef HRG_MID_SHIFT
#define HRG_MID_SHIFT -1
#endif
#ifndef HRG_ELEM_WRITE
#define HRG_ELEM_WRITE 1
#endif
#ifndef HRG_COMPACT_MINB
#define HRG_COMPACT_MINB 5
#endif
#ifndef HRG_SEGCAP
#define HRG_SEGCAP 12
#endif
#ifndef HRG_LIGHT_MAX
#define HRG_LIGHT_MAX 2048
#endif
#ifndef HRG_WARP_BUCKET_MAX
#define HRG_WARP_BUCKET_MAX 512
#endif
#ifndef HRG_TILE_HITS
#define HRG_TILE_HITS 2048
#endif
#ifndef HRG_SORTWARP_MINB
#define HRG_SORTWARP_MINB 6
#endif
#ifndef HRG_SORT_GRID
#define HRG_SORT_GRID 12
#endif
#ifndef HRG_HEAVY_MINB
#define HRG_HEAVY_MINB 3
#endif
#ifndef HRG_HEAVY_BATCH
#define HRG_HEAVY_BATCH 4
#endif
#ifndef HRG_LIGHT_MINBLOCKS
#define HRG_LIGHT_MINBLOCKS 8
#endif

constexpr int kMaxBands = 32;     // one warp lane per radial band
constexpr int kTrigLibm = 0;      // glibc's sin/cos, bit for bit (hrgen's arithmetic; default)
constexpr int kTrigCR = 1;        // correctly rounded sin/cos

// cos/sin of an angle in [0, 2pi) as the context's trig mode asks
__device__ __forceinline__ void trig_sincos(int trig, double x, double* sn, double* cs) {
  if (trig == kTrigLibm) {
    *sn = libm::sin(x);
    *cs = libm::cos(x);
  } else {
    sincos_crf(x, sn, cs);
  }
}
constexpr int kQBits = 53;
constexpr uint64_t kQMask = (1ull << kQBits) - 1;
constexpr double kTwoPi = 6.283185307179586;  // == 2.0 * math.pi (geometry.py:19)

struct Band {
  int32_t start, end;      // sorted positions of the band
  int32_t qstart, qend;    // query positions (this shard's angular sector)
  int64_t dir_base;        // offset of the band's directory in dir[]
  int32_t shift;           // bucket(q) = q >> shift
  int32_t nb;              // buckets (power of two); directory has nb + 1 entries
  double pmin;             // innermost Poincare radius of the band's points
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

// The same count by binary search over the thresholds staged in shared
// memory (thr non-decreasing; entries past L hold +inf).
__device__ __forceinline__ int band_of_smem(const double* thr, double rp) {
  int b = 0;
#pragma unroll
  for (int st = 16; st > 0; st >>= 1)
    if (thr[b + st] <= rp) b += st;
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

// Sort key: band << 27 | top 27 bits of the angular key.  Points are ordered
// by (band, angle) to 2^-27 of a turn; ties keep draw order (stable sort).
// Everything that relies on the order works at that granularity or coarser:
// directory buckets (shift >= kSortShift), shard sector bounds (multiples of
// 2^kSortShift) and the exact key trims, which drop a point only on its own
// full key and so stay correct on any order.
constexpr int kSortShift = kQBits - 27;
constexpr int kDirExtra = HRG_DIR_EXTRA;  // directory buckets per point: 1-2 x 2^kDirExtra
__device__ __forceinline__ uint32_t sort_key32(int band, uint64_t q) {
  return ((uint32_t)band << 27) | (uint32_t)(q >> kSortShift);
}

// hrgen generator.py:160-179 with a counter-based stream: vertex i draws its
// angle from the first and its radius from the second 53-bit uniform of
// Philox4x32-10(counter = i, key = seed).
__device__ __forceinline__ void philox_u53(int64_t i, uint64_t seed, uint64_t& a, uint64_t& b) {
  uint32_t c[4] = {(uint32_t)i, (uint32_t)((uint64_t)i >> 32), 0u, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  a = (((uint64_t)c[1] << 32) | c[0]) >> 11;
  b = (((uint64_t)c[3] << 32) | c[2]) >> 11;
}

__device__ __forceinline__ double angle_from_u53(uint64_t a) {
  return __dmul_rn(kTwoPi, (double)a * 0x1.0p-53);                    // :170
}

__device__ __forceinline__ void radius_from_u53(uint64_t b, const SampleParams& P, double& r,
                                                double& p) {
  const double u2 = (double)b * 0x1.0p-53;
  r = __dmul_rn(P.two_over_alpha, asinh(__dmul_rn(__dsqrt_rn(u2), P.sinh_half)));
  r = fmin(r, P.r_cap);                                                // :174
  p = fmin(tanh(__dmul_rn(r, 0.5)), P.rp_cap);                        // :175-178
}

__device__ __forceinline__ void sample_point(int64_t i, const SampleParams& P, double& ph,
                                             double& r, double& p) {
  uint64_t a, b;
  philox_u53(i, P.seed, a, b);
  ph = angle_from_u53(a);
  radius_from_u53(b, P, r, p);
}

// The pipeline's sampler: packed (phi, r_p), sort key and id per vertex; the
// API's coordinate arrays only when asked for (a generation materialises
// them later, on request, with k_sample_coords -- same stream, same bits).
__global__ void __launch_bounds__(256) k_sample(int64_t n, SampleParams P, BandSpec S,
                                                double* __restrict__ phi, double* __restrict__ rn,
                                                double* __restrict__ rp,
                                                uint32_t* __restrict__ keys,
                                                int32_t* __restrict__ vals,
                                                double2* __restrict__ pr) {
  __shared__ double s_thr[kMaxBands];
  if (threadIdx.x < kMaxBands)
    s_thr[threadIdx.x] =
        threadIdx.x < S.L ? S.thr[threadIdx.x] : __longlong_as_double(0x7ff0000000000000ll);
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ph, r, p;
  sample_point(i, P, ph, r, p);
  if (phi) phi[i] = ph;
  if (rn) rn[i] = r;
  if (rp) rp[i] = p;
  pr[i] = make_double2(ph, p);
  keys[i] = sort_key32(band_of_smem(s_thr, p), qkey(ph, P.C));
  vals[i] = (int32_t)i;
}

__global__ void __launch_bounds__(256) k_sample_coords(int64_t n, SampleParams P,
                                                       double* __restrict__ phi,
                                                       double* __restrict__ rn,
                                                       double* __restrict__ rp) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ph, r, p;
  sample_point(i, P, ph, r, p);
  phi[i] = ph; rn[i] = r; rp[i] = p;
}

// smallest Poincare radius (positive doubles order like their bit patterns)
__global__ void __launch_bounds__(256) k_min_rp(int64_t n, const double2* __restrict__ pr,
                                                unsigned long long* __restrict__ out) {
  unsigned long long m = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = min(m, (unsigned long long)__double_as_longlong(pr[i].y));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

// Keys for caller-supplied coordinates; flags points outside the tree region
// (hrgen quadtree.py:293-299 raises OutOfBoundsError for those).
__global__ void __launch_bounds__(256) k_keys_from_coords(int64_t n, const double* __restrict__ phi,
                                                          const double* __restrict__ rp,
                                                          double max_r, double C, BandSpec S,
                                                          double* __restrict__ rn,
                                                          uint32_t* __restrict__ keys,
                                                          int32_t* __restrict__ vals,
                                                          int* __restrict__ bad,
                                                          double2* __restrict__ pr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ph = phi[i], p = rp[i];
  if (!(ph >= 0.0 && ph < kTwoPi && p >= 0.0 && p < max_r)) { atomicOr(bad, 1); p = 0.0; ph = 0.0; }
  rn[i] = 2.0 * atanh(p);  // geometry.py:121 to_native_radius
  pr[i] = make_double2(ph, p);
  keys[i] = sort_key32(band_of(S, p), qkey(ph, C));
  vals[i] = (int32_t)i;
}

// Per-point records, split so a pair test fetches only what it needs: the
// point (p_x, p_y), 16 B, for pred(v -> w) -- every candidate -- and the circle
// (c_x, c_y, rad^2), 32 B, for the query side and for pred(w -> v) inside the
// rounding margin; the vertex id (4 B, the sort permutation) beside them.
struct __align__(16) Circ {
  double cx, cy, rsq;
  float rf;    // a lower bound of the hyperbolic radius 2 atanh(r) (window-table row)
  float invd;  // an upper bound of 1 / D, D = a (1 - r)(1 + r) + 2 (the pair test's margin)
};

struct Recs {
  double2* pt;          // the point (p_x, p_y): what a pair test reads of a candidate
  Circ* circ;           // the query circle: the query side, and the rare other orientation
  const int32_t* ids;   // sorted position -> vertex id (sample order)
};

struct QRec {          // query-side extras, per sorted position
  double* phi;
};

// Gather into (band, angle) order and precompute every per-point quantity the
// query needs.  p_x/p_y: quadtree.py:474-475; c_x/c_y/rad^2: quadtree.py:516-518
// with center_r/rad from geometry.py:141-157.
// (phi, r_p) arrive packed (one 16 B random read per point, the DRAM burst
// granularity, instead of one per array); the full key is rebuilt from the
// band bits of the sort key and qkey(phi), the same function k_sample used.
template <bool kSampleIds>
__global__ void __launch_bounds__(256) k_gather(int64_t n, const int32_t* perm,
                                                const uint32_t* __restrict__ k32,
                                                uint64_t* __restrict__ keys_out, double C,
                                                const double2* __restrict__ pr,
                                                const double* __restrict__ rn, double a,
                                                Recs rec, QRec q,
                                                double* __restrict__ s_rp,
                                                double* __restrict__ s_rn,
                                                const int32_t* __restrict__ gid,
                                                int32_t* ids_out,
                                                unsigned long long* __restrict__ band_pmin,
                                                int trig) {
  // innermost Poincare radius per band (non-negative doubles order like
  // their bits): warp reduction when a warp's points share a band (sorted
  // positions: nearly always), shared memory, one global atomic per band
  // per block
  __shared__ unsigned long long s_pmin[kMaxBands];
  if (threadIdx.x < kMaxBands) s_pmin[threadIdx.x] = ~0ull;
  __syncthreads();
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = p < n;
  {
    const int band = ok ? (int)(k32[p] >> 27) : -1;
    unsigned long long v = ok ? (unsigned long long)__double_as_longlong(pr[perm[p]].y) : ~0ull;
    const unsigned FULL = 0xffffffffu;
    const int b0 = __shfl_sync(FULL, band, 0);
    if (__all_sync(FULL, band == b0)) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
      if ((threadIdx.x & 31) == 0 && b0 >= 0) atomicMin(&s_pmin[b0], v);
    } else if (ok) {
      atomicMin(&s_pmin[band], v);
    }
  }
  __syncthreads();
  if (threadIdx.x < kMaxBands && s_pmin[threadIdx.x] != ~0ull)
    atomicMin(band_pmin + threadIdx.x, s_pmin[threadIdx.x]);
  if (!ok) return;
  const int32_t i = perm[p];
  // sharded sampling: perm holds compact indices; ids_out (== perm) gets
  // the global vertex id in place (same element, same thread)
  const int32_t id = gid ? __ldg(gid + i) : i;
  if (gid) ids_out[p] = id;
  const double2 q2 = pr[i];
  const double ph = q2.x, r = q2.y;
  keys_out[p] = ((uint64_t)(k32[p] >> 27) << kQBits) | qkey(ph, C);
  double sn, cs;
  trig_sincos(trig, ph, &sn, &cs);  // quadtree.py:474-475 / 516-517
  double cr, rad;
  circle_params(r, a, &cr, &rad);
  const double px = __dmul_rn(r, cs), py = __dmul_rn(r, sn);
  const double cx = __dmul_rn(cr, cs), cy = __dmul_rn(cr, sn), rsq = __dmul_rn(rad, rad);
  rec.pt[p] = make_double2(px, py);
  Circ ci;
  ci.cx = cx; ci.cy = cy; ci.rsq = rsq;
  {
    // 1 / D rounded up (float) with 2^-18 of slack: D = a b + 2 errs by a few
    // ulps here, the walk's margin only needs an upper bound
    const double D = a * ((1.0 - r) * (1.0 + r)) + 2.0;
    ci.invd = __double2float_ru(1.0 / D) * (1.0f + 0x1p-18f);
  }
  q.phi[p] = ph;
  // a lower bound of the hyperbolic radius of the stored Poincare point,
  // only used to pick the window-table row (a smaller radius picks a row
  // of wider windows): 2 atanh(r) = log((1 + r)/(1 - r)) in float, with
  // 1 - r exact in double (r <= 1 - 2^-53), then 1e-5 relative and 1e-5
  // absolute taken off (float log and division err by < 1e-6 relative)
  const float lr = __logf(__fdividef((float)(1.0 + r), (float)(1.0 - r)));
  ci.rf = fmaxf(0.0f, lr * (1.0f - 1e-5f) - 1e-5f);
  rec.circ[p] = ci;
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

// Warp-cooperative lower bound: 32 probes per step, so ~log32(n) dependent
// loads instead of log2(n) (each a DRAM round trip on a cold array).
__device__ __forceinline__ int64_t warp_lower_bound_u64(const uint64_t* a, int64_t n, uint64_t key,
                                                        int lane) {
  const unsigned FULL = 0xffffffffu;
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + (int64_t)lane * step;
    const bool pred = p < hi && a[p] < key;
    const int c = __popc(__ballot_sync(FULL, pred));
    if (c == 0) return lo;
    const int64_t nlo = lo + (int64_t)(c - 1) * step + 1;
    const int64_t nhi = min(hi, lo + (int64_t)c * step);
    lo = nlo;
    hi = nhi;
  }
  const int64_t p = lo + lane;
  const bool pred = p < hi && a[p] < key;
  return lo + __popc(__ballot_sync(FULL, pred));
}

// One block: band position ranges, shard query ranges, directory sizing.
__global__ void k_band_setup(const uint64_t* __restrict__ keys, int64_t n, int L,
                             uint64_t qsec_lo, uint64_t qsec_hi, Band* __restrict__ bands,
                             int64_t* __restrict__ dir_total,
                             const float* __restrict__ cover,
                             const unsigned long long* __restrict__ band_pmin) {
  // searches by warp (block of 32 warps): band starts, then sector bounds
  __shared__ int64_t st[kMaxBands + 1], sq0[kMaxBands], sq1[kMaxBands];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = w; t < 3 * (kMaxBands + 1); t += nw) {
    const int which = t / (kMaxBands + 1), b = t % (kMaxBands + 1);
    if (b > L || (which > 0 && b >= L)) continue;
    const uint64_t base = (uint64_t)b << kQBits;
    if (which == 0) {
      const int64_t r = warp_lower_bound_u64(keys, n, base, lane);
      if (lane == 0) st[b] = r;
    } else if (which == 1) {
      const int64_t r = warp_lower_bound_u64(keys, n, base | qsec_lo, lane);
      if (lane == 0) sq0[b] = r;
    } else if (qsec_hi <= kQMask) {
      const int64_t r = warp_lower_bound_u64(keys, n, base | qsec_hi, lane);
      if (lane == 0) sq1[b] = r;
    }
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < L) {
    Band B;
    B.start = (int32_t)st[j];
    B.end = (int32_t)st[j + 1];
    B.qstart = (int32_t)sq0[j];
    B.qend = qsec_hi > kQMask ? B.end : (int32_t)sq1[j];
    int64_t cnt = B.end - B.start;
    // a sharded run's subset covers only part of the circle: size the
    // directory for the band's density, not its count
    if (cover && cnt > 0) cnt = (int64_t)ceil((double)cnt / fmax((double)cover[j], 1e-6));
    int lg = 0;
    while ((1ll << lg) < cnt && lg < kQBits - kSortShift) ++lg;  // nb = next pow2 >= cnt
    lg = min(lg + kDirExtra, kQBits - kSortShift);                // (x 2^kDirExtra)
    B.nb = 1 << lg;
    B.shift = kQBits - lg;

    // innermost radius from k_gather (+inf for an empty band)
    B.pmin = B.end > B.start ? __longlong_as_double((long long)band_pmin[j])
                             : __longlong_as_double(0x7ff0000000000000ll);
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


// dir[base + k] = first position of the band whose bucket >= k.
// dir[b] = first position of the band whose bucket is >= b: every point
// fills the buckets between its predecessor's and its own.  Gaps longer than
// kDirGapInline buckets (empty angular stretches: sparse inner bands, the
// region outside a sharded run's sector) are queued for k_dir_gaps.
constexpr int kDirGapInline = 64;
struct DirGap {
  int64_t begin, end;
  int32_t value, pad;
};

__global__ void __launch_bounds__(256) k_dir_fill(int64_t n, const uint64_t* __restrict__ keys,
                                                  const Band* __restrict__ bands,
                                                  int32_t* __restrict__ dir,
                                                  DirGap* __restrict__ gaps,
                                                  unsigned* __restrict__ ngaps) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint64_t key = keys[p];
  int j = (int)(key >> kQBits);
  Band B = bands[j];
  int64_t b = (int64_t)((key & kQMask) >> B.shift);
  int64_t bprev = -1;
  if (p > B.start) bprev = (int64_t)((keys[p - 1] & kQMask) >> B.shift);
  if (b - bprev <= kDirGapInline) {
    for (int64_t k = bprev + 1; k <= b; ++k) dir[B.dir_base + k] = (int32_t)p;
  } else {
    const unsigned g = atomicAdd(ngaps, 1u);
    gaps[g].begin = bprev + 1;
    gaps[g].end = b + 1;
    gaps[g].value = (int32_t)p;
    gaps[g].pad = j;
  }
}

// Sharded subset: only the buckets of a band's needed range (+1 either side,
// circular) are ever looked up; the rest of a gap is left unwritten.
struct ShardRanges {
  const int64_t* lo;  // 27-bit key units, see k_shard_ranges
  const int64_t* hi;
  const int* mode;    // -1 none, 0 [lo, hi), 1 whole band
};

__device__ __forceinline__ void fill_range(int32_t* dir, const Band& B, int64_t b0, int64_t b1,
                                           int32_t value, const ShardRanges* R, int j, int t0,
                                           int nt) {
  if (R && R->mode[j] == 0) {
    const int64_t bl = ((R->lo[j] << kSortShift) >> B.shift) - 1;
    const int64_t bh = ((R->hi[j] << kSortShift) >> B.shift) + 2;
    int64_t lo[2], hi[2];
    int m = 0;
    if (R->lo[j] <= R->hi[j]) { lo[0] = bl; hi[0] = bh; m = 1; }
    else { lo[0] = bl; hi[0] = B.nb + 1; lo[1] = 0; hi[1] = bh; m = 2; }
    for (int r = 0; r < m; ++r) {
      const int64_t a = max(b0, lo[r]), e = min(b1, hi[r]);
      for (int64_t k = a + t0; k < e; k += nt) dir[B.dir_base + k] = value;
    }
  } else {
    for (int64_t k = b0 + t0; k < b1; k += nt) dir[B.dir_base + k] = value;
  }
}

__global__ void __launch_bounds__(256) k_dir_gaps(const DirGap* __restrict__ gaps,
                                                  const unsigned* __restrict__ ngaps,
                                                  const Band* __restrict__ bands,
                                                  int32_t* __restrict__ dir, ShardRanges R,
                                                  bool sharded) {
  const unsigned ng = *ngaps;
  for (unsigned g = blockIdx.x; g < ng; g += gridDim.x) {
    const DirGap G = gaps[g];
    const Band B = bands[G.pad];
    fill_range(dir, B, G.begin, G.end, G.value, sharded ? &R : nullptr, G.pad, threadIdx.x,
               blockDim.x);
  }
}

__global__ void k_dir_tail(const uint64_t* __restrict__ keys, const Band* __restrict__ bands,
                           int32_t* __restrict__ dir, ShardRanges R, bool sharded) {
  Band B = bands[blockIdx.x];
  int64_t last = -1;
  if (B.end > B.start) last = (int64_t)((keys[B.end - 1] & kQMask) >> B.shift);
  fill_range(dir, B, last + 1, (int64_t)B.nb + 1, B.end, sharded ? &R : nullptr, blockIdx.x,
             threadIdx.x, blockDim.x);
}

constexpr int kLightMax = HRG_LIGHT_MAX;  // queries with more candidates take the heavy path
constexpr int kSegCap = HRG_SEGCAP;  // non-empty band segments a light query may hold
constexpr int kChunk = 2048;       // heavy-path work item: candidates of one query
constexpr int kLightThreads = 128;
constexpr float kRowStep = 1.0f / 16.0f;  // window table: query-radius row height

struct QueryArgs {
  Recs rec;
  QRec q;
  const Band* bands;
  const int32_t* dir;
  const uint64_t* keys;      // sorted (band << 53 | angular key)
  const float* wtab;         // window half-width per (query-radius row, band); >= pi: whole band
  const uint32_t* wtab_q;    // the same in 2^-32 turns (window_units)
  int wrows;
  int L;
  double C;                  // 2^53 / (2 pi)
  double a;                  // 2 sinh^2(R/2) = cosh R - 1 (geometry.py:149)
  int32_t light_max;         // queries with more candidates are deferred (<= kLightMax)
  // staging: every light query owns one slot per candidate (hit id or -1);
  // a heavy query's slice holds its chunks' compacted hits at chunk * kChunk
  int32_t* stage;
  int64_t stage_cap;
  unsigned long long* bump;  // staging allocator
  int64_t* stage_off;        // per sorted position
  int32_t* slots;            // per sorted position: candidates (= slots for light)
  int* overflow;
  // heavy queries (hubs), deferred by the light pass
  int32_t* heavy_v;          // entry -> sorted position
  int32_t* heavy_c;          // entry -> candidates
  unsigned* heavy_n;
  int32_t* heavy_of;         // sorted position -> entry, or -1
  const int64_t* chunk_start;// entry -> first chunk (exclusive scan, H + 1)
  const int32_t* chunk_entry;// chunk -> entry
  const int64_t* total_chunks;  // device scalar (k_heavy_prep)
  int32_t* chunk_hits;
  int32_t* deg;              // row length per output row
  // output row of a sorted position: nullptr = the vertex id (ids[] in
  // sample order, the position itself in angular order); sharded runs:
  // compact rows, one per query of the sector, in position order
  const int32_t* rowidx;
  unsigned long long* cand_total;
  // query tiles: 32 consecutive positions of one band (start | end << 32;
  // ~0 = no tile)
  const uint64_t* tiles;
  int64_t ntiles;            // entries (an upper bound on the tiles)
  unsigned long long* tile_next;  // dynamic tile counters: k_light, k_compact_light
};

template <bool kSampleIds>
__device__ __forceinline__ int32_t row_of(const QueryArgs& A, int32_t v) {
  return A.rowidx ? __ldg(A.rowidx + v) : (kSampleIds ? __ldg(A.rec.ids + v) : v);
}

// Compact rows of a sharded run: row k = the k-th query position of the
// sector (bands in order), rowidx[pos] = k, row_ids[k] = its vertex id;
// nq = the row count.
__global__ void k_rowidx(const Band* __restrict__ bands, int L, const int32_t* __restrict__ ids,
                         int32_t* __restrict__ rowidx, int32_t* __restrict__ row_ids,
                         int64_t* __restrict__ nq) {
  // base[j]: first row of band j (+inf past L, for the search)
  __shared__ int64_t base[kMaxBands], s_total;
  __shared__ int32_t qs0[kMaxBands];
  if (threadIdx.x == 0) {
    int64_t a = 0;
    for (int j = 0; j < kMaxBands; ++j) {
      base[j] = j < L ? a : INT64_MAX;
      qs0[j] = j < L ? bands[j].qstart : 0;
      if (j < L) a += max(0, bands[j].qend - bands[j].qstart);
    }
    s_total = a;
    if (blockIdx.x == 0) *nq = a;
  }
  __syncthreads();
  const int64_t total = s_total;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;  // last band with base[j] <= k (binary search; bands past L are +inf)
#pragma unroll
    for (int st = 16; st > 0; st >>= 1)
      if (base[j + st] <= k) j += st;
    const int32_t pos = qs0[j] + (int32_t)(k - base[j]);
    rowidx[pos] = (int32_t)k;
    row_ids[k] = ids[pos];
  }
}

// Tile table: every band's query range cut into tiles of 32 positions.  The
// light pass takes tiles in table order.  Bands below first_mixed come band
// after band (the inner bands' tiles are the expensive ones and start first);
// the tiles of the outer bands, which hold nearly all points, are interleaved
// by their relative position in the band -- their angle, up to sampling noise --
// so the tiles in flight share one angular sector of every band and the L2
// serves the sweep (one pass over the records instead of one per query band).
// The interleave is a rank, not a sort: tile t of nt_j precedes tile t' of
// nt_j' iff (2t + 1) nt_j' < (2t' + 1) nt_j, ties by band -- a total order on
// exact integers, so the ranks are a permutation.
#ifndef HRG_TILE_MIX
#define HRG_TILE_MIX 5
#endif
constexpr int kTileMixBands = HRG_TILE_MIX;  // outermost bands whose tiles interleave
__global__ void k_tile_table(const Band* __restrict__ bands, int L, int64_t ntmax,
                             uint64_t* __restrict__ tval, int first_mixed) {
  __shared__ int64_t pre[kMaxBands + 1];
  if (threadIdx.x == 0) {
    int64_t a = 0;
    for (int j = 0; j < L; ++j) {
      pre[j] = a;
      a += max(0, bands[j].qend - bands[j].qstart + 31) / 32;
    }
    pre[L] = a;
  }
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ntmax;
       k += (int64_t)gridDim.x * blockDim.x) {
    if (k >= pre[L]) {
      tval[k] = ~0ull;
      continue;
    }
    int j = 0;
    while (j + 1 < L && pre[j + 1] <= k) ++j;
    const int64_t t = k - pre[j];
    const int64_t s = bands[j].qstart + t * 32;
    const int64_t e = min(s + 32, (int64_t)bands[j].qend);
    int64_t rank = k;
    if (j >= first_mixed) {
      const int64_t nt = pre[j + 1] - pre[j];
      rank = pre[first_mixed];
      for (int jj = first_mixed; jj < L; ++jj) {
        const int64_t ntj = pre[jj + 1] - pre[jj];
        if (jj == j) { rank += t; continue; }
        // tiles t' of band jj ahead of (j, t): (2t' + 1) nt < (2t + 1) ntj,
        // or <= when jj < j
        const int64_t B = (2 * t + 1) * ntj;
        const int64_t q = jj < j ? B / nt : (B - 1) / nt;  // 2t' + 1 <= q
        rank += min(ntj, (q + 1) / 2);
      }
    }
    tval[rank] = (uint64_t)s | ((uint64_t)e << 32);
  }
}

// drop leading positions whose angular key is below ql / trailing ones above qh
__device__ __forceinline__ void trim_lo(const uint64_t* keys, int32_t& s, int32_t e, uint64_t ql) {
  while (s < e && (__ldg(keys + s) & kQMask) < ql) ++s;
}
__device__ __forceinline__ void trim_hi(const uint64_t* keys, int32_t s, int32_t& e, uint64_t qh) {
  while (e > s && (__ldg(keys + e - 1) & kQMask) > qh) --e;
}

// ------------------------------------------------------------ window table
//
// For query v (Poincare radius r, circle centre c, radius rad from
// geometry.py:141-157) and a point w at Poincare radius p >= p1 and angle
// offset psi, hrgen's exact test is |P_w - C_v|^2 - rad^2 < 0 with
// |P_w - C_v|^2 = p^2 + c^2 - 2pc cos psi.  With F = 2|P_v-P_w|^2 - a b_v b_w
// (b = (1-r)(1+r), D = a b + 2) one has |P_w - C_v|^2 - rad_v^2 = F / D_v, and
// the fp64 evaluation of either orientation of the predicate errs by at most
// e = 2^-45 in its own frame (all operands <= 1 in magnitude), so a pair that
// either orientation accepts has F < e * max(D_v, D_w), i.e. in v's frame
//   cos psi > (p^2 + c^2 - rad^2 - e * max(1, D_w / D_v)) / (2 p c).
// The right side increases with p (c^2 - rad^2 < 0: every query circle holds
// the origin), so p = p1, the band's innermost point, bounds the window; D_w
// is largest there and D_v smallest at the row's outer edge.  The pad is a
// fixed fraction of the window's size in cos-space across bands (both scale
// like e^(r_v - r_w)), so windows stay tight at every disk radius.
__device__ __forceinline__ double poincare_halfwidth(double a, double e, double r_native,
                                                     double p1) {
  const double pi = 3.141592653589793;
  const double rh = tanh(0.5 * r_native);
  const double b = (1.0 - rh) * (1.0 + rh);
  const double denom = a * b + 2.0;
  const double c = 2.0 * rh / denom;
  const double diff = (2.0 * rh * rh - a * b) / denom;  // c^2 - rad^2, without cancellation
  if (!(p1 * c > 0.0)) return diff - e < 0.0 ? 4.0 : -1.0;
  const double cl = (p1 * p1 + diff - e) / (2.0 * p1 * c);
  if (cl <= -1.0) return 4.0;
  if (cl >= 1.0) return -1.0;
  const double d = acos(cl) * (1.0 + 1e-9) + 1e-15;
  return d >= pi ? 4.0 : d;
}

// The same half-width in units of 2^-32 of a turn, rounded up, for the
// per-query windows' integer arithmetic on the top 32 bits q32 of the 53-bit
// angular keys.  qkey floors a rounded product, so a point within dlt of the
// query's angle -- and every key in [qkey(phi - dlt), qkey(phi + dlt)], the
// fp64 window of the union / heavy path -- lies within dlt * C + 5 of the
// query's key; q32 * 2^21 is up to 2^21 - 1 below that key, and
// dq = floor(dlt * 2^32 / 2 pi) + 3 covers both: dq * 2^21 >= dlt * C + 2^22.
constexpr uint32_t kWinWhole = 0xffffffffu, kWinEmpty = 0xfffffffeu;
__device__ __forceinline__ uint32_t window_units(float dlt) {
  if (dlt < 0.0f) return kWinEmpty;
  if (dlt >= 3.14159f) return kWinWhole;
  const double u = floor((double)dlt * (4294967296.0 / kTwoPi)) + 3.0;
  return u >= 2147483648.0 ? kWinWhole : (uint32_t)u;
}

// Row s covers query (hyperbolic) radii [s*kRowStep, (s+1)*kRowStep); entry
// < 0: no vertex of the band can be a neighbour; >= pi: the whole band.
__global__ void k_window_table(const Band* __restrict__ bands, int L, int rows, double a,
                               double E, float* __restrict__ wtab,
                               uint32_t* __restrict__ wtab_q = nullptr) {
  const int s = blockIdx.x, j = threadIdx.x;
  if (s >= rows || j >= L) return;
  const Band B = bands[j];
  float out = -1.0f;
  if (B.end > B.start) {
    const double r_lo = s * (double)kRowStep;
    const double r_hi = (s + 1) * (double)kRowStep + 1e-5;  // + fp32 slack of the row index
    const double ch = cosh(0.5 * r_hi);
    const double Dv = a * (0.99 / (ch * ch)) + 2.0;       // smallest D of the row's queries
    const double bw = (1.0 - B.pmin) * (1.0 + B.pmin);
    const double Dw = a * bw + 2.0;                       // largest D of the band's points
    const double e = E * fmax(1.0, Dw / Dv) * 1.01;
    // the window shrinks across the row; take both ends plus slack
    const double d = fmax(poincare_halfwidth(a, e, r_lo, B.pmin),
                          poincare_halfwidth(a, e, r_hi, B.pmin));
    out = d < 0.0 ? -1.0f : (d >= 3.14159 ? 4.0f : __double2float_ru(d * 1.01));
  }
  wtab[s * L + j] = out;
  if (wtab_q) wtab_q[s * L + j] = window_units(out);
}

// Sharded runs: the angular range of each band that any query of this
// rank's sector can reach.  wtab was built on bands whose innermost radius is
// the band's threshold (a lower bound, so windows only widen); windows shrink
// with the query radius, so rows from the smallest query radius on bound
// every query.  Output per band, in 27-bit sort-key units: [lo, hi) of
// needed keys (circular; lo > hi wraps), or whole = 1, or none = -1.
__global__ void k_shard_ranges(const float* __restrict__ wtab, int L, int rows,
                               const unsigned long long* __restrict__ pmin_bits,
                               int64_t sec_lo, int64_t sec_hi, int64_t* __restrict__ lo,
                               int64_t* __restrict__ hi, int* __restrict__ mode,
                               float* __restrict__ cover) {
  // row of the smallest query radius present (rounded down); the widest
  // window of each band over rows s0.. (blockDim = 32 x groups of rows)
  __shared__ float part[32][33];
  const int j = threadIdx.x & 31, g = threadIdx.x >> 5, ng = blockDim.x >> 5;
  const double pmin = __longlong_as_double((long long)*pmin_bits);
  const double rmin = fmax(0.0, 2.0 * atanh(pmin) * (1.0 - 1e-12) - 1e-9);
  const int s0 = (int)floor(rmin / (double)kRowStep);
  float dm = -1.0f;
  if (j < L)
    for (int s = max(s0, 0) + g; s < rows; s += ng) dm = fmaxf(dm, wtab[s * L + j]);
  part[g][j] = dm;
  __syncthreads();
  if (g != 0 || j >= L) return;
  float d = -1.0f;
  for (int k = 0; k < ng; ++k) d = fmaxf(d, part[k][j]);
  const int64_t span = (int64_t)1 << 27;
  cover[j] = 1.0f;
  if (d < 0.0f) { mode[j] = -1; return; }
  const double w = (double)d * (double)span / kTwoPi;
  const int64_t dk = (int64_t)ceil(w * (1.0 + 1e-9)) + 2;
  if (d >= 3.14159f || 2 * dk + (sec_hi - sec_lo) >= span) { mode[j] = 1; return; }
  mode[j] = 0;
  lo[j] = ((sec_lo - dk) % span + span) % span;
  hi[j] = (sec_hi + dk) % span;
  cover[j] = (float)((double)(2 * dk + (sec_hi - sec_lo)) / (double)span);
}

// Does band b's reachable range (k_shard_ranges) hold 27-bit angle q?
__device__ __forceinline__ bool shard_keep(int b, int64_t q, const int64_t* lo,
                                           const int64_t* hi, const int* mode) {
  const int md = mode[b];
  bool ok = md > 0;
  if (md == 0) ok = lo[b] <= hi[b] ? (q >= lo[b] && q < hi[b]) : (q >= lo[b] || q < hi[b]);
  return ok;
}

__global__ void k_shard_flags(int64_t n, const uint32_t* __restrict__ k32,
                              const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                              const int* __restrict__ mode, uint8_t* __restrict__ keep) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t k = k32[i];
  keep[i] = shard_keep((int)(k >> 27), (int64_t)(k & ((1u << 27) - 1)), lo, hi, mode) ? 1 : 0;
}

// ---- sharded sampling (sample ids).  A rank needs only the points its
// sector's queries can reach, and those are decided by the angle and the
// band alone, so the radius (asinh + tanh, the sampler's FP64 cost) is
// evaluated for the kept points only.  Bands are cut on the radial uniform:
// band(b) = #{ j in [1, L) : b >= ub[j] } on the 53-bit integer b behind u2,
// any increasing ub works; k_shard_prep bounds each band's innermost radius
// from below by evaluating the sampler at ub[j].
struct ShardSample {
  uint64_t ub[kMaxBands];  // band thresholds on the 53-bit radial uniform
  int L;
  int64_t sec_lo, sec_hi;  // this rank's sector, 27-bit angle units
};

// Pass 1 over all draws: every vertex's 32-bit sort key (band from the
// radial uniform, binary search over ub[] in shared memory; angle from the
// first uniform) and the smallest radial uniform among the sector's vertices
// (its queries' widest windows come from the smallest radius, which is
// monotone in it).  The keep decision then reads 4 B per draw instead of
// evaluating Philox a second time.
__global__ void __launch_bounds__(256) k_shard_keys(int64_t n, SampleParams P, ShardSample S,
                                                    uint32_t* __restrict__ keys,
                                                    unsigned long long* __restrict__ out) {
  __shared__ uint64_t s_ub[kMaxBands];
  if (threadIdx.x < kMaxBands) s_ub[threadIdx.x] = threadIdx.x < S.L ? S.ub[threadIdx.x] : ~0ull;
  __syncthreads();
  unsigned long long m = ~0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t a, b;
    philox_u53(i, P.seed, a, b);
    const uint64_t q = qkey(angle_from_u53(a), P.C);
    int band = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1)
      if (b >= s_ub[band + st]) band += st;
    keys[i] = sort_key32(band, q);
    const int64_t q27 = (int64_t)(q >> kSortShift);
    if (q27 >= S.sec_lo && q27 < S.sec_hi) m = min(m, (unsigned long long)b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(out, m);
}

// Lower bounds of each band's innermost Poincare radius (the sampler at the
// band's threshold, 16 ulps down: asinh/tanh are monotone to a few ulps) as
// window-table bands, and the smallest query radius of the sector (0 when
// the sector is empty: the widest windows, always safe).
__global__ void k_shard_prep(SampleParams P, ShardSample S,
                             const unsigned long long* __restrict__ umin, Band* __restrict__ tb,
                             unsigned long long* __restrict__ pmin_bits) {
  const int j = threadIdx.x;
  if (j < S.L) {
    double r, p = 0.0;
    if (j > 0) {
      radius_from_u53(S.ub[j], P, r, p);
      for (int k = 0; k < 16; ++k) p = nextafter(p, 0.0);
    }
    Band B;
    memset(&B, 0, sizeof(B));
    B.start = 0; B.end = 1; B.pmin = p;
    tb[j] = B;
  }
  if (j == 0) {
    double r, p = 0.0;
    if (*umin != ~0ull) radius_from_u53(*umin, P, r, p);
    *pmin_bits = (unsigned long long)__double_as_longlong(p);
  }
}

// Pass 2: the kept draws' sort keys, compact indices (the sort's values)
// and global ids.  A block takes kShardPer draws per thread and reserves its
// output with one atomic (one per warp serialises on the counter).  The
// order of kept points is arbitrary: ties of the 32-bit sort key may land in
// any order, which changes no row (rows are sorted by id) and no window
// (exact trims hold on any order).
constexpr int kShardPer = 16;
__global__ void __launch_bounds__(256) k_shard_select(int64_t n, int L,
                                                      const uint32_t* __restrict__ keys_all,
                                                      const int64_t* __restrict__ lo,
                                                      const int64_t* __restrict__ hi,
                                                      const int* __restrict__ mode,
                                                      uint32_t* __restrict__ keys,
                                                      int32_t* __restrict__ vals,
                                                      int32_t* __restrict__ gid,
                                                      unsigned* __restrict__ count) {
  __shared__ unsigned wcnt[8], wbase[8], bbase;
  // per band: (lo, hi | (mode + 1) << 28) in 27-bit angle units, one load
  __shared__ uint2 s_rng[kMaxBands];
  if (threadIdx.x < kMaxBands) {
    const int j = threadIdx.x;
    const int md = j < L ? mode[j] : -1;
    s_rng[j] = make_uint2(md == 0 ? (unsigned)lo[j] : 0u,
                          (md == 0 ? (unsigned)hi[j] : 0u) | ((unsigned)(md + 1) << 28));
  }
  __syncthreads();
  auto keep_of = [&](uint32_t k) {
    const uint2 g = s_rng[k >> 27];
    const unsigned q = k & ((1u << 27) - 1), h = g.y & 0x0fffffffu;
    const int md = (int)(g.y >> 28) - 1;
    return md > 0 || (md == 0 && (g.x <= h ? (q >= g.x && q < h) : (q >= g.x || q < h)));
  };
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * (256 * kShardPer) + threadIdx.x;
  uint32_t kk[kShardPer];
  unsigned ballots[kShardPer];
  unsigned warp_tot = 0;
#pragma unroll
  for (int k = 0; k < kShardPer; ++k) {  // all loads in flight first
    const int64_t i = i0 + 256 * k;
    kk[k] = i < n ? __ldg(keys_all + i) : 0u;
  }
#pragma unroll
  for (int k = 0; k < kShardPer; ++k) {
    const bool keep = i0 + 256 * k < n && keep_of(kk[k]);
    ballots[k] = __ballot_sync(0xffffffffu, keep);
    warp_tot += __popc(ballots[k]);
  }
  if (lane == 0) wcnt[w] = warp_tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int k = 0; k < 8; ++k) { wbase[k] = t; t += wcnt[k]; }
    bbase = t ? atomicAdd(count, t) : 0u;
  }
  __syncthreads();
  unsigned pos = bbase + wbase[w];
#pragma unroll
  for (int k = 0; k < kShardPer; ++k) {
    if ((ballots[k] >> lane) & 1u) {
      const unsigned at = pos + __popc(ballots[k] & ((1u << lane) - 1u));
      keys[at] = kk[k];
      vals[at] = (int32_t)at;
      gid[at] = (int32_t)(i0 + 256 * k);
    }
    pos += __popc(ballots[k]);
  }
}

// Pass 3, dense over the kept points: (phi, r_p) from the vertex's own draws
// (Philox again for a quarter of the draws; asinh + tanh only here).
__global__ void __launch_bounds__(256) k_shard_points(SampleParams P,
                                                      const unsigned* __restrict__ count,
                                                      const int32_t* __restrict__ gid,
                                                      double2* __restrict__ pr) {
  const int64_t m = *count;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    double ph, r, p;
    sample_point(__ldg(gid + i), P, ph, r, p);
    pr[i] = make_double2(ph, p);
  }
}

// Window of band B for a query at angle phi with table half-width dlt, as
// <= 2 sorted-position segments [sA, eA) then [sB, eB).
__device__ __forceinline__ void band_segments(const QueryArgs& A, const Band& B, double phi,
                                              float dlt_f, int32_t& sA, int32_t& eA,
                                              int32_t& sB, int32_t& eB) {
  sA = eA = sB = eB = 0;
  if (B.end <= B.start || dlt_f < 0.0f) return;
  if (dlt_f >= 3.14159265f) { sA = B.start; eA = B.end; return; }
  const double dlt = (double)dlt_f;
  const double lo = phi - dlt, hi = phi + dlt;
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

__device__ __forceinline__ const float* wtab_row(const QueryArgs& A, float rv) {
  int row = (int)(rv * (1.0f / kRowStep));
  row = min(max(row, 0), A.wrows - 1);
  return A.wtab + row * A.L;
}

__device__ __forceinline__ double2 load_pt(const Recs& R, int32_t w) { return __ldg(R.pt + w); }

__device__ __forceinline__ Circ load_circ(const Recs& R, int32_t w) {
  const double2* q = reinterpret_cast<const double2*>(R.circ + w);
  const double2 a = __ldg(q), b = __ldg(q + 1);
  Circ c;
  c.cx = a.x; c.cy = a.y; c.rsq = b.x;
  const long long bits = __double_as_longlong(b.y);  // (rf, invd) as two floats
  c.rf = __int_as_float((int)(bits & 0xffffffffll));
  c.invd = __int_as_float((int)(bits >> 32));
  return c;
}

struct QFull {
  double px, py, cx, cy, rsq;
  int32_t pos, idv;
};

template <bool kSampleIds>
__device__ __forceinline__ QFull load_query(const QueryArgs& A, int32_t v) {
  QFull f;
  f.pos = v;
  const double2 p = load_pt(A.rec, v);
  const Circ c = load_circ(A.rec, v);
  f.px = p.x; f.py = p.y; f.cx = c.cx; f.cy = c.cy; f.rsq = c.rsq;
  f.idv = kSampleIds ? __ldg(A.rec.ids + v) : v;  // angular ids are positions
  return f;
}

__device__ __forceinline__ void load_bands(const QueryArgs& A, Band* sb) {
  if (threadIdx.x < A.L) sb[threadIdx.x] = A.bands[threadIdx.x];
  __syncthreads();
}

// Raw (directory-resolved) window of band B: segments [sA,eA) and [sB,eB)
// cover whole buckets; tlA/thA/tlB are the angular keys the exact trim
// enforces (0 / kQMask+1 = no trim on that side).
struct RawWin {
  int32_t sA, eA, sB, eB;
  uint64_t tlA, thA, tlB;
};

__device__ __forceinline__ RawWin raw_window(const QueryArgs& A, const Band& B, double phi,
                                             float dlt_f) {
  RawWin r;
  r.sA = r.eA = r.sB = r.eB = 0;
  r.tlA = 0; r.thA = kQMask + 1; r.tlB = 0;
  if (B.end <= B.start || dlt_f < 0.0f) return r;
  if (dlt_f >= 3.14159265f) { r.sA = B.start; r.eA = B.end; return r; }
  const double dlt = (double)dlt_f;
  const double lo = phi - dlt, hi = phi + dlt;
  const int32_t* d = A.dir + B.dir_base;
  if (lo < 0.0 || hi >= kTwoPi) {
    const uint64_t qh = qkey(lo < 0.0 ? hi : hi - kTwoPi, A.C);
    const uint64_t ql = qkey(lo < 0.0 ? lo + kTwoPi : lo, A.C);
    r.sA = B.start; r.eA = __ldg(d + (qh >> B.shift) + 1); r.thA = qh;
    r.sB = __ldg(d + (ql >> B.shift)); r.eB = B.end; r.tlB = ql;
  } else {
    const uint64_t ql = qkey(lo, A.C), qh = qkey(hi, A.C);
    r.sA = __ldg(d + (ql >> B.shift)); r.eA = __ldg(d + (qh >> B.shift) + 1);
    r.tlA = ql; r.thA = qh;
  }
  return r;
}

// One trim step with the boundary keys already loaded, then finish (rare:
// two or more out-of-window points in one boundary bucket) with a loop.
__device__ __forceinline__ void finish_trim(const uint64_t* keys, RawWin& r, uint64_t kA0,
                                            uint64_t kA1, uint64_t kB0) {
  if (r.sA < r.eA && (kA0 & kQMask) < r.tlA) { ++r.sA; trim_lo(keys, r.sA, r.eA, r.tlA); }
  if (r.sA < r.eA && (kA1 & kQMask) > r.thA) { --r.eA; trim_hi(keys, r.sA, r.eA, r.thA); }
  if (r.sB < r.eB && (kB0 & kQMask) < r.tlB) { ++r.sB; trim_lo(keys, r.sB, r.eB, r.tlB); }
}

// Band B's part of a union window centred at `mid` with half-width dlt_f
// (the window table's value, widened by the sub-tile's half span): <= 2
// sorted-position segments [sA, eA), [sB, eB) with sB >= eA, trimmed to
// exact angular keys.  Also the heavy pass's per-query window (span 0), so
// both paths see the same candidates for a deferred query.
__device__ __forceinline__ void union_window(const QueryArgs& A, const Band& B, double mid,
                                             float dlt_f, int32_t& sA, int32_t& eA,
                                             int32_t& sB, int32_t& eB) {
  RawWin r = raw_window(A, B, mid, dlt_f);
  if (HRG_TRIM_UNION) {
    const uint64_t kA0 = (r.sA < r.eA && r.tlA) ? __ldg(A.keys + r.sA) : 0;
    const uint64_t kA1 = (r.sA < r.eA && r.thA <= kQMask) ? __ldg(A.keys + r.eA - 1) : 0;
    const uint64_t kB0 = (r.sB < r.eB && r.tlB) ? __ldg(A.keys + r.sB) : 0;
    finish_trim(A.keys, r, kA0, kA1, kB0);
  }
  if (r.sB < r.eB && r.sB < r.eA) {  // the window wraps onto itself: whole band
    r.sA = B.start; r.eA = B.end; r.sB = r.eB = 0;
  }
  if (r.eA < r.sA) r.eA = r.sA;
  if (r.eB < r.sB) r.eB = r.sB;
  sA = r.sA; eA = r.eA; sB = r.sB; eB = r.eB;
}

constexpr int kBandGroup = HRG_BAND_GROUP;    // bands resolved together (loads in flight)
constexpr bool kTrimUnion = HRG_TRIM_UNION;   // ... and of the tile's union windows
constexpr int kUnionSmall = HRG_UNION_SMALL;  // union windows this small are shared by the tile
constexpr int kDenseMax = HRG_DENSE_MAX;      // ... and up to this size tested as a dense block
constexpr int kDenseBig = HRG_DENSE_BIG;      // ... or up to this size if the windows cover
constexpr float kDenseRatio = HRG_DENSE_RATIO;  //     this fraction of the union
constexpr int kDenseCap = 64;                 // dense candidates per tile (one bit each)

constexpr int kWalkUnroll = HRG_WALK_UNROLL;  // walk steps whose loads are in flight together
// flat entry, second word: flat index of the segment's first candidate
// (16 bits) | query lane << 16 | band << 21 | the query's first segment << 31
constexpr int kFirstSeg = INT32_MIN;
constexpr int kFlatMask = 0xffff;
constexpr int kFlatLaneShift = 16;
static_assert(kLightMax * 32 <= (1 << 16), "a tile's flat candidate index must fit 16 bits");

// The walk's pair test with a fixed orientation.  hrgen decides {v, w} with the
// circle of the smaller id (generator.py:182-187).  The walk always evaluates
// pred(v -> w): S = |P_w - C_v|^2 in ref_pred's own operation order against
// rad_v^2, so a candidate costs one 16 B point (+ its id) instead of the 48 B
// record.  For id_v < id_w that is hrgen's decision itself.  For id_w < id_v
// hrgen evaluates pred(w -> v); with g_x = F / D_x the exact value of
// orientation x (see "window table" above) and every fp64 evaluation within
// e = 2^-45 of it, |S - rad_v^2| > e (1 + D_w / D_v) implies both evaluations
// have the sign of F; only inside that margin (D_w bounded by the band's
// innermost point) is the other orientation evaluated from w's full record.
struct __align__(16) QHot {   // per query, shared memory: the walk's operands
  double cx, cy, rsq;
  float invd;                 // >= 1 / D_v
  int32_t idv;                // vertex id (sample order) or position (angular)
};
struct __align__(16) QCold {  // per query: its point, for the other orientation
  double px, py;
};
constexpr float kPredErrF = 0x1.000008p-45f;  // e, rounded up

// Per-lane segment slots (kCap + 1 stride, padded against bank conflicts).
// Two variants: kSegCap slots at 5 blocks/SM, and kSegCapWide slots at 4
// blocks/SM for models whose queries reach most of the 32 bands (small
// alpha: every band populated, so a light query holds up to 32 segments plus
// wrap-around splits; with the narrow variant nearly all of them would be
// deferred to the per-query heavy path).
#ifndef HRG_WIDE_CAP
#define HRG_WIDE_CAP 36
#endif
#ifndef HRG_WIDE_MINB
#define HRG_WIDE_MINB 4
#endif
constexpr int kSegCapWide = HRG_WIDE_CAP;   // static shared memory stays under 48 KB
constexpr int kWideMinBlocks = HRG_WIDE_MINB;
constexpr int kWideBands = 26;   // populated bands from which the wide variant is used
template <int kCap>
struct LightSmem {
  static constexpr int kStride = kCap + 1;
  int2 flat[kLightThreads / 32][32 * kStride];  // per warp: the tile's band segments
  QHot qh[kLightThreads];
  QCold qc[kLightThreads];
  int32_t hits[kLightThreads];
  int32_t dsh[kLightThreads];                    // dense hits of the warp's queries up to this one
  int32_t dids[kLightThreads / 32][kDenseCap];   // per warp: ids of the tile's dense candidates
  float dband[kMaxBands];  // e * D of each band's innermost point, rounded up
};

// w's circle (c_x, c_y, rad^2), for pred(w -> v): the walk's margin case
template <bool kSampleIds>
__device__ __forceinline__ void load_other(const Recs& R, int32_t w, double2& cxy, double& rsq) {
  const Circ* c = R.circ + w;
  cxy = __ldg(reinterpret_cast<const double2*>(&c->cx));
  rsq = __ldg(&c->rsq);
}

template <int kCap>
constexpr size_t light_smem() { return sizeof(LightSmem<kCap>); }

// Queries with more than kLightMax candidates or kCap segments are deferred
// to k_heavy.
template <bool kSampleIds, int kCap, int kMinBlocks>
__global__ void __launch_bounds__(kLightThreads, kMinBlocks) k_light(QueryArgs A) {
  constexpr int kSegCap = kCap;
  constexpr int kSegStride = LightSmem<kCap>::kStride;
  __shared__ Band sb[kMaxBands];
  __shared__ LightSmem<kCap> sm;  // static: compile-time shared addresses
  load_bands(A, sb);
  if (threadIdx.x < kMaxBands) {
    const Band B = sb[threadIdx.x];
    float d = 0.0f;
    if (threadIdx.x < A.L && B.end > B.start) {
      const double D = A.a * ((1.0 - B.pmin) * (1.0 + B.pmin)) + 2.0;
      d = __double2float_ru(0x1p-45 * D) * (1.0f + 0x1p-18f);
    }
    sm.dband[threadIdx.x] = d;
  }
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int wb = tid - lane;  // first thread of this warp
  unsigned long long cand_local = 0;
  // tiles handed out dynamically (their cost varies by orders of magnitude
  // between inner and outer bands): first one by warp id, then a counter
  // every tile from the counter, the first one included: a block that only
  // becomes resident late (the grid may exceed what fits beside the shared
  // carve-out) must not hold back a tile from the head of the list
  int64_t tk = __shfl_sync(FULL, lane == 0 ? (int64_t)atomicAdd(A.tile_next, 1ull) : 0, 0);
  for (; tk < A.ntiles;
       tk = __shfl_sync(FULL, lane == 0 ? (int64_t)atomicAdd(A.tile_next, 1ull) : 0, 0)) {
    const uint64_t tv = __ldg(A.tiles + tk);
    if (tv == ~0ull) break;
    const int32_t v0 = (int32_t)(tv & 0xffffffffu) + lane;
    const bool active = v0 < (int32_t)(tv >> 32);
    const int32_t v = active ? v0 : 0;
    int nseg = 0;
    int2* fl_own = sm.flat[tid >> 5] + lane * kSegStride;
    int32_t c = 0;
    bool ovf = false;
    const double phi = active ? A.q.phi[v] : 0.0;
    const float rvq = active ? __ldg(&A.rec.circ[v].rf) : 3.0e38f;
    const uint32_t q32 = (uint32_t)(qkey(phi, A.C) >> (kQBits - 32));
    const uint32_t* wrowq = A.wtab_q + (wtab_row(A, rvq) - A.wtab);
    // ---- tile-level union windows (lane = band): the 32 queries are
    // angular neighbours, so in bands where their windows are wide relative
    // to the tile's angular span the union of the 32 windows is barely larger
    // than one of them.  Bands whose union is empty are skipped; a union of
    // at most kDenseMax candidates is tested against all 32 queries as a
    // dense block (lane = query, the candidates broadcast: no per-query
    // window, no segment, ~20 instructions per candidate for 32 tests);
    // the other bands are resolved per query and walked.
    unsigned cheap = 0, dense = 0, skip = 0;
    int32_t uA = 0, uAe = 0, uB = 0, uBe = 0;
    int32_t dex = 0, Dn = 0;  // lane = band: first dense-list index of its candidates; their total
    bool dense_big = false;  // a larger union of which every query needs a good part
    {
      double pmin = active ? phi : 1e300, pmax = active ? phi : -1e300;
      float rmin = rvq, rmax = active ? rvq : 0.0f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        pmin = fmin(pmin, __shfl_xor_sync(FULL, pmin, o));
        pmax = fmax(pmax, __shfl_xor_sync(FULL, pmax, o));
        rmin = fminf(rmin, __shfl_xor_sync(FULL, rmin, o));
        rmax = fmaxf(rmax, __shfl_xor_sync(FULL, rmax, o));
      }
      int32_t un = -1;  // union size; -1: not resolved (the tile spans a wide arc)
      if (pmax >= pmin && pmax - pmin < 0.5 && lane < A.L) {
        const float dlt = __ldg(wtab_row(A, rmin) + lane);
        const double half = 0.5 * (pmax - pmin);
        RawWin r = raw_window(A, sb[lane], 0.5 * (pmin + pmax),
                              (dlt < 0.0f || dlt >= 3.14159265f)
                                  ? dlt : __double2float_ru((double)dlt + half));
        if (kTrimUnion) {
          const uint64_t kA0 = (r.sA < r.eA && r.tlA) ? __ldg(A.keys + r.sA) : 0;
          const uint64_t kA1 = (r.sA < r.eA && r.thA <= kQMask) ? __ldg(A.keys + r.eA - 1) : 0;
          const uint64_t kB0 = (r.sB < r.eB && r.tlB) ? __ldg(A.keys + r.sB) : 0;
          finish_trim(A.keys, r, kA0, kA1, kB0);
        }
        if (r.sB < r.eB && r.sB < r.eA) { r.sA = sb[lane].start; r.eA = sb[lane].end; r.sB = r.eB = 0; }
        if (r.eA < r.sA) r.eA = r.sA;
        if (r.eB < r.sB) r.eB = r.sB;
        uA = r.sA; uAe = r.eA; uB = r.sB; uBe = r.eB;
        un = (uAe - uA) + (uBe - uB);
        // the narrowest window of the tile (its outermost query), in points
        const float dn = __ldg(wtab_row(A, rmax) + lane);
        const float nb = (float)(sb[lane].end - sb[lane].start);
        const float w_est = dn < 0.0f ? 0.0f : (dn >= 3.14159265f ? nb : dn * nb * 0.31830988f);
        if (un <= kUnionSmall) cheap = 1;
        // a dense test costs ~0.65 instructions per pair against ~3 in the
        // walk (plus the window and flatten work of a segment), so a union of
        // up to kDenseBig candidates is also tested densely when the tile's
        // narrowest window covers at least kDenseRatio of it
        dense_big = kDenseBig > 0 && un <= kDenseBig && w_est >= kDenseRatio * (float)un;
      }
      cheap = __ballot_sync(FULL, cheap != 0);
      skip = __ballot_sync(FULL, un == 0 || lane >= A.L);
      bool dn_ok = kDenseMax > 0 && un > 0 && (un <= kDenseMax || dense_big);
      if (!kSampleIds) {
        // positions are ids and rows leave sorted: dense hits are written
        // ahead of a row's walked hits, so dense bands must lie inside every
        // band that is walked
        const unsigned walked = __ballot_sync(FULL, lane < A.L && un != 0 && !dn_ok);
        dn_ok = dn_ok && (walked == 0 || lane < __ffs(walked) - 1);
      }
      int32_t dincl = dn_ok ? un : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, dincl, o);
        if (lane >= o) dincl += y;
      }
      // the cap keeps a prefix of the dense bands (indices stay contiguous;
      // with positions as ids the dropped bands lie outside the kept ones)
      dn_ok = dn_ok && dincl <= kDenseCap;
      dense = __ballot_sync(FULL, dn_ok);
      // non-decreasing over the lanes, for the search below; a band that is
      // not dense owns no index (it ties with the next dense band, which the
      // search prefers, or lies past Dn)
      dex = dincl - (dn_ok ? un : 0);
      Dn = dense ? __shfl_sync(FULL, dincl, 31 - __clz(dense)) : 0;
    }
    // bands still to resolve per query (or shared as a small union)
    for (unsigned todo = ~(skip | dense); todo;) {
      int jj[kBandGroup];
#pragma unroll
      for (int u = 0; u < kBandGroup; ++u) {
        jj[u] = todo ? __ffs(todo) - 1 : -1;
        todo &= todo - 1;
      }
      // union segments of the group's bands, from their lanes
      int32_t gA[kBandGroup], gAe[kBandGroup], gB[kBandGroup], gBe[kBandGroup];
#pragma unroll
      for (int u = 0; u < kBandGroup; ++u) {
        const int j = max(jj[u], 0);
        gA[u] = __shfl_sync(FULL, uA, j); gAe[u] = __shfl_sync(FULL, uAe, j);
        gB[u] = __shfl_sync(FULL, uB, j); gBe[u] = __shfl_sync(FULL, uBe, j);
      }
      if (!active) continue;
      {
        // per-query windows at directory granularity, in integer arithmetic
        // on the top 32 bits of the query's angular key: [q - dq, q + dq]
        // wraps mod 2^32 like the angle; two directory reads per band
        RawWin w[kBandGroup];
#pragma unroll
        for (int u = 0; u < kBandGroup; ++u) {
          const int j = jj[u];
          w[u] = RawWin{0, 0, 0, 0, 0, kQMask + 1, 0};
          if (j < 0 || ((cheap >> j) & 1u)) continue;
          const uint32_t dq = __ldg(wrowq + j);
          const int32_t bs = sb[j].start, be = sb[j].end;
          if (dq == kWinEmpty || be <= bs) continue;
          if (dq == kWinWhole) { w[u].sA = bs; w[u].eA = be; continue; }
          const uint32_t ql = q32 - dq, qh = q32 + dq;
          const int sh = sb[j].shift - (kQBits - 32);
          const int32_t* d = A.dir + sb[j].dir_base;
          const int32_t lo = __ldg(d + (sh < 32 ? ql >> sh : 0u));
          const int32_t hi = __ldg(d + (sh < 32 ? qh >> sh : 0u) + 1);
          if (q32 < dq || qh < q32) { w[u].sA = bs; w[u].eA = hi; w[u].sB = lo; w[u].eB = be; }
          else { w[u].sA = lo; w[u].eA = hi; }
        }
#pragma unroll
        for (int u = 0; u < kBandGroup; ++u) {
          const int j = jj[u];
          if (j < 0) continue;
          RawWin& r = w[u];
          if ((cheap >> j) & 1u) {
            r.sA = gA[u]; r.eA = gAe[u]; r.sB = gB[u]; r.eB = gBe[u];
          } else {
            if (r.sB < r.eB && r.sB < r.eA) {  // window wraps onto itself: whole band
              r.sA = sb[j].start; r.eA = sb[j].end; r.sB = r.eB = 0;
            }
          }
          if (r.eA > r.sA) {
            if (nseg < kSegCap) fl_own[nseg++] = make_int2(r.sA, (c & 0xffff) | (j << 16));
            else ovf = true;
            c += r.eA - r.sA;
          }
          if (r.eB > r.sB) {
            if (nseg < kSegCap) fl_own[nseg++] = make_int2(r.sB, (c & 0xffff) | (j << 16));
            else ovf = true;
            c += r.eB - r.sB;
          }
        }
      }
    }
    // every query of the tile also tests the Dn dense candidates
    cand_local += active ? (unsigned long long)(c + Dn) : 0ull;
    const bool heavy = active && (c + Dn > A.light_max || ovf);
    const bool light = active && !heavy;
    const int32_t want = light ? c : 0, nsl = light ? nseg : 0;
    int32_t incl = want, sincl = nsl;  // inclusive scans: candidates, segments
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, incl, o), z = __shfl_up_sync(FULL, sincl, o);
      if (lane >= o) { incl += y; sincl += z; }
    }
    const int32_t T = __shfl_sync(FULL, incl, 31), S = __shfl_sync(FULL, sincl, 31);
    const int32_t excl = incl - want;
    int2* fl = sm.flat[tid >> 5];
    QFull f;
    float invd = 0.0f;
    if (light) {
      f = load_query<kSampleIds>(A, v);
      invd = __ldg(&A.rec.circ[v].invd);
      QHot h;
      h.cx = f.cx; h.cy = f.cy; h.rsq = f.rsq; h.invd = invd; h.idv = f.idv;
      sm.qh[tid] = h;
      QCold k;
      k.px = f.px; k.py = f.py;
      sm.qc[tid] = k;
    }
    // ---- dense block: lane k of each half holds dense candidate k (its band
    // from a search over the bands' first indices), every candidate is
    // broadcast and tested by all lanes against their own query.  Bit k of
    // dm: candidate k is a neighbour of this lane's query.
    unsigned long long dm = 0;
    for (int h0 = 0; h0 < Dn; h0 += 32) {
      const int k = h0 + lane;
      int l = 0;  // owner band: the last lane with dex <= k
#pragma unroll
      for (int st = 16; st > 0; st >>= 1)
        if (__shfl_sync(FULL, dex, l + st) <= k) l += st;
      const int32_t t = k - __shfl_sync(FULL, dex, l);
      const int32_t la = __shfl_sync(FULL, uAe - uA, l);
      const int32_t pa = __shfl_sync(FULL, uA, l), pb = __shfl_sync(FULL, uB, l);
      const int32_t pos = k < Dn ? (t < la ? pa + t : pb + (t - la)) : 0;
      const double2 cp = __ldg(A.rec.pt + pos);
      const int32_t cid = kSampleIds ? __ldg(A.rec.ids + pos) : pos;
      const float ced = sm.dband[l];
      if (k < Dn) sm.dids[tid >> 5][k] = cid;
      const int nk = min(32, Dn - h0);
      for (int kk = 0; kk < nk; ++kk) {
        const double px = __shfl_sync(FULL, cp.x, kk), py = __shfl_sync(FULL, cp.y, kk);
        const int32_t idw = __shfl_sync(FULL, cid, kk);
        const float ed = __shfl_sync(FULL, ced, kk);
        const int32_t pw = __shfl_sync(FULL, pos, kk);
        if (light) {
          const double dx = __dsub_rn(px, f.cx), dy = __dsub_rn(py, f.cy);
          const double s2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
          bool hit = s2 < f.rsq;  // quadtree.py:611-613 with v's circle
          if (idw < f.idv &&
              fabsf(__double2float_rn(__dsub_rn(s2, f.rsq))) <= fmaf(ed, invd, kPredErrF)) {
            double2 oc;
            double orsq;
            load_other<kSampleIds>(A.rec, pw, oc, orsq);
            hit = ref_pred(f.px, f.py, oc.x, oc.y, orsq);  // w's circle decides
          }
          if (hit && idw != f.idv) dm |= 1ull << (h0 + kk);
        }
      }
    }
    const int32_t dh = __popcll(dm);
    int32_t dhi = dh;  // inclusive scan of the dense hits over the tile's queries
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, dhi, o);
      if (lane >= o) dhi += y;
    }
    sm.dsh[tid] = dhi;
    // staging for the tile's light rows: walked candidates + dense hits
    const int32_t Talloc = T + __shfl_sync(FULL, dhi, 31);
    unsigned long long base = 0;
    if (lane == 31 && Talloc > 0) base = atomicAdd(A.bump, (unsigned long long)Talloc);
    base = __shfl_sync(FULL, base, 31);
    sm.hits[tid] = 0;
    if (heavy) {
      unsigned long long hoff = atomicAdd(A.bump, (unsigned long long)(c + Dn));
      unsigned e = atomicAdd(A.heavy_n, 1u);
      A.heavy_v[e] = v;
      A.heavy_c[e] = c + Dn;
      A.heavy_of[v] = (int32_t)e;
      A.stage_off[v] = (int64_t)hoff;
      A.slots[v] = c + Dn;
    } else if (active) {
      A.heavy_of[v] = -1;
    }
    const bool fits = (int64_t)base + Talloc <= A.stage_cap;
    if (!fits && lane == 0) atomicOr(A.overflow, 1);
    // ---- flatten: lane l's segments sit at fl[l * kSegStride + k] as (first
    // record, offset in the query).  Pack them, in query order, to fl[0, S)
    // as (first record, kFirstSeg | flat index of the first candidate << 5 |
    // lane).  Rounds run over destinations; every entry moves down (dest <=
    // source), so a round's writes never hit a source still to be read.
    {
      const int32_t sb = sincl - nsl;
      for (int e0 = 0; e0 < S; e0 += 32) {
        const int e = e0 + lane;
        int l = 0;  // owner: the last lane with sb <= e
#pragma unroll
        for (int st = 16; st > 0; st >>= 1)
          if (__shfl_sync(FULL, sb, l + st) <= e) l += st;
        const int k = e - __shfl_sync(FULL, sb, l);
        const int32_t own_ex = __shfl_sync(FULL, excl, l);
        int2 g = make_int2(0, 0);
        if (e < S) g = fl[l * kSegStride + k];
        __syncwarp();
        if (e < S)
          fl[e] = make_int2(g.x, (k == 0 ? kFirstSeg : 0) | ((g.y >> 16) << (kFlatLaneShift + 5)) |
                                     (l << kFlatLaneShift) | (own_ex + (g.y & 0xffff)));
        __syncwarp();
      }
    }
    __syncwarp();
    // ---- walk: lane l takes flat candidate i0 + l, so a warp reads 32
    // consecutive records of one or a few segments per step.  The segment of
    // each lane comes from a bit mask of the segment starts inside the step.
    // Only hits are written, compacted, so a query's hits are one contiguous
    // run; the running hit prefix at a query's first and past its last
    // candidate bound that run.  A query's dense hits go in front of its
    // walked ones: a walked hit moves up by the dense hits of the queries up
    // to and including its own.
    if (fits) {
      int32_t* out = A.stage + base;
      int s0 = 0;          // segment holding flat index i0
      int32_t pre = 0;     // hits before i0
      // the segment lookup of a group of steps: each lane's candidate (wv),
      // its query lane | band << 5 (qv), first candidate of its query (qs)
      int32_t wv[kWalkUnroll], nwv[kWalkUnroll];
      int qv[kWalkUnroll], nqv[kWalkUnroll];
      bool qs[kWalkUnroll], nqs[kWalkUnroll];
      auto lookup = [&](int32_t i0, int32_t (&w)[kWalkUnroll], int (&q)[kWalkUnroll],
                        bool (&first)[kWalkUnroll]) {
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u) {
          const int32_t ib = i0 + 32 * u;
          const int sl = s0 + 1 + lane;
          const int32_t st = sl < S ? (fl[sl].y & kFlatMask) : INT32_MAX;
          const unsigned rel = (unsigned)(st - ib);
          const unsigned mask = __reduce_or_sync(FULL, rel < 32u ? 1u << rel : 0u);
          const int my = min(s0 + __popc(mask & ((2u << lane) - 1u)), max(S - 1, 0));
          s0 += __popc(mask);
          const int2 e = fl[my];
          const int32_t off = ib + lane - (e.y & kFlatMask);
          q[u] = (e.y >> kFlatLaneShift) & 1023;
          first[u] = off == 0 && e.y < 0;
          w[u] = e.x + off;
        }
      };
      lookup(0, nwv, nqv, nqs);
      for (int32_t i0 = 0; i0 < T; i0 += 32 * kWalkUnroll) {
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u) { wv[u] = nwv[u]; qv[u] = nqv[u]; qs[u] = nqs[u]; }
        double2 pt[kWalkUnroll];
        int32_t idw[kWalkUnroll];
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u)
          if (i0 + 32 * u + lane < T) {
            pt[u] = __ldg(A.rec.pt + wv[u]);
            idw[u] = kSampleIds ? __ldg(A.rec.ids + wv[u]) : wv[u];
          }
        // the next group's lookup (shared memory) runs under these loads
        if (i0 + 32 * kWalkUnroll < T) lookup(i0 + 32 * kWalkUnroll, nwv, nqv, nqs);
        bool hit[kWalkUnroll], unc[kWalkUnroll];
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u) {
          hit[u] = unc[u] = false;
          if (i0 + 32 * u + lane < T) {
            const QHot f = sm.qh[wb + (qv[u] & 31)];
            const double dx = __dsub_rn(pt[u].x, f.cx), dy = __dsub_rn(pt[u].y, f.cy);
            const double s2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
            hit[u] = s2 < f.rsq && idw[u] != f.idv;  // quadtree.py:611-613 with v's circle
            const float g = fabsf(__double2float_rn(__dsub_rn(s2, f.rsq)));
            unc[u] = idw[u] < f.idv && g <= fmaf(sm.dband[qv[u] >> 5], f.invd, kPredErrF);
          }
        }
        // margin cases (rare: one group of steps in ~4 holds any): w's circle
        // decides.  Their loads are issued together and waited for once.
        bool any_unc = false;
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u) any_unc = any_unc || unc[u];
        if (__any_sync(FULL, any_unc)) {
          double2 oc[kWalkUnroll];
          double orsq[kWalkUnroll];
#pragma unroll
          for (int u = 0; u < kWalkUnroll; ++u)
            if (unc[u]) load_other<kSampleIds>(A.rec, wv[u], oc[u], orsq[u]);
#pragma unroll
          for (int u = 0; u < kWalkUnroll; ++u)
            if (unc[u]) {
              const QCold k = sm.qc[wb + (qv[u] & 31)];
              hit[u] = ref_pred(k.px, k.py, oc[u].x, oc[u].y, orsq[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kWalkUnroll; ++u) {
          const int32_t i = i0 + 32 * u + lane;
          // hits only, compacted: the tile's rows end up back to back
          const unsigned hm = __ballot_sync(FULL, hit[u]);
          const int32_t at = pre + __popc(hm & ((1u << lane) - 1u));
          if (hit[u]) out[at + sm.dsh[wb + (qv[u] & 31)]] = idw[u];
          if (qs[u] && i < T) sm.hits[wb + (qv[u] & 31)] = at;
          pre += __popc(hm);
        }
      }
      // walked hits of query q = prefix at the next non-empty query (or the
      // end) minus the prefix at q; the row is its dense hits, then those
      __syncwarp();
      const unsigned ne = __ballot_sync(FULL, want > 0) & ~((2u << lane) - 1u);
      const int32_t end = ne ? sm.hits[wb + __ffs(ne) - 1] : pre;
      const int32_t mine = want > 0 ? sm.hits[tid] : end;
      __syncwarp();
      const int32_t row0 = mine + dhi - dh;  // the row's first slot in the tile's range
      sm.hits[tid] = end - mine + dh;
      {
        // the dense hits, in candidate order (32-bit halves of the mask)
        const int32_t* dids = sm.dids[tid >> 5];
        int32_t at = row0;
        for (unsigned m = (unsigned)dm; m; m &= m - 1) out[at++] = dids[__ffs(m) - 1];
        for (unsigned m = (unsigned)(dm >> 32); m; m &= m - 1) out[at++] = dids[31 + __ffs(m)];
      }
      if (light) {  // the row's hits: stage[stage_off, stage_off + slots)
        A.stage_off[v] = (int64_t)base + row0;
        A.slots[v] = end - mine + dh;
      }
    }
    __syncwarp();
    if (light) A.deg[row_of<kSampleIds>(A, v)] = fits ? sm.hits[tid] : 0;
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cand_local += __shfl_xor_sync(FULL, cand_local, o);
  if (lane == 0 && cand_local) atomicAdd(A.cand_total, cand_local);
}

// Exclusive scan of a device-sized int32 array into int64 out[0, count],
// one block (the counts here are the deferred queries' chunks: small).
__device__ void block_scan_i64(const int32_t* in, int64_t count, int64_t* out) {
  __shared__ int64_t s_w[32];
  __shared__ int64_t s_run;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_run = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < count; b0 += blockDim.x) {
    const int64_t i = b0 + tid;
    const int64_t x = i < count ? (int64_t)in[i] : 0;
    int64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const int64_t w = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
      int64_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < (int)(blockDim.x >> 5)) s_w[lane] = wi - w;
    }
    __syncthreads();
    const int64_t ex = s_run + s_w[warp] + inc - x;
    if (i < count) out[i] = ex;
    __syncthreads();
    if (tid == blockDim.x - 1) s_run = ex + x;
    __syncthreads();
  }
  if (tid == 0) out[count] = s_run;
}

// Deferred (heavy) queries, on the device so no host round trip sits between
// the light pass and the heavy one: chunks per query, their exclusive scan
// (chunk_start, total), and the chunk -> query map.
__global__ void __launch_bounds__(1024) k_heavy_prep(const int32_t* __restrict__ heavy_c,
                                                     const unsigned* __restrict__ heavy_n,
                                                     int32_t* __restrict__ nchunks,
                                                     int64_t* __restrict__ chunk_start,
                                                     int32_t* __restrict__ chunk_entry,
                                                     int64_t* __restrict__ total,
                                                     const int* __restrict__ overflow) {
  // a staging overflow voids the pass (re-run by the host); nothing after
  // the light pass may then touch buffers sized by the staging capacity
  if (*overflow) { if (threadIdx.x == 0) *total = 0; return; }
  const int64_t H = *heavy_n;
  for (int64_t e = threadIdx.x; e < H; e += blockDim.x)
    nchunks[e] = (heavy_c[e] + kChunk - 1) / kChunk;
  __syncthreads();
  block_scan_i64(nchunks, H, chunk_start);
  __syncthreads();
  if (threadIdx.x == 0) *total = chunk_start[H];
  for (int64_t e = threadIdx.x; e < H; e += blockDim.x)
    for (int64_t c = chunk_start[e]; c < chunk_start[e + 1]; ++c) chunk_entry[c] = (int32_t)e;
}

// Exclusive scan of the heavy chunks' hit counts (count on the device).
__global__ void __launch_bounds__(1024) k_scan_chunks(const int32_t* __restrict__ in,
                                                      const int64_t* __restrict__ count,
                                                      int64_t* __restrict__ out,
                                                      const int* __restrict__ overflow) {
  if (*overflow) return;
  block_scan_i64(in, *count, out);
}

// Heavy pass: one warp per chunk of kChunk candidates of one deferred query;
// lanes own bands for the window phase, then stride the chunk 32 candidates
// at a time (4 batches in flight) with ballot-ordered writes into the
// chunk's slot of the query's staging slice.
template <bool kSampleIds>
__global__ void __launch_bounds__(256, HRG_HEAVY_MINB) k_heavy(QueryArgs A, int64_t H) {
  constexpr int HB = HRG_HEAVY_BATCH;  // batches of 32 candidates in flight
  if (*A.overflow) return;  // void pass, re-run by the host
  __shared__ Band sb[kMaxBands];
  if (threadIdx.x < A.L) sb[threadIdx.x] = A.bands[threadIdx.x];
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t total_chunks = *A.total_chunks;
  // chunks from a counter (tile_next[2]): a hub's chunks cost far more than
  // a barely-deferred query's, and a static stride left the pass in its tail
  auto next_chunk = [&]() {
    return __shfl_sync(FULL, lane == 0 ? (int64_t)atomicAdd(A.tile_next + 2, 1ull) : 0, 0);
  };
  for (int64_t c = next_chunk(); c < total_chunks; c = next_chunk()) {
    const int64_t e = __ldg(A.chunk_entry + c);
    const int32_t v = A.heavy_v[e];
    const int64_t local = c - A.chunk_start[e];
    QFull f = load_query<kSampleIds>(A, v);
    const float invd = __ldg(&A.rec.circ[v].invd);
    int32_t sA = 0, eA = 0, sB = 0, eB = 0;
    float ed = 0.0f;  // lane = band: e * D of its innermost point (the walk's margin)
    if (lane < A.L) {
      const float* wrow = wtab_row(A, __ldg(&A.rec.circ[v].rf));
      union_window(A, sb[lane], A.q.phi[v], __ldg(wrow + lane), sA, eA, sB, eB);
      const double D = A.a * ((1.0 - sb[lane].pmin) * (1.0 + sb[lane].pmin)) + 2.0;
      ed = __double2float_ru(0x1p-45 * D) * (1.0f + 0x1p-18f);
    }
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
    for (int32_t base = beg; base < end; base += 32 * HB) {
      int32_t wv[HB];
      bool ok[HB];
      float edw[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u) {
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
        edw[u] = __shfl_sync(FULL, ed, o);
        wv[u] = tt < la ? sa + tt : sbb + (tt - la);
        ok[u] = i < end;
      }
      // the walk's test (see QHot): v's circle against w's point, the other
      // orientation only inside the rounding margin
      double2 pt[HB];
      int32_t idw[HB];
#pragma unroll
      for (int u = 0; u < HB; ++u)
        if (ok[u]) {
          pt[u] = __ldg(A.rec.pt + wv[u]);
          idw[u] = kSampleIds ? __ldg(A.rec.ids + wv[u]) : wv[u];
        }
#pragma unroll
      for (int u = 0; u < HB; ++u) {
        bool hit = false;
        if (ok[u]) {
          const double dx = __dsub_rn(pt[u].x, f.cx), dy = __dsub_rn(pt[u].y, f.cy);
          const double s2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
          hit = s2 < f.rsq;
          if (idw[u] < f.idv &&
              fabsf(__double2float_rn(__dsub_rn(s2, f.rsq))) <= fmaf(edw[u], invd, kPredErrF)) {
            double2 oc;
            double orsq;
            load_other<kSampleIds>(A.rec, wv[u], oc, orsq);
            hit = ref_pred(f.px, f.py, oc.x, oc.y, orsq);
          }
          hit = hit && idw[u] != f.idv;
        }
        unsigned bal = __ballot_sync(FULL, hit);
        if (hit && fits) out[hits + __popc(bal & ((1u << lane) - 1u))] = idw[u];
        hits += __popc(bal);
      }
    }
    if (lane == 0) {
      if (!fits) atomicOr(A.overflow, 1);
      A.chunk_hits[c] = hits;
      atomicAdd(&A.deg[row_of<kSampleIds>(A, v)], hits);
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

// Batcher's odd-even merge sort network over a register array, ascending:
// 63 / 191 / 543 comparators for 16 / 32 / 64 keys against bitonic's 80 /
// 240 / 672.  oe_idx enumerates the comparators at compile time; the fold
// below instantiates each with constant register indices.
template <int N>
__host__ __device__ constexpr int oe_idx(int c, bool hi) {
  int m = 0;
  for (int p = 1; p < N; p <<= 1)
    for (int k = p; k >= 1; k >>= 1)
      for (int j = k % p; j + k < N; j += 2 * k)
        for (int i = 0; i < k && i + j + k < N; ++i)
          if ((i + j) / (2 * p) == (i + j + k) / (2 * p)) {
            if (m == c) return hi ? i + j + k : i + j;
            ++m;
          }
  return m;  // past the last comparator: their count
}

template <int Lo, int Hi, int N>
__device__ __forceinline__ void cmpx(int32_t (&x)[N]) {
  const int32_t a = x[Lo], b = x[Hi];
  x[Lo] = min(a, b);
  x[Hi] = max(a, b);
}

template <int N, int... C>
__device__ __forceinline__ void oe_apply(int32_t (&x)[N], std::integer_sequence<int, C...>) {
  (cmpx<oe_idx<N>(C, false), oe_idx<N>(C, true)>(x), ...);
}

template <int N>
__device__ __forceinline__ void reg_oddeven(int32_t (&x)[N]) {
  oe_apply<N>(x, std::make_integer_sequence<int, oe_idx<N>(1 << 30, false)>{});
}

// Bitonic network over a register array (compile-time indices throughout).
template <int N>
__device__ __forceinline__ void reg_bitonic(int32_t (&x)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const int32_t a = x[i], b = x[l];
          if ((i & k) == 0) { x[i] = min(a, b); x[l] = max(a, b); }
          else { x[i] = max(a, b); x[l] = min(a, b); }
        }
      }
    }
  }
}

// Misses (-1) sort to the end; hits are non-negative ids.
__device__ __forceinline__ int32_t miss_last(int32_t x) { return x < 0 ? INT32_MAX : x; }

// Register network over one row's slots held in shared memory: ids
// ascending, misses (-1) last; the first `len` values are the row, written
// back in place.  In angular order ids are the candidates' positions, already
// ascending, so this is an order-preserving compaction; in sample order it is
// hrgen's sorted row (graph.py:69-71).
template <int N>
__device__ __forceinline__ void thread_sort_smem(int32_t* sm, int32_t ns, int32_t len) {
  int32_t x[N];
#pragma unroll
  for (int t = 0; t < N; ++t) x[t] = t < ns ? miss_last(sm[t]) : INT32_MAX;
  reg_oddeven<N>(x);
#pragma unroll
  for (int t = 0; t < N; ++t)
    if (t < len) sm[t] = x[t];
}

template <int E>
__device__ __forceinline__ void warp_sort_slots(const int32_t* src, int32_t ns, int32_t* dst,
                                                int32_t len, int lane) {
  int32_t x[E];
#pragma unroll
  for (int t = 0; t < E; ++t) {
    const int e = lane * E + t;
    x[t] = e < ns ? miss_last(src[e]) : INT32_MAX;
  }
  warp_bitonic<E>(x, lane);
  __syncwarp();  // in-place jobs: every lane has read before anyone writes
#pragma unroll
  for (int t = 0; t < E; ++t) {
    const int e = lane * E + t;
    if (e < len) dst[e] = x[t];
  }
}

// A list of rows to sort: [off, off + len) of a source array, sorted into
// the same range of a destination array (the same array when in place).
struct RowList {
  int64_t* off;
  int32_t* len;
  unsigned* n;
};

__device__ __forceinline__ void push_row(const RowList& R, int64_t off, int32_t len) {
  const unsigned k = atomicAdd(R.n, 1u);
  R.off[k] = off;
  R.len[k] = len;
}

// Rows queued for an in-place sort of idx[dst, dst + len): every row is
// contiguous by then (k_light compacts light rows, heavy rows are compacted
// chunk by chunk), so a job is just its range.
constexpr int kWarpBucketMax = HRG_WARP_BUCKET_MAX;   // rows a warp sorts in shared memory
constexpr int kBucketMax = 4096;       // rows a 256-thread block sorts
constexpr int kLargeMax = 24576;       // rows a 1024-thread block sorts (in + out: 221 KB)

// Rows are queued by length straight into the list of the kernel that sorts
// them, so the sort kernels are independent (they run on separate streams).
struct SortJobs {
  RowList rows;    // queued rows, for k_sort_warp
  RowList mid;     // rows above kWarpBucketMax: k_sort_rows<256, kBucketMax>
  RowList large;   // rows above kBucketMax: k_sort_rows<1024, kLargeMax>
  RowList giant;   // rows above kLargeMax: split by value first (k_giant_*)
};

// Queue a row; called by every lane of a warp (want = this lane has a row),
// one atomic per warp.
__device__ __forceinline__ void push_job_warp(const SortJobs& J, bool want, int64_t dst,
                                              int32_t len) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const bool big = want && len > kWarpBucketMax;  // rare: one atomic each
  if (big) push_row(len <= kBucketMax ? J.mid : (len <= kLargeMax ? J.large : J.giant), dst, len);
  want = want && !big;
  const unsigned bal = __ballot_sync(FULL, want);
  if (!bal) return;
  unsigned base = 0;
  if (lane == __ffs(bal) - 1) base = atomicAdd(J.rows.n, (unsigned)__popc(bal));
  base = __shfl_sync(FULL, base, __ffs(bal) - 1);
  if (want) {
    const unsigned k = base + __popc(bal & ((1u << lane) - 1u));
    J.rows.off[k] = dst;
    J.rows.len[k] = len;
  }
}

constexpr int kCompactThreads = 128;
constexpr bool kElemWrite = HRG_ELEM_WRITE;  // compaction writes rows element-parallel
constexpr int kSmallSlots = HRG_SMALL_SLOTS;    // rows sorted by one thread (32 or 64)
constexpr int kTileHits = HRG_TILE_HITS;                 // smem hits per warp
constexpr int kCopyUnroll = 8;                  // loads in flight per lane

// 4-byte global -> shared copy that bypasses registers (LDGSTS).
__device__ __forceinline__ void cp_async4(int32_t* smem, const int32_t* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP) signalled on an mbarrier.
// HRG_COMPACT_TMA=1 stages each compaction group with one bulk copy instead
// of per-lane cp.async: correct (parity suite) but measured 1.7% slower
// (k_compact_light 1.492 -> 1.518 ms at config 2: one serialised bulk copy
// per group against 32 lanes' copies in flight), so off by default.
#ifndef HRG_COMPACT_TMA
#define HRG_COMPACT_TMA 0
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// generic-proxy accesses of this thread's shared memory before async-proxy
// (TMA) writes into it
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Compaction of light rows.  A warp owns the same 32 consecutive queries as
// in k_light, whose hits k_light left back to back in the staging buffer,
// row after row in candidate order.  With angular ids and no deferred query
// in the tile the rows are also consecutive in the CSR: one straight copy.
// Otherwise the warp stages groups of rows in shared memory; with
// sample-order ids each lane then sorts its row (<= kSmallSlots hits) with a
// register network -- hrgen's Graph keeps rows sorted by id
// (graph.py:69-71); longer rows are queued for an in-place sort.  With
// angular ids candidate order is id order and nothing is sorted.
template <bool kSampleIds>
__global__ void __launch_bounds__(kCompactThreads, HRG_COMPACT_MINB) k_compact_light(
    QueryArgs A, const int64_t* __restrict__ rowptr, int32_t* __restrict__ idx, SortJobs J) {
  if (*A.overflow) return;  // void pass, re-run by the host
  __shared__ Band sb[kMaxBands];
  // per warp: the group buffer (+ 8 ids: a TMA copy starts at the 16-byte
  // boundary below the group's first hit) and its mbarrier
  __shared__ __align__(16) int32_t buf[kCompactThreads / 32][kTileHits + 8];
  __shared__ __align__(8) uint64_t s_bar[kCompactThreads / 32];
  load_bands(A, sb);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int32_t* const smraw = buf[threadIdx.x >> 5];
  uint64_t* const bar = s_bar + (threadIdx.x >> 5);
  unsigned bar_phase = 0;
  if (HRG_COMPACT_TMA && lane == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncwarp();
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // The per-row loads of a tile (its entry in the tile table, then heavy
  // flag, row, hit count, staging offset, then the row's CSR offset) are
  // dependent DRAM round trips; the next tile's are issued while this one is
  // copied and sorted (software pipelining across the dynamic tile loop).
  struct Pro { uint64_t tv; int32_t hv, idv, sl; int64_t so; };
  auto fetch = [&](int64_t t) {
    Pro P;
    P.tv = t < A.ntiles ? __ldg(A.tiles + t) : ~0ull;
    const int32_t v0 = (int32_t)(P.tv & 0xffffffffu) + lane;
    const bool act = P.tv != ~0ull && v0 < (int32_t)(P.tv >> 32);
    const int32_t vv = act ? v0 : 0;
    P.hv = act ? A.heavy_of[vv] : 0;
    P.idv = act ? row_of<kSampleIds>(A, vv) : 0;
    P.sl = act ? A.slots[vv] : 0;
    P.so = act ? A.stage_off[vv] : INT64_MAX;
    return P;
  };
  int64_t tk = wid;
  Pro cur = fetch(tk);
  while (tk < A.ntiles && cur.tv != ~0ull) {
    const int64_t tn =
        __shfl_sync(FULL, lane == 0 ? (int64_t)(nw + atomicAdd(A.tile_next + 1, 1ull)) : 0, 0);
    const uint64_t tv = cur.tv;
    const int32_t v0 = (int32_t)(tv & 0xffffffffu) + lane;
    const bool active = v0 < (int32_t)(tv >> 32);
    // a light row's length is its hit count k_light left in slots[]
    const bool light = active && cur.hv < 0;
    const int32_t ns = light ? cur.sl : 0, len = ns;
    const int64_t dst = light ? rowptr[cur.idv] : 0, src = light ? cur.so : INT64_MAX;
    const Pro nxt = fetch(tn);
    int64_t base = src;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) base = min(base, (int64_t)__shfl_xor_sync(FULL, base, o));
    int32_t hi = len, si = ns;  // inclusive scans of hits and slots
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, hi, o), z = __shfl_up_sync(FULL, si, o);
      if (lane >= o) { hi += y; si += z; }
    }
    const int32_t Htot = __shfl_sync(FULL, hi, 31), T = __shfl_sync(FULL, si, 31);
    const int32_t hexcl = hi - len;
    if (!kSampleIds && __all_sync(FULL, !active || light)) {
      // angular ids, every query light: staging range == CSR range
      const int64_t d0 = __shfl_sync(FULL, dst, 0);
      constexpr int U = 2 * kCopyUnroll;
      for (int32_t i0 = 0; i0 < T; i0 += 32 * U) {
        int32_t x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t i = i0 + 32 * u + lane;
          x[u] = i < T ? __ldg(A.stage + base + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int32_t i = i0 + 32 * u + lane;
          if (i < T) idx[d0 + i] = x[u];
        }
      }
    } else {
      // Rows in groups of consecutive lanes whose hits fit in shared memory
      // (one group for all but hub-heavy tiles): one coalesced copy of the
      // group's staging range, row q at [hexcl_q - start, ...), the small
      // rows sorted in registers (sample ids), rows written one at a time,
      // 32 lanes wide.  A row above kTileHits alone is copied straight
      // through.
      __shared__ int64_t s_dst[kCompactThreads], r_dst[kCompactThreads];
      __shared__ int32_t s_len[kCompactThreads], s_off[kCompactThreads], r_off[kCompactThreads];
      const int wb = threadIdx.x - lane;
      s_dst[threadIdx.x] = dst;
      s_len[threadIdx.x] = len;
      if (kSampleIds) push_job_warp(J, len > kSmallSlots, dst, len);
      int l0 = 0;
      while (l0 < 32) {
        const int32_t start = __shfl_sync(FULL, hexcl, l0);
        const unsigned fit = __ballot_sync(FULL, lane >= l0 && hi - start <= kTileHits);
        if (!fit) {  // row l0 alone exceeds shared memory
          const int64_t d = s_dst[wb + l0];
          const int32_t n0 = s_len[wb + l0];
          const int64_t s0 = base + start;
          for (int32_t k0 = 0; k0 < n0; k0 += 32 * kCopyUnroll) {
            int32_t x[kCopyUnroll];
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
              const int32_t k = k0 + 32 * u + lane;
              x[u] = k < n0 ? __ldg(A.stage + s0 + k) : 0;
            }
#pragma unroll
            for (int u = 0; u < kCopyUnroll; ++u) {
              const int32_t k = k0 + 32 * u + lane;
              if (k < n0) idx[d + k] = x[u];
            }
          }
          ++l0;
          continue;
        }
        const int l1 = 32 - __clz(fit);  // hits are non-decreasing: fit = lanes [l0, l1)
        const int32_t G = __shfl_sync(FULL, hi, l1 - 1) - start;
        const bool ing = lane >= l0 && lane < l1;
        const int32_t* gsrc = A.stage + base + start;
        int32_t* sm = smraw;
        if (HRG_COMPACT_TMA) {
          // one 1-D TMA bulk copy of the group's staging range, widened to
          // 16-byte boundaries (the staging buffer has 64 bytes of slack);
          // the group's first hit sits sh ids into the buffer
          const uintptr_t g0 = (uintptr_t)gsrc & ~(uintptr_t)15;
          const int sh = (int)(((uintptr_t)gsrc - g0) >> 2);
          const unsigned bytes =
              (unsigned)((((uintptr_t)(gsrc + G) + 15) & ~(uintptr_t)15) - g0);
          sm = smraw + sh;
          __syncwarp();  // the previous group's reads and in-place sorts are done
          if (G > 0) {
            if (lane == 0) {
              fence_proxy_async_smem();
              mbar_expect_tx(bar, bytes);
              bulk_g2s(smraw, (const void*)g0, bytes, bar);
            }
            mbar_wait(bar, bar_phase);
            bar_phase ^= 1u;
          }
        } else {
          // asynchronous copies (no registers held): the whole group in flight
          for (int32_t i = lane; i < G; i += 32) cp_async4(sm + i, gsrc + i);
          cp_async_wait_all();
        }
        s_off[threadIdx.x] = hexcl - start;
        __syncwarp();
        if (kSampleIds) {
          const bool small = ing && len > 1 && len <= kSmallSlots;
          const int32_t mx = __reduce_max_sync(FULL, small ? len : 0);
          int32_t* row = sm + (hexcl - start);
          if (mx <= 16) {
            if (small) thread_sort_smem<16>(row, len, len);
          } else if (mx <= 32) {
            if (small) thread_sort_smem<32>(row, len, len);
          } else if (kSmallSlots > 32) {
            if (small) thread_sort_smem<kSmallSlots>(row, len, len);
          }
          __syncwarp();
        }
        if (kElemWrite) {
          // write out element-parallel: lane l takes element i0 + l; its row
          // (by rank among the group's non-empty rows) from a bit mask of the
          // row starts inside the step
          const bool nz = ing && len > 0;
          const unsigned nzm = __ballot_sync(FULL, nz);
          const int nr = __popc(nzm);
          if (nz) {
            const int rk = __popc(nzm & ((1u << lane) - 1u));
            r_dst[wb + rk] = dst;
            r_off[wb + rk] = hexcl - start;
          }
          __syncwarp();
          int k0 = 0;  // rank of the row holding element i0
          for (int32_t i0 = 0; i0 < G; i0 += 32) {
            const int sl = k0 + 1 + lane;
            const int32_t st = sl < nr ? r_off[wb + sl] : INT32_MAX;
            const unsigned rel = (unsigned)(st - i0);
            const unsigned mask = __reduce_or_sync(FULL, rel < 32u ? 1u << rel : 0u);
            const int my = k0 + __popc(mask & ((2u << lane) - 1u));
            k0 += __popc(mask);
            const int32_t i = i0 + lane;
            if (i < G) idx[r_dst[wb + my] + (i - r_off[wb + my])] = sm[i];
          }
        } else {
          unsigned todo = __ballot_sync(FULL, ing && len > 0);
          while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t d = s_dst[wb + l];
            const int32_t n0 = s_len[wb + l], e0 = s_off[wb + l];
            for (int32_t k = lane; k < n0; k += 32) idx[d + k] = sm[e0 + k];
          }
        }
        __syncwarp();
        l0 = l1;
      }
    }
    tk = tn;
    cur = nxt;
  }
}

constexpr int kSkewBucket = 32;    // a value bucket this full means non-uniform ids

// Ascending sort of a[0, n) by a group of threads (a warp, kGroup = 32, or
// the block), any n: the bitonic network in its "mirror, then half-cleaners"
// form, where every comparator puts the minimum at the lower index, so the
// positions past n act as +inf padding and their comparators are skipped.
// O(n log^2 n); the order-robust fallback of the bucket sorts below.
template <int kGroup>
__device__ void group_bitonic(int32_t* a, int n, int t0) {
  int P = 1;
  while (P < n) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = t0; t < (P >> 1); t += kGroup) {
        const int r = t & (j - 1);
        const int lo = (t - r) * 2 + r;
        const int hi = j == (k >> 1) ? lo - r + k - 1 - r : lo + j;  // mirror : half-cleaner
        if (hi < n) {
          const int32_t x = a[lo], y = a[hi];
          if (y < x) { a[lo] = y; a[hi] = x; }
        }
      }
      if (kGroup == 32) __syncwarp(); else __syncthreads();
    }
  }
}

// Bucket sort of one row held in shared memory (in[0, len)) by a group of
// kGroup threads, written to dst[0, len) (global; may be the row itself).
// len >> kShift buckets split the row's own [min, max]: for the i.i.d.-uniform
// sample-order ids that is O(len) -- count, scan, scatter into tmp, then
// every id finds its final place by ranking itself inside its (small)
// bucket.  Returns false (nothing written) if a bucket overflows
// kSkewBucket, i.e. the ids are far from uniform; the caller then sorts with
// the bitonic network.  cnt holds (len >> kShift) + 1 counters.  Ids in a
// row are distinct.  Every thread of the group calls it.
template <int kGroup, int kShift>
__device__ bool group_bucket_sort(const int32_t* in, int32_t* tmp, int32_t* cnt, int32_t* dst,
                                  int len, int t0, int32_t mn, int32_t mx, int* s_flag,
                                  int32_t* s_wsum) {
  const unsigned FULL = 0xffffffffu;
  const int lane = t0 & 31;
  const int B = max(1, len >> kShift);
  for (int b = t0; b < B; b += kGroup) cnt[b] = 0;
  if (t0 == 0) *s_flag = 0;
  if (kGroup == 32) __syncwarp(); else __syncthreads();
  const float scale = (float)B / ((float)(mx - mn) + 1.0f);
  for (int i = t0; i < len; i += kGroup) {
    const int b = min((int)((float)(in[i] - mn) * scale), B - 1);
    if (atomicAdd(&cnt[b], 1) == kSkewBucket) *s_flag = 1;
  }
  if (kGroup == 32) __syncwarp(); else __syncthreads();
  if (*s_flag) return false;
  // exclusive scan of cnt[0, B): thread t takes counters [t * per, t * per + per)
  const int per = (B + kGroup - 1) / kGroup;
  int32_t acc = 0;
  for (int q = 0; q < per; ++q) {
    const int b = t0 * per + q;
    if (b < B) acc += cnt[b];
  }
  int32_t inc = acc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += y;
  }
  int32_t woff = 0;
  if (kGroup > 32) {
    const int warp = t0 >> 5;
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const int32_t w = lane < kGroup / 32 ? s_wsum[lane] : 0;
      int32_t wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, wi, o);
        if (lane >= o) wi += y;
      }
      if (lane < kGroup / 32) s_wsum[lane] = wi - w;
    }
    __syncthreads();
    woff = s_wsum[warp];
  }
  int32_t run = woff + inc - acc;
  for (int q = 0; q < per; ++q) {
    const int b = t0 * per + q;
    if (b < B) { const int32_t c = cnt[b]; cnt[b] = run; run += c; }
  }
  if (kGroup == 32) __syncwarp(); else __syncthreads();
  for (int i = t0; i < len; i += kGroup) {
    const int32_t x = in[i];
    const int b = min((int)((float)(x - mn) * scale), B - 1);
    tmp[atomicAdd(&cnt[b], 1)] = x;
  }
  if (kGroup == 32) __syncwarp(); else __syncthreads();
  // cnt[b] is now the end of bucket b: rank each id inside its bucket
  for (int i = t0; i < len; i += kGroup) {
    const int32_t x = tmp[i];
    const int b = min((int)((float)(x - mn) * scale), B - 1);
    const int beg = b == 0 ? 0 : cnt[b - 1], end = cnt[b];
    int r = beg;
    for (int j = beg; j < end; ++j) r += tmp[j] < x;
    dst[r] = x;
  }
  if (kGroup == 32) __syncwarp(); else __syncthreads();
  return true;
}

constexpr int kSortWarpThreads = 256;
struct SortWarpSmem {
  int32_t in[kWarpBucketMax], tmp[kWarpBucketMax], cnt[32];
  int flag;
};
constexpr size_t kSortWarpSmem = sizeof(SortWarpSmem) * (kSortWarpThreads / 32);

// One lane sorts its bucket b[0, c), c <= N, in registers (in place).
template <int N>
__device__ __forceinline__ void lane_sort_bucket(int32_t* b, int32_t c) {
  int32_t x[N];
#pragma unroll
  for (int t = 0; t < N; ++t) x[t] = t < c ? b[t] : INT32_MAX;
  reg_oddeven<N>(x);
#pragma unroll
  for (int t = 0; t < N; ++t)
    if (t < c) b[t] = x[t];
}

// Queued rows (sample-order ids), one warp per row: up to 64 ids by a
// register network, up to kWarpBucketMax by a bucket sort in shared memory;
// longer rows go on to k_sort_rows.
__global__ void __launch_bounds__(kSortWarpThreads, HRG_SORTWARP_MINB) k_sort_warp(int32_t* __restrict__ idx,
                                                                SortJobs J) {
  extern __shared__ __align__(16) unsigned char sort_smem[];
  SortWarpSmem& S = reinterpret_cast<SortWarpSmem*>(sort_smem)[threadIdx.x >> 5];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned nj = *J.rows.n;
  for (int64_t k = warp; k < nj; k += nwarps) {
    const int64_t d = J.rows.off[k];
    const int32_t len = J.rows.len[k];
    int32_t* row = idx + d;
    if (len <= 64) {
      warp_sort_slots<2>(row, len, row, len, lane);
      continue;
    }
    if (len > kWarpBucketMax) {
      if (lane == 0) push_row(J.mid, d, len);
      continue;
    }
    int32_t mn = INT32_MAX, mx = 0;
    for (int i = lane; i < len; i += 32) {
      const int32_t x = row[i];
      S.in[i] = x;
      mn = min(mn, x);
      mx = max(mx, x);
    }
    mn = __reduce_min_sync(FULL, mn);
    mx = __reduce_max_sync(FULL, mx);
    // 32 value buckets over [mn, mx], one per lane: count, scan, scatter into
    // tmp, then each lane sorts its bucket (~len/32 ids) with a register
    // network.  A bucket above 32 ids (far from uniform) -> bitonic fallback.
    S.cnt[lane] = 0;
    __syncwarp();
    const float scale = 32.0f / ((float)(mx - mn) + 1.0f);
    for (int i = lane; i < len; i += 32)
      atomicAdd(&S.cnt[min((int)((float)(S.in[i] - mn) * scale), 31)], 1);
    __syncwarp();
    const int32_t c = S.cnt[lane];
    const int32_t cmax = __reduce_max_sync(FULL, c);
    if (cmax > 32) {
      group_bitonic<32>(S.in, len, lane);
      for (int i = lane; i < len; i += 32) row[i] = S.in[i];
      __syncwarp();
      continue;
    }
    int32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, inc, o);
      if (lane >= o) inc += y;
    }
    const int32_t off = inc - c;
    __syncwarp();
    S.cnt[lane] = off;  // scatter cursors
    __syncwarp();
    for (int i = lane; i < len; i += 32) {
      const int32_t x = S.in[i];
      S.tmp[atomicAdd(&S.cnt[min((int)((float)(x - mn) * scale), 31)], 1)] = x;
    }
    __syncwarp();
    if (cmax <= 8) lane_sort_bucket<8>(S.tmp + off, c);
    else if (cmax <= 16) lane_sort_bucket<16>(S.tmp + off, c);
    else lane_sort_bucket<32>(S.tmp + off, c);
    __syncwarp();
    for (int i = lane; i < len; i += 32) row[i] = S.tmp[i];
    __syncwarp();
  }
}

constexpr int kMidShift = HRG_MID_SHIFT;  // < 0: one bucket per thread, register networks
template <int kCap, int kShift>
constexpr size_t sort_rows_smem() {
  return sizeof(int32_t) * (2 * kCap + (kShift < 0 ? 1024 : (kCap >> kShift) + 1));
}

// Rows of up to kCap ids, one block of kThreads per row, in shared memory
// (bucket sort, bitonic fallback).  Rows above kCap are pushed to `over`
// (when given); without one -- a sub-bucket of a giant row that still
// exceeds the block, only for far-from-uniform ids -- the block sorts the
// row by the bitonic network in global memory.
template <int kThreads, int kCap, int kShift>
__global__ void __launch_bounds__(kThreads) k_sort_rows(const int32_t* src_base,
                                                        int32_t* dst_base, RowList R,
                                                        RowList over) {
  extern __shared__ __align__(16) unsigned char rows_smem[];
  int32_t* in = reinterpret_cast<int32_t*>(rows_smem);
  int32_t* out = in + kCap;
  int32_t* cnt = out + kCap;  // (kCap >> kShift) + 1
  __shared__ int32_t s_wsum[32];
  __shared__ int s_min, s_max, s_flag;
  const int tid = threadIdx.x, lane = tid & 31;
  const unsigned nr = *R.n;
  for (unsigned r = blockIdx.x; r < nr; r += gridDim.x) {
    const int64_t off = R.off[r];
    const int32_t len = R.len[r];
    const int32_t* src = src_base + off;
    int32_t* dst = dst_base + off;
    if (len > kCap) {
      if (over.n) {
        if (tid == 0) push_row(over, off, len);
        continue;
      }
      if (src != dst)
        for (int i = tid; i < len; i += kThreads) dst[i] = src[i];
      __syncthreads();
      group_bitonic<kThreads>(dst, len, tid);
      continue;
    }
    if (len <= 1) {
      if (len == 1 && tid == 0) dst[0] = src[0];
      continue;
    }
    if (tid == 0) { s_min = INT32_MAX; s_max = 0; }
    __syncthreads();
    int32_t mn = INT32_MAX, mx = 0;
    for (int i = tid; i < len; i += kThreads) {
      const int32_t x = src[i];
      in[i] = x;
      mn = min(mn, x);
      mx = max(mx, x);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) { atomicMin(&s_min, mn); atomicMax(&s_max, mx); }
    __syncthreads();
    if (kShift < 0) {
      // one value bucket per thread (~len / kThreads ids), sorted by that
      // thread with a register network
      mn = s_min;
      const float scale = (float)kThreads / ((float)(s_max - mn) + 1.0f);
      cnt[tid] = 0;
      if (tid == 0) s_flag = 0;
      __syncthreads();
      for (int i = tid; i < len; i += kThreads)
        atomicAdd(&cnt[min((int)((float)(in[i] - mn) * scale), kThreads - 1)], 1);
      __syncthreads();
      const int32_t c = cnt[tid];
      const int32_t cm = __reduce_max_sync(0xffffffffu, c);
      if (lane == 0) atomicMax(&s_flag, cm);
      int32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) s_wsum[tid >> 5] = inc;
      __syncthreads();
      if (tid < 32) {
        const int32_t w = tid < kThreads / 32 ? s_wsum[tid] : 0;
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
          if (tid >= o) wi += y;
        }
        if (tid < kThreads / 32) s_wsum[tid] = wi - w;
      }
      __syncthreads();
      const int32_t cmax = s_flag;
      const int32_t boff = s_wsum[tid >> 5] + inc - c;
      if (cmax <= 32) {
        cnt[tid] = boff;
        __syncthreads();
        for (int i = tid; i < len; i += kThreads) {
          const int32_t x = in[i];
          out[atomicAdd(&cnt[min((int)((float)(x - mn) * scale), kThreads - 1)], 1)] = x;
        }
        __syncthreads();
        if (cmax <= 8) lane_sort_bucket<8>(out + boff, c);
        else if (cmax <= 16) lane_sort_bucket<16>(out + boff, c);
        else lane_sort_bucket<32>(out + boff, c);
        __syncthreads();
        for (int i = tid; i < len; i += kThreads) dst[i] = out[i];
      } else {
        group_bitonic<kThreads>(in, len, tid);
        for (int i = tid; i < len; i += kThreads) dst[i] = in[i];
      }
    } else if (!group_bucket_sort<kThreads, kShift < 0 ? 0 : kShift>(
                   in, out, cnt, dst, len, tid, s_min, s_max, &s_flag, s_wsum)) {
      group_bitonic<kThreads>(in, len, tid);
      for (int i = tid; i < len; i += kThreads) dst[i] = in[i];
    }
    __syncthreads();
  }
}

// Giant rows (above kLargeMax ids): split by value into sub-buckets of about
// kGiantTarget ids through a scratch array, kGiantChunk ids per block pass.
struct Giant {
  RowList rows;     // the giant rows (in place in idx)
  RowList sub;      // their sub-buckets: scratch -> idx, same offsets
  int32_t* nb;      // per giant row: sub-bucket count,
  int32_t* bbase;   //   first sub-bucket,
  int32_t* cbase;   //   first chunk
  int32_t* chunk_row;
  unsigned* nchunks;
  unsigned long long* cur;  // per sub-bucket: scatter cursor
};
constexpr int kGiantTarget = 16384;
constexpr int kGiantChunk = 16384;
constexpr int kGiantMaxB = 4096;   // sub-buckets per giant row (smem counters)

__device__ __forceinline__ int giant_nb(int32_t len) {
  return min(kGiantMaxB, max(1, (len + kGiantTarget - 1) / kGiantTarget));
}

// Giant rows, step 1 (one block): sub-bucket and chunk layout per row, the
// sub-bucket list (offsets are filled by k_giant_scan), zeroed counters.
__global__ void __launch_bounds__(1024) k_giant_plan(Giant G) {
  __shared__ int32_t wb[32], wc[32];
  __shared__ int32_t s_b, s_c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned ng = *G.rows.n;
  if (tid == 0) { s_b = 0; s_c = 0; }
  __syncthreads();
  for (unsigned g0 = 0; g0 < ng; g0 += 1024) {
    const unsigned g = g0 + tid;
    const int32_t len = g < ng ? G.rows.len[g] : 0;
    const int32_t nb = g < ng ? giant_nb(len) : 0;
    const int32_t nc = g < ng ? (len + kGiantChunk - 1) / kGiantChunk : 0;
    int32_t ib = nb, ic = nc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, ib, o), z = __shfl_up_sync(0xffffffffu, ic, o);
      if (lane >= o) { ib += y; ic += z; }
    }
    if (lane == 31) { wb[warp] = ib; wc[warp] = ic; }
    __syncthreads();
    if (warp == 0) {
      int32_t a = wb[lane], c = wc[lane], ia = a, icc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, ia, o), z = __shfl_up_sync(0xffffffffu, icc, o);
        if (lane >= o) { ia += y; icc += z; }
      }
      wb[lane] = ia - a;
      wc[lane] = icc - c;
    }
    __syncthreads();
    const int32_t b0 = s_b + wb[warp] + ib - nb, c0 = s_c + wc[warp] + ic - nc;
    if (g < ng) {
      G.nb[g] = nb;
      G.bbase[g] = b0;
      G.cbase[g] = c0;
      for (int32_t q = 0; q < nc; ++q) G.chunk_row[c0 + q] = (int32_t)g;
      for (int32_t q = 0; q < nb; ++q) G.cur[b0 + q] = 0;
    }
    __syncthreads();
    if (tid == 1023) { s_b = b0 + nb; s_c = c0 + nc; }
    __syncthreads();
  }
  if (tid == 0) { *G.sub.n = (unsigned)s_b; *G.nchunks = (unsigned)s_c; }
}

__device__ __forceinline__ int giant_bucket(int32_t x, float scale, int nb) {
  return min((int)((float)x * scale), nb - 1);
}

// Giant rows, step 2: per-chunk histograms into the sub-bucket counters.
__global__ void __launch_bounds__(1024) k_giant_hist(const int32_t* __restrict__ idx, Giant G,
                                                     int64_t n_ids) {
  __shared__ int32_t h[kGiantMaxB];
  const unsigned nc = *G.nchunks;
  for (unsigned c = blockIdx.x; c < nc; c += gridDim.x) {
    const int32_t g = G.chunk_row[c];
    const int nb = G.nb[g];
    const float scale = (float)nb / (float)n_ids;
    const int64_t off = G.rows.off[g] + (int64_t)(c - G.cbase[g]) * kGiantChunk;
    const int32_t m = min(kGiantChunk, (int32_t)(G.rows.off[g] + G.rows.len[g] - off));
    for (int b = threadIdx.x; b < nb; b += 1024) h[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += 1024) atomicAdd(&h[giant_bucket(idx[off + i], scale, nb)], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += 1024)
      if (h[b]) atomicAdd(G.cur + G.bbase[g] + b, (unsigned long long)h[b]);
    __syncthreads();
  }
}

// Giant rows, step 3: counts -> sub-bucket ranges (absolute offsets) and
// scatter cursors; one block per giant row.
__global__ void __launch_bounds__(1024) k_giant_scan(Giant G) {
  __shared__ int64_t s_run;
  const unsigned ng = *G.rows.n;
  const int tid = threadIdx.x, lane = tid & 31;
  __shared__ int64_t ws[32];
  for (unsigned g = blockIdx.x; g < ng; g += gridDim.x) {
    const int nb = G.nb[g], b0 = G.bbase[g];
    if (tid == 0) s_run = G.rows.off[g];
    __syncthreads();
    for (int q0 = 0; q0 < nb; q0 += 1024) {
      const int q = q0 + tid;
      const int64_t c = q < nb ? (int64_t)G.cur[b0 + q] : 0;
      int64_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (lane == 31) ws[tid >> 5] = inc;
      __syncthreads();
      if (tid < 32) {
        int64_t w = ws[lane], wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane >= o) wi += y;
        }
        ws[lane] = wi - w;
      }
      __syncthreads();
      const int64_t start = s_run + ws[tid >> 5] + inc - c;
      if (q < nb) {
        G.cur[b0 + q] = (unsigned long long)start;
        G.sub.off[b0 + q] = start;
        G.sub.len[b0 + q] = (int32_t)c;
      }
      __syncthreads();
      if (tid == 1023) s_run = start + c;
      __syncthreads();
    }
  }
}

// Giant rows, step 4: scatter each chunk into its sub-buckets of the scratch
// array (order inside a sub-bucket is fixed by k_sort_rows).
__global__ void __launch_bounds__(1024) k_giant_scatter(const int32_t* __restrict__ idx,
                                                        int32_t* __restrict__ scratch, Giant G,
                                                        int64_t n_ids) {
  __shared__ int32_t h[kGiantMaxB];
  __shared__ int32_t base[kGiantMaxB];  // relative to the row's offset
  const unsigned nc = *G.nchunks;
  for (unsigned c = blockIdx.x; c < nc; c += gridDim.x) {
    const int32_t g = G.chunk_row[c];
    const int nb = G.nb[g];
    const float scale = (float)nb / (float)n_ids;
    const int64_t off = G.rows.off[g] + (int64_t)(c - G.cbase[g]) * kGiantChunk;
    const int32_t m = min(kGiantChunk, (int32_t)(G.rows.off[g] + G.rows.len[g] - off));
    for (int b = threadIdx.x; b < nb; b += 1024) h[b] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += 1024) atomicAdd(&h[giant_bucket(idx[off + i], scale, nb)], 1);
    __syncthreads();
    const int64_t row0 = G.rows.off[g];
    for (int b = threadIdx.x; b < nb; b += 1024)
      base[b] = h[b] ? (int32_t)((int64_t)atomicAdd(G.cur + G.bbase[g] + b,
                                                    (unsigned long long)h[b]) - row0)
                     : 0;
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += 1024) {
      const int32_t x = idx[off + i];
      scratch[row0 + atomicAdd(&base[giant_bucket(x, scale, nb)], 1)] = x;
    }
    __syncthreads();
  }
}

// Compaction of heavy rows: one warp per chunk; the chunk's hits go to
// rowptr[id] + (hits of the row's earlier chunks).
__global__ void __launch_bounds__(256) k_compact_heavy(QueryArgs A, int64_t H,
                                                       const int64_t* __restrict__ chunk_off,
                                                       const int64_t* __restrict__ rowptr,
                                                       int32_t* __restrict__ idx,
                                                       bool sample_ids) {
  if (*A.overflow) return;  // void pass, re-run by the host
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t total_chunks = *A.total_chunks;
  for (int64_t c = warp; c < total_chunks; c += nwarps) {
    const int64_t e = __ldg(A.chunk_entry + c);
    const int32_t v = A.heavy_v[e];
    const int32_t idv = sample_ids ? row_of<true>(A, v) : row_of<false>(A, v);
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

// Sample-order ids: heavy rows arrive in (band, angle) order of their
// neighbours; queue each for an in-place sort.
__global__ void k_queue_heavy_rows(QueryArgs A, const int64_t* __restrict__ rowptr,
                                   SortJobs J) {
  if (*A.overflow) return;  // void pass, re-run by the host
  const int64_t H = *A.heavy_n;
  for (int64_t e0 = blockIdx.x * (int64_t)blockDim.x; e0 < H;
       e0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = e0 + threadIdx.x;
    int64_t b = 0;
    int32_t len = 0;
    if (e < H) {
      const int32_t idv = row_of<true>(A, A.heavy_v[e]);
      b = rowptr[idv];
      len = (int32_t)(rowptr[idv + 1] - b);
    }
    push_job_warp(J, len > 1, b, len);
  }
}

__global__ void __launch_bounds__(256) k_sincos(int64_t n, const double* __restrict__ x,
                                                double* __restrict__ s, double* __restrict__ c,
                                                int mode) {
  // mode 0: glibc's sin/cos (the product default), 1: correctly rounded
  // (fast path + rounding test), 2: correctly rounded, full evaluation
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    if (mode == 2) sincos_cr(x[i], s + i, c + i);
    else trig_sincos(mode, x[i], s + i, c + i);
  }
}

// Fast path (with its rounding test) against the full double-double
// evaluation on n Philox angles in [0, 2pi) plus, every 4th one, an angle
// within 2^-20 of a multiple of pi/4: mismatches and fast-path rejections.
__global__ void __launch_bounds__(256) k_sincos_compare(int64_t n, uint64_t seed,
                                                        unsigned long long* __restrict__ out) {
  unsigned long long bad = 0, slow = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t a, b;
    philox_u53(i, seed, a, b);
    double x = angle_from_u53(a);
    if ((i & 3) == 3) {
      const double m = (double)(b & 7) * 0.7853981633974483;
      x = fabs(m + ((double)(a >> 20) * 0x1.0p-33 - 0.5) * 0x1.0p-19);
    }
    double s0, c0, s1, c1;
    sincos_cr(x, &s0, &c0);
    slow += !sincos_crf(x, &s1, &c1);
    bad += (__double_as_longlong(s0) != __double_as_longlong(s1)) ||
           (__double_as_longlong(c0) != __double_as_longlong(c1));
  }
  atomicAdd(out, bad);
  atomicAdd(out + 1, slow);
}

// ---- all-pairs reference (hrgen generator.py:249-274, generate_brute_force):
// x = r cos(phi), y = r sin(phi), b = (1 - r)(1 + r); {i, j} is an edge iff
// 2 asinh(sqrt(d2 / (b_i b_j))) < R with d2 = dx*dx + dy*dy, evaluated in that
// order.  The predicate is symmetric (fl(a - b) = -fl(b - a)), so every row
// scans all columns in ascending order and comes out sorted.  A pair far from
// the threshold is decided by d2 against (sinh(R/2)(1 -+ 1e-9))^2 b_i b_j
// (no division, sqrt or asinh); the others by hrgen's own sequence, and those
// within 4 ulps of R -- where CUDA's asinh and glibc's may round differently
// -- are counted as near ties.
__global__ void __launch_bounds__(256) k_bf_points(int64_t n, const double* __restrict__ phi,
                                                   const double* __restrict__ rp,
                                                   double* __restrict__ x, double* __restrict__ y,
                                                   double* __restrict__ b, int trig) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sn, cs;
  trig_sincos(trig, phi[i], &sn, &cs);
  const double r = rp[i];
  x[i] = __dmul_rn(r, cs);
  y[i] = __dmul_rn(r, sn);
  b[i] = __dmul_rn(__dsub_rn(1.0, r), __dadd_rn(1.0, r));
}

template <bool kWrite>
__global__ void __launch_bounds__(256) k_bf_pairs(int64_t n, const double* __restrict__ x,
                                                  const double* __restrict__ y,
                                                  const double* __restrict__ b, double t_lo,
                                                  double t_hi, double R, double tie,
                                                  int32_t* __restrict__ deg,
                                                  const int64_t* __restrict__ rowptr,
                                                  int32_t* __restrict__ idx,
                                                  unsigned long long* __restrict__ ties) {
  __shared__ double sx[256], sy[256], sbb[256];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool ok = i < n;
  const double xi = ok ? x[i] : 0.0, yi = ok ? y[i] : 0.0, bi = ok ? b[i] : 0.0;
  int32_t cnt = 0;
  int64_t at = (kWrite && ok) ? rowptr[i] : 0;
  unsigned long long nt = 0;
  for (int64_t j0 = 0; j0 < n; j0 += 256) {
    __syncthreads();
    const int64_t jj = j0 + threadIdx.x;
    sx[threadIdx.x] = jj < n ? x[jj] : 0.0;
    sy[threadIdx.x] = jj < n ? y[jj] : 0.0;
    sbb[threadIdx.x] = jj < n ? b[jj] : 0.0;
    __syncthreads();
    const int m = (int)min((int64_t)256, n - j0);
    if (!ok) continue;
    for (int t = 0; t < m; ++t) {
      const int64_t j = j0 + t;
      const double dx = __dsub_rn(xi, sx[t]), dy = __dsub_rn(yi, sy[t]);
      const double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      const double bb = __dmul_rn(bi, sbb[t]);
      bool hit;
      if (d2 < __dmul_rn(t_lo, bb)) {
        hit = true;
      } else if (d2 > __dmul_rn(t_hi, bb)) {
        hit = false;
      } else {  // hrgen's sequence (generator.py:266)
        const double dist = __dmul_rn(2.0, asinh(__dsqrt_rn(__ddiv_rn(d2, bb))));
        hit = dist < R;
        if (j != i && fabs(dist - R) <= tie) ++nt;
      }
      if (hit && j != i) {
        if (kWrite) idx[at++] = (int32_t)j;
        else ++cnt;
      }
    }
  }
  if (ok && !kWrite) deg[i] = cnt;
  if (kWrite && nt) atomicAdd(ties, nt);
}

// Compact rows -> the n-row CSR of the API (on request): degrees by vertex
// id, then every row copied to its place, a warp per row.
__global__ void __launch_bounds__(256) k_expand_deg(int64_t nq, const int64_t* __restrict__ rp_c,
                                                    const int32_t* __restrict__ row_ids,
                                                    int32_t* __restrict__ deg) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nq;
       k += (int64_t)gridDim.x * blockDim.x)
    deg[row_ids[k]] = (int32_t)(rp_c[k + 1] - rp_c[k]);
}

__global__ void __launch_bounds__(256) k_expand_rows(int64_t nq, const int64_t* __restrict__ rp_c,
                                                     const int32_t* __restrict__ row_ids,
                                                     const int32_t* __restrict__ idx_c,
                                                     const int64_t* __restrict__ rp,
                                                     int32_t* __restrict__ idx) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = w0; k < nq; k += nw) {
    const int64_t s = rp_c[k], len = rp_c[k + 1] - s, d = rp[row_ids[k]];
    for (int64_t i = lane; i < len; i += 32) idx[d + i] = idx_c[s + i];
  }
}

// Ids below 2^24 as 3 little-endian bytes each (the result copy's transfer
// format when n <= 2^24): a thread packs 4 ids into 3 words.  `in` need not
// be 16-byte aligned (it starts anywhere in the index array).
__global__ void __launch_bounds__(256) k_pack3(int64_t n, const int32_t* __restrict__ in,
                                               uint32_t* __restrict__ out) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t i = 4 * g;
  if (i >= n) return;
  uint32_t x[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) x[t] = i + t < n ? (uint32_t)in[i + t] & 0xffffffu : 0u;
  out[3 * g] = x[0] | (x[1] << 24);
  out[3 * g + 1] = (x[1] >> 8) | (x[2] << 16);
  out[3 * g + 2] = (x[2] >> 16) | (x[3] << 8);
}

__global__ void __launch_bounds__(256) k_widen(int64_t n, const int32_t* __restrict__ in,
                                               int64_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace hrg

#include "hrg_block.cuh"
