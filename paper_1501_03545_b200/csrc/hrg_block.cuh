// hrg_block.cuh -- the range query as dense blocks: a count pass and a
// write pass over query sub-tiles (included at the end of hrg_kernels.cuh).
//
// Replaces hrgen's leaf scan (quadtree.py:596-615: a query tests every point
// of its angular window in each leaf) and generator.py:182-225.
//
// A warp takes a tile (32 consecutive positions of one radial band) and cuts
// it into sub-tiles of T' queries.  For a sub-tile, lane j resolves band j's
// UNION window: the angular span of the T' queries widened by the window of
// their smallest radius, directory-resolved and trimmed to exact keys
// (<= 2 sorted-position segments per band; the same conservative windows as
// the per-query ones, so every neighbour of every query of the sub-tile lies
// in the union).  The union's U records are then tested against all T'
// queries as a dense T' x U block: lane l holds record l of a 32-record
// chunk in registers (one coalesced 48-byte load per lane, straight from
// HBM/L2), the queries are broadcast from shared memory, and each (query,
// chunk) pair is one ballot.  Testing a record outside a query's own window
// is harmless -- hrgen's predicate (quadtree.py:611-613, circle of the smaller
// id, generator.py:182-187) decides every pair exactly -- and costs ~20
// instructions per 32 tests, with no per-query window resolution, segment
// lists or scattered loads.
//
// T' trades union overhead against per-chunk setup: the sub-tile's angular
// span covers about T' * n / N_i points summed over all bands (N_i the points
// of the tile's band), so T'_i = pow2floor(G * N_i / n) keeps that overhead
// near G records per sub-tile (G = HRG_BLOCK_G).  A sub-tile whose T' * U
// exceeds the write pass's shared row buffer, or whose span is >= 0.5 rad, is
// halved; a single query with more than kLightMax candidates (hubs near the
// centre) is deferred to k_heavy, exactly as the walk path defers it.
//
// Count pass (kWrite = false): row lengths -> deg[].  After the scan of deg,
// the write pass (kWrite = true) recomputes the same blocks (the same
// decisions, deterministically), gathers each query's hits in shared memory,
// sorts rows of <= kSmallSlots ids in registers (sample-order ids; hrgen's
// Graph rows are sorted, graph.py:69-71), queues longer rows for the
// in-place sorts, and writes every row straight into its CSR range: no
// staging buffer, no compaction pass.  Angular ids come out sorted (the
// union is walked band by band in position order).
#pragma once

namespace hrg {

#ifndef HRG_BLOCK_G
#define HRG_BLOCK_G 64
#endif
#ifndef HRG_BLOCK_HITCAP
#define HRG_BLOCK_HITCAP 2048
#endif
#ifndef HRG_BLOCK_MINB_COUNT
#define HRG_BLOCK_MINB_COUNT 8
#endif
#ifndef HRG_BLOCK_MINB_WRITE
#define HRG_BLOCK_MINB_WRITE 4
#endif
#ifndef HRG_BLOCK_TILECAP
#define HRG_BLOCK_TILECAP 2048
#endif

#ifdef HRG_BLOCK_PROFILE
// per band of the tile: [0] clock cycles, [1] tiles, [2] sub-tiles, [3] chunks,
// [4] (query, chunk) iterations, [5] tests; [6] union rounds (experiments only)
__device__ unsigned long long g_bprof[2][kMaxBands][8];
#endif
constexpr int kBlockThreads = 128;
constexpr int kBlockG = HRG_BLOCK_G;        // union overhead target, records per sub-tile
constexpr int kHitCap = HRG_BLOCK_HITCAP;   // T' * U bound: the write pass's row buffer per warp
constexpr int kTileCap = HRG_BLOCK_TILECAP;  // write pass: a tile's rows buffered per warp

// A query (or candidate) as the pair test needs it.
struct __align__(16) QB {
  double px, py, cx, cy, rsq;
  int32_t id, pad;
};

template <bool kSampleIds>
__device__ __forceinline__ QB load_qb(const QueryArgs& A, int32_t v) {
  QB b;
  {
    const double2 p = load_pt(A.rec, v);
    const Circ ci = load_circ(A.rec, v);
    b.px = p.x; b.py = p.y; b.cx = ci.cx; b.cy = ci.cy; b.rsq = ci.rsq;
    b.id = kSampleIds ? __ldg(A.rec.ids + v) : v;  // angular ids are positions
  }
  b.pad = 0;
  return b;
}

// One pair test, operands selected first (no divergent branch): the circle
// of the smaller id decides (generator.py:182-187).
__device__ __forceinline__ bool block_test(const QB& q, const QB& r) {
  const bool lower = r.id < q.id;  // r's circle decides
  const double x = lower ? q.px : r.px, y = lower ? q.py : r.py;
  const double cx = lower ? r.cx : q.cx, cy = lower ? r.cy : q.cy;
  const double rs = lower ? r.rsq : q.rsq;
  // non-short-circuit: no branch (and no reconvergence around the ballot)
  return ref_pred(x, y, cx, cy, rs) & (r.id != q.id);
}

// A sub-tile's union as the chunk loop needs it (per lane = band j): the
// exclusive prefix of the band's union size, its A-part length and the
// starts of both parts; U = the union's total size (warp-uniform).
struct SubUnion {
  int32_t excl, lenA, sA, sB, U;
};

// Record of flat union index c0 + lane (band = last lane j with excl_j <= i;
// id -1 past the end).
template <bool kSampleIds>
__device__ __forceinline__ QB fetch_rec(const QueryArgs& A, const SubUnion& S, int32_t c0) {
  const unsigned FULL = 0xffffffffu;
  const int32_t i = c0 + (int32_t)(threadIdx.x & 31);
  int o = 0;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1)
    if (__shfl_sync(FULL, S.excl, o + s) <= i) o += s;
  const int32_t off = i - __shfl_sync(FULL, S.excl, o);
  const int32_t la = __shfl_sync(FULL, S.lenA, o);
  const int32_t sa = __shfl_sync(FULL, S.sA, o), sbb = __shfl_sync(FULL, S.sB, o);
  QB r;
  if (i < S.U) {
    r = load_qb<kSampleIds>(A, off < la ? sa + off : sbb + (off - la));
  } else {
    r.px = r.py = r.cx = r.cy = r.rsq = 0.0;
    r.id = -1;
  }
  return r;
}

// The T x U block of one sub-tile (queries q0 .. q0 + T - 1 of the tile):
// kIn chunks of 32 records in flight per step, the T queries unrolled with
// their hit counts in registers.  cnt (this lane's query) receives its
// count; the write pass stores each query's hits at obase[oofs_q + k].
template <int T, bool kSampleIds, bool kWrite>
__device__ __forceinline__ void block_chunks(const QueryArgs& A, const SubUnion& S, const QB* qs,
                                             int q0, int32_t& cnt, int32_t* obase, int64_t oofs) {
  constexpr int kIn = T == 1 ? 4 : (T <= 4 ? 2 : 1);
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int32_t cq[T];
#pragma unroll
  for (int t = 0; t < T; ++t) cq[t] = 0;
  // T = 1: the query stays in registers
  QB Q1;
  if (T == 1) Q1 = qs[q0];
  for (int32_t c0 = 0; c0 < S.U; c0 += 32 * kIn) {
    QB r[kIn];
#pragma unroll
    for (int k = 0; k < kIn; ++k) r[k] = fetch_rec<kSampleIds>(A, S, c0 + 32 * k);
#pragma unroll
    for (int k = 0; k < kIn; ++k) {
      if (c0 + 32 * k >= S.U) break;
      const bool ok = r[k].id >= 0;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const QB Q = T == 1 ? Q1 : qs[q0 + t];
        const bool hit = ok & block_test(Q, r[k]);
        const unsigned m = __ballot_sync(FULL, hit);
        if (kWrite) {
          const int64_t at = __shfl_sync(FULL, oofs, q0 + t) + cq[t];
          if (hit) obase[at + __popc(m & lt)] = r[k].id;
        }
        cq[t] += __popc(m);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t)
    if (lane == q0 + t) cnt = cq[t];
}

template <bool kSampleIds, bool kWrite>
__global__ void __launch_bounds__(kBlockThreads, kWrite ? HRG_BLOCK_MINB_WRITE : HRG_BLOCK_MINB_COUNT)
k_block(QueryArgs A, const int64_t* __restrict__ rowptr, int64_t nrows, int32_t* __restrict__ idx,
        int64_t idx_cap, SortJobs J) {
  constexpr int kW = kBlockThreads / 32;
  __shared__ Band sb[kMaxBands];
  __shared__ int32_t s_tsub[kMaxBands];
  __shared__ QB s_q[kW][32];
  __shared__ int32_t s_hb[kWrite ? kW : 1][kWrite ? kTileCap : 1];
  if (kWrite) {
    // a staging overflow of the heavy pass or a CSR larger than idx voids
    // the pass (re-run by the host with the capacities it then knows)
    if (*A.overflow) return;
    if (rowptr[nrows] > idx_cap) {
      if (threadIdx.x == 0 && blockIdx.x == 0) atomicOr(A.overflow, 2);
      return;
    }
  }
  if (threadIdx.x < A.L) sb[threadIdx.x] = A.bands[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < kMaxBands) {
    // sub-tile size of band i: T' * n / N_i ~ G records of union overhead
    int64_t tot = 0;
    for (int j = 0; j < A.L; ++j) tot += max(0, sb[j].end - sb[j].start);
    const int i = threadIdx.x;
    const int64_t ni = i < A.L ? max(0, sb[i].end - sb[i].start) : 0;
    const double t = tot > 0 ? (double)kBlockG * (double)ni / (double)tot : 1.0;
    int ts = 1;
    while (ts < 16 && 2.0 * ts <= t) ts <<= 1;
    s_tsub[i] = ts;
  }
  __syncthreads();
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  QB* qs = s_q[threadIdx.x >> 5];
  int32_t* hb = s_hb[kWrite ? (threadIdx.x >> 5) : 0];
  unsigned long long* counter = A.tile_next + (kWrite ? 1 : 0);
  unsigned long long tests = 0;
  for (int64_t tk = __shfl_sync(FULL, lane == 0 ? (int64_t)atomicAdd(counter, 1ull) : 0, 0);
       tk < A.ntiles;
       tk = __shfl_sync(FULL, lane == 0 ? (int64_t)atomicAdd(counter, 1ull) : 0, 0)) {
#ifdef HRG_BLOCK_PROFILE
    const long long clk0 = clock64();
    unsigned long long pf_sub = 0, pf_chunks = 0, pf_iter = 0, pf_rounds = 0;
#endif
    const uint64_t tv = __ldg(A.tiles + tk);
    if (tv == ~0ull) break;
    const int32_t v0 = (int32_t)(tv & 0xffffffffu);
    const int nq = (int)((int32_t)(tv >> 32) - v0);
    const bool act = lane < nq;
    const int32_t v = v0 + (act ? lane : 0);
    __syncwarp();
    if (act) qs[lane] = load_qb<kSampleIds>(A, v);
    const double phi = act ? A.q.phi[v] : 0.0;
    const float rf = act ? __ldg(&A.rec.circ[v].rf) : 3.0e38f;
    const int32_t row = act ? row_of<kSampleIds>(A, v) : 0;
    // write pass: the tile's rows (lengths known from the count pass) go to
    // a shared buffer at exact offsets when they fit -- then every lane sorts
    // one row and the tile is written out as one stream -- else straight
    // to their CSR ranges (and queued for the in-place sorts)
    int64_t dst = 0;
    int32_t rlen = 0, roff = 0, ttot = 0;
    if (kWrite) {
      if (act) {
        dst = rowptr[row];
        rlen = A.heavy_of[v] < 0 ? (int32_t)(rowptr[row + 1] - dst) : 0;
      }
      int32_t incl = rlen;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      roff = incl - rlen;
      ttot = __shfl_sync(FULL, incl, 31);
    }
    const bool buffered = kWrite && ttot <= kTileCap;
    int32_t* const obase = buffered ? hb : idx;       // warp-uniform (shared or global)
    const int64_t oofs = buffered ? (int64_t)roff : dst;  // this lane's row in obase
    const int bi = __ffs(__ballot_sync(FULL, lane < A.L && sb[lane].start <= v0 &&
                                                 v0 < sb[lane].end)) - 1;
    const int t0 = bi >= 0 ? s_tsub[bi] : 1;
    __syncwarp();
    int32_t cnt = 0;  // this lane's query: hits so far
    int q0 = 0;
    while (q0 < nq) {
      int T = t0;  // a power of two <= 16
      while (T > nq - q0) T >>= 1;
      int32_t sA = 0, eA = 0, sB = 0, eB = 0, U = 0;
      for (;;) {
        const bool in = lane >= q0 && lane < q0 + T;
        double pmin = in ? phi : 1e300, pmax = in ? phi : -1e300;
        float rmin = in ? rf : 3.0e38f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          pmin = fmin(pmin, __shfl_xor_sync(FULL, pmin, o));
          pmax = fmax(pmax, __shfl_xor_sync(FULL, pmax, o));
          rmin = fminf(rmin, __shfl_xor_sync(FULL, rmin, o));
        }
#ifdef HRG_BLOCK_PROFILE
        pf_rounds += 1;
#endif
        if (T > 1 && pmax - pmin >= 0.5) { T >>= 1; continue; }
        sA = eA = sB = eB = 0;
        if (lane < A.L) {
          const float dlt = __ldg(wtab_row(A, rmin) + lane);
          const double half = 0.5 * (pmax - pmin);
          union_window(A, sb[lane], 0.5 * (pmin + pmax),
                       (dlt < 0.0f || dlt >= 3.14159265f) ? dlt
                                                          : __double2float_ru((double)dlt + half),
                       sA, eA, sB, eB);
        }
        U = __reduce_add_sync(FULL, (eA - sA) + (eB - sB));
        if (T > 1 && T * U > kHitCap) { T >>= 1; continue; }
        break;
      }
      if (T == 1 && U > kLightMax) {
        // a hub: deferred to k_heavy (the count pass queues it; both passes
        // skip it here)
        if (!kWrite && lane == q0) {
          const unsigned long long hoff = atomicAdd(A.bump, (unsigned long long)U);
          const unsigned e = atomicAdd(A.heavy_n, 1u);
          A.heavy_v[e] = v;
          A.heavy_c[e] = U;
          A.heavy_of[v] = (int32_t)e;
          A.stage_off[v] = (int64_t)hoff;
        }
        q0 += 1;
        continue;
      }
      if (lane == 0) tests += (unsigned long long)T * (unsigned long long)U;
#ifdef HRG_BLOCK_PROFILE
      pf_sub += 1; pf_chunks += (U + 31) / 32; pf_iter += (unsigned long long)((U + 31) / 32) * T;
#endif
      const int32_t lenA = eA - sA, len = lenA + (eB - sB);
      int32_t incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
      }
      const SubUnion S{incl - len, lenA, sA, sB, U};
      switch (T) {
        case 1: block_chunks<1, kSampleIds, kWrite>(A, S, qs, q0, cnt, obase, oofs); break;
        case 2: block_chunks<2, kSampleIds, kWrite>(A, S, qs, q0, cnt, obase, oofs); break;
        case 4: block_chunks<4, kSampleIds, kWrite>(A, S, qs, q0, cnt, obase, oofs); break;
        case 8: block_chunks<8, kSampleIds, kWrite>(A, S, qs, q0, cnt, obase, oofs); break;
        default: block_chunks<16, kSampleIds, kWrite>(A, S, qs, q0, cnt, obase, oofs); break;
      }
      if (!kWrite && lane >= q0 && lane < q0 + T) {
        A.deg[row] = cnt;
        A.heavy_of[v] = -1;
      }
      q0 += T;
    }
#ifdef HRG_BLOCK_PROFILE
    if (lane == 0 && bi >= 0) {
      unsigned long long* P = g_bprof[kWrite ? 1 : 0][bi];
      atomicAdd(P + 0, (unsigned long long)(clock64() - clk0));
      atomicAdd(P + 1, 1ull); atomicAdd(P + 2, pf_sub); atomicAdd(P + 3, pf_chunks);
      atomicAdd(P + 4, pf_iter); atomicAdd(P + 6, pf_rounds);
    }
#endif
    if (kWrite) {
      // the recomputed row must have the count pass's length (a mismatch
      // would be a bug: fail the generation loudly instead of writing it)
      if (act && A.heavy_of[v] < 0 && cnt != rlen) atomicOr(A.overflow, 4);
      __syncwarp();
      if (buffered) {
        if (kSampleIds) {
          // every lane sorts its own row (<= kSmallSlots ids) in registers
          const bool small = cnt > 1 && cnt <= kSmallSlots;
          const int32_t mx = __reduce_max_sync(FULL, small ? cnt : 0);
          int32_t* myrow = hb + roff;
          if (mx > 0) {
            if (mx <= 16) {
              if (small) thread_sort_smem<16>(myrow, cnt, cnt);
            } else if (mx <= 32) {
              if (small) thread_sort_smem<32>(myrow, cnt, cnt);
            } else {
              if (small) thread_sort_smem<kSmallSlots>(myrow, cnt, cnt);
            }
          }
          push_job_warp(J, cnt > kSmallSlots, dst, cnt);
          __syncwarp();
        }
        // the tile's rows as one stream: element i belongs to the last row
        // whose offset is <= i (binary search over the lanes' offsets)
        for (int32_t i0 = 0; i0 < ttot; i0 += 32) {
          const int32_t i = i0 + lane;
          int o = 0;
#pragma unroll
          for (int s = 16; s > 0; s >>= 1)
            if (__shfl_sync(FULL, roff, o + s) <= i) o += s;
          const int64_t d = __shfl_sync(FULL, dst, o);
          const int32_t ro = __shfl_sync(FULL, roff, o);
          if (i < ttot) idx[d + (i - ro)] = hb[i];
        }
      } else if (kSampleIds) {
        push_job_warp(J, cnt > 1, dst, cnt);  // rows written in union order
      }
      __syncwarp();
    }
  }
  if (!kWrite && lane == 0 && tests) atomicAdd(A.cand_total, tests);
}

}  // namespace hrg
