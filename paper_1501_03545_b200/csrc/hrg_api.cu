// hrg_api.cu -- C ABI (include/hrgen_b200.h) over the sm_100a kernels.
//
// Host orchestration of one generation on one stream.  The only host<->device
// synchronisation inside a generation is reading the CSR size after the count
// pass (to size the index buffer); everything else is queued asynchronously.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#if defined(__SSE2__)
#include <emmintrin.h>
#endif
#if defined(__x86_64__)
#include <tmmintrin.h>
#endif
#include <string>
#include <thread>
#include <vector>

#include "../../include/hrgen_b200.h"
#include "../../include/hrgen_b200_debug.h"
#include "hrg_kernels.cuh"

using namespace hrg;

namespace {

thread_local std::string g_err;

hrg_status fail(hrg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail(HRG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t b = std::max<size_t>(want, 256);
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

struct ToI64 {
  __host__ __device__ __forceinline__ long long operator()(const int32_t& x) const { return x; }
};

}  // namespace

struct hrg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int sm_count = 148;
  // coordinates in vertex-id order
  Buf phi, rn, rp;
  // sort
  Buf keys_out, vals_in, vals_out;
  // sorted records
  Buf pt, circ, s_phi, s_rp, s_rn, pr;
  // staging + heavy queries
  Buf stage, stage_off, counters, heavy_v, heavy_c, heavy_of, nchunks, chunk_start, chunk_hits, chunk_entry,
      chunk_off, slots, large_off, large_len, giant_off, giant_len, giant_meta,
      sub_off, sub_len, sub_cur, chunk_row, tv0, wtab, job_dst, job_len, mid_off, mid_len;
  int64_t stage_cap = 0;
  // index
  Buf bands, dir, dir_total, bad, dir_gaps, band_pmin;
  // CSR
  Buf deg, rowptr, idx, cand, rowidx, row_ids, rowptr_c, nq_buf;
  bool compact_result = false;  // sharded: rows in sector-position order (expanded on request)
  int64_t nq = 0;
  Buf temp, k32_in, k32_out, sh_buf, sh_bands, sh_wtab, sh_keep, sh_gid;
  bool sh_sampled = false;  // sharded sampling: vals are compact indices, sh_gid the ids
  Buf widen, pack;
  int32_t* h_stage = nullptr;      // pinned int32 staging of the indices (host widening)
  size_t h_stage_bytes = 0;
  std::vector<cudaEvent_t> h_ev;   // one per staged chunk
  int64_t n = 0, np = 0, nnz = 0;
  const float* sh_cover = nullptr;  // sharded subset: per-band circle coverage,
  const int64_t* sh_lo = nullptr;   //   needed key ranges (k_shard_ranges)
  const int64_t* sh_hi = nullptr;
  const int* sh_mode = nullptr;
  bool have_result = false;
  bool coords_sorted = false;  // angular order: coordinates live in s_phi/s_rn/s_rp
  bool coords_pending = false; // sample order: phi/rn/rp not yet materialised
  SampleParams pending{};
  int32_t* idx_final = nullptr;
  cudaEvent_t ev[9] = {};  // see enum Ev
  int query_blocks_per_sm = 0;
  cudaStream_t aux[2] = {nullptr, nullptr};  // side streams of the row sorts
  cudaEvent_t fork = nullptr, join[2] = {nullptr, nullptr};
  unsigned char* h_rb = nullptr;  // mapped pinned readback area (kReadback bytes)
  unsigned char* d_rb = nullptr;  // its device alias
  int64_t launches = 0;  // this library's kernel launches (CUB's not included)
  int trig = kTrigLibm;  // sin/cos of the Poincare coordinates (hrg_context_set_trig)
  int grid_block_count = 0, grid_block_write = 0;
  int grid_light = 0, grid_light_wide = 0, grid_heavy = 0, grid_compact = 0, grid_compact_heavy = 0;
};

namespace {

enum Ev { E_START, E_SAMPLED, E_SORTED, E_INDEXED, E_PLANNED, E_COUNTED, E_WRITE0, E_WRITTEN,
          E_ROWSORTED };

hrg_status check_model(const hrg_model* m) {
  if (!m) return fail(HRG_ERR_PARAMETER_DOMAIN, "model is NULL");
  if (m->n < 1) return fail(HRG_ERR_PARAMETER_DOMAIN, "n must be at least 1");
  if (m->n >= (int64_t)1 << 30) return fail(HRG_ERR_PARAMETER_DOMAIN, "n must be below 2^30");
  if (!(m->alpha > 0.0)) return fail(HRG_ERR_PARAMETER_DOMAIN, "alpha must be positive");
  if (!(m->R > 0.0)) return fail(HRG_ERR_PARAMETER_DOMAIN, "radius must be positive");
  if (!(m->max_r > 0.0 && m->max_r < 1.0))
    return fail(HRG_ERR_PARAMETER_DOMAIN, "max_r must be in (0, 1)");  // quadtree.py:260
  if (!(m->cosh_r_minus_1 > 0.0)) return fail(HRG_ERR_PARAMETER_DOMAIN, "bad cosh(R)-1");
  return HRG_OK;
}

BandSpec make_bands(double R, int* L_out) {
  BandSpec S;
  memset(&S, 0, sizeof(S));
  int L = kMaxBands;
  S.L = L;
  for (int j = 0; j < L; ++j) S.thr[j] = std::tanh(R * j / L / 2.0);
  *L_out = L;
  return S;
}

hrg_status ensure_point_buffers(hrg_context* c, int64_t n) {
  size_t d = sizeof(double) * (size_t)n, f = sizeof(float) * (size_t)n, i32 = 4 * (size_t)n;
  size_t u64 = 8 * (size_t)n;
  CUDA_TRY(c->phi.ensure(d)); CUDA_TRY(c->rn.ensure(d)); CUDA_TRY(c->rp.ensure(d));
  CUDA_TRY(c->keys_out.ensure(u64));
  CUDA_TRY(c->k32_in.ensure(i32)); CUDA_TRY(c->k32_out.ensure(i32));
  CUDA_TRY(c->vals_in.ensure(i32)); CUDA_TRY(c->vals_out.ensure(i32));
  for (Buf* b : {&c->s_phi, &c->s_rp, &c->s_rn}) CUDA_TRY(b->ensure(d));
  CUDA_TRY(c->pr.ensure(2 * d));
  CUDA_TRY(c->pt.ensure(16 * (size_t)n));
  CUDA_TRY(c->circ.ensure(sizeof(Circ) * (size_t)n));
  CUDA_TRY(c->stage_off.ensure(8 * (size_t)n)); CUDA_TRY(c->counters.ensure(128));
  CUDA_TRY(c->heavy_v.ensure(i32)); CUDA_TRY(c->heavy_c.ensure(i32));
  CUDA_TRY(c->heavy_of.ensure(i32)); CUDA_TRY(c->slots.ensure(i32));
  CUDA_TRY(c->bands.ensure(sizeof(Band) * kMaxBands));
  CUDA_TRY(c->dir.ensure(4 * (size_t)((2 * n << kDirExtra) + 2 * kMaxBands + 64)));
  CUDA_TRY(c->dir_total.ensure(16)); CUDA_TRY(c->bad.ensure(8)); CUDA_TRY(c->cand.ensure(8));
  CUDA_TRY(c->deg.ensure(i32)); CUDA_TRY(c->rowptr.ensure(8 * (size_t)(n + 1)));
  return HRG_OK;
}

inline unsigned blocks_for(int64_t n, int t = 256) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// Small device->host readbacks through mapped pinned memory (a kernel
// stores, the host reads after the stream sync): no copy-engine command, so a
// readback never queues behind another context's multi-GB result copy.
constexpr size_t kReadback = 256;
struct RbItem { const void* src; size_t bytes; };
__global__ void k_readback(RbItem a, RbItem b, RbItem e, unsigned char* dst) {
  for (size_t i = threadIdx.x; i < a.bytes; i += blockDim.x)
    dst[i] = static_cast<const unsigned char*>(a.src)[i];
  for (size_t i = threadIdx.x; i < b.bytes; i += blockDim.x)
    dst[a.bytes + i] = static_cast<const unsigned char*>(b.src)[i];
  for (size_t i = threadIdx.x; i < e.bytes; i += blockDim.x)
    dst[a.bytes + b.bytes + i] = static_cast<const unsigned char*>(e.src)[i];
}

hrg_status readback(hrg_context* c, const void* src_a, size_t na, void* dst_a,
                    const void* src_b = nullptr, size_t nb = 0, void* dst_b = nullptr,
                    const void* src_e = nullptr, size_t ne = 0, void* dst_e = nullptr) {
  ++c->launches, k_readback<<<1, 128, 0, c->stream>>>(RbItem{src_a, na}, RbItem{src_b, nb}, RbItem{src_e, ne},
                                       c->d_rb);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  memcpy(dst_a, c->h_rb, na);
  if (nb) memcpy(dst_b, c->h_rb + na, nb);
  if (ne) memcpy(dst_e, c->h_rb + na + nb, ne);
  return HRG_OK;
}

double ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Sort keys -> permutation; build the sorted SoA, band table and directory.
hrg_status build_index(hrg_context* c, const hrg_model* M, const BandSpec& S, int L,
                       const hrg_shard* shard, double C, bool sample_ids) {
  const int64_t n = c->np;  // indexed points (all, or a sharded run's subset)
  cudaStream_t st = c->stream;
  size_t tb = 0;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, c->k32_in.as<uint32_t>(),
                                           c->k32_out.as<uint32_t>(), c->vals_in.as<int32_t>(),
                                           c->vals_out.as<int32_t>(), (int)n, 0, 32, st));
  CUDA_TRY(c->temp.ensure(tb));
  tb = c->temp.bytes;
  CUDA_TRY(cub::DeviceRadixSort::SortPairs(c->temp.p, tb, c->k32_in.as<uint32_t>(),
                                           c->k32_out.as<uint32_t>(), c->vals_in.as<int32_t>(),
                                           c->vals_out.as<int32_t>(), (int)n, 0, 32, st));
  CUDA_TRY(cudaEventRecord(c->ev[E_SORTED], st));
  QRec q{c->s_phi.as<double>()};
  const Recs recs{c->pt.as<double2>(), c->circ.as<Circ>(),
                  c->vals_out.as<int32_t>()};
  CUDA_TRY(c->band_pmin.ensure(8 * kMaxBands));
  unsigned long long* band_pmin = c->band_pmin.as<unsigned long long>();
  CUDA_TRY(cudaMemsetAsync(band_pmin, 0xff, 8 * kMaxBands, st));
  if (sample_ids)
    ++c->launches, k_gather<true><<<blocks_for(n), 256, 0, st>>>(
        n, c->vals_out.as<int32_t>(), c->k32_out.as<uint32_t>(), c->keys_out.as<uint64_t>(), C,
        c->pr.as<double2>(), c->rn.as<double>(), M->cosh_r_minus_1, recs, q, nullptr,
        nullptr, c->sh_sampled ? c->sh_gid.as<int32_t>() : nullptr, c->vals_out.as<int32_t>(),
        band_pmin, c->trig);
  else
    ++c->launches, k_gather<false><<<blocks_for(n), 256, 0, st>>>(
        n, c->vals_out.as<int32_t>(), c->k32_out.as<uint32_t>(), c->keys_out.as<uint64_t>(), C,
        c->pr.as<double2>(), c->rn.as<double>(), M->cosh_r_minus_1, recs, q, c->s_rp.as<double>(),
        c->s_rn.as<double>(), nullptr, nullptr, band_pmin, c->trig);
  uint64_t qlo = 0, qhi = (uint64_t)1 << kQBits;
  if (shard && shard->count > 1) {
    // sector bounds on the sort granularity (multiples of 2^kSortShift)
    const uint64_t span = (uint64_t)1 << (kQBits - kSortShift);
    qlo = ((uint64_t)shard->index * span + (uint64_t)shard->count - 1) / (uint64_t)shard->count;
    qhi = ((uint64_t)(shard->index + 1) * span + (uint64_t)shard->count - 1) /
          (uint64_t)shard->count;
    if (shard->index + 1 == shard->count) qhi = span;
    qlo <<= kSortShift;
    qhi <<= kSortShift;
  }
  ++c->launches, k_band_setup<<<1, 1024, 0, st>>>(c->keys_out.as<uint64_t>(), n, L, qlo, qhi, c->bands.as<Band>(),
                                 c->dir_total.as<int64_t>(), c->np < M->n ? c->sh_cover : nullptr,
                                 band_pmin);
  CUDA_TRY(c->dir_gaps.ensure(sizeof(DirGap) * (size_t)(n / 16 + 2 * kMaxBands + 8)));
  unsigned* ngaps = reinterpret_cast<unsigned*>(c->dir_total.as<char>() + 8);
  CUDA_TRY(cudaMemsetAsync(ngaps, 0, 4, st));
  ++c->launches, k_dir_fill<<<blocks_for(n), 256, 0, st>>>(n, c->keys_out.as<uint64_t>(), c->bands.as<Band>(),
                                            c->dir.as<int32_t>(), c->dir_gaps.as<DirGap>(), ngaps);
  const bool sharded = c->np < M->n;
  const ShardRanges R{c->sh_lo, c->sh_hi, c->sh_mode};
  ++c->launches, k_dir_gaps<<<4 * c->sm_count, 256, 0, st>>>(c->dir_gaps.as<DirGap>(), ngaps,
                                              c->bands.as<Band>(), c->dir.as<int32_t>(), R,
                                              sharded);
  ++c->launches, k_dir_tail<<<L, 256, 0, st>>>(c->keys_out.as<uint64_t>(), c->bands.as<Band>(),
                                c->dir.as<int32_t>(), R, sharded);
  CUDA_TRY(cudaGetLastError());
  return HRG_OK;
}

template <class K>
int occupancy_grid(hrg_context* c, K kernel, int threads = 256, size_t smem = 0) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem);
  return std::max(1, nb) * c->sm_count;
}

// inclusive scan of int32 in[0..n) into out[1..n], out[0] = 0 (int64)
hrg_status scan_i32_to_i64(hrg_context* c, const int32_t* in, int64_t* out, int64_t n) {
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemsetAsync(out, 0, 8, st));
  if (n == 0) return HRG_OK;
  auto it = thrust::make_transform_iterator(in, ToI64());
  size_t tb = 0;
  CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tb, it, (long long*)out + 1, (int)n, st));
  CUDA_TRY(c->temp.ensure(tb));
  tb = c->temp.bytes;
  CUDA_TRY(cub::DeviceScan::InclusiveSum(c->temp.p, tb, it, (long long*)out + 1, (int)n, st));
  return HRG_OK;
}

// Light query pass, heavy (hub) pass, scans, compaction (+ row sort when ids
// are not positions).
hrg_status emit_edges(hrg_context* c, const hrg_model* M, int L, double C, bool sample_ids,
                      bool compact, int shard_count, hrg_stats* stats) {
  const int64_t n = M->n;   // vertex ids (rows)
  const int64_t np = c->np; // indexed positions
  cudaStream_t st = c->stream;
  QueryArgs A;
  memset(&A, 0, sizeof(A));
  A.rec = Recs{c->pt.as<double2>(), c->circ.as<Circ>(),
                c->vals_out.as<int32_t>()};
  A.q = QRec{c->s_phi.as<double>()};
  A.a = M->cosh_r_minus_1;
  // one warp walks a whole tile, so a tile of 32 queries at the limit bounds
  // the light pass from below (~0.35 ms at 2048): sharded runs, whose light
  // pass is that short, defer earlier (the heavy pass spreads a query's
  // chunks over the machine)
  A.light_max = kLightMax;
  if (shard_count > 1) A.light_max = std::min(kLightMax, std::max(512, 2 * kLightMax / shard_count));
  if (const char* e = getenv("HRG_LIGHT_MAX")) A.light_max = std::min(kLightMax, std::max(32, atoi(e)));
  A.bands = c->bands.as<Band>();
  A.dir = c->dir.as<int32_t>();
  A.keys = c->keys_out.as<uint64_t>();
  A.L = L;
  A.C = C;
  A.bump = c->counters.as<unsigned long long>();
  A.cand_total = c->counters.as<unsigned long long>() + 1;
  A.tile_next = c->counters.as<unsigned long long>() + 11;
  A.heavy_n = reinterpret_cast<unsigned*>(c->counters.as<unsigned long long>() + 2);
  A.overflow = reinterpret_cast<int*>(c->counters.as<unsigned long long>() + 3);
  A.stage_off = c->stage_off.as<int64_t>();
  A.slots = c->slots.as<int32_t>();
  A.heavy_v = c->heavy_v.as<int32_t>();
  A.heavy_c = c->heavy_c.as<int32_t>();
  A.heavy_of = c->heavy_of.as<int32_t>();
  A.deg = c->deg.as<int32_t>();
  A.rowidx = nullptr;
  // sharded runs: compact rows, one per query of the sector in position
  // order (the n-row CSR of the API is assembled on request); the row
  // count is bounded by the indexed points
  const int64_t nrows = compact ? np : n;
  int64_t* rowbuf = c->rowptr.as<int64_t>();
  if (compact) {
    CUDA_TRY(c->rowidx.ensure(4 * (size_t)np));
    CUDA_TRY(c->row_ids.ensure(4 * (size_t)np));
    CUDA_TRY(c->rowptr_c.ensure(8 * (size_t)(np + 1)));
    CUDA_TRY(c->nq_buf.ensure(8));
    ++c->launches, k_rowidx<<<4 * c->sm_count, 256, 0, st>>>(A.bands, L, c->vals_out.as<int32_t>(),
                                              c->rowidx.as<int32_t>(), c->row_ids.as<int32_t>(),
                                              c->nq_buf.as<int64_t>());
    A.rowidx = c->rowidx.as<int32_t>();
    rowbuf = c->rowptr_c.as<int64_t>();
  }

  // window table: one row per 1/16 of query radius, one column per band.
  // 2^-45 bounds the absolute fp64 error of dx*dx+dy*dy and rad^2 (all
  // operands <= 1 in magnitude); see DESIGN.md "window padding".
  const int rows = (int)std::ceil(M->R / (double)kRowStep) + 2;
  CUDA_TRY(c->wtab.ensure(2 * sizeof(float) * (size_t)rows * L));
  A.wtab = c->wtab.as<float>();
  A.wtab_q = reinterpret_cast<const uint32_t*>(A.wtab + (size_t)rows * L);
  A.wrows = rows;
  ++c->launches, k_window_table<<<rows, 32, 0, st>>>(
      A.bands, L, rows, M->cosh_r_minus_1, std::ldexp(1.0, -45), c->wtab.as<float>(),
      reinterpret_cast<uint32_t*>(c->wtab.as<float>() + (size_t)rows * L));

  // query tiles: 32 consecutive positions of one band; inner bands in band
  // order, the outermost kTileMixBands interleaved by angle (k_tile_table)
  {
    const int64_t ntmax = np / 32 + L + 1;
    CUDA_TRY(c->tv0.ensure(8 * (size_t)ntmax));
    int first_mixed = std::max(0, L - kTileMixBands);
    if (const char* e = getenv("HRG_TILE_MIX")) first_mixed = std::max(0, L - atoi(e));
    ++c->launches, k_tile_table<<<(unsigned)std::min<int64_t>(blocks_for(ntmax), 4 * c->sm_count), 256, 0, st>>>(
        A.bands, L, ntmax, c->tv0.as<uint64_t>(), first_mixed);
    A.tiles = c->tv0.as<uint64_t>();
    A.ntiles = ntmax;
  }

  if (c->grid_light == 0) {
#ifdef HRG_LIGHT_CARVEOUT
    for (auto kern : {k_light<true, kSegCap, HRG_LIGHT_MINBLOCKS>,
                      k_light<false, kSegCap, HRG_LIGHT_MINBLOCKS>})
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    HRG_LIGHT_CARVEOUT));
#endif
    c->grid_light = occupancy_grid(c, k_light<true, kSegCap, HRG_LIGHT_MINBLOCKS>, kLightThreads);
    c->grid_light_wide = occupancy_grid(c, k_light<true, kSegCapWide, kWideMinBlocks>, kLightThreads);
    c->grid_heavy = occupancy_grid(c, k_heavy<true>);
    c->grid_compact_heavy = occupancy_grid(c, k_compact_heavy);
#ifdef HRG_COMPACT_CARVEOUT
    for (auto kern : {k_compact_light<true>, k_compact_light<false>})
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    HRG_COMPACT_CARVEOUT));
#endif
    c->grid_compact = occupancy_grid(c, k_compact_light<true>, kCompactThreads);
    c->grid_block_count = occupancy_grid(c, k_block<true, false>, kBlockThreads);
    c->grid_block_write = occupancy_grid(c, k_block<true, true>, kBlockThreads);
    CUDA_TRY(cudaFuncSetAttribute(k_sort_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSortWarpSmem));
    CUDA_TRY(cudaFuncSetAttribute(k_sort_rows<256, kBucketMax, kMidShift>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sort_rows_smem<kBucketMax, kMidShift>()));
    CUDA_TRY(cudaFuncSetAttribute(k_sort_rows<1024, kLargeMax, 2>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sort_rows_smem<kLargeMax, 2>()));
  }
  // range query: the per-query window walk (k_light + staging + compaction;
  // the default) or dense blocks (HRG_QUERY=block: count pass + write pass
  // straight into the CSR, hrg_block.cuh -- measured slower)
  bool block = false;
  if (const char* e = getenv("HRG_QUERY")) block = strcmp(e, "block") == 0;
  // segment slots per light query: the wide variant when most of the 32
  // bands hold points (expected >= 1 point per band, from the radial CDF
  // (cosh(alpha r) - 1) / (cosh(alpha R) - 1)), so light queries reach them all
  bool wide = false;
  {
    int populated = 0;
    const double den = std::cosh(M->alpha * M->R) - 1.0;
    for (int j = 0; j < L; ++j) {
      const double f0 = (std::cosh(M->alpha * M->R * j / L) - 1.0) / den;
      const double f1 = (std::cosh(M->alpha * M->R * (j + 1) / L) - 1.0) / den;
      populated += (double)n * (f1 - f0) >= 1.0;
    }
    wide = populated >= kWideBands;
    if (const char* e = getenv("HRG_LIGHT_WIDE")) wide = atoi(e) != 0;
  }
  unsigned gq = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(blocks_for(np, kLightThreads),
                           wide ? c->grid_light_wide : c->grid_light));
  unsigned gc = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>(blocks_for(np, kCompactThreads), c->grid_compact));
  // staging capacity: the previous call's use on this context, else a
  // generous estimate.  Everything after the light pass runs without a host
  // round trip (buffers sized by upper bounds, counts read on the device);
  // one synchronisation at the end checks for a staging overflow, in which
  // case the pass is re-run with the capacity the bump allocator reached.
  if (c->stage_cap == 0) {
    // first call on this context: the model's expected degree (hrgen
    // geometry.py:170-190, power-law regime) with 30% headroom, so dense
    // graphs do not void their first pass
    int64_t cap = std::max<int64_t>(64 * np, 1 << 20);
    if (M->alpha > 0.5) {
      double kexp = 0.0;
      if (hrg_expected_avg_degree(M->n, M->alpha, M->R, &kexp) == HRG_OK && std::isfinite(kexp) &&
          kexp > 0.0)
        cap = std::max<int64_t>(cap, (int64_t)(1.3 * kexp * (double)np) + (1 << 20));
    }
    c->stage_cap = cap;
  }
  unsigned long long ctr[16];
  int64_t nnz = 0, total_chunks = 0;
  for (int attempt = 0; attempt < 3; ++attempt) {
    const int64_t cap = c->stage_cap;  // also bounds hits, chunks, rows to sort
    CUDA_TRY(c->stage.ensure(4 * (size_t)cap + 64));  // + slack: the compaction's TMA copies
                                                       // round up to 16-byte boundaries
    A.stage = c->stage.as<int32_t>();
    A.stage_cap = cap;
    const int64_t hcap = np + 1;                     // deferred queries
    const int64_t ccap = cap / kChunk + np + 1;      // their chunks
    CUDA_TRY(c->nchunks.ensure(4 * (size_t)hcap));
    CUDA_TRY(c->chunk_start.ensure(8 * (size_t)(hcap + 1)));
    CUDA_TRY(c->chunk_hits.ensure(4 * (size_t)ccap));
    CUDA_TRY(c->chunk_entry.ensure(4 * (size_t)ccap));
    CUDA_TRY(c->chunk_off.ensure(8 * (size_t)(ccap + 1)));
    CUDA_TRY(c->idx.ensure(4 * (size_t)cap));
    unsigned long long* ctrs = c->counters.as<unsigned long long>();
    int64_t* d_chunks = reinterpret_cast<int64_t*>(ctrs + 14);  // 11, 12: tile counters
    A.chunk_start = c->chunk_start.as<int64_t>();
    A.chunk_entry = c->chunk_entry.as<int32_t>();
    A.chunk_hits = c->chunk_hits.as<int32_t>();
    A.total_chunks = d_chunks;

    CUDA_TRY(cudaMemsetAsync(c->deg.p, 0, sizeof(int32_t) * nrows, st));
    CUDA_TRY(cudaMemsetAsync(c->counters.p, 0, 128, st));
    CUDA_TRY(cudaEventRecord(c->ev[E_INDEXED], st));
    if (block) {
      // count pass of the block range query (hrg_block.cuh)
      const unsigned gbc = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>(blocks_for(np, kBlockThreads), c->grid_block_count));
      if (sample_ids)
        ++c->launches, k_block<true, false><<<gbc, kBlockThreads, 0, st>>>(A, rowbuf, nrows, nullptr, 0, SortJobs{});
      else
        ++c->launches, k_block<false, false><<<gbc, kBlockThreads, 0, st>>>(A, rowbuf, nrows, nullptr, 0, SortJobs{});
    } else {
      constexpr int MB = HRG_LIGHT_MINBLOCKS;
      if (sample_ids && !wide) ++c->launches, k_light<true, kSegCap, MB><<<gq, kLightThreads, 0, st>>>(A);
      else if (!wide) ++c->launches, k_light<false, kSegCap, MB><<<gq, kLightThreads, 0, st>>>(A);
      else if (sample_ids) ++c->launches, k_light<true, kSegCapWide, kWideMinBlocks><<<gq, kLightThreads, 0, st>>>(A);
      else ++c->launches, k_light<false, kSegCapWide, kWideMinBlocks><<<gq, kLightThreads, 0, st>>>(A);
    }
    CUDA_TRY(cudaEventRecord(c->ev[E_PLANNED], st));
    ++c->launches, k_heavy_prep<<<1, 1024, 0, st>>>(A.heavy_c, A.heavy_n, c->nchunks.as<int32_t>(),
                                     c->chunk_start.as<int64_t>(), c->chunk_entry.as<int32_t>(),
                                     d_chunks, A.overflow);
    if (sample_ids) ++c->launches, k_heavy<true><<<c->grid_heavy, 256, 0, st>>>(A, 0);
    else ++c->launches, k_heavy<false><<<c->grid_heavy, 256, 0, st>>>(A, 0);
    CUDA_TRY(cudaEventRecord(c->ev[E_COUNTED], st));
    CUDA_TRY(cudaGetLastError());
    hrg_status s = scan_i32_to_i64(c, c->deg.as<int32_t>(), rowbuf, nrows);
    if (s != HRG_OK) return s;

    int32_t* idx = c->idx.as<int32_t>();
    const int64_t* rp = rowbuf;
    // sort jobs (sample order): light rows above kSmallSlots ids, heavy rows
    const int64_t jcap = 2 * np + 1;
    const int64_t mcap = cap / (kWarpBucketMax + 1) + 1;
    const int64_t lcap = cap / (kBucketMax + 1) + 1;
    CUDA_TRY(c->job_dst.ensure(8 * (size_t)jcap));
    CUDA_TRY(c->job_len.ensure(4 * (size_t)jcap));
    CUDA_TRY(c->mid_off.ensure(8 * (size_t)mcap));
    CUDA_TRY(c->mid_len.ensure(4 * (size_t)mcap));
    CUDA_TRY(c->large_off.ensure(8 * (size_t)lcap));
    CUDA_TRY(c->large_len.ensure(4 * (size_t)lcap));
    const int64_t gcap = cap / (kLargeMax + 1) + 1;          // giant rows
    const int64_t bcap = cap / kGiantTarget + gcap + 1;      // their sub-buckets / chunks
    CUDA_TRY(c->giant_off.ensure(8 * (size_t)gcap));
    CUDA_TRY(c->giant_len.ensure(4 * (size_t)gcap));
    CUDA_TRY(c->giant_meta.ensure(4 * 3 * (size_t)gcap));
    CUDA_TRY(c->sub_off.ensure(8 * (size_t)bcap));
    CUDA_TRY(c->sub_len.ensure(4 * (size_t)bcap));
    CUDA_TRY(c->sub_cur.ensure(8 * (size_t)bcap));
    CUDA_TRY(c->chunk_row.ensure(4 * (size_t)bcap));
    SortJobs J;
    J.rows = RowList{c->job_dst.as<int64_t>(), c->job_len.as<int32_t>(),
                     reinterpret_cast<unsigned*>(ctrs + 4)};
    J.mid = RowList{c->mid_off.as<int64_t>(), c->mid_len.as<int32_t>(),
                    reinterpret_cast<unsigned*>(ctrs + 5)};
    unsigned* uctr = reinterpret_cast<unsigned*>(ctrs + 6);  // 4 more 32-bit counters
    J.large = RowList{c->large_off.as<int64_t>(), c->large_len.as<int32_t>(), uctr};
    Giant G;
    G.rows = RowList{c->giant_off.as<int64_t>(), c->giant_len.as<int32_t>(), uctr + 1};
    G.sub = RowList{c->sub_off.as<int64_t>(), c->sub_len.as<int32_t>(), uctr + 2};
    G.nchunks = uctr + 3;
    G.nb = c->giant_meta.as<int32_t>();
    G.bbase = G.nb + gcap;
    G.cbase = G.nb + 2 * gcap;
    G.chunk_row = c->chunk_row.as<int32_t>();
    G.cur = c->sub_cur.as<unsigned long long>();
    J.giant = G.rows;
    CUDA_TRY(cudaEventRecord(c->ev[E_WRITE0], st));
    if (block) {
      // write pass: rows straight into the CSR (light rows sorted on the way)
      const unsigned gbw = (unsigned)std::max<int64_t>(
          1, std::min<int64_t>(blocks_for(np, kBlockThreads), c->grid_block_write));
      if (sample_ids)
        ++c->launches, k_block<true, true><<<gbw, kBlockThreads, 0, st>>>(A, rp, nrows, idx, cap, J);
      else
        ++c->launches, k_block<false, true><<<gbw, kBlockThreads, 0, st>>>(A, rp, nrows, idx, cap, J);
    } else if (sample_ids) {
      ++c->launches, k_compact_light<true><<<gc, kCompactThreads, 0, st>>>(A, rp, idx, J);
    } else {
      ++c->launches, k_compact_light<false><<<gc, kCompactThreads, 0, st>>>(A, rp, idx, J);
    }
    ++c->launches, k_scan_chunks<<<1, 1024, 0, st>>>(c->chunk_hits.as<int32_t>(), d_chunks,
                                      c->chunk_off.as<int64_t>(), A.overflow);
    ++c->launches, k_compact_heavy<<<c->grid_compact_heavy, 256, 0, st>>>(A, 0, c->chunk_off.as<int64_t>(), rp, idx,
                                                   sample_ids);
    if (sample_ids) ++c->launches, k_queue_heavy_rows<<<2 * c->sm_count, 256, 0, st>>>(A, rp, J);
    CUDA_TRY(cudaEventRecord(c->ev[E_WRITTEN], st));
    c->idx_final = idx;
    if (sample_ids) {
      // rows by length: a warp (<= kWarpBucketMax), a 256-thread block
      // (<= kBucketMax), a 1024-thread block (<= kLargeMax); giant (hub) rows
      // are first split by value into sub-buckets through the scratch array
      // scratch of the giant-row split: the staging buffer, dead once the
      // compaction has run (saves a cap-sized buffer: 8 GB at n = 1e8)
      int32_t* scratch = c->stage.as<int32_t>();
      const RowList none{nullptr, nullptr, nullptr};
      const unsigned sm = (unsigned)c->sm_count;
      // the length classes are independent (rows were queued straight into
      // their class): warp rows on the context's stream, block rows and the
      // giant split on two side streams, joined before the readback
      cudaStream_t s1 = c->aux[0], s2 = c->aux[1];
      CUDA_TRY(cudaEventRecord(c->fork, st));
      CUDA_TRY(cudaStreamWaitEvent(s1, c->fork, 0));
      CUDA_TRY(cudaStreamWaitEvent(s2, c->fork, 0));
      ++c->launches, k_sort_warp<<<HRG_SORT_GRID * sm, kSortWarpThreads, kSortWarpSmem, st>>>(idx, J);
      ++c->launches, k_sort_rows<256, kBucketMax, kMidShift>
          <<<HRG_SORT_GRID * sm, 256, sort_rows_smem<kBucketMax, kMidShift>(), s1>>>(idx, idx, J.mid,
                                                                                J.large);
      ++c->launches, k_sort_rows<1024, kLargeMax, 2><<<sm, 1024, sort_rows_smem<kLargeMax, 2>(), s2>>>(
          idx, idx, J.large, G.rows);
      ++c->launches, k_giant_plan<<<1, 1024, 0, s2>>>(G);
      ++c->launches, k_giant_hist<<<2 * sm, 1024, 0, s2>>>(idx, G, n);
      ++c->launches, k_giant_scan<<<sm, 1024, 0, s2>>>(G);
      ++c->launches, k_giant_scatter<<<2 * sm, 1024, 0, s2>>>(idx, scratch, G, n);
      ++c->launches, k_sort_rows<1024, kLargeMax, 2><<<sm, 1024, sort_rows_smem<kLargeMax, 2>(), s2>>>(
          scratch, idx, G.sub, none);
      CUDA_TRY(cudaEventRecord(c->join[0], s1));
      CUDA_TRY(cudaEventRecord(c->join[1], s2));
      CUDA_TRY(cudaStreamWaitEvent(st, c->join[0], 0));
      CUDA_TRY(cudaStreamWaitEvent(st, c->join[1], 0));
    }
    CUDA_TRY(cudaEventRecord(c->ev[E_ROWSORTED], st));
    CUDA_TRY(cudaGetLastError());
    // the one synchronisation: counters, edge total, overflow flag
    {
      hrg_status rs = readback(c, c->counters.p, 128, ctr, rowbuf + nrows, 8, &nnz,
                               compact ? c->nq_buf.p : nullptr, compact ? 8 : 0, &c->nq);
      if (rs != HRG_OK) return rs;
    }
    total_chunks = (int64_t)ctr[14];
    if ((ctr[3] & 0xffffffffull) == 0) break;
    if (ctr[3] & 4) return fail(HRG_ERR_INTERNAL, "block query: write pass disagrees with count pass");
    // staging (or, block query, the CSR) overflowed: size it from the bump
    // allocator's final value / the CSR size
    {
      const int64_t need = std::max<int64_t>((int64_t)ctr[0], nnz);
      c->stage_cap = need + need / 8 + 4096;
    }
    if (attempt == 2) return fail(HRG_ERR_INTERNAL, "staging buffer overflow");
  }
  // next call: keep ~10% headroom over this call's staging use
  {
    const int64_t used = std::max<int64_t>((int64_t)ctr[0], nnz);
    c->stage_cap = std::max<int64_t>(c->stage_cap, used + used / 10 + 4096);
  }
  c->nnz = nnz;
  c->compact_result = compact;
  if (stats) {
    stats->nnz = nnz;
    stats->m = nnz / 2;
    stats->candidates = (int64_t)ctr[1];
    stats->heavy_queries = (int64_t)(ctr[2] & 0xffffffffull);
    stats->heavy_chunks = total_chunks;
  }
  return HRG_OK;
}

// Sharded runs (sample ids): index only the points some query of this
// rank's sector can reach -- per band, the sector widened by the widest
// window of any query radius present.  Keys and ids
// of the kept points are compacted in draw order, so the sort and everything
// after it see a smaller, identically ordered point set; ids stay global.
hrg_status shard_subset(hrg_context* c, const hrg_model* M, const BandSpec& S, int L,
                        const hrg_shard* shard) {
  const int64_t n = M->n;
  cudaStream_t st = c->stream;
  // smallest Poincare radius present (the widest windows)
  CUDA_TRY(c->sh_buf.ensure(1024));
  unsigned long long* d_min = reinterpret_cast<unsigned long long*>(c->sh_buf.p);
  CUDA_TRY(cudaMemsetAsync(d_min, 0xff, 8, st));
  ++c->launches, k_min_rp<<<4 * c->sm_count, 256, 0, st>>>(n, c->pr.as<double2>(), d_min);
  size_t tb = 0;
  // window table on bands whose innermost radius is their threshold
  std::vector<Band> tbands(L);
  for (int j = 0; j < L; ++j) {
    memset(&tbands[j], 0, sizeof(Band));
    tbands[j].start = 0;
    tbands[j].end = 1;
    tbands[j].pmin = j == 0 ? 0.0 : S.thr[j];
  }
  const int rows = (int)std::ceil(M->R / (double)kRowStep) + 2;
  CUDA_TRY(c->sh_bands.ensure(sizeof(Band) * L));
  CUDA_TRY(c->sh_wtab.ensure(sizeof(float) * (size_t)rows * L));
  CUDA_TRY(cudaMemcpyAsync(c->sh_bands.p, tbands.data(), sizeof(Band) * L,
                           cudaMemcpyHostToDevice, st));
  ++c->launches, k_window_table<<<rows, 32, 0, st>>>(c->sh_bands.as<Band>(), L, rows, M->cosh_r_minus_1,
                                      std::ldexp(1.0, -45), c->sh_wtab.as<float>());
  const int64_t span = (int64_t)1 << 27;
  const int64_t sec_lo = ((int64_t)shard->index * span + shard->count - 1) / shard->count;
  const int64_t sec_hi = shard->index + 1 == shard->count
                             ? span
                             : ((int64_t)(shard->index + 1) * span + shard->count - 1) /
                                   shard->count;
  int64_t* lo = reinterpret_cast<int64_t*>(c->sh_buf.as<char>() + 64);
  int64_t* hi = lo + kMaxBands;
  int* mode = reinterpret_cast<int*>(hi + kMaxBands);
  float* cover = reinterpret_cast<float*>(mode + kMaxBands);
  ++c->launches, k_shard_ranges<<<1, 1024, 0, st>>>(c->sh_wtab.as<float>(), L, rows, d_min, sec_lo, sec_hi, lo,
                                   hi, mode, cover);
  c->sh_cover = cover;
  c->sh_lo = lo;
  c->sh_hi = hi;
  c->sh_mode = mode;
  // directories sized for density (k_band_setup): up to ~4x the global count
  CUDA_TRY(c->dir.ensure(4 * (size_t)((4 * n << kDirExtra) + 2 * kMaxBands + 64)));
  CUDA_TRY(c->sh_keep.ensure((size_t)n));
  ++c->launches, k_shard_flags<<<blocks_for(n), 256, 0, st>>>(n, c->k32_in.as<uint32_t>(), lo, hi, mode,
                                               c->sh_keep.as<uint8_t>());
  // order-preserving compaction of (key, id) into the sort's output buffers,
  // then back
  int* d_cnt = reinterpret_cast<int*>(c->sh_buf.as<char>() + 960);
  tb = 0;
  CUDA_TRY(cub::DeviceSelect::Flagged(nullptr, tb, c->k32_in.as<uint32_t>(),
                                      c->sh_keep.as<uint8_t>(), c->k32_out.as<uint32_t>(), d_cnt,
                                      (int)n, st));
  CUDA_TRY(c->temp.ensure(tb));
  tb = c->temp.bytes;
  CUDA_TRY(cub::DeviceSelect::Flagged(c->temp.p, tb, c->k32_in.as<uint32_t>(),
                                      c->sh_keep.as<uint8_t>(), c->k32_out.as<uint32_t>(), d_cnt,
                                      (int)n, st));
  tb = c->temp.bytes;
  CUDA_TRY(cub::DeviceSelect::Flagged(c->temp.p, tb, c->vals_in.as<int32_t>(),
                                      c->sh_keep.as<uint8_t>(), c->vals_out.as<int32_t>(), d_cnt,
                                      (int)n, st));
  int np = 0;
  {
    hrg_status rs = readback(c, d_cnt, 4, &np);
    if (rs != HRG_OK) return rs;
  }
  CUDA_TRY(cudaMemcpyAsync(c->k32_in.p, c->k32_out.p, 4 * (size_t)np, cudaMemcpyDeviceToDevice,
                           st));
  CUDA_TRY(cudaMemcpyAsync(c->vals_in.p, c->vals_out.p, 4 * (size_t)np, cudaMemcpyDeviceToDevice,
                           st));
  c->np = np;
  return HRG_OK;
}

// Sharded runs sampling their own points (sample ids): the sector's
// smallest radius, the reachable range of every band, then one sampling
// pass that keeps (and evaluates the radius of) only the reachable points
// (DESIGN.md "Multi-GPU").  Replaces k_sample + shard_subset.
hrg_status shard_sample(hrg_context* c, const hrg_model* M, int L, const hrg_shard* shard,
                        const SampleParams& P) {
  const int64_t n = M->n;
  cudaStream_t st = c->stream;
  ShardSample S;
  memset(&S, 0, sizeof(S));
  S.L = L;
  // band thresholds on the radial uniform: the inverse CDF at r_j = R j / L
  // (any increasing sequence is correct; this one matches the radial bands)
  const double two53 = std::ldexp(1.0, 53);
  for (int j = 1; j < L; ++j) {
    const double rj = M->R * j / L;
    const double u = std::pow(std::sinh(M->alpha * rj / 2.0) / M->sinh_half_alpha_r, 2.0);
    double b = std::ceil(u * two53);
    if (!(b < two53)) b = two53;
    S.ub[j] = std::max<uint64_t>((uint64_t)b, S.ub[j - 1] + 1);
  }
  const int64_t span = (int64_t)1 << 27;
  S.sec_lo = ((int64_t)shard->index * span + shard->count - 1) / shard->count;
  S.sec_hi = shard->index + 1 == shard->count
                 ? span
                 : ((int64_t)(shard->index + 1) * span + shard->count - 1) / shard->count;
  CUDA_TRY(c->sh_buf.ensure(1024));
  unsigned long long* d_umin = reinterpret_cast<unsigned long long*>(c->sh_buf.p);
  unsigned long long* d_pmin = d_umin + 1;
  unsigned* d_cnt = reinterpret_cast<unsigned*>(c->sh_buf.as<char>() + 960);
  CUDA_TRY(cudaMemsetAsync(d_umin, 0xff, 8, st));
  CUDA_TRY(cudaMemsetAsync(d_cnt, 0, 4, st));
  ++c->launches, k_shard_keys<<<8 * c->sm_count, 256, 0, st>>>(n, P, S, c->k32_out.as<uint32_t>(), d_umin);
  const int rows = (int)std::ceil(M->R / (double)kRowStep) + 2;
  CUDA_TRY(c->sh_bands.ensure(sizeof(Band) * L));
  CUDA_TRY(c->sh_wtab.ensure(sizeof(float) * (size_t)rows * L));
  ++c->launches, k_shard_prep<<<1, 32, 0, st>>>(P, S, d_umin, c->sh_bands.as<Band>(), d_pmin);
  ++c->launches, k_window_table<<<rows, 32, 0, st>>>(c->sh_bands.as<Band>(), L, rows, M->cosh_r_minus_1,
                                      std::ldexp(1.0, -45), c->sh_wtab.as<float>());
  int64_t* lo = reinterpret_cast<int64_t*>(c->sh_buf.as<char>() + 64);
  int64_t* hi = lo + kMaxBands;
  int* mode = reinterpret_cast<int*>(hi + kMaxBands);
  float* cover = reinterpret_cast<float*>(mode + kMaxBands);
  ++c->launches, k_shard_ranges<<<1, 1024, 0, st>>>(c->sh_wtab.as<float>(), L, rows, d_pmin, S.sec_lo, S.sec_hi,
                                   lo, hi, mode, cover);
  c->sh_cover = cover;
  c->sh_lo = lo;
  c->sh_hi = hi;
  c->sh_mode = mode;
  CUDA_TRY(c->dir.ensure(4 * (size_t)((4 * n << kDirExtra) + 2 * kMaxBands + 64)));
  CUDA_TRY(c->sh_gid.ensure(4 * (size_t)n));
  ++c->launches, k_shard_select<<<blocks_for(n, 256 * kShardPer), 256, 0, st>>>(
      n, L, c->k32_out.as<uint32_t>(), lo, hi, mode, c->k32_in.as<uint32_t>(),
      c->vals_in.as<int32_t>(), c->sh_gid.as<int32_t>(), d_cnt);
  ++c->launches, k_shard_points<<<8 * c->sm_count, 256, 0, st>>>(P, d_cnt, c->sh_gid.as<int32_t>(),
                                                  c->pr.as<double2>());
  CUDA_TRY(cudaGetLastError());
  unsigned np = 0;
  {
    hrg_status rs = readback(c, d_cnt, 4, &np);
    if (rs != HRG_OK) return rs;
  }
  c->np = np;
  c->sh_sampled = true;
  return HRG_OK;
}

hrg_status run_pipeline(hrg_context* c, const hrg_model* M, const hrg_shard* shard,
                        bool sample_ids, bool from_coords, uint64_t seed, hrg_stats* stats) {
  int64_t n = M->n;
  cudaStream_t st = c->stream;
  int L = 0;
  BandSpec S = make_bands(M->R, &L);
  double C = std::ldexp(1.0, kQBits) / kTwoPi;
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->n = n;
    stats->radius = M->R;
    stats->alpha = M->alpha;
    stats->n_bands = L;
  }
  const int64_t launches0 = c->launches;
  CUDA_TRY(cudaEventRecord(c->ev[E_START], st));
  c->sh_sampled = false;
  const bool shard_sampling = !from_coords && shard && shard->count > 1 && sample_ids;
  if (shard_sampling) {
    SampleParams P{seed, M->two_over_alpha, M->sinh_half_alpha_r, M->r_cap, M->rp_cap, C};
    hrg_status s0 = shard_sample(c, M, L, shard, P);
    if (s0 != HRG_OK) return s0;
    c->coords_pending = true;
    c->pending = P;
  } else if (!from_coords) {
    SampleParams P{seed, M->two_over_alpha, M->sinh_half_alpha_r, M->r_cap, M->rp_cap, C};
    // coordinates on request only (hrg_result_device_ptrs); angular order
    // gathers r_native into its sorted copy, so that one is written
    ++c->launches, k_sample<<<blocks_for(n), 256, 0, st>>>(n, P, S, nullptr,
                                            sample_ids ? nullptr : c->rn.as<double>(), nullptr,
                                            c->k32_in.as<uint32_t>(), c->vals_in.as<int32_t>(),
                                            c->pr.as<double2>());
    c->coords_pending = sample_ids;
    c->pending = P;
  } else {
    c->coords_pending = false;
    CUDA_TRY(cudaMemsetAsync(c->bad.p, 0, 4, st));
    ++c->launches, k_keys_from_coords<<<blocks_for(n), 256, 0, st>>>(
        n, c->phi.as<double>(), c->rp.as<double>(), M->max_r, C, S, c->rn.as<double>(),
        c->k32_in.as<uint32_t>(), c->vals_in.as<int32_t>(), c->bad.as<int>(),
        c->pr.as<double2>());
    int bad = 0;
    hrg_status rs = readback(c, c->bad.p, 4, &bad);
    if (rs != HRG_OK) return rs;
    if (bad) return fail(HRG_ERR_OUT_OF_BOUNDS, "point outside the tree region");
  }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaEventRecord(c->ev[E_SAMPLED], st));
  if (!shard_sampling) c->np = n;
  hrg_status s = HRG_OK;
  if (!shard_sampling && shard && shard->count > 1 && sample_ids) {
    s = shard_subset(c, M, S, L, shard);
    if (s != HRG_OK) return s;
  }
  s = build_index(c, M, S, L, shard, C, sample_ids);
  if (s != HRG_OK) return s;
  s = emit_edges(c, M, L, C, sample_ids, shard && shard->count > 1 && sample_ids,
                 shard ? shard->count : 1, stats);
  if (s != HRG_OK) return s;
  CUDA_TRY(cudaStreamSynchronize(st));
  c->n = n;
  c->have_result = true;
  c->coords_sorted = !sample_ids;
  if (stats) {
    stats->t_sample_ms = ev_ms(c->ev[E_START], c->ev[E_SAMPLED]);
    stats->t_build_ms = ev_ms(c->ev[E_SAMPLED], c->ev[E_INDEXED]);
    stats->t_edges_ms = ev_ms(c->ev[E_INDEXED], c->ev[E_ROWSORTED]);
    stats->t_sort_ms = ev_ms(c->ev[E_SAMPLED], c->ev[E_SORTED]);
    stats->t_light_ms = ev_ms(c->ev[E_INDEXED], c->ev[E_PLANNED]);
    stats->t_heavy_ms = ev_ms(c->ev[E_PLANNED], c->ev[E_COUNTED]);
    stats->t_compact_ms = ev_ms(c->ev[E_WRITE0], c->ev[E_WRITTEN]);
    stats->t_rowsort_ms = ev_ms(c->ev[E_WRITTEN], c->ev[E_ROWSORTED]);
    stats->kernel_launches = (int32_t)(c->launches - launches0);
  }
  return HRG_OK;
}

// Sharded result: compact rows -> the n-row CSR of the API, once, on request.
hrg_status expand_rows(hrg_context* c) {
  if (!c->compact_result) return HRG_OK;
  cudaStream_t st = c->stream;
  const int64_t n = c->n;
  CUDA_TRY(cudaMemsetAsync(c->deg.p, 0, sizeof(int32_t) * n, st));
  ++c->launches, k_expand_deg<<<4 * c->sm_count, 256, 0, st>>>(c->nq, c->rowptr_c.as<int64_t>(),
                                                c->row_ids.as<int32_t>(), c->deg.as<int32_t>());
  hrg_status s = scan_i32_to_i64(c, c->deg.as<int32_t>(), c->rowptr.as<int64_t>(), n);
  if (s != HRG_OK) return s;
  // the compact rows are in idx (the compaction's output); the staging
  // buffer (>= nnz ids: every hit had a staging slot) is dead by now and
  // takes the expanded rows
  if (c->stage.bytes < 4 * (size_t)std::max<int64_t>(c->nnz, 1))
    return fail(HRG_ERR_INTERNAL, "staging smaller than the result");
  int32_t* out = c->stage.as<int32_t>();
  ++c->launches, k_expand_rows<<<8 * c->sm_count, 256, 0, st>>>(c->nq, c->rowptr_c.as<int64_t>(),
                                                 c->row_ids.as<int32_t>(), c->idx_final,
                                                 c->rowptr.as<int64_t>(), out);
  CUDA_TRY(cudaGetLastError());
  c->idx_final = out;
  c->compact_result = false;
  return HRG_OK;
}

}  // namespace

extern "C" {

const char* hrg_version(void) { return "hrgen_b200 1 (sm_100a)"; }
const char* hrg_last_error(void) { return g_err.c_str(); }

hrg_status hrg_context_create(int device, void* cuda_stream, hrg_context** out) {
  if (!out) return fail(HRG_ERR_PARAMETER_DOMAIN, "out is NULL");
  CUDA_TRY(cudaSetDevice(device));
  hrg_context* c = new hrg_context();
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  for (auto& e : c->ev) {
    cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) { delete c; return fail(HRG_ERR_CUDA, cudaGetErrorString(r)); }
  }
  {
    cudaError_t r = cudaHostAlloc(reinterpret_cast<void**>(&c->h_rb), kReadback,
                                  cudaHostAllocMapped);
    if (r == cudaSuccess)
      r = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->d_rb), c->h_rb, 0);
    if (r != cudaSuccess) { delete c; return fail(HRG_ERR_CUDA, cudaGetErrorString(r)); }
  }
  {
    cudaError_t r = cudaSuccess;
    for (auto& a : c->aux)
      if (r == cudaSuccess) r = cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    if (r == cudaSuccess) r = cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming);
    for (auto& e : c->join)
      if (r == cudaSuccess) r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) { delete c; return fail(HRG_ERR_CUDA, cudaGetErrorString(r)); }
  }
  // the sin/cos table of the fast path (device-global, idempotent)
  ++c->launches, k_sincos_table<<<1, 256, 0, c->stream>>>();
  cudaError_t r = cudaStreamSynchronize(c->stream);
  if (r == cudaSuccess) r = cudaGetLastError();
  if (r != cudaSuccess) { delete c; return fail(HRG_ERR_CUDA, cudaGetErrorString(r)); }
  *out = c;
  return HRG_OK;
}

hrg_status hrg_context_destroy(hrg_context* c) {
  if (!c) return HRG_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (Buf* b : {&c->phi, &c->rn, &c->rp, &c->keys_out, &c->vals_in, &c->vals_out,
                 &c->pt, &c->circ, &c->s_phi, &c->s_rp, &c->s_rn, &c->pr, &c->stage,
                 &c->stage_off, &c->counters, &c->heavy_v, &c->heavy_c, &c->heavy_of,
                 &c->nchunks, &c->chunk_start, &c->chunk_hits, &c->chunk_entry, &c->chunk_off,
                 &c->slots,
                 &c->large_off, &c->large_len, &c->giant_off, &c->giant_len, &c->giant_meta, &c->sub_off, &c->sub_len, &c->sub_cur,
                 &c->chunk_row, &c->tv0, &c->wtab, &c->job_dst, &c->job_len,
                 &c->mid_off, &c->mid_len, &c->bands, &c->dir, &c->dir_total, &c->bad, &c->dir_gaps, &c->band_pmin,
                 &c->deg, &c->rowptr, &c->idx, &c->cand, &c->rowidx, &c->row_ids, &c->rowptr_c, &c->nq_buf, &c->temp, &c->k32_in, &c->k32_out, &c->sh_buf, &c->sh_bands, &c->sh_wtab, &c->sh_keep, &c->sh_gid,
                 &c->widen, &c->pack})
    b->release();
  if (c->h_rb) cudaFreeHost(c->h_rb);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (auto e : c->h_ev) cudaEventDestroy(e);
  for (auto a : c->aux)
    if (a) cudaStreamDestroy(a);
  if (c->fork) cudaEventDestroy(c->fork);
  for (auto e : c->join)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev) if (e) cudaEventDestroy(e);
  delete c;
  return HRG_OK;
}

hrg_status hrg_context_set_stream(hrg_context* c, void* s) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  c->stream = (cudaStream_t)s;
  return HRG_OK;
}

hrg_status hrg_context_launches(hrg_context* c, int64_t* out) {
  if (!c || !out) return fail(HRG_ERR_PARAMETER_DOMAIN, "bad arguments");
  *out = c->launches;
  return HRG_OK;
}

hrg_status hrg_context_set_trig(hrg_context* c, int mode) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  if (mode != HRG_TRIG_LIBM && mode != HRG_TRIG_CR)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "trig mode must be HRG_TRIG_LIBM or HRG_TRIG_CR");
  c->trig = mode;
  return HRG_OK;
}

hrg_status hrg_expected_avg_degree(int64_t n, double alpha, double radius, double* out) {
  // hrgen geometry.py:170-190
  if (!(alpha > 0.5)) return fail(HRG_ERR_PARAMETER_DOMAIN, "alpha must be > 0.5");
  if (!(radius > 0.0)) return fail(HRG_ERR_PARAMETER_DOMAIN, "radius must be > 0");
  if (n < 1) return fail(HRG_ERR_PARAMETER_DOMAIN, "n must be >= 1");
  const double pi = 3.141592653589793;
  double xi = alpha / (alpha - 0.5);
  double inner = alpha * (radius / 2.0) *
                     ((pi / 4.0) / (alpha * alpha) - (pi - 1.0) / alpha + (pi - 2.0)) - 1.0;
  *out = (2.0 / pi) * xi * xi * (double)n *
         (std::exp(-radius / 2.0) + std::exp(-alpha * radius) * inner);
  return HRG_OK;
}

hrg_status hrg_target_radius(int64_t n, double k, double alpha, double rel_tol, double* out) {
  // hrgen geometry.py:197-232 (geometric grid, peak, bisection on the decaying branch)
  if (!(alpha > 0.5)) return fail(HRG_ERR_PARAMETER_DOMAIN, "alpha must be > 0.5");
  if (!(k > 0.0 && k < (double)(n - 1)))
    return fail(HRG_ERR_PARAMETER_DOMAIN, "target average degree must be in (0, n-1)");
  const double lo_r = 1e-6, hi_r = 200.0;
  double best = -INFINITY, lo = lo_r;
  for (int i = 0; i < 512; ++i) {
    double r = std::pow(10.0, std::log10(lo_r) + (std::log10(hi_r) - std::log10(lo_r)) * i / 511.0);
    if (i == 0) r = lo_r;
    if (i == 511) r = hi_r;
    double v;
    hrg_expected_avg_degree(n, alpha, r, &v);
    if (v > best) { best = v; lo = r; }
  }
  double hi = hi_r, vhi;
  hrg_expected_avg_degree(n, alpha, hi, &vhi);
  if (best < k || vhi > k) return fail(HRG_ERR_INFEASIBLE, "no radius yields that average degree");
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi), v;
    hrg_expected_avg_degree(n, alpha, mid, &v);
    if (std::fabs(v - k) <= rel_tol * k) { *out = mid; return HRG_OK; }
    if (v > k) lo = mid; else hi = mid;
  }
  return fail(HRG_ERR_INFEASIBLE, "bisection failed to reach tolerance");
}

hrg_status hrg_model_init(int64_t n, double alpha, double R, hrg_model* out) {
  if (!out) return fail(HRG_ERR_PARAMETER_DOMAIN, "out is NULL");
  out->n = n;
  out->alpha = alpha;
  out->R = R;
  double s = std::sinh(R / 2.0);
  out->cosh_r_minus_1 = 2.0 * (s * s);
  out->max_r = std::tanh(R / 2.0);
  out->rp_cap = std::nextafter(out->max_r, 0.0);
  out->r_cap = std::nextafter(R, 0.0);
  out->two_over_alpha = 2.0 / alpha;
  out->sinh_half_alpha_r = std::sinh(alpha * R / 2.0);
  return check_model(out);
}

hrg_status hrg_generate(hrg_context* c, const hrg_model* M, uint64_t seed, int order,
                        const hrg_shard* shard, hrg_stats* stats) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  hrg_status s = check_model(M);
  if (s != HRG_OK) return s;
  if (order != HRG_ORDER_SAMPLE && order != HRG_ORDER_ANGULAR)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "unknown vertex order");
  if (shard && (shard->count < 1 || shard->index < 0 || shard->index >= shard->count))
    return fail(HRG_ERR_PARAMETER_DOMAIN, "bad shard");
  CUDA_TRY(cudaSetDevice(c->device));
  c->have_result = false;
  s = ensure_point_buffers(c, M->n);
  if (s != HRG_OK) return s;
  return run_pipeline(c, M, shard, order == HRG_ORDER_SAMPLE, false, seed, stats);
}

hrg_status hrg_sample_points(hrg_context* c, const hrg_model* M, uint64_t seed, int order,
                             int mem_kind, double* phi, double* rn, double* rp) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  hrg_status s = check_model(M);
  if (s != HRG_OK) return s;
  if (order != HRG_ORDER_SAMPLE && order != HRG_ORDER_ANGULAR)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "unknown vertex order");
  CUDA_TRY(cudaSetDevice(c->device));
  c->have_result = false;
  s = ensure_point_buffers(c, M->n);
  if (s != HRG_OK) return s;
  int64_t n = M->n;
  cudaStream_t st = c->stream;
  int L = 0;
  BandSpec S = make_bands(M->R, &L);
  double C = std::ldexp(1.0, kQBits) / kTwoPi;
  SampleParams P{seed, M->two_over_alpha, M->sinh_half_alpha_r, M->r_cap, M->rp_cap, C};
  ++c->launches, k_sample<<<blocks_for(n), 256, 0, st>>>(n, P, S, c->phi.as<double>(), c->rn.as<double>(),
                                          c->rp.as<double>(), c->k32_in.as<uint32_t>(),
                                          c->vals_in.as<int32_t>(), c->pr.as<double2>());
  CUDA_TRY(cudaGetLastError());
  const double *sp = c->phi.as<double>(), *sn = c->rn.as<double>(), *sr = c->rp.as<double>();
  if (order == HRG_ORDER_ANGULAR) {
    // build_index sizes everything from c->np and reads the shard state of
    // the previous call: this call indexes all n points, unsharded
    c->np = n;
    c->sh_sampled = false;
    c->sh_cover = nullptr;
    c->sh_lo = c->sh_hi = nullptr;
    c->sh_mode = nullptr;
    s = build_index(c, M, S, L, nullptr, C, false);
    if (s != HRG_OK) return s;
    sp = c->s_phi.as<double>(); sn = c->s_rn.as<double>(); sr = c->s_rp.as<double>();
  }
  cudaMemcpyKind k = mem_kind == HRG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  size_t d = sizeof(double) * (size_t)n;
  if (phi) CUDA_TRY(cudaMemcpyAsync(phi, sp, d, k, st));
  if (rn) CUDA_TRY(cudaMemcpyAsync(rn, sn, d, k, st));
  if (rp) CUDA_TRY(cudaMemcpyAsync(rp, sr, d, k, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return HRG_OK;
}

hrg_status hrg_edges_from_coords(hrg_context* c, const hrg_model* M, const double* phi,
                                 const double* rp, int mem_kind, const hrg_shard* shard,
                                 hrg_stats* stats) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  hrg_status s = check_model(M);
  if (s != HRG_OK) return s;
  if (!phi || !rp) return fail(HRG_ERR_PARAMETER_DOMAIN, "coordinate pointer is NULL");
  if (shard && (shard->count < 1 || shard->index < 0 || shard->index >= shard->count))
    return fail(HRG_ERR_PARAMETER_DOMAIN, "bad shard");
  CUDA_TRY(cudaSetDevice(c->device));
  c->have_result = false;
  s = ensure_point_buffers(c, M->n);
  if (s != HRG_OK) return s;
  cudaMemcpyKind k = mem_kind == HRG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUDA_TRY(cudaMemcpyAsync(c->phi.p, phi, sizeof(double) * M->n, k, c->stream));
  CUDA_TRY(cudaMemcpyAsync(c->rp.p, rp, sizeof(double) * M->n, k, c->stream));
  return run_pipeline(c, M, shard, true, true, 0, stats);
}

hrg_status hrg_edges_brute_force(hrg_context* c, int64_t n, const double* phi, const double* rp,
                                 int mem_kind, double R, int64_t* near_ties) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  if (n < 1) return fail(HRG_ERR_PARAMETER_DOMAIN, "n must be at least 1");
  if (n >= (int64_t)1 << 30) return fail(HRG_ERR_PARAMETER_DOMAIN, "n must be below 2^30");
  if (!(R > 0.0)) return fail(HRG_ERR_PARAMETER_DOMAIN, "radius must be positive");
  if (!phi || !rp) return fail(HRG_ERR_PARAMETER_DOMAIN, "coordinate pointer is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  c->have_result = false;
  hrg_status s = ensure_point_buffers(c, n);
  if (s != HRG_OK) return s;
  cudaStream_t st = c->stream;
  cudaMemcpyKind k = mem_kind == HRG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  CUDA_TRY(cudaMemcpyAsync(c->phi.p, phi, sizeof(double) * n, k, st));
  CUDA_TRY(cudaMemcpyAsync(c->rp.p, rp, sizeof(double) * n, k, st));
  // x, y, b in the sorted-record buffers (free outside a generation)
  double* x = c->s_phi.as<double>();
  double* y = c->s_rn.as<double>();
  double* b = c->s_rp.as<double>();
  ++c->launches, k_bf_points<<<blocks_for(n), 256, 0, st>>>(n, c->phi.as<double>(), c->rp.as<double>(), x, y, b,
                                             c->trig);
  const double S = std::sinh(R / 2.0);
  const double t_lo = (S * (1.0 - 1e-9)) * (S * (1.0 - 1e-9));
  const double t_hi = (S * (1.0 + 1e-9)) * (S * (1.0 + 1e-9));
  const double tie = 4.0 * (std::nextafter(R, INFINITY) - R);
  CUDA_TRY(c->cand.ensure(8));
  unsigned long long* d_ties = c->cand.as<unsigned long long>();
  CUDA_TRY(cudaMemsetAsync(d_ties, 0, 8, st));
  ++c->launches, k_bf_pairs<false><<<blocks_for(n), 256, 0, st>>>(n, x, y, b, t_lo, t_hi, R, tie,
                                                    c->deg.as<int32_t>(), nullptr, nullptr,
                                                    nullptr);
  s = scan_i32_to_i64(c, c->deg.as<int32_t>(), c->rowptr.as<int64_t>(), n);
  if (s != HRG_OK) return s;
  int64_t nnz = 0;
  s = readback(c, c->rowptr.as<int64_t>() + n, 8, &nnz);
  if (s != HRG_OK) return s;
  CUDA_TRY(c->idx.ensure(4 * (size_t)std::max<int64_t>(nnz, 1)));
  ++c->launches, k_bf_pairs<true><<<blocks_for(n), 256, 0, st>>>(n, x, y, b, t_lo, t_hi, R, tie, nullptr,
                                                   c->rowptr.as<int64_t>(), c->idx.as<int32_t>(),
                                                   d_ties);
  CUDA_TRY(cudaGetLastError());
  unsigned long long ties = 0;
  s = readback(c, d_ties, 8, &ties);
  if (s != HRG_OK) return s;
  if (near_ties) *near_ties = (int64_t)ties;
  c->n = n;
  c->nnz = nnz;
  c->idx_final = c->idx.as<int32_t>();
  c->compact_result = false;
  c->coords_pending = false;
  c->coords_sorted = false;
  c->have_result = true;
  return HRG_OK;
}

hrg_status hrg_result_sizes(hrg_context* c, int64_t* n, int64_t* nnz) {
  if (!c || !c->have_result) return fail(HRG_ERR_NO_RESULT, "no result");
  if (n) *n = c->n;
  if (nnz) *nnz = c->nnz;
  return HRG_OK;
}

hrg_status hrg_result_device_ptrs(hrg_context* c, const double** phi, const double** rn,
                                  const double** rp, const int64_t** indptr,
                                  const int32_t** indices) {
  if (!c || !c->have_result) return fail(HRG_ERR_NO_RESULT, "no result");
  if ((phi || rn || rp) && c->coords_pending) {
    CUDA_TRY(cudaSetDevice(c->device));
    ++c->launches, k_sample_coords<<<blocks_for(c->n), 256, 0, c->stream>>>(
        c->n, c->pending, c->phi.as<double>(), c->rn.as<double>(), c->rp.as<double>());
    CUDA_TRY(cudaGetLastError());
    c->coords_pending = false;
  }
  if (indptr || indices) {
    CUDA_TRY(cudaSetDevice(c->device));
    hrg_status es = expand_rows(c);
    if (es != HRG_OK) return es;
  }
  if (phi) *phi = c->coords_sorted ? c->s_phi.as<double>() : c->phi.as<double>();
  if (rn) *rn = c->coords_sorted ? c->s_rn.as<double>() : c->rn.as<double>();
  if (rp) *rp = c->coords_sorted ? c->s_rp.as<double>() : c->rp.as<double>();
  if (indptr) *indptr = c->rowptr.as<int64_t>();
  if (indices) *indices = c->idx_final;
  return HRG_OK;
}

namespace {

// 8-byte ids into HOST memory: int32 ids cross PCIe (half the bytes of int64)
// into pinned staging, chunk by chunk with all copies queued at once,
// and the host threads widen each chunk into the caller's array as soon as
// its copy has landed (every thread takes a slice of every chunk, so the
// widening trails the copy by one chunk).
// ids per staged chunk (64 MB; 16 MB chunks or spinning on the chunk events
// instead of blocking measured the same 38 ms per copy, 4 MB chunks 48 ms)
constexpr size_t kWidenChunk = (size_t)1 << 24;
#ifndef HRG_PINNED_DEVICE_FRAC
#define HRG_PINNED_DEVICE_FRAC 0.1
#endif
constexpr double kPinnedDeviceFrac = HRG_PINNED_DEVICE_FRAC;

// Measured (config 2, 3.2e8 ids, 16 host cores): into PAGEABLE memory the
// host widening takes 51 ms against 157 ms for the int64 copy (which stages
// through the driver's bounce buffers).  Into PINNED memory the PCIe link and
// the host's memory bandwidth are both busy, so the ids can be split: the
// first fraction f is widened on the device and copied as int64, the rest
// crosses as int32 and is widened by the host threads while the copies run
// (PCIe bytes 4 (1 + f) per id, host widening (1 - f) of the ids).  With the
// host widening writing through non-temporal stores (widen_ids: 12 instead of
// 20 bytes of memory traffic per id) the host keeps up with most of the link
// (tools/e2e_copy_ab.py, libraries alternating, 3 rounds, ms per copy:
// f = 1: 51, 0.6: 46, 0.45: 45, 0.3: 45, 0.15: 42, 0: 40; with plain stores
// 51 / 48 / 50 / 47 / 51 / 53; the two-context e2e of bench.py: 42-43 ms/step
// at f <= 0.25 against 48-49 at 0.45).  Times vary by +-10% between runs and
// boxes; HRG_WIDEN_DEVICE_FRAC overrides f.
// The balance between the two paths is the host's (its memory bandwidth and
// what else runs on it) against the link's, and differs between machines
// (one all-host widening copy: 38 ms on one box of this pool, 73 ms on another,
// where the plain int64 copy's 51 ms wins).  So the share adapts, in steps of
// 10%, from what each split copy observed: the host threads done well before
// the DMA -> more for the host; the host threads never waiting for a chunk
// and finishing last -> more for the device.  Process-wide, pinned
// destinations only; HRG_WIDEN_DEVICE_FRAC pins it.
constexpr int kWidenMaxPct = 60;  // bounds the device-side widening buffer
std::atomic<int> g_widen_pct{(int)(kPinnedDeviceFrac * 100.0 + 0.5)};

double device_widen_frac(const hrg_context* c, const void* dst, bool* adaptive = nullptr) {
  if (adaptive) *adaptive = false;
  if (const char* e = getenv("HRG_WIDEN_DEVICE_FRAC")) return std::min(1.0, std::max(0.0, atof(e)));
  if ((size_t)c->nnz < ((size_t)1 << 22)) return 1.0;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, dst) != cudaSuccess) {
    cudaGetLastError();  // clear the query's error
    return 0.0;
  }
  if (at.type == cudaMemoryTypeUnregistered) return 0.0;
  if (adaptive) *adaptive = true;
  return g_widen_pct.load() / 100.0;
}

// int32 -> int64 of n non-negative ids on the host.  The destination is
// written once and not read back here, so it is written with non-temporal
// stores: a plain store first reads its cache line for ownership, and the
// result copy is bound by the host's memory bandwidth (4 B read + 8 B written
// per id instead of 4 + 8 + 8).
void widen_ids(const int32_t* src, int64_t* dst, size_t n) {
  size_t i = 0;
#if defined(__SSE2__)
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15u)) { dst[i] = src[i]; ++i; }
  const __m128i zero = _mm_setzero_si128();
  for (; i + 4 <= n; i += 4) {
    const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_unpacklo_epi32(x, zero));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2), _mm_unpackhi_epi32(x, zero));
  }
  _mm_sfence();
#endif
  for (; i < n; ++i) dst[i] = src[i];
}

// 3-byte ids (k_pack3) -> int64, the same way.  src + 3 n may be read up to
// 16 bytes past the last id's bytes only where the caller's buffer has them
// (the last 8 ids are unpacked byte by byte).
#if defined(__x86_64__)
__attribute__((target("ssse3")))
#endif
void widen_ids3(const uint8_t* src, int64_t* dst, size_t n) {
  size_t i = 0;
  auto one = [&](size_t k) {
    dst[k] = (int64_t)src[3 * k] | ((int64_t)src[3 * k + 1] << 8) | ((int64_t)src[3 * k + 2] << 16);
  };
#if defined(__x86_64__)
  while (i < n && (reinterpret_cast<uintptr_t>(dst + i) & 15u)) { one(i); ++i; }
  const __m128i lo = _mm_setr_epi8(0, 1, 2, -1, -1, -1, -1, -1, 3, 4, 5, -1, -1, -1, -1, -1);
  const __m128i hi = _mm_setr_epi8(6, 7, 8, -1, -1, -1, -1, -1, 9, 10, 11, -1, -1, -1, -1, -1);
  for (; i + 12 <= n; i += 4) {  // 16 bytes loaded, 12 used: stay 8 ids inside the slice
    const __m128i x = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 3 * i));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), _mm_shuffle_epi8(x, lo));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 2), _mm_shuffle_epi8(x, hi));
  }
  _mm_sfence();
#endif
  for (; i < n; ++i) one(i);
}

bool use_pack3(const hrg_context* c) {
  if (c->n > ((int64_t)1 << 24)) return false;
  if (const char* e = getenv("HRG_PACK3")) return atoi(e) != 0;
#if defined(__x86_64__)
  return __builtin_cpu_supports("ssse3");
#else
  return false;
#endif
}

// ids [0, first) widened on the device and copied as int64; ids [first, nnz)
// copied as int32 -- or, when every id fits 24 bits, as 3 bytes each -- in
// chunks and widened by the host threads as each lands.
hrg_status copy_indices_split(hrg_context* c, int64_t* dst, size_t first, bool adaptive) {
  const size_t nnz = (size_t)c->nnz;
  cudaStream_t st = c->stream;
  const size_t nh = nnz - first;
  // both staging buffers are sized for any share the adaptation may pick
  // (re-allocating a pinned gigabyte costs more than many copies)
  const size_t wcap = adaptive ? std::max(first, (size_t)(0.01 * kWidenMaxPct * (double)nnz) + 1) : first;
  const size_t hcap = adaptive ? nnz : nh;
  if (first > 0) {
    CUDA_TRY(c->widen.ensure(8 * wcap));
    ++c->launches, k_widen<<<blocks_for((int64_t)first), 256, 0, st>>>((int64_t)first, c->idx_final,
                                                                       c->widen.as<int64_t>());
  }
  if (c->h_stage_bytes < 4 * hcap) {
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->h_stage_bytes = 0;
    CUDA_TRY(cudaMallocHost(&c->h_stage, std::max<size_t>(4 * hcap, 4)));
    c->h_stage_bytes = std::max<size_t>(4 * hcap, 4);
  }
  const size_t nch = (nh + kWidenChunk - 1) / kWidenChunk;
  while (c->h_ev.size() < nch) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    c->h_ev.push_back(e);
  }
  const bool pack3 = use_pack3(c) && nh >= 64;
  uint8_t* const h_bytes = reinterpret_cast<uint8_t*>(c->h_stage);
  if (pack3) {
    CUDA_TRY(c->pack.ensure(3 * (adaptive ? nnz : nh) + 64));
    ++c->launches, k_pack3<<<blocks_for((int64_t)((nh + 3) / 4)), 256, 0, st>>>(
        (int64_t)nh, c->idx_final + first, c->pack.as<uint32_t>());
  }
  for (size_t ch = 0; ch < nch; ++ch) {
    const size_t a = ch * kWidenChunk, b = std::min(nh, a + kWidenChunk);
    if (pack3)
      CUDA_TRY(cudaMemcpyAsync(h_bytes + 3 * a, c->pack.as<uint8_t>() + 3 * a, 3 * (b - a),
                               cudaMemcpyDeviceToHost, st));
    else
      CUDA_TRY(cudaMemcpyAsync(c->h_stage + a, c->idx_final + first + a, 4 * (b - a),
                               cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaEventRecord(c->h_ev[ch], st));
  }
  if (first > 0)
    CUDA_TRY(cudaMemcpyAsync(dst, c->widen.p, 8 * first, cudaMemcpyDeviceToHost, st));
  const unsigned T = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::atomic<int> err{0};
  using clk = std::chrono::steady_clock;
  const clk::time_point t0 = clk::now();
  double waited = 0.0;  // thread 0: seconds blocked on chunks after the first
  auto work = [&](unsigned t) {
    for (size_t ch = 0; ch < nch; ++ch) {
      const clk::time_point w0 = clk::now();
      if (cudaEventSynchronize(c->h_ev[ch]) != cudaSuccess) { err = 1; return; }
      if (t == 0 && ch > 0) waited += std::chrono::duration<double>(clk::now() - w0).count();
      const size_t a = ch * kWidenChunk, b = std::min(nh, a + kWidenChunk);
      const size_t lo = a + (b - a) * t / T, hi = a + (b - a) * (t + 1) / T;
      if (pack3) widen_ids3(h_bytes + 3 * lo, dst + first + lo, hi - lo);
      else widen_ids(c->h_stage + lo, dst + first + lo, hi - lo);
    }
  };
  if (nch > 0) {
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < T; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  if (err) return fail(HRG_ERR_CUDA, "index copy failed");
  if (adaptive && nch > 1) {
    const double t_host = std::chrono::duration<double>(clk::now() - t0).count();
    CUDA_TRY(cudaStreamSynchronize(st));
    const double t_all = std::chrono::duration<double>(clk::now() - t0).count();
    int pct = g_widen_pct.load();
    if (t_all - t_host > 0.08 * t_all) pct -= 10;        // the DMA finished last
    else if (waited < 0.05 * t_host) pct += 10;           // the host never waited and finished last
    g_widen_pct.store(std::min(kWidenMaxPct, std::max(0, pct)));
    if (getenv("HRG_WIDEN_TRACE"))
      fprintf(stderr, "[hrg] result copy: device share %d%% host %.1f ms (waited %.1f) all %.1f ms -> %d%%\n",
              (int)(100.0 * (double)first / (double)nnz + 0.5), 1e3 * t_host, 1e3 * waited, 1e3 * t_all,
              g_widen_pct.load());
  }
  return HRG_OK;
}

}  // namespace

hrg_status hrg_copy_result(hrg_context* c, int mem_kind, double* phi, double* rn, double* rp,
                           int64_t* indptr, void* indices, int index_bytes) {
  if (!c || !c->have_result) return fail(HRG_ERR_NO_RESULT, "no result");
  if (indices && index_bytes != 4 && index_bytes != 8)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "index_bytes must be 4 or 8");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st = c->stream;
  cudaMemcpyKind k = mem_kind == HRG_MEM_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  size_t d = sizeof(double) * (size_t)c->n;
  const double *sp = nullptr, *sn = nullptr, *sr = nullptr;
  if (indptr || indices) {
    hrg_status es = expand_rows(c);
    if (es != HRG_OK) return es;
  }
  hrg_status s = hrg_result_device_ptrs(c, phi ? &sp : nullptr, rn ? &sn : nullptr,
                                        rp ? &sr : nullptr, nullptr, nullptr);
  if (s != HRG_OK) return s;
  if (phi) CUDA_TRY(cudaMemcpyAsync(phi, sp, d, k, st));
  if (rn) CUDA_TRY(cudaMemcpyAsync(rn, sn, d, k, st));
  if (rp) CUDA_TRY(cudaMemcpyAsync(rp, sr, d, k, st));
  if (indptr) CUDA_TRY(cudaMemcpyAsync(indptr, c->rowptr.p, 8 * (size_t)(c->n + 1), k, st));
  if (indices && c->nnz > 0) {
    if (index_bytes == 4) {
      CUDA_TRY(cudaMemcpyAsync(indices, c->idx_final, 4 * (size_t)c->nnz, k, st));
    } else if (mem_kind == HRG_MEM_HOST && device_widen_frac(c, indices) < 1.0) {
      bool adaptive = false;
      const size_t first = (size_t)(device_widen_frac(c, indices, &adaptive) * (double)c->nnz);
      hrg_status ws = copy_indices_split(c, static_cast<int64_t*>(indices), first, adaptive);
      if (ws != HRG_OK) return ws;
    } else {
      // widen on the device in one pass, then one copy: the copy engine then
      // never waits for SMs (another context's generation may hold them all)
      CUDA_TRY(c->widen.ensure(8 * (size_t)c->nnz));
      ++c->launches, k_widen<<<blocks_for(c->nnz), 256, 0, st>>>(c->nnz, c->idx_final, c->widen.as<int64_t>());
      CUDA_TRY(cudaMemcpyAsync(indices, c->widen.p, 8 * (size_t)c->nnz, k, st));
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return HRG_OK;
}

hrg_status hrg_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(HRG_ERR_PARAMETER_DOMAIN, "out is NULL");
  CUDA_TRY(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
  return HRG_OK;
}

hrg_status hrg_host_free(void* p) {
  if (p) CUDA_TRY(cudaFreeHost(p));
  return HRG_OK;
}

hrg_status hrg_debug_sincos_compare(hrg_context* c, int64_t n, uint64_t seed,
                                    int64_t* mismatches, int64_t* rejected) {
  if (!c || n < 0 || !mismatches || !rejected)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "bad arguments");
  CUDA_TRY(cudaSetDevice(c->device));
  Buf b;
  CUDA_TRY(b.ensure(16));
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemsetAsync(b.p, 0, 16, st));
  ++c->launches, k_sincos_compare<<<8 * c->sm_count, 256, 0, st>>>(n, seed, b.as<unsigned long long>());
  CUDA_TRY(cudaGetLastError());
  unsigned long long h[2];
  CUDA_TRY(cudaMemcpyAsync(h, b.p, 16, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  *mismatches = (int64_t)h[0];
  *rejected = (int64_t)h[1];
  return HRG_OK;
}

hrg_status hrg_debug_sincos(hrg_context* c, int64_t n, const double* x, int mode, double* s,
                            double* co) {
  if (!c || n < 0 || !x || !s || !co || mode < 0 || mode > 2)
    return fail(HRG_ERR_PARAMETER_DOMAIN, "bad arguments");
  if (n == 0) return HRG_OK;
  CUDA_TRY(cudaSetDevice(c->device));
  Buf b;
  CUDA_TRY(b.ensure(24 * (size_t)n));
  double* d = b.as<double>();
  cudaStream_t st = c->stream;
  CUDA_TRY(cudaMemcpyAsync(d, x, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
  ++c->launches, k_sincos<<<blocks_for(n), 256, 0, st>>>(n, d, d + n, d + 2 * n, mode);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(s, d + n, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(co, d + 2 * n, 8 * (size_t)n, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  b.release();
  return HRG_OK;
}

#ifdef HRG_BLOCK_PROFILE
// experiments: per-band counters of the block query (reset after reading)
hrg_status hrg_debug_block_profile(hrg_context* c, unsigned long long* out) {
  CUDA_TRY(cudaSetDevice(c->device));
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  CUDA_TRY(cudaMemcpyFromSymbol(out, g_bprof, sizeof(g_bprof)));
  std::vector<unsigned long long> z(sizeof(g_bprof) / 8, 0ull);
  CUDA_TRY(cudaMemcpyToSymbol(g_bprof, z.data(), sizeof(g_bprof)));
  return HRG_OK;
}
#endif

hrg_status hrg_synchronize(hrg_context* c) {
  if (!c) return fail(HRG_ERR_PARAMETER_DOMAIN, "ctx is NULL");
  CUDA_TRY(cudaStreamSynchronize(c->stream));
  return HRG_OK;
}

}  // extern "C"
