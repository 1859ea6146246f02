/*
 * hrgen_b200.h -- C ABI of the B200 random-hyperbolic-graph generator.
 *
 * Drop-in boundary for the reference package hrgen
 * (/root/reference/pkg/src/hrgen).  Every entry point names the reference
 * interface it replaces.  Plain pointers and sizes only; no torch types.
 * Host bindings: paper_1501_03545_b200/_lib.py (ctypes); see INTEGRATION.md
 * for the stub a maintainer would add on the reference side.
 *
 * Vertex ids and edge semantics are the reference's:
 *   - vertex i of generate() is the i-th draw of the seeded stream
 *     (hrgen generator.py:160-179), unless HRG_ORDER_ANGULAR is requested;
 *   - {v, w} with v < w is an edge iff w lies strictly inside the Euclidean
 *     image of v's hyperbolic disk of radius R in the Poincare model
 *     (generator.py:182-187, quadtree.py:611-613, geometry.py:141-157);
 *   - the result is the CSR of hrgen.Graph (graph.py:52-77): both
 *     orientations, rows sorted ascending.
 */
#ifndef HRGEN_B200_H
#define HRGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HRGEN_B200_ABI_VERSION 1

/* Status codes.  Parameter / bounds errors mirror hrgen.errors (errors.py). */
typedef enum {
  HRG_OK = 0,
  HRG_ERR_PARAMETER_DOMAIN = 1,   /* hrgen.ParameterDomainError */
  HRG_ERR_INFEASIBLE = 2,         /* hrgen.InfeasibleParametersError */
  HRG_ERR_OUT_OF_BOUNDS = 3,      /* hrgen.OutOfBoundsError (quadtree.py:293-299) */
  HRG_ERR_CUDA = 10,
  HRG_ERR_NO_RESULT = 11,
  HRG_ERR_INTERNAL = 12
} hrg_status;

/* Vertex labelling of hrg_generate. */
enum {
  HRG_ORDER_SAMPLE = 0,   /* reference semantics: id = draw index */
  HRG_ORDER_ANGULAR = 1   /* id = rank in (radial band, angle) order; rows come out sorted
                             without a sort pass.  The same point set with hrgen's edge
                             rule applied to these labels (the circle of the smaller
                             label decides a pair): NOT exactly a relabelling of the
                             sample-order graph -- borderline pairs can be decided
                             differently (1601 of 1.6e8 pairs at config 2). */
};

/* sin/cos behind the Poincare coordinates p_x = r cos(phi), p_y = r sin(phi)
 * (quadtree.py:474-475, 516-517). */
enum {
  HRG_TRIG_LIBM = 0,  /* default: glibc 2.39's dbl-64 sin/cos bit for bit -- what
                         numpy evaluates on x86-64 glibc hosts, i.e. hrgen's own
                         arithmetic; the edge set is then hrgen's exactly */
  HRG_TRIG_CR = 1     /* correctly rounded sin/cos (libm-independent) */
};

/* Memory kinds for user buffers. */
enum { HRG_MEM_HOST = 0, HRG_MEM_DEVICE = 1 };

/* Resolved model (hrgen geometry.py:82-101 ModelParams) plus the derived
 * scalars the reference evaluates with numpy.  hrg_model_init fills the
 * derived fields with libm; the Python host layer overwrites them with the
 * numpy-evaluated values so results are bit-identical to hrgen. */
typedef struct {
  int64_t n;
  double alpha;
  double R;
  /* derived */
  double cosh_r_minus_1;   /* a = 2*sinh(R/2)^2          (geometry.py:150) */
  double max_r;            /* tanh(R/2)                  (generator.py:203) */
  double rp_cap;           /* nextafter(max_r, 0)        (generator.py:176-178) */
  double r_cap;            /* nextafter(R, 0)            (generator.py:174) */
  double two_over_alpha;   /* 2/alpha                    (generator.py:156) */
  double sinh_half_alpha_r;/* sinh(alpha*R/2)            (generator.py:156) */
} hrg_model;

/* Angular sector of query vertices this call emits rows for (multi-GPU
 * sharding): rows are produced for vertices whose angle lies in
 * [2*pi*index/count, 2*pi*(index+1)/count).  {0, 1} = everything. */
typedef struct { int32_t index, count; } hrg_shard;

typedef struct {
  int64_t n, m;            /* vertices, undirected edges (over all rows emitted) */
  int64_t nnz;             /* CSR entries emitted = sum of emitted row lengths */
  int64_t candidates;      /* pair tests performed by the range query */
  double radius, alpha;
  int64_t heavy_queries, heavy_chunks;  /* hub queries split across warps */
  /* CUDA-event phase times: sample | build (key sort + records + index) |
   * edges (light query, heavy query, compaction, row ordering) */
  double t_sample_ms, t_build_ms, t_edges_ms;
  double t_sort_ms, t_light_ms, t_heavy_ms, t_compact_ms, t_rowsort_ms;
  int32_t n_bands;
  int32_t kernel_launches;
} hrg_stats;

typedef struct hrg_context hrg_context;

const char *hrg_version(void);
/* Thread-local message for the last non-OK status. */
const char *hrg_last_error(void);

/* Context = device + stream + device workspace + the last result. */
hrg_status hrg_context_create(int device, void *cuda_stream, hrg_context **out);
hrg_status hrg_context_destroy(hrg_context *ctx);
hrg_status hrg_context_set_stream(hrg_context *ctx, void *cuda_stream);
/* Trig mode (HRG_TRIG_LIBM, the default, or HRG_TRIG_CR) for later calls. */
hrg_status hrg_context_set_trig(hrg_context *ctx, int mode);
/* Kernel launches this library has queued on ctx so far (library kernels
 * such as CUB's sort and scan passes not included). */
hrg_status hrg_context_launches(hrg_context *ctx, int64_t *out);

/* hrgen geometry.py:170-190 expected_avg_degree / 197-232 target_radius
 * (libm evaluation; the Python layer uses numpy for bit-identical R). */
hrg_status hrg_expected_avg_degree(int64_t n, double alpha, double radius, double *out);
hrg_status hrg_target_radius(int64_t n, double avg_degree, double alpha, double rel_tol,
                             double *out);
hrg_status hrg_model_init(int64_t n, double alpha, double R, hrg_model *out);

/* hrgen generator.py:190-239 generate_with_stats / 242-246 generate:
 * sample n points from seed (counter-based Philox4x32-10), index them, and
 * emit the CSR of the graph.  Result stays on the device in ctx. */
hrg_status hrg_generate(hrg_context *ctx, const hrg_model *model, uint64_t seed, int order,
                        const hrg_shard *shard, hrg_stats *stats);

/* hrgen generator.py:160-179 sample_points: only the coordinates (vertex-id
 * order for the given labelling), copied to phi / r_native / r_poincare
 * (n doubles each; mem_kind says where they live; NULL skips an array). */
hrg_status hrg_sample_points(hrg_context *ctx, const hrg_model *model, uint64_t seed, int order,
                             int mem_kind, double *phi, double *r_native, double *r_poincare);

/* hrgen generator.py:249-274 generate_brute_force(coords, R) signature with
 * the quadtree edge semantics of generate(): edges among caller-supplied
 * Poincare coordinates (phi in [0,2pi), r_poincare in [0, max_r)).
 * mem_kind says where phi / r_poincare live.  Ids = array index. */
hrg_status hrg_edges_from_coords(hrg_context *ctx, const hrg_model *model, const double *phi,
                                 const double *r_poincare, int mem_kind, const hrg_shard *shard,
                                 hrg_stats *stats);

/* hrgen generator.py:249-274 generate_brute_force(coords, R) itself: all
 * pairs, edge iff 2 asinh(sqrt(d2 / (b_i b_j))) < R with x = r cos(phi),
 * y = r sin(phi), b = (1 - r)(1 + r), d2 = dx*dx + dy*dy (hrgen's sequence).
 * O(n^2), for validation.  *near_ties (optional) receives the number of
 * ordered pairs whose distance is within 4 ulps of R, where the device's asinh
 * and libm's may round differently.  Ids = array index; result as for
 * hrg_generate. */
hrg_status hrg_edges_brute_force(hrg_context *ctx, int64_t n, const double *phi,
                                 const double *r_poincare, int mem_kind, double R,
                                 int64_t *near_ties);

/* Sizes of the last result. */
hrg_status hrg_result_sizes(hrg_context *ctx, int64_t *n, int64_t *nnz);

/* Copy the last result out.  Any pointer may be NULL to skip that array.
 * indices are written as int64 when index_bytes == 8, int32 when 4.
 * Coordinates (in vertex-id order) are available after hrg_generate. */
hrg_status hrg_copy_result(hrg_context *ctx, int mem_kind, double *phi, double *r_native,
                           double *r_poincare, int64_t *indptr, void *indices,
                           int index_bytes);

/* Device pointers of the last result (valid until the next generate call). */
hrg_status hrg_result_device_ptrs(hrg_context *ctx, const double **phi, const double **r_native,
                                  const double **r_poincare, const int64_t **indptr,
                                  const int32_t **indices);

/* Pinned host memory helpers (for callers without a CUDA runtime binding). */
hrg_status hrg_host_alloc(size_t bytes, void **out);
hrg_status hrg_host_free(void *p);

/* Wait for all work queued by ctx. */
hrg_status hrg_synchronize(hrg_context *ctx);

#ifdef __cplusplus
}
#endif
#endif
