/*
 * hrg_oracle.h -- CPU restatement of the reference generator's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1501_03545_b200/)
 * links, loads or calls this library.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may use it, and only as
 * the checker or as the timed CPU baseline.
 *
 * Every function cites the reference file:line it restates
 * (reference = /root/reference/pkg/src/hrgen, "hrgen" below).
 */
#ifndef HRG_ORACLE_H
#define HRG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Trigonometry used for the Poincare-disk x/y coordinates.
 *   ORC_TRIG_LIBM : libm cos/sin -- what numpy's float64 cos/sin evaluate to on
 *                   glibc hosts (checked in tests/test_oracle.py), i.e. the
 *                   reference's own arithmetic.
 *   ORC_TRIG_CR   : correctly rounded cos/sin (__float128 evaluation rounded
 *                   once to double).  The CUDA path computes correctly rounded
 *                   values, so this mode is the bit-exact twin of the GPU. */
enum { ORC_TRIG_LIBM = 0, ORC_TRIG_CR = 1 };

/* One Philox4x32-10 block (for known-answer tests). */
void orc_philox_raw(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Counter-based Philox4x32-10 uniforms: u1[i], u2[i] in [0,1) with 53 bits. */
void orc_philox_uniforms(int64_t n, uint64_t seed, uint64_t offset, double *u1, double *u2);

/* hrgen generator.py:142-179 (radial_inverse_cdf + sample_points) on given uniforms. */
void orc_sample_from_uniforms(int64_t n, const double *u1, const double *u2,
                              double two_over_alpha, double sinh_half_alpha_r,
                              double r_cap, double rp_cap,
                              double *phi, double *r_native, double *r_poincare);

/* hrgen geometry.py:141-157 circle_params; a = cosh(R) - 1 as the reference computes it. */
void orc_circle_params(int64_t n, const double *rp, double a, double *center_r, double *rad);

/* p_x = r*cos(phi), p_y = r*sin(phi)  (quadtree.py:474-475, 516-517). */
void orc_xy(int64_t n, const double *phi, const double *r, int trig, double *x, double *y);

/* One correctly rounded cos/sin (for pinning the GPU's sincos). */
void orc_sincos_cr(int64_t n, const double *x, double *s, double *c);

/* All-pairs reference edge set {(v,w): v<w, pred(v->w)}, pred being the
 * quadtree leaf test quadtree.py:611-613 against the circle of the smaller id
 * (generator.py:182-187).  Returns m; writes up to cap pairs (u<v, sorted by
 * u then v) when u/v are non-NULL.  O(n^2); nthreads<=0 means all cores. */
int64_t orc_edges_brute(int64_t n, const double *phi, const double *rp, double a, int trig,
                        int nthreads, int64_t cap, int64_t *u, int64_t *v);

/* Same edge set through a restatement of the reference's polar quadtree
 * (quadtree.py: build 303-340, pack 399-495, query_many 499-631).
 * Output pairs are sorted (u<v lexicographic).  Returns m, or -1 on error. */
typedef struct orc_qt_timing { double t_build_s, t_query_s, t_csr_s; } orc_qt_timing;
int64_t orc_edges_quadtree(int64_t n, const double *phi, const double *rp, double a, double alpha,
                           double max_r, int capacity, int trig, int nthreads,
                           int64_t query_lo, int64_t query_hi,
                           int64_t cap, int64_t *u, int64_t *v, orc_qt_timing *timing);

/* Full rows of the vertices qids[0..nq) by all-pairs tests: row k holds every
 * w != qids[k] with pred(min -> max) (generator.py:182-187, quadtree.py:611-613),
 * ascending.  For full-size parity checks of sampled rows.  Returns the total
 * entry count; fills indptr (nq+1) and indices (up to cap) when non-NULL. */
int64_t orc_rows_brute(int64_t n, const double *phi, const double *rp, double a, int trig,
                       int nthreads, int64_t nq, const int64_t *qids, int64_t cap,
                       int64_t *indptr, int64_t *indices);

/* |cosh d - cosh R| / cosh R for pairs (u[k], v[k]), in __float128 (the
 * north star's exception band for pairs on which two edge sets differ). */
void orc_cosh_gap(int64_t m, const int64_t *u, const int64_t *v, const double *phi,
                  const double *rp, double R, double *gap);

/* hrgen graph.py:52-77 Graph.from_edge_arrays for u<v pairs: symmetric CSR,
 * rows sorted.  indptr has n+1 entries, indices 2m. */
void orc_csr_from_pairs(int64_t n, int64_t m, const int64_t *u, const int64_t *v,
                        int64_t *indptr, int64_t *indices);

#ifdef __cplusplus
}
#endif
#endif
