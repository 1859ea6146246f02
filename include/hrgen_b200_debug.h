/*
 * hrgen_b200_debug.h -- diagnostic entry points of libhrgen_b200.so.
 *
 * Not part of the drop-in boundary (include/hrgen_b200.h): they exist so the
 * parity tests can check the device arithmetic in isolation.
 */
#ifndef HRGEN_B200_DEBUG_H
#define HRGEN_B200_DEBUG_H

#include "hrgen_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* The device's sin/cos (the values behind p_x = r*cos(phi), quadtree.py:474)
 * for n host angles in [0, 2pi).  mode: 0 = glibc's (HRG_TRIG_LIBM, what
 * generations use by default), 1 = correctly rounded (HRG_TRIG_CR: fast
 * path + rounding test), 2 = correctly rounded, full double-double
 * evaluation. */
hrg_status hrg_debug_sincos(hrg_context *ctx, int64_t n, const double *x, int mode, double *s,
                            double *c);

/* The correctly rounded fast sin/cos (table + short series + rounding test)
 * against the full double-double evaluation on n seeded angles (every 4th
 * within 2^-20 of a multiple of pi/4): values that differ, and values the
 * fast path's rounding test sent to the full evaluation. */
hrg_status hrg_debug_sincos_compare(hrg_context *ctx, int64_t n, uint64_t seed,
                                    int64_t *mismatches, int64_t *rejected);

#ifdef __cplusplus
}
#endif
#endif
