/* gpbo_test.h -- test and diagnostic hooks of libgpbo (the same shared library as gpbo.h).
 *
 * Not part of the hot path's interface (SURVEY.md §8(b) names gp_fit, gp_posterior,
 * ei_score_argmax, bo_suggest_batch): these entry points let tests force an implementation,
 * deliberately break the argmax filter's error bounds to exercise its soundness fallback, trace
 * the tcgen05 pipeline, microbenchmark the MMA path and pin the host Nelder-Mead optimiser.
 * Conventions (status codes, ctx, streams, ownership) as in gpbo.h. */
#ifndef GPBO_TEST_H
#define GPBO_TEST_H

#include "gpbo.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host-only test hook (no GPU needed): run gp_fit_ml2's Nelder-Mead state machine on a caller
 * objective f (evaluated in request order) from x0 in the box [lo, hi]; returns the best vertex,
 * its f, f(x0) and the number of evaluations.  Lets CPU tests pin the optimiser itself. */
gpbo_status gpbo_nm_selftest(int dim, const double *x0, const double *lo, const double *hi,
                             double step, int iters, double (*f)(const double *x, void *user),
                             void *user, double *best_x, double *best_f, double *start_f,
                             int64_t *nevals);

/* Test hook: multiply the fast phase's error bounds (dmu, dvar) by `scale` (default 1; 0 makes
 * the EI bracket nearly zero-width).  A negative scale keeps the bounds but halves every EI
 * bracket -- deliberately unsound, so the violation path above is exercised.  GPBO_EINVAL for a
 * non-finite scale. */
gpbo_status gpbo_debug_bound_scale(gpbo_ctx *ctx, float scale);

/* Test hook: one CTA computes D[128 x N] = A[128 x K] B[N x K]^T (fp16 row-major device inputs,
 * fp32 output) through the same tcgen05 path the scoring kernel uses: K-major operands in the
 * `row_bytes` (32/64/128) swizzle layout, one MMA per 16-wide k step, B read from a row offset
 * `b_row_off` (multiple of 8) of its shared-memory tile, accumulator in TMEM.  Synchronous. */
gpbo_status gpbo_tc_selftest(const void *A, const void *B, float *D, int N, int K, int row_bytes,
                             int b_row_off);
/* Same, followed by `reps` back-to-back accumulate MMAs of shape 128 x N x 16 issued by one warp;
 * cycles[0] = clock64 cycles to issue them, cycles[1] = until the last one completed (host). */
gpbo_status gpbo_tc_bench(const void *A, const void *B, float *D, int N, int K, int row_bytes,
                          int b_row_off, int reps, long long *cycles);

/* Test hook: if dev_buf (device, >= 98304 uint64) is non-NULL, the tcgen05 kernel of later
 * scoring calls records clock64 pipeline events of CTA 0 into it (entry 0 = count, then
 * (tag << 56 | role << 48 | panel) / clock pairs).  NULL disables. */
gpbo_status gpbo_debug_trace(gpbo_ctx *ctx, void *dev_buf);

/* Scoring implementation for this ctx: 0 = auto (the tcgen05 kernels wherever their envelope
 * covers every search of the call, else the CUDA-core kernel), 1 = CUDA-core kernel only,
 * 2 = tcgen05 only (calls outside its envelope fail with GPBO_ENOTSUP), 3 = as 2, and models
 * fitted while it is set use the streamed operand layout (the kernel for n > 256 / large d,
 * forced on small searches for testing), 4 = the float64 direct kernel (one thread per
 * candidate, every row scored exactly; n <= 64; auto picks it when sum over searches of
 * rows x n16^2 <= 2^24).  Models whose resident shared-memory image would not fit (n rounded to
 * 16 > 256, or a large d) always use the streamed layout.  Diagnostic/testing. */
gpbo_status gpbo_set_score_impl(gpbo_ctx *ctx, int impl);

/* Test hook: run only the fast phase of the scoring path on M device-resident candidates of
 * search s and write, per candidate (device float32 arrays of M, standardised units): the fast
 * mean mu~, its error bound dmu, the latent variance s2~, its error bound dvar, and the EI
 * bracket [ei_lo, ei_hi] the argmax filter uses.  Tests check the bracket contains the oracle. */
gpbo_status gpbo_debug_fast_phase(gpbo_ctx *ctx, const gpbo_model *model, int32_t s,
                                  const float *Xstar_dev, int64_t M, float *mu, float *dmu,
                                  float *var, float *dvar, float *ei_lo, float *ei_hi);

#ifdef __cplusplus
}
#endif
#endif /* GPBO_TEST_H */
