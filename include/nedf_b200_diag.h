/*
 * nedf_b200_diag.h -- diagnostics entry points of libnedf_b200 (not part of
 * the reference-facing boundary).  Used by the GPU tests to pin the tcgen05
 * operand layouts and to calibrate the near-tie guard.
 */
#ifndef NEDF_B200_DIAG_H
#define NEDF_B200_DIAG_H

#include <stdint.h>

#include "nedf_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One-CTA tcgen05 GEMM D[128][N] = A[128][K] * B[N][K]^T (fp16 in, fp32 out),
 * K in {64,128,192,256}, N in {64,...,256} step 16.  a_in_tmem selects the TS
 * form (A staged in tensor memory) instead of SS; d_col offsets the
 * accumulator columns in TMEM. */
int nedf_diag_umma(const void* a_dev, const void* b_dev, float* d_dev, int k, int n, int a_in_tmem, int d_col,
                   void* stream);

/* Raw network logits for local rays (rows that miss the box are left
 * untouched): precision NEDF_PREC_TENSOR (tcgen05 kernel) or NEDF_PREC_FP32. */
int nedf_diag_ray_logits(NedfContext* ctx, const NedfModel* m, const double* origins_dev, const double* dirs_dev,
                         int64_t n, float* coarse_dev, float* fine_dev, float* alpha_logit_dev, int precision,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif
