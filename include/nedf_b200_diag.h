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

/* One-CTA kind::tf32 (bf16 = 0) or kind::f16 bf16 (bf16 = 1) tcgen05 GEMM of fp32 A[m][k],
 * B[n][k] (m = 64 or 128), SW128 K-major: writes the raw accumulator, TMEM lanes 0..127 x
 * n columns, to draw[128][n] (pins the M = 64 layout of the guard kernel). */
int nedf_diag_umma32(const float* a_dev, const float* b_dev, float* draw_dev, int m, int n, int k, int bf16,
                     void* stream);

/* The trainer's fp32-accurate split-tf32 tcgen05 GEMM: C[m][n] = op(A)[m][k] op(B)[n][k]^T
 * (+ beta C); ta / tb = 1: that operand is stored transposed (A[k][m], B[k][n]); ws: optional
 * split-K workspace of ws_floats floats. */
int nedf_diag_gemm(const float* a, int lda, int ta, const float* b, int ldb, int tb, float* c, int ldc, int m, int n,
                   int k, float beta, float* ws, int64_t ws_floats, void* stream);

/* clock64 stamps of the GEMM's CTA (0, 0, 0): [0] start, [1] set up, [2 + c] chunk c ready
 * (c < 8), [10] accumulators complete, [11] stored; enable >= 0 switches tracing. */
int nedf_diag_gemm_trace(int enable, unsigned long long* out);

/* Raw network logits for local rays (rows that miss the box are left
 * untouched): precision NEDF_PREC_TENSOR (tcgen05 kernel), NEDF_PREC_FP32, or
 * 16 + NEDF_GUARD_* (only that near-tie guard kernel, on every ray). */
int nedf_diag_ray_logits(NedfContext* ctx, const NedfModel* m, const double* origins_dev, const double* dirs_dev,
                         int64_t n, float* coarse_dev, float* fine_dev, float* alpha_logit_dev, int precision,
                         void* stream);

/* Timeline of CTA 0's second tile in the tensor-core kernel (clock64 stamps):
 * enable >= 0 sets tracing on/off for later launches; out (host, n <= 1024
 * entries) receives the stamps: [L] / [40+L] MMA layer start / issued,
 * [100+8L+s] / [104+8L+s] epilogue slice ready / done, [400+p] / [420+p]
 * encoder point written / slot acquired, [450+L] producer layer start. */
int nedf_diag_tc_trace(int enable, unsigned long long* out, int n);

/* Timeline of cluster 0 / CTA 0 of the cluster-split fp32 guard kernel (clock64):
 * per tile i < 4, [64 i] start, [64 i + 1] rays set up, [64 i + 2] features
 * landed, [64 i + 3 + L] layer L landed, [64 i + 40] decoded; n <= 256. */
int nedf_diag_cl_trace(int enable, unsigned long long* out, int n);

/* Timeline of cluster 0 / CTA 0's first tile in the tcgen05 guard kernel (clock64): [L] layer
 * L's MMAs start, [40+L] issued, [80+L] epilogue has the accumulators, [120+L] slab sent,
 * [160+L] layer landed, [200+L] next B tiles written, [240+q] weight stage q issued; n <= 320. */
int nedf_diag_guard_trace(int enable, unsigned long long* out, int n);

/* Timeline of CTA 0's first tile in the guard's throughput kernel (mlp_precise.cu, clock64):
 * [L] layer L's MMAs start, [40+L] issued, [80+L] epilogue has the accumulators, [120+L]
 * epilogue done, [160+p] head point p encoded; n <= 200. */
int nedf_diag_precise_trace(int enable, unsigned long long* out, int n);

/* tcgen05 issue-rate probe: `iters` M=128 x N MMAs (ts: A from TMEM) from one
 * warp, committing every `per_commit`; writes elapsed clock64 cycles to out_dev. */
int nedf_diag_mma_rate(int ts, int n, int iters, int per_commit, unsigned long long* out_dev);

/* L2 -> shared memory bulk-copy bandwidth probe: `ctas` CTAs each stream `total`
 * bytes of `src` (wrapping within `span`) through `depth` x `stage`-byte
 * buffers; out_dev[cta] = clock64 cycles. */
int nedf_diag_bulk_rate(const void* src, size_t span, int stage, int depth, size_t total, int ctas,
                        unsigned long long* out_dev);

#ifdef __cplusplus
}
#endif
#endif
