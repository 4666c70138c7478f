// Diagnostic CTA-pair tcgen05 GEMM: D[256][N] = A[256][K] * B[N][K]^T with
// cta_group::2 (M = 256).  CTA r of the pair stages A rows [128r, 128r+128)
// (shared memory, or TMEM for the TS form) and B rows [r N/2, (r+1) N/2); the
// even CTA issues the MMAs and a multicast commit releases both CTAs.  Pins
// the operand split the paired network kernel relies on.
#include "common.cuh"
#include "tc_ptx.cuh"
#include "../../include/nedf_b200_diag.h"

namespace nedf {

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
umma2_unit_kernel(const __half* __restrict__ A, const __half* __restrict__ B, float* __restrict__ D, int K, int N,
                  int a_in_tmem) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = smem;                 // 4 x 16 KB [128 rows x 64 K]
  unsigned char* sb = smem + 4 * 16384;     // 4 x 16 KB [<=128 rows x 64 K]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t rank = tc::cluster_rank();
  const int nkc = K / 64, nh = N / 2;
  const int arow = 128 * rank + tid;
  for (int kc = 0; kc < nkc; ++kc) {
    for (int j = 0; j < 8; ++j) {
      const uint4 v = *reinterpret_cast<const uint4*>(A + (size_t)arow * K + kc * 64 + j * 8);
      *reinterpret_cast<uint4*>(sa + kc * 16384 + tc::sw128_offset(tid, j)) = v;
    }
    for (int r = tid; r < nh; r += 128)
      for (int j = 0; j < 8; ++j) {
        const uint4 v = *reinterpret_cast<const uint4*>(B + (size_t)(rank * nh + r) * K + kc * 64 + j * 8);
        *reinterpret_cast<uint4*>(sb + kc * 16384 + tc::sw128_offset(r, j)) = v;
      }
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc2<512>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const uint32_t a_col = 256;
  if (a_in_tmem) {
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) {
        __half lo = A[(size_t)arow * K + 2 * (c0 + j)], hi = A[(size_t)arow * K + 2 * (c0 + j) + 1];
        r[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tc::tmem_st16(tbase + lane_base + a_col + c0, r);
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (rank == 0 && warp == 0) {
    const uint32_t idesc = tc::idesc_f16(256, N);
    if (tc::elect_one()) {
      for (int kc = 0; kc < nkc; ++kc)
        for (int k = 0; k < 4; ++k) {
          const uint64_t bdesc = tc::sw128_desc(tc::smem_u32(sb + kc * 16384) + k * 32);
          const uint32_t acc = (kc | k) ? 1u : 0u;
          if (a_in_tmem) tc::mma2_ts(tbase, tbase + a_col + kc * 32 + k * 8, bdesc, idesc, acc);
          else tc::mma2_ss(tbase, tc::sw128_desc(tc::smem_u32(sa + kc * 16384) + k * 32), bdesc, idesc, acc);
        }
      tc::mma2_commit_both(&bar);
    }
    __syncwarp();
  }
  tc::mbar_wait_cluster(&bar, 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tc::tmem_ld16(tbase + lane_base + c0, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(size_t)arow * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc2<512>(tbase);
}

// Issue-rate probe for the pair form: the even CTA issues `iters` M = 256 x N
// MMAs (K = 16 each, 4 per elect), one commit at the end; out[0] = cycles.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
mma2_rate_kernel(int ts, int N, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t rank = tc::cluster_rank();
  for (int i = tid; i < ((ts & 2) ? 16384 + 32768 + 8 * 16384 : 16384 + 32768) / 16; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc2<512>(&tmem_base_s);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  if (rank == 0 && warp == 0) {
    const uint32_t idesc = tc::idesc_f16(256, N);
    const uint64_t adesc = tc::sw128_desc(tc::smem_u32(smem));
    const uint64_t bdesc = tc::sw128_desc(tc::smem_u32(smem + 16384));
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // ts & 2: B cycles through eight 16 KB slots (no operand reuse between stages)
          const uint64_t bd = (ts & 2) ? tc::sw128_desc(tc::smem_u32(smem + 49152 + ((i >> 2) & 7) * 16384)) : bdesc;
          if (ts & 1) tc::mma2_ts(tbase, tbase + 256 + 8 * k, bd + 2 * k, idesc, 1u);
          else tc::mma2_ss(tbase, adesc + 2 * k, bd + 2 * k, idesc, 1u);
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) tc::mma2_commit_both(&bar);
    __syncwarp();
    tc::mbar_wait_cluster(&bar, 0);
    if (tid == 0) out[0] = clock64() - t0;
  } else if (tid == 0) {
    tc::mbar_wait_cluster(&bar, 0);
  }
  __syncwarp();
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc2<512>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_mma2_rate(int ts, int n, int iters, unsigned long long* out_dev) {
  using namespace nedf;
  if (!out_dev || n < 32 || n > 256 || n % 32 || iters < 4) return NEDF_ERR_INVALID;
  const size_t smem = 16384 + 32768 + 1024 + ((ts & 2) ? 8 * 16384 : 0);
  cudaFuncSetAttribute(mma2_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma2_rate_kernel<<<2, 128, smem>>>(ts, n, iters, out_dev);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}

extern "C" int nedf_diag_umma2(const void* a, const void* b, float* d, int k, int n, int a_in_tmem, void* stream) {
  using namespace nedf;
  if (!a || !b || !d || k < 64 || k > 256 || k % 64 || n < 32 || n > 256 || n % 32) return NEDF_ERR_INVALID;
  const size_t smem = 8 * 16384 + 1024;
  cudaFuncSetAttribute(umma2_unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma2_unit_kernel<<<2, 128, smem, (cudaStream_t)stream>>>((const __half*)a, (const __half*)b, d, k, n, a_in_tmem);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}
