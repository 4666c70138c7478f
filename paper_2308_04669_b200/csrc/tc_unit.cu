// Diagnostic one-CTA tcgen05 GEMM used by the GPU tests to pin the operand
// layouts the fused network kernel relies on: 128B-swizzled K-major shared
// tiles (SS form), A staged in TMEM as packed f16x2 columns (TS form), and
// the 32x32b TMEM load of the fp32 accumulator.
#include <cstdio>

#include <cuda_bf16.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "../../include/nedf_b200_diag.h"

namespace nedf {

__global__ void __launch_bounds__(128, 1)
umma_unit_kernel(const __half* __restrict__ A, const __half* __restrict__ B, float* __restrict__ D, int K, int N,
                 int a_in_tmem, int d_col) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* sa = smem;                 // 4 x 16 KB  [128 rows x 64 K] per K chunk
  unsigned char* sb = smem + 4 * 16384;     // 4 x 32 KB  [256 rows x 64 K]
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nkc = K / 64;
  // stage A rows (thread = row) and B rows into swizzled tiles
  for (int kc = 0; kc < nkc; ++kc) {
    for (int j = 0; j < 8; ++j) {
      const uint4 v = *reinterpret_cast<const uint4*>(A + (size_t)tid * K + kc * 64 + j * 8);
      *reinterpret_cast<uint4*>(sa + kc * 16384 + tc::sw128_offset(tid, j)) = v;
    }
    for (int r = tid; r < N; r += 128)
      for (int j = 0; j < 8; ++j) {
        const uint4 v = *reinterpret_cast<const uint4*>(B + (size_t)r * K + kc * 64 + j * 8);
        *reinterpret_cast<uint4*>(sb + kc * 32768 + tc::sw128_offset(r, j)) = v;
      }
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const uint32_t a_col = 256;
  if (a_in_tmem) {
    // row tid -> lane tid; column c holds (A[k=2c], A[k=2c+1]) as (lo, hi)
    for (int c0 = 0; c0 < K / 2; c0 += 16) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) {
        __half lo = A[(size_t)tid * K + 2 * (c0 + j)], hi = A[(size_t)tid * K + 2 * (c0 + j) + 1];
        r[j] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
      }
      tc::tmem_st16(tbase + lane_base + a_col + c0, r);
    }
    tc::tmem_st_wait();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_f16(128, N);
    for (int kc = 0; kc < nkc; ++kc)
      for (int k = 0; k < 4; ++k) {
        uint64_t bdesc = tc::sw128_desc(tc::smem_u32(sb + kc * 32768) + k * 32);
        uint32_t acc = (kc | k) ? 1u : 0u;
        if (a_in_tmem) {
          tc::mma_ts(tbase + d_col, tbase + a_col + kc * 32 + k * 8, bdesc, idesc, acc);
        } else {
          uint64_t adesc = tc::sw128_desc(tc::smem_u32(sa + kc * 16384) + k * 32);
          tc::mma_ss(tbase + d_col, adesc, bdesc, idesc, acc);
        }
      }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    tc::tmem_ld16(tbase + lane_base + d_col + c0, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(size_t)tid * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_umma(const void* a, const void* b, float* d, int k, int n, int a_in_tmem, int d_col,
                              void* stream) {
  using namespace nedf;
  if (!a || !b || !d || k < 64 || k > 256 || k % 64 || n < 16 || n > 256 || n % 16 || d_col < 0 ||
      d_col + n > 256)
    return NEDF_ERR_INVALID;
  size_t smem = 4 * 16384 + 4 * 32768 + 1024;
  cudaFuncSetAttribute(umma_unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma_unit_kernel<<<1, 128, smem, (cudaStream_t)stream>>>((const __half*)a, (const __half*)b, d, k, n, a_in_tmem,
                                                           d_col);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}

namespace nedf {

// kind::tf32 / kind::f16(bf16) unit GEMM, A [M][K] and B [N][K] given as fp32 (bf16: rounded
// on staging), 128B-swizzled K-major tiles of 32 fp32 (or 64 bf16) K per atom; writes the raw
// TMEM accumulator, all 128 lanes x N columns, to Draw[lane][n] (pins the M = 64 D layout).
__global__ void __launch_bounds__(128, 1)
umma32_unit_kernel(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ Draw, int M, int N,
                   int K, int bf16, int d_lane) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int esz = bf16 ? 2 : 4, per_atom = 128 / esz, n_atoms = K / per_atom;
  unsigned char* sa = smem;                            // n_atoms x [M rows x 128 B]
  unsigned char* sb = smem + (size_t)n_atoms * M * 128;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < (M + N) * K; e += 128) {
    const bool isa = e < M * K;
    const int r = isa ? e / K : (e - M * K) / K, k = isa ? e % K : (e - M * K) % K;
    const float v = isa ? A[(size_t)r * K + k] : B[(size_t)r * K + k];
    const int atom = k / per_atom, kin = k % per_atom;
    unsigned char* base = (isa ? sa + (size_t)atom * M * 128 : sb + (size_t)atom * N * 128);
    const uint32_t off = tc::sw128_offset(r, (kin * esz) >> 4) + ((kin * esz) & 15);
    if (bf16) *reinterpret_cast<__nv_bfloat16*>(base + off) = __float2bfloat16_rn(v);
    else *reinterpret_cast<float*>(base + off) = v;
  }
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_s);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_fence_init();
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  if (tid == 0) {
    const uint32_t idesc = bf16 ? tc::idesc_bf16(M, N) : tc::idesc_tf32(M, N);
    const int steps = K / (bf16 ? 16 : 8);
    for (int s = 0; s < steps; ++s) {
      const int atom = s / 4, within = (s % 4) * 32;
      const uint64_t ad = tc::sw128_desc(tc::smem_u32(sa + (size_t)atom * M * 128) + within);
      const uint64_t bd = tc::sw128_desc(tc::smem_u32(sb + (size_t)atom * N * 128) + within);
      const uint32_t dt = tbase + ((uint32_t)d_lane << 16);
      if (bf16) tc::mma_ss(dt, ad, bd, idesc, s > 0);
      else tc::mma_ss_tf32(dt, ad, bd, idesc, s > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    tc::tmem_ld8(tbase + ((uint32_t)(warp * 32) << 16) + c0, r);
    tc::tmem_ld_wait();
    for (int j = 0; j < 8; ++j) Draw[(size_t)tid * N + c0 + j] = __uint_as_float(r[j]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_umma32(const float* a, const float* b, float* draw, int m, int n, int k, int bf16,
                                void* stream) {
  using namespace nedf;
  const int d_lane = bf16 >> 8;                 // bits 8+: TMEM lane offset of the accumulator (layout probe)
  bf16 &= 0xFF;
  const int per_atom = bf16 ? 64 : 32;
  if (!a || !b || !draw || (m != 64 && m != 128) || n < 8 || n > 256 || n % 8 || k < per_atom || k > 256 ||
      k % per_atom)
    return NEDF_ERR_INVALID;
  const size_t smem = (size_t)(k / per_atom) * (m + n) * 128 + 1024;
  cudaFuncSetAttribute(umma32_unit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  umma32_unit_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(a, b, draw, m, n, k, bf16, d_lane);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}

namespace nedf {

// Throughput probe: one thread issues `iters` back-to-back M=128 MMAs of width N
// (SS: A and B from shared memory; TS: A from TMEM) accumulating into TMEM,
// and records clock64 from first issue to commit completion.
__device__ unsigned char g_rate_src[8 * 16384];

__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int ts, int N, int iters, int per_commit,
                                                          unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // warp-uniform for the compiler
  for (int i = tid; i < (16384 + 32768) / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  tc::fence_proxy_async_smem();
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_s);
  if (tid == 0) { tc::mbar_init(&bar, 1); tc::mbar_fence_init(); }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  __shared__ volatile int stop_flag;
  if (tid == 0) stop_flag = 0;
  __syncthreads();
  if ((per_commit == -5 || per_commit == -6) && warp == 1) {
    // variant -5: lanes 0-7 of warp 1 stream 16 KB bulk copies global -> shared (L2-resident source)
    // into a separate 128 KB region while warp 0 issues MMAs: smem write-port contention
    __shared__ uint64_t cbar[8];
    const int l = tid & 31;
    if (l < 8) {
      tc::mbar_init(&cbar[l], 1);
      tc::mbar_fence_init();
      unsigned char* dst = smem + 49152 + l * 16384;
      uint32_t ph = 0;
      long long copies = 0;
      while (!stop_flag) {
        tc::mbar_expect_tx(&cbar[l], 16384);
        tc::bulk_g2s(dst, g_rate_src + l * 16384, 16384, &cbar[l]);
        tc::mbar_wait(&cbar[l], ph);
        ph ^= 1;
        ++copies;
      }
      if (l == 0) out[1] = copies;
    }
    __syncwarp();
  }
  if (per_commit <= -3 && per_commit >= -4 && warp != 0) {
    // variant -3 / -4: the other warps hammer TMEM (-3: tcgen05.ld 32 cols + st 16 cols per round
    // on columns the MMA does not touch; -4: plain FMA work) while warp 0 issues MMAs
    const uint32_t lane_addr = tbase + ((uint32_t)(32 * warp) << 16);
    float acc = 0.f;
    while (!stop_flag) {
      if (per_commit == -3) {
        uint32_t v[32];
        tc::tmem_ld32(lane_addr + 384, v);
        tc::tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = v[2 * j] ^ v[2 * j + 1];
        tc::tmem_st16(lane_addr + 448, pk);
        tc::tmem_st_wait();
      } else {
#pragma unroll 8
        for (int j = 0; j < 64; ++j) acc = fmaf(acc, 1.0001f, 0.5f);
      }
    }
    if (acc == 12345.f) out[1] = 1;
  }
  if (warp == 0) {
    const uint32_t idesc = tc::idesc_f16(128, N);
    const uint64_t adesc = tc::sw128_desc(tc::smem_u32(smem));
    const uint64_t bdesc = tc::sw128_desc(tc::smem_u32(smem + 16384));
    unsigned long long t0 = clock64();
    uint32_t phase = 0;
    if (per_commit <= -2) {
      // variant: whole warp runs the loop (uniform values), elect.sync issues
      if (per_commit == -6) {          // no MMAs: copies alone for iters * 74 cycles
        while (clock64() - t0 < (unsigned long long)iters * 74) {
        }
      } else
      if (per_commit <= -12 && per_commit >= -14) {
        // -12: per 8 MMAs one wait + fence and one commit; -13: per 8 MMAs two waits and two commits;
        // -14: per 16 MMAs one wait + fence and one commit
        __shared__ uint64_t dbar2, cbar2[8];
        if (tc::elect_one()) {
          tc::mbar_init(&dbar2, 1);
          for (int j = 0; j < 8; ++j) tc::mbar_init(&cbar2[j], 1);
          tc::mbar_fence_init();
          tc::mbar_arrive(&dbar2);
        }
        __syncwarp();
        const int group = per_commit == -14 ? 16 : 8;
        t0 = clock64();
        for (int i = 0; i < iters; i += group) {
          tc::mbar_wait(&dbar2, 0);
          if (per_commit == -13) tc::mbar_wait(&dbar2, 0);
          tc::tc_fence_after();
          const uint64_t bslot = tc::sw128_desc(tc::smem_u32(smem + 16384));
          if (tc::elect_one()) {
            for (int k = 0; k < group; ++k)
              tc::mma_ts(tbase, tbase + 256 + 8 * (k & 3), bslot + 2 * (k & 3), idesc, 1u);
            tc::mma_commit(&cbar2[(i / group) & 7]);
            if (per_commit == -13) tc::mma_commit(&cbar2[((i / group) + 4) & 7]);
          }
          __syncwarp();
        }
      } else
      if (per_commit <= -8 && per_commit >= -11 || per_commit == -17 || per_commit == -19 || per_commit == -20) {
        // variants -8 / -9: the network kernel's per-stage issue pattern -- a (satisfied) mbarrier
        // wait, tcgen05 fence, elect, 4 MMAs, a commit per stage; -9 also alternates the
        // accumulator slice every 4 stages and restarts accumulation like the body layers
        __shared__ uint64_t dbar, cbar[8];
        if (tc::elect_one()) {
          tc::mbar_init(&dbar, 1);
          for (int j = 0; j < 8; ++j) tc::mbar_init(&cbar[j], 1);
          tc::mbar_fence_init();
          tc::mbar_arrive(&dbar);
        }
        __syncwarp();
        t0 = clock64();
        for (int i = 0; i < iters; i += 4) {
          if (per_commit != -10) {            // -10: commit only
            if (per_commit == -19) tc::mbar_spin(&dbar, 0);   // -19: mbarrier.test_wait spin
            else tc::mbar_wait(&dbar, 0);
            if (per_commit != -17) tc::tc_fence_after();   // -17: wait + commit without the fence
          }
          const uint64_t bslot = tc::sw128_desc(tc::smem_u32(smem + 16384)) + (uint64_t)(((i >> 2) & 1) * 1024);
          const int st = (i >> 2) & 7;
          const uint32_t dcol = per_commit == -9 ? 128u * ((i >> 4) & 1) : 0u;
          const bool first = per_commit == -9 && ((i >> 2) & 3) == 0;
          if (tc::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc::mma_ts(tbase + dcol, tbase + 256 + 8 * k, bslot + 2 * k, idesc, (first && k == 0) ? 0u : 1u);
            if (per_commit == -20)              // -20: commit with a shared::cta address operand
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
                               (unsigned long long)__cvta_generic_to_shared(&cbar[st]))
                           : "memory");
            else if (per_commit != -11) tc::mma_commit(&cbar[st]);   // -11: wait + fence only
          }
          __syncwarp();
        }
      } else
      for (int i = 0; i < iters; i += 4) {
        if (tc::elect_one()) {
#pragma unroll
          // variant -7: B cycles through eight 16 KB slots (no operand reuse between stages)
          const uint64_t bslot =
              per_commit == -7 ? tc::sw128_desc(tc::smem_u32(smem + 49152 + ((i >> 2) & 7) * 16384)) : bdesc;
          for (int k = 0; k < 4; ++k) {
            const uint64_t bd = bslot + 2 * k;
            const uint64_t ad = adesc + 2 * k;
            const uint32_t at = tbase + 256 + 8 * k;
            if (ts) tc::mma_ts(tbase, at, bd, idesc, 1u);
            else tc::mma_ss(tbase, ad, bd, idesc, 1u);
          }
        }
        __syncwarp();
      }
      if (tc::elect_one()) tc::mma_commit(&bar);
      __syncwarp();
      tc::mbar_wait(&bar, 0);
      unsigned long long t1 = clock64();
      if (tid == 0) out[0] = t1 - t0;
      if (tid == 0) stop_flag = 1;
    } else if (per_commit < 0) {
      // variant: single thread, unrolled x4 with distinct K offsets, one commit
      if (tid == 0) {
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (ts) tc::mma_ts(tbase, tbase + 256 + 8 * k, bdesc + 2 * k, idesc, 1u);
            else tc::mma_ss(tbase, adesc + 2 * k, bdesc + 2 * k, idesc, 1u);
          }
        }
        tc::mma_commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, 0);
      unsigned long long t1 = clock64();
      if (tid == 0) out[0] = t1 - t0;
    } else
    for (int i = 0; i < iters; ++i) {
      if (tc::elect_one()) {
        if (ts) tc::mma_ts(tbase, tbase + 256, bdesc, idesc, 1u);
        else tc::mma_ss(tbase, adesc, bdesc, idesc, 1u);
        if ((i + 1) % per_commit == 0) tc::mma_commit(&bar);
      }
      __syncwarp();
      if ((i + 1) % per_commit == 0 && per_commit < iters) { tc::mbar_wait(&bar, phase); phase ^= 1; }
    }
    if (per_commit >= iters) { tc::mbar_wait(&bar, 0); }
    if (per_commit >= 0) {
      unsigned long long t1 = clock64();
      if (tid == 0) out[0] = t1 - t0;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

}  // namespace nedf

extern "C" int nedf_diag_mma_rate(int ts, int n, int iters, int per_commit, unsigned long long* out_dev) {
  using namespace nedf;
  size_t smem = 16384 + 32768 + 1024 + (per_commit <= -5 ? 8 * 16384 : 0);
  cudaFuncSetAttribute(mma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_rate_kernel<<<1, 128, smem>>>(ts, n, iters, per_commit, out_dev);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}

namespace nedf {

// L2 -> shared bulk-copy bandwidth probe: each CTA streams `total` bytes of
// `src` (wrapping inside `span` bytes) through a ring of `depth` stages of
// `stage` bytes with cp.async.bulk; out[blockIdx] = cycles taken.
__global__ void __launch_bounds__(32, 1) bulk_rate_kernel(const unsigned char* src, size_t span, int stage,
                                                           int depth, size_t total, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) tc::mbar_init(&bars[i], 1);
    tc::mbar_fence_init();
  }
  __syncwarp();
  const size_t n = total / stage;
  unsigned long long t0 = clock64();
  if (depth < 0) {
    // variant: `-depth` lanes each own one stage and stream independently
    const int lanes = -depth;
    if ((int)threadIdx.x < lanes) {
      const int slot = threadIdx.x;
      size_t off = ((size_t)(blockIdx.x * 7919 + slot * 131) * stage) % span;
      uint32_t ph = 0;
      for (size_t i = slot; i < n; i += lanes) {
        tc::mbar_expect_tx(&bars[slot], stage);
        tc::bulk_g2s(smem_raw + (size_t)slot * stage, src + off, stage, &bars[slot]);
        tc::mbar_wait(&bars[slot], ph);
        ph ^= 1;
        off += (size_t)lanes * stage;
        if (off + stage > span) off = (size_t)slot * stage;
      }
    }
    __syncwarp();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    return;
  }
  if (threadIdx.x == 0) {
    size_t off = ((size_t)blockIdx.x * 7919 * stage) % span;
    for (size_t i = 0; i < n + depth; ++i) {
      if (i >= (size_t)depth) {
        const size_t j = i - depth;
        tc::mbar_wait(&bars[j % depth], (j / depth) & 1);
      }
      if (i < n) {
        const int slot = i % depth;
        tc::mbar_expect_tx(&bars[slot], stage);
        tc::bulk_g2s(smem_raw + (size_t)slot * stage, src + off, stage, &bars[slot]);
        off += stage;
        if (off + stage > span) off = 0;
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

}  // namespace nedf

extern "C" int nedf_diag_bulk_rate(const void* src, size_t span, int stage, int depth, size_t total, int ctas,
                                   unsigned long long* out_dev) {
  using namespace nedf;
  size_t smem = (size_t)stage * (depth < 0 ? -depth : depth);
  if (depth > 16 || depth < -16 || smem > 200 * 1024) return NEDF_ERR_INVALID;
  cudaFuncSetAttribute(bulk_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  bulk_rate_kernel<<<ctas, 32, smem>>>((const unsigned char*)src, span, stage, depth, total, out_dev);
  return cudaGetLastError() == cudaSuccess ? NEDF_OK : NEDF_ERR_CUDA;
}
