// fp32-accurate GEMM on the 5th-generation tensor cores for the trainer
// (train.cu): C[M][N] (+)= op(A)[M][K] . op(B)[N][K]^T, fp32 in and out.
//
// The reference trains in float64 numpy (nn.py:138-232); the trainer's
// gradients must stay at fp32 accuracy (tests/test_train.py), so every product
// is split like the near-tie guard's (guard_tc.cu): x = x_hi + x_lo with x_hi =
// x truncated to tf32 (what kind::tf32 reads from the raw fp32 value) and x_lo
// the remainder rounded to tf32; three MMAs per k-step accumulate
//   A_hi B_hi              into two alternating "main" accumulators (by K chunk:
//                          fewer additions per accumulator keep the tensor
//                          core's accumulation rounding at the fp32 level)
//   A_hi B_lo + A_lo B_hi  into a "cross" accumulator
// and the epilogue sums them in fp32.  The dropped A_lo B_lo term is ~2^-22 of
// a product.
//
// Operands are row-major fp32 with either layout (op = transpose or not): the
// loader threads read them with vector loads, split each value into its hi /
// lo tiles and store both into 128B-swizzled K-major shared-memory atoms (32
// fp32 of K per 128-byte row), so no transposed copy is ever written to global
// memory.  One CTA computes a 128 x 64 tile: 8 loader warps stream 32-wide K
// chunks (global -> registers -> split -> a 4-stage shared-memory ring, mbarrier
// full / empty handshakes), one warp issues the M128 x N64 x K8 MMAs, and warps
// 0-3 read the accumulators back with tcgen05.ld for a coalesced store.  Long K
// (the weight gradients reduce over the batch) is split across CTAs into a
// workspace and summed in a fixed order by a second kernel (deterministic).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "frame.cuh"
#include "tc_ptx.cuh"

namespace nedf {
namespace {

constexpr int kBM = 128, kBN = 64, kBK = 32;
constexpr uint32_t kATile = kBM * 128;          // 16 KB: [128 rows][32 fp32]
constexpr uint32_t kBTile = kBN * 128;          // 8 KB
constexpr uint32_t kStage = 2 * kATile + 2 * kBTile;   // A_raw, A_lo, B_raw, B_lo: 48 KB
constexpr int kStages = 4;                      // 192 KB ring
static_assert(kStages * kStage >= kBM * (kBN + 1) * 4, "epilogue tile fits the ring");
constexpr int kLoadWarps = 8;
constexpr int kThreads = 32 * kLoadWarps;       // loader threads (+ one MMA warp)

struct GemmArgs {
  const float* A;
  const float* B;
  float* C;                  // C, or the split-K workspace [splits][M][N]
  int M, N, K;
  int lda, ldb, ldc;
  int ta, tb;                // 1: op(A)[m][k] = A[k * lda + m] (else A[m * lda + k]); same for B
  float beta;                // C = acc + beta * C (no split)
  int k_per_split;           // multiple of kBK
};

__device__ __forceinline__ float tf32_lo(float x) {
  const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  return __uint_as_float((__float_as_uint(x - hi) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ uint32_t sw_off(int row, int k) {
  return (uint32_t)row * 128u + (((uint32_t)(k >> 2) ^ (uint32_t)(row & 7)) << 4) + ((k & 3) << 2);
}

// One operand's K chunk [rows][kBK], fetched into registers (rows beyond `rows_total` and K
// beyond `k_end` read as zero) and later stored into its raw / lo tiles.  Non-transposed:
// each item is 4 consecutive K of a row (one float4 when aligned); transposed: 4
// consecutive rows of one K.
template <int ROWS>
struct Chunk {
  static constexpr int kItems = ROWS * kBK / 4 / kThreads;   // float4 items per thread
  float4 v[kItems];

  __device__ __forceinline__ void fetch(const float* __restrict__ P, int ld, int trans, int row0, int rows_total,
                                        int k0, int k_end) {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int it = threadIdx.x + j * kThreads;
      int gr, gk;
      const float* src;
      bool full;
      if (!trans) {
        gr = row0 + it / (kBK / 4);
        gk = k0 + (it % (kBK / 4)) * 4;
        src = P + (size_t)gr * ld + gk;
        full = gr < rows_total && gk + 3 < k_end;
      } else {
        gk = k0 + it / (ROWS / 4);
        gr = row0 + (it % (ROWS / 4)) * 4;
        src = P + (size_t)gk * ld + gr;
        full = gk < k_end && gr + 3 < rows_total;
      }
      if (full && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        v[j] = __ldg(reinterpret_cast<const float4*>(src));
      } else {
        float t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool ok = trans ? (gk < k_end && gr + i < rows_total) : (gr < rows_total && gk + i < k_end);
          t[i] = ok ? src[trans ? i : i] : 0.f;
        }
        v[j] = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
  }

  __device__ __forceinline__ void put(int trans, unsigned char* raw, unsigned char* lo) const {
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int it = threadIdx.x + j * kThreads;
      if (!trans) {
        const int r = it / (kBK / 4), kk = (it % (kBK / 4)) * 4;
        const uint32_t o = sw_off(r, kk);
        *reinterpret_cast<float4*>(raw + o) = v[j];
        *reinterpret_cast<float4*>(lo + o) = make_float4(tf32_lo(v[j].x), tf32_lo(v[j].y), tf32_lo(v[j].z), tf32_lo(v[j].w));
      } else {
        const int kk = it / (ROWS / 4), r = (it % (ROWS / 4)) * 4;
        const float t[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t o = sw_off(r + i, kk);
          *reinterpret_cast<float*>(raw + o) = t[i];
          *reinterpret_cast<float*>(lo + o) = tf32_lo(t[i]);
        }
      }
    }
  }
};

}  // namespace

__global__ void __launch_bounds__(kThreads + 32, 1) gemm_tf32x3_kernel(GemmArgs g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full_bar[kStages], empty_bar[kStages], done_bar;
  __shared__ uint32_t tmem_base_s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * kBN, split = blockIdx.z;
  const int k_begin = split * g.k_per_split;
  const int k_end = min(g.K, k_begin + g.k_per_split);
  const int n_chunks = max(0, (k_end - k_begin + kBK - 1) / kBK);
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&full_bar[i], kLoadWarps);
      tc::mbar_init(&empty_bar[i], 1);
    }
    tc::mbar_init(&done_bar, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<256>(&tmem_base_s);      // main 0 / main 1 / cross: 3 x 64 columns
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  auto stage = [&](int s) { return smem + (size_t)s * kStage; };
  if (warp < kLoadWarps) {
    // ---- loaders: chunk c -> registers -> (wait for the slot) -> raw / lo tiles, kStages ahead
    Chunk<kBM> ra;
    Chunk<kBN> rb;
    for (int c = 0; c < n_chunks; ++c) {
      const int s = c % kStages;
      const int k0 = k_begin + c * kBK;
      ra.fetch(g.A, g.lda, g.ta, m0, g.M, k0, k_end);
      rb.fetch(g.B, g.ldb, g.tb, n0, g.N, k0, k_end);
      if (c >= kStages) tc::mbar_wait(&empty_bar[s], ((c / kStages) - 1) & 1);
      unsigned char* st = stage(s);
      ra.put(g.ta, st, st + kATile);
      rb.put(g.tb, st + 2 * kATile, st + 2 * kATile + kBTile);
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[s]);
    }
  } else {
    // ---- MMA issuer (warp kLoadWarps)
    const uint32_t idesc = tc::idesc_tf32(kBM, kBN);
    for (int c = 0; c < n_chunks; ++c) {
      const int s = c % kStages;
      tc::mbar_wait(&full_bar[s], (c / kStages) & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t sa = tc::smem_u32(stage(s));
        const uint64_t a_raw = tc::sw128_desc(sa), a_lo = tc::sw128_desc(sa + kATile);
        const uint64_t b_raw = tc::sw128_desc(sa + 2 * kATile), b_lo = tc::sw128_desc(sa + 2 * kATile + kBTile);
        const uint32_t d_main = tbase + 64 * (c & 1), d_cross = tbase + 128;
#pragma unroll
        for (int ks = 0; ks < kBK / 8; ++ks) {
          const uint32_t o = (ks * 32) >> 4;
          tc::mma_ss_tf32(d_main, a_raw + o, b_raw + o, idesc, (c < 2 && ks == 0) ? 0u : 1u);
          tc::mma_ss_tf32(d_cross, a_raw + o, b_lo + o, idesc, (c == 0 && ks == 0) ? 0u : 1u);
          tc::mma_ss_tf32(d_cross, a_lo + o, b_raw + o, idesc, 1u);
        }
        tc::mma_commit(&empty_bar[s]);
        if (c == n_chunks - 1) tc::mma_commit(&done_bar);
      }
      __syncwarp();
    }
  }
  if (n_chunks > 0) tc::mbar_wait(&done_bar, 0);
  tc::tc_fence_after();
  __syncthreads();
  // ---- epilogue: TMEM -> registers (warps 0-3, thread = row) -> a padded shared tile (the
  // ring is free now) -> coalesced row stores by all loader warps
  constexpr int kLd = kBN + 1;
  float* tile = reinterpret_cast<float*>(smem);
  if (warp < 4) {
    const int r = 32 * warp + lane;
    const uint32_t lb = (uint32_t)(32 * warp) << 16;
    for (int j0 = 0; j0 < kBN; j0 += 16) {
      uint32_t r0[16], r1[16], rc[16];
      tc::tmem_ld16(tbase + lb + j0, r0);
      tc::tmem_ld16(tbase + lb + 64 + j0, r1);
      tc::tmem_ld16(tbase + lb + 128 + j0, rc);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j)
        tile[r * kLd + j0 + j] = n_chunks == 0 ? 0.f
                                 : (__uint_as_float(r0[j]) + (n_chunks > 1 ? __uint_as_float(r1[j]) : 0.f)) +
                                       __uint_as_float(rc[j]);
    }
  }
  __syncthreads();
  float* out = g.C + (size_t)split * ((size_t)g.M * g.ldc);
  const bool use_beta = gridDim.z == 1 && g.beta != 0.f;
  for (int e = tid; e < kBM * kBN; e += kThreads + 32) {
    const int r = e / kBN, col = e % kBN;
    const int gr = m0 + r, gc = n0 + col;
    if (gr < g.M && gc < g.N) {
      float* dst = out + (size_t)gr * g.ldc + gc;
      const float v = tile[r * kLd + col];
      *dst = use_beta ? v + g.beta * *dst : v;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<256>(tbase);
}

// C[m][n] = sum over splits of ws[s][m][n] (+ beta C), in split order
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ C, int M, int N, int ldc,
                                     int splits, float beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i % N);
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += ws[((size_t)k * M + m) * ldc + n];
    float* dst = C + (size_t)m * ldc + n;
    *dst = beta != 0.f ? s + beta * *dst : s;
  }
}

// C[M][N] (+)= op(A) op(B)^T.  ws: workspace of at least ws_floats floats for split K (may be
// NULL: no split).
cudaError_t gemm_tf32x3(const float* A, int lda, int ta, const float* B, int ldb, int tb, float* C, int ldc, int M,
                        int N, int K, float beta, float* ws, size_t ws_floats, int n_sms, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  static bool configured[kMaxDevices] = {};
  const size_t smem = kStages * kStage + 1024;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!configured[dev % kMaxDevices]) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tf32x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured[dev % kMaxDevices] = true;
  }
  const int gm = (M + kBM - 1) / kBM, gn = (N + kBN - 1) / kBN;
  // split K until the grid covers the SMs (chunks of at least 4 x kBK)
  int splits = 1;
  if (ws != nullptr && ldc == N) {
    while (gm * gn * splits * 2 <= n_sms && (K + splits * 2 - 1) / (splits * 2) >= 4 * kBK &&
           (size_t)(splits * 2) * M * N <= ws_floats)
      splits *= 2;
  }
  int kps = (K + splits - 1) / splits;
  kps = (kps + kBK - 1) / kBK * kBK;
  splits = (K + kps - 1) / kps;
  if (splits < 1) splits = 1;
  GemmArgs g;
  g.A = A; g.B = B; g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc; g.ta = ta; g.tb = tb;
  g.beta = beta;
  g.k_per_split = kps;
  g.C = splits > 1 ? ws : C;
  gemm_tf32x3_kernel<<<dim3(gm, gn, splits), kThreads + 32, smem, st>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = (int64_t)M * N;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)n_sms * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, C, M, N, ldc, splits, beta);
  return cudaGetLastError();
}

}  // namespace nedf
