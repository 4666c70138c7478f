// fp32-accurate GEMM on the 5th-generation tensor cores for the trainer
// (train.cu): C[M][N] (+)= op(A)[M][K] . op(B)[N][K]^T, fp32 in and out.
//
// The reference trains in float64 numpy (nn.py:138-232); the trainer's
// gradients must stay at fp32 accuracy (tests/test_train.py), so every product
// is split like the near-tie guard's (guard_tc.cu): x = x_hi + x_lo with x_hi =
// x truncated to tf32 (what kind::tf32 reads from the raw fp32 value) and x_lo
// the remainder rounded to tf32; three MMAs per k-step accumulate
//   A_hi B_hi              into 1-7 rotating "main" accumulators (by K chunk:
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
#ifndef NEDF_GEMM_REGBUFS
#define NEDF_GEMM_REGBUFS 2
#endif
constexpr int kRegBufs = NEDF_GEMM_REGBUFS;     // K chunks in flight per loader thread (2 measured best: 3 and 4 are slower)
constexpr int kMaxMains = 7;                    // main accumulators (rotating by K chunk) + 1 cross: 512 TMEM columns
constexpr int kChunksPerMain = 16;              // at most ~64 MMAs accumulate into one
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
  GemmEpi epi;               // fused elementwise epilogue
};

// the fused epilogue on one output element (row r, column c) with v = acc (+ beta C)
__device__ __forceinline__ void epi_store(const GemmEpi& e, float* C, int ldc, int r, int c, float v) {
  const size_t i = (size_t)r * ldc + c;
  switch (e.mode) {
    case GEMM_EPI_BIAS: C[i] = v + e.bias[c]; break;
    case GEMM_EPI_BIAS_RELU: { const float a = v + e.bias[c]; C[i] = a; e.aux[i] = fmaxf(a, 0.f); break; }
    case GEMM_EPI_RESIDUAL: { const float a = v + e.bias[c]; C[i] = a; e.aux[i] = e.in[i] + fmaxf(a, 0.f); break; }
    case GEMM_EPI_MASK: C[i] = e.in[i] > 0.f ? v : 0.f; break;
    case GEMM_EPI_MASK_AUX: C[i] = v; e.aux[i] = e.in[i] > 0.f ? v : 0.f; break;
    default: C[i] = v;
  }
}

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

// The output tile (in shared memory, [kBM][kBN + 1]) to C / the split-K workspace with the
// fused epilogue MODE (-1: raw partial), 4 consecutive columns of a row per item: float4
// loads / stores when the run is whole and aligned, scalar otherwise.
template <int MODE>
__device__ __forceinline__ void store_tile(const GemmArgs& g, const float* tile, int m0, int n0, int split) {
  constexpr int kLd = kBN + 1, kNT = kThreads + 32;
  constexpr bool kIn = MODE == GEMM_EPI_RESIDUAL || MODE == GEMM_EPI_MASK || MODE == GEMM_EPI_MASK_AUX;
  constexpr bool kBias = MODE == GEMM_EPI_BIAS || MODE == GEMM_EPI_BIAS_RELU || MODE == GEMM_EPI_RESIDUAL;
  constexpr bool kAux = MODE == GEMM_EPI_BIAS_RELU || MODE == GEMM_EPI_RESIDUAL || MODE == GEMM_EPI_MASK_AUX;
  const GemmEpi& ep = g.epi;
  float* out = g.C + (size_t)split * ((size_t)g.M * g.ldc);
  const bool beta = MODE >= 0 && g.beta != 0.f;
  auto f = [&](float x, float cold, float xin, float bb, float& aux) {
    if (beta) x += g.beta * cold;
    if (MODE == GEMM_EPI_BIAS) return x + bb;
    if (MODE == GEMM_EPI_BIAS_RELU) { const float a = x + bb; aux = fmaxf(a, 0.f); return a; }
    if (MODE == GEMM_EPI_RESIDUAL) { const float a = x + bb; aux = xin + fmaxf(a, 0.f); return a; }
    if (MODE == GEMM_EPI_MASK) return xin > 0.f ? x : 0.f;
    if (MODE == GEMM_EPI_MASK_AUX) { aux = xin > 0.f ? x : 0.f; return x; }
    return x;
  };
  const bool vec_ok = (g.ldc & 3) == 0 && ((reinterpret_cast<uintptr_t>(out) | (kIn ? reinterpret_cast<uintptr_t>(ep.in) : 0) |
                                            (kAux ? reinterpret_cast<uintptr_t>(ep.aux) : 0)) & 15) == 0 &&
                      (!kBias || (reinterpret_cast<uintptr_t>(ep.bias) & 15) == 0);
  for (int e = threadIdx.x; e < kBM * kBN / 4; e += kNT) {
    const int r = e / (kBN / 4), c4 = (e % (kBN / 4)) * 4;
    const int gr = m0 + r, gc = n0 + c4;
    if (gr >= g.M || gc >= g.N) continue;
    const size_t at = (size_t)gr * g.ldc + gc;
    const float* t = tile + r * kLd + c4;
    if (vec_ok && gc + 4 <= g.N) {
      float4 cold = make_float4(0.f, 0.f, 0.f, 0.f), xin = cold, bb = cold, aux = cold;
      if (beta) cold = *reinterpret_cast<const float4*>(out + at);
      if (kIn) xin = *reinterpret_cast<const float4*>(ep.in + at);
      if (kBias) bb = *reinterpret_cast<const float4*>(ep.bias + gc);
      float4 o;
      o.x = f(t[0], cold.x, xin.x, bb.x, aux.x);
      o.y = f(t[1], cold.y, xin.y, bb.y, aux.y);
      o.z = f(t[2], cold.z, xin.z, bb.z, aux.z);
      o.w = f(t[3], cold.w, xin.w, bb.w, aux.w);
      *reinterpret_cast<float4*>(out + at) = o;
      if (kAux) *reinterpret_cast<float4*>(ep.aux + at) = aux;
    } else {
      for (int j = 0; j < 4 && gc + j < g.N; ++j) {
        float aux = 0.f;
        const float o = f(t[j], beta ? out[at + j] : 0.f, kIn ? ep.in[at + j] : 0.f, kBias ? ep.bias[gc + j] : 0.f, aux);
        out[at + j] = o;
        if (kAux) ep.aux[at + j] = aux;
      }
    }
  }
}

__device__ unsigned long long g_gemm_trace[16];
__device__ int g_gemm_trace_on;
#define GEMM_TRACE(i)                                                                                 \
  do {                                                                                                \
    if (g_gemm_trace_on && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) g_gemm_trace[i] = clock64(); \
  } while (0)

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
  if (tid == 0) GEMM_TRACE(0);
  const int mains = max(1, min(kMaxMains, (n_chunks + kChunksPerMain - 1) / kChunksPerMain));
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      tc::mbar_init(&full_bar[i], kLoadWarps);
      tc::mbar_init(&empty_bar[i], 1);
    }
    tc::mbar_init(&done_bar, 1);
    tc::mbar_fence_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_s);      // kMains main accumulators + cross: 8 x 64 columns
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = tmem_base_s;
  if (tid == 0) GEMM_TRACE(1);
  auto stage = [&](int s) { return smem + (size_t)s * kStage; };
  if (warp < kLoadWarps) {
    // ---- loaders: chunk c -> registers -> (wait for the slot) -> raw / lo tiles, kStages ahead;
    // kRegBufs register buffers, so chunks c + 1 .. c + kRegBufs are in flight while chunk c is
    // stored (the loads are latency-bound: a chunk is ~24 B of global reads per thread)
    Chunk<kBM> ra[kRegBufs];
    Chunk<kBN> rb[kRegBufs];
    auto fetch = [&](int c, Chunk<kBM>& a, Chunk<kBN>& b) {
      const int k0 = k_begin + c * kBK;
      a.fetch(g.A, g.lda, g.ta, m0, g.M, k0, k_end);
      b.fetch(g.B, g.ldb, g.tb, n0, g.N, k0, k_end);
    };
    auto store = [&](int c, const Chunk<kBM>& a, const Chunk<kBN>& b) {
      const int s = c % kStages;
      if (c >= kStages) tc::mbar_wait(&empty_bar[s], ((c / kStages) - 1) & 1);
      unsigned char* st = stage(s);
      a.put(g.ta, st, st + kATile);
      b.put(g.tb, st + 2 * kATile, st + 2 * kATile + kBTile);
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full_bar[s]);
    };
#pragma unroll
    for (int i = 0; i < kRegBufs; ++i)
      if (i < n_chunks) fetch(i, ra[i], rb[i]);
    for (int c = 0; c < n_chunks; c += kRegBufs) {
#pragma unroll
      for (int i = 0; i < kRegBufs; ++i) {
        if (c + i < n_chunks) {
          store(c + i, ra[i], rb[i]);
          if (c + i + kRegBufs < n_chunks) fetch(c + i + kRegBufs, ra[i], rb[i]);
        }
      }
    }
  } else {
    // ---- MMA issuer (warp kLoadWarps)
    const uint32_t idesc = tc::idesc_tf32(kBM, kBN);
    for (int c = 0; c < n_chunks; ++c) {
      const int s = c % kStages;
      tc::mbar_wait(&full_bar[s], (c / kStages) & 1);
      tc::tc_fence_after();
      if (lane == 0 && c < 8) GEMM_TRACE(2 + c);
      if (tc::elect_one()) {
        const uint32_t sa = tc::smem_u32(stage(s));
        const uint64_t a_raw = tc::sw128_desc(sa), a_lo = tc::sw128_desc(sa + kATile);
        const uint64_t b_raw = tc::sw128_desc(sa + 2 * kATile), b_lo = tc::sw128_desc(sa + 2 * kATile + kBTile);
        const uint32_t d_main = tbase + 64 * (1 + c % mains), d_cross = tbase;
#pragma unroll
        for (int ks = 0; ks < kBK / 8; ++ks) {
          const uint32_t o = (ks * 32) >> 4;
          tc::mma_ss_tf32(d_main, a_raw + o, b_raw + o, idesc, (c < mains && ks == 0) ? 0u : 1u);
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
  if (tid == 0) GEMM_TRACE(10);
  __syncthreads();
  // ---- epilogue: TMEM -> registers (warps 0-3, thread = row) -> a padded shared tile (the
  // ring is free now) -> coalesced row stores by all loader warps
  constexpr int kLd = kBN + 1;
  float* tile = reinterpret_cast<float*>(smem);
  if (warp < 4) {
    const int r = 32 * warp + lane;
    const uint32_t lb = (uint32_t)(32 * warp) << 16;
    const int used = min(n_chunks, mains);                    // main accumulators written
    for (int j0 = 0; j0 < kBN; j0 += 16) {
      // the cross accumulator and up to three mains per wait
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
      for (int i0 = 0; i0 <= used; i0 += 4) {
        uint32_t rv[4][16];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i0 + q <= used) tc::tmem_ld16(tbase + lb + 64 * (i0 + q) + j0, rv[q]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (i0 + q <= used && n_chunks > 0) {
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] += __uint_as_float(rv[q][j]);
          }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) tile[r * kLd + j0 + j] = acc[j];
    }
    if (tid == 0) GEMM_TRACE(12);
  }
  __syncthreads();
  if (tid == 0) GEMM_TRACE(13);
  const GemmEpi& ep = g.epi;
  switch (gridDim.z > 1 ? -1 : ep.mode) {
    case -1: store_tile<-1>(g, tile, m0, n0, split); break;     // split-K partial: the reduce kernel finishes
    case GEMM_EPI_BIAS: store_tile<GEMM_EPI_BIAS>(g, tile, m0, n0, split); break;
    case GEMM_EPI_BIAS_RELU: store_tile<GEMM_EPI_BIAS_RELU>(g, tile, m0, n0, split); break;
    case GEMM_EPI_RESIDUAL: store_tile<GEMM_EPI_RESIDUAL>(g, tile, m0, n0, split); break;
    case GEMM_EPI_MASK: store_tile<GEMM_EPI_MASK>(g, tile, m0, n0, split); break;
    case GEMM_EPI_MASK_AUX: store_tile<GEMM_EPI_MASK_AUX>(g, tile, m0, n0, split); break;
    default: store_tile<GEMM_EPI_NONE>(g, tile, m0, n0, split);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tid == 0) GEMM_TRACE(11);
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

extern "C" int nedf_diag_gemm_trace(int enable, unsigned long long* out) {
  if (enable >= 0 && cudaMemcpyToSymbol(g_gemm_trace_on, &enable, sizeof(int)) != cudaSuccess) return NEDF_ERR_CUDA;
  if (out && cudaMemcpyFromSymbol(out, g_gemm_trace, 16 * sizeof(unsigned long long)) != cudaSuccess)
    return NEDF_ERR_CUDA;
  return NEDF_OK;
}

// C[m][n] = sum over splits of ws[s][m][n] (+ beta C), in split order
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, float* __restrict__ C, int M, int N, int ldc,
                                     int splits, float beta, GemmEpi epi) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / N), n = (int)(i % N);
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += ws[((size_t)k * M + m) * ldc + n];
    if (beta != 0.f) s += beta * C[(size_t)m * ldc + n];
    epi_store(epi, C, ldc, m, n, s);
  }
}

// C[M][N] (+)= op(A) op(B)^T.  ws: workspace of at least ws_floats floats for split K (may be
// NULL: no split).
cudaError_t gemm_tf32x3(const float* A, int lda, int ta, const float* B, int ldb, int tb, float* C, int ldc, int M,
                        int N, int K, float beta, float* ws, size_t ws_floats, int n_sms, cudaStream_t st,
                        const GemmEpi& epi) {
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
  g.epi = epi;
  g.C = splits > 1 ? ws : C;
  gemm_tf32x3_kernel<<<dim3(gm, gn, splits), kThreads + 32, smem, st>>>(g);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = (int64_t)M * N;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)n_sms * 8);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(ws, C, M, N, ldc, splits, beta, epi);
  return cudaGetLastError();
}

}  // namespace nedf

// diagnostics / tests: C[M][N] = op(A) op(B)^T with the trainer's GEMM (ws may be NULL)
extern "C" int nedf_diag_gemm(const float* a, int lda, int ta, const float* b, int ldb, int tb, float* c, int ldc,
                              int m, int n, int k, float beta, float* ws, int64_t ws_floats, void* stream) {
  using namespace nedf;
  if (!a || !b || !c || m < 0 || n < 0 || k < 0) return NEDF_ERR_INVALID;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return gemm_tf32x3(a, lda, ta, b, ldb, tb, c, ldc, m, n, k, beta, ws, ws ? (size_t)ws_floats : 0, sms,
                     (cudaStream_t)stream) == cudaSuccess
             ? NEDF_OK
             : NEDF_ERR_CUDA;
}
