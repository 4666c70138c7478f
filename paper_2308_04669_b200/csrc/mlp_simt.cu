// fp32 CUDA-core evaluation of the NeDF intersection network.
//
// Role: (1) the near-tie guard's re-evaluation path for rays the tensor-core
// kernel flags, (2) the path for model shapes the tcgen05 kernel does not
// cover, (3) NEDF_PREC_FP32.  Weights are the .nedm float32 values exactly
// (nn.py:245 stores f32; the reference widens them to f64 losslessly), the
// encoding is float64-accurate, activations and accumulation are fp32.
//
// Network (nn.py:115-135): x = W_h f + b_h ; 16 x { x += relu(W2 relu(W1 x + b1) + b2) } ;
// tail_a = W_a x + b_a (N_c coarse + alpha last), tail_b = W_b x + b_b (N_f fine).
//
// Tile: 32 rays x 128 threads; thread t owns output columns t and t+128 for all
// 32 rays (64 accumulators); activations live in shared memory, weights are
// read transposed [in][out] so a warp's weight loads are coalesced.
#include "common.cuh"
#include "encode.cuh"
#include "frame.cuh"

namespace nedf {

constexpr int kSimtRays = 32;
constexpr int kSimtThreads = 128;
constexpr int kLd = 256;

struct SimtSmem {
  float x[kSimtRays][kLd];
  float h[kSimtRays][kLd];
  float f[kSimtRays][64];
  double lray[kSimtRays][8];     // local o[3], d[3], t0, t1
  double wray[kSimtRays][6];     // world o[3], d[3]
  uint32_t pix[kSimtRays];
  uint32_t obj[kSimtRays];
  int valid[kSimtRays];
};

// acc[j][r] += sum_k in[r][k] * WT[k][o_j], k in [0, n_in) (n_in % 4 == 0)
__device__ __forceinline__ void dense_acc(const float (*in)[kLd], int n_in, const float* __restrict__ WT,
                                          int n_out, float acc[2][kSimtRays]) {
  const int o0 = threadIdx.x, o1 = threadIdx.x + kSimtThreads;
  const bool v0 = o0 < n_out, v1 = o1 < n_out;
  for (int k = 0; k < n_in; k += 4) {
    float w0[4], w1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w0[j] = v0 ? __ldg(WT + (size_t)(k + j) * n_out + o0) : 0.f;
      w1[j] = v1 ? __ldg(WT + (size_t)(k + j) * n_out + o1) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < kSimtRays; ++r) {
      float4 a = *reinterpret_cast<const float4*>(&in[r][k]);
      acc[0][r] = fmaf(a.x, w0[0], acc[0][r]);
      acc[0][r] = fmaf(a.y, w0[1], acc[0][r]);
      acc[0][r] = fmaf(a.z, w0[2], acc[0][r]);
      acc[0][r] = fmaf(a.w, w0[3], acc[0][r]);
      acc[1][r] = fmaf(a.x, w1[0], acc[1][r]);
      acc[1][r] = fmaf(a.y, w1[1], acc[1][r]);
      acc[1][r] = fmaf(a.z, w1[2], acc[1][r]);
      acc[1][r] = fmaf(a.w, w1[3], acc[1][r]);
    }
  }
}

// same with a [32][64] feature tile (head chunk)
__device__ __forceinline__ void dense_acc_feat(const float (*in)[64], const float* __restrict__ WT,
                                               int n_out, float acc[2][kSimtRays]) {
  const int o0 = threadIdx.x, o1 = threadIdx.x + kSimtThreads;
  const bool v0 = o0 < n_out, v1 = o1 < n_out;
  for (int k = 0; k < 64; k += 4) {
    float w0[4], w1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      w0[j] = v0 ? __ldg(WT + (size_t)(k + j) * n_out + o0) : 0.f;
      w1[j] = v1 ? __ldg(WT + (size_t)(k + j) * n_out + o1) : 0.f;
    }
#pragma unroll
    for (int r = 0; r < kSimtRays; ++r) {
      float4 a = *reinterpret_cast<const float4*>(&in[r][k]);
      acc[0][r] = fmaf(a.x, w0[0], acc[0][r]);
      acc[0][r] = fmaf(a.y, w0[1], acc[0][r]);
      acc[0][r] = fmaf(a.z, w0[2], acc[0][r]);
      acc[0][r] = fmaf(a.w, w0[3], acc[0][r]);
      acc[1][r] = fmaf(a.x, w1[0], acc[1][r]);
      acc[1][r] = fmaf(a.y, w1[1], acc[1][r]);
      acc[1][r] = fmaf(a.z, w1[2], acc[1][r]);
      acc[1][r] = fmaf(a.w, w1[3], acc[1][r]);
    }
  }
}

__device__ __forceinline__ void zero_acc(float acc[2][kSimtRays]) {
#pragma unroll
  for (int r = 0; r < kSimtRays; ++r) { acc[0][r] = 0.f; acc[1][r] = 0.f; }
}

// Evaluate one tile of <= 32 items of one model.
__device__ void simt_tile(SimtSmem& S, const DevModel& m, const RayJob& job, const OutSpec& out,
                          const uint32_t* pix_list, const uint32_t* obj_list, int n_items) {
  const int tid = threadIdx.x;
  const int F = m.d_feat;
  const bool logits_mode = out.feats != nullptr;          // features given instead of rays
  const bool logits_out = out.mode == OUT_LOGITS;
  if (tid < kSimtRays) {
    int v = tid < n_items;
    S.valid[tid] = v;
    uint32_t p = v ? pix_list[tid] : 0u, o = v ? obj_list[tid] : 0u;
    S.pix[tid] = p;
    S.obj[tid] = o;
    if (v && !logits_mode) {
      double wo[3], wd[3], lo[3], ld[3], t0 = 0, t1 = 0;
      item_local_ray(job, p, o, wo, wd, lo, ld);
      slab_clip(lo, ld, m.bmin, m.bmax, t0, t1);
      for (int a = 0; a < 3; ++a) {
        S.lray[tid][a] = lo[a]; S.lray[tid][3 + a] = ld[a];
        S.wray[tid][a] = wo[a]; S.wray[tid][3 + a] = wd[a];
      }
      S.lray[tid][6] = t0; S.lray[tid][7] = t1;
    }
  }
  __syncthreads();

  float acc[2][kSimtRays];
  zero_acc(acc);
  // ---- head: 16 chunks of 63 features (+1 zero pad column) ----
  for (int pt = 0; pt < kPoints; ++pt) {
    if (logits_mode) {
      for (int e = tid; e < kSimtRays * 64; e += kSimtThreads) {
        int r = e >> 6, k = e & 63;
        float v = 0.f;
        if (k < kPerPoint && S.valid[r]) v = out.feats[(size_t)S.pix[r] * kDin + pt * kPerPoint + k];
        S.f[r][k] = v;
      }
    } else if (tid < kSimtRays * 3) {
      int r = tid / 3, a = tid % 3;
      double enc[21];
      if (S.valid[r]) {
        double t0 = S.lray[r][6], t1 = S.lray[r][7];
        double t = t0 + (t1 - t0) * lin16(pt);
        double p = ((S.lray[r][a] + t * S.lray[r][3 + a]) - m.c[a]) / m.h[a];
        encode_coord_f64(p, enc);
      } else {
#pragma unroll
        for (int j = 0; j < 21; ++j) enc[j] = 0.0;
      }
#pragma unroll
      for (int j = 0; j < 21; ++j) S.f[r][21 * a + j] = (float)enc[j];
      if (a == 0) S.f[r][63] = 0.f;
    }
    __syncthreads();
    dense_acc_feat(S.f, m.wT + m.wT_off[0] + (size_t)pt * kPerPoint * F, F, acc);
    __syncthreads();
  }
  {
    const float* b = m.bias + m.b_off[0];
    for (int j = 0; j < 2; ++j) {
      int o = tid + j * kSimtThreads;
      if (o < F) {
        float bb = b[o];
        for (int r = 0; r < kSimtRays; ++r) S.x[r][o] = acc[j][r] + bb;
      }
    }
  }
  __syncthreads();
  // ---- residual blocks ----
  for (int blk = 0; blk < m.n_blocks; ++blk) {
    int l1 = 1 + 2 * blk, l2 = 2 + 2 * blk;
    zero_acc(acc);
    dense_acc(S.x, F, m.wT + m.wT_off[l1], F, acc);
    const float* b1 = m.bias + m.b_off[l1];
    for (int j = 0; j < 2; ++j) {
      int o = tid + j * kSimtThreads;
      if (o < F) {
        float bb = b1[o];
        for (int r = 0; r < kSimtRays; ++r) S.h[r][o] = fmaxf(acc[j][r] + bb, 0.f);
      }
    }
    __syncthreads();
    zero_acc(acc);
    dense_acc(S.h, F, m.wT + m.wT_off[l2], F, acc);
    const float* b2 = m.bias + m.b_off[l2];
    __syncthreads();
    for (int j = 0; j < 2; ++j) {
      int o = tid + j * kSimtThreads;
      if (o < F) {
        float bb = b2[o];
        for (int r = 0; r < kSimtRays; ++r) S.x[r][o] += fmaxf(acc[j][r] + bb, 0.f);
      }
    }
    __syncthreads();
  }
  // ---- tails: coarse+alpha -> h[:, 0:n_c+1], fine -> h[:, 128:128+n_f] ----
  const int la = m.n_layers - 2, lb = m.n_layers - 1;
  const int na = m.n_coarse + 1, nf = m.n_fine;
  zero_acc(acc);
  dense_acc(S.x, F, m.wT + m.wT_off[la], na, acc);
  for (int j = 0; j < 2; ++j) {
    int o = tid + j * kSimtThreads;
    if (o < na) {
      float bb = m.bias[m.b_off[la] + o];
      for (int r = 0; r < kSimtRays; ++r) S.h[r][o] = acc[j][r] + bb;
    }
  }
  zero_acc(acc);
  dense_acc(S.x, F, m.wT + m.wT_off[lb], nf, acc);
  for (int j = 0; j < 2; ++j) {
    int o = tid + j * kSimtThreads;
    if (o < nf) {
      float bb = m.bias[m.b_off[lb] + o];
      for (int r = 0; r < kSimtRays; ++r) S.h[r][128 + o] = acc[j][r] + bb;
    }
  }
  __syncthreads();
  // ---- decode (model.py:288-292): first maximum wins ----
  if (tid < kSimtRays && S.valid[tid]) {
    const int r = tid;
    if (logits_out) {
      size_t row = S.pix[r];
      for (int k = 0; k < m.n_coarse; ++k) out.lc[row * m.n_coarse + k] = S.h[r][k];
      for (int k = 0; k < nf; ++k) out.lf[row * nf + k] = S.h[r][128 + k];
      out.la[row] = S.h[r][m.n_coarse];
    } else {
      int c = 0;
      float best = S.h[r][0];
      for (int k = 1; k < m.n_coarse; ++k) if (S.h[r][k] > best) { best = S.h[r][k]; c = k; }
      int f = 0;
      best = S.h[r][128];
      for (int k = 1; k < nf; ++k) if (S.h[r][128 + k] > best) { best = S.h[r][128 + k]; f = k; }
      double wo[3] = {S.wray[r][0], S.wray[r][1], S.wray[r][2]};
      double wd[3] = {S.wray[r][3], S.wray[r][4], S.wray[r][5]};
      finish_ray(m, job, out, S.pix[r], S.obj[r], c, f, (double)S.h[r][m.n_coarse], wo, wd);
    }
  }
  __syncthreads();
}

// Grid-stride over the 32-item tiles of every group's list.
__global__ void __launch_bounds__(kSimtThreads)
mlp_fp32_kernel(GroupTable gt, ListSet ls, RayJob job, OutSpec out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SimtSmem& S = *reinterpret_cast<SimtSmem*>(smem_raw);
  __shared__ int s_tiles[65];
  if (threadIdx.x == 0) {
    int cum = 0;
    s_tiles[0] = 0;
    for (int g = 0; g < ls.n_groups && g < 64; ++g) {
      cum += (ls.count[g] + kSimtRays - 1) / kSimtRays;
      s_tiles[g + 1] = cum;
    }
  }
  __syncthreads();
  const int ng = ls.n_groups < 64 ? ls.n_groups : 64;
  const int total = s_tiles[ng];
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int g = 0;
    while (t >= s_tiles[g + 1]) ++g;
    int lt = t - s_tiles[g];
    int n = ls.count[g] - lt * kSimtRays;
    n = n < kSimtRays ? n : kSimtRays;
    const int64_t base = ls.offset[g] + (int64_t)lt * kSimtRays;
    simt_tile(S, gt.models[g], job, out, ls.pix + base, ls.obj + base, n);
  }
}

size_t simt_smem_bytes() { return sizeof(SimtSmem); }

cudaError_t launch_mlp_fp32(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                            int n_sms, cudaStream_t stream) {
  static bool configured_dev[kMaxDevices] = {};
  bool& configured = configured_dev[current_device()];
  size_t smem = sizeof(SimtSmem);
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(mlp_fp32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  int grid = n_sms * 3;
  mlp_fp32_kernel<<<grid, kSimtThreads, smem, stream>>>(gt, ls, job, out);
  return cudaGetLastError();
}

}  // namespace nedf
