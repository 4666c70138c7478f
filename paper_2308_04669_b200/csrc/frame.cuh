// Host-visible declarations of the frame kernels and the network launchers.
#pragma once

#include "common.cuh"

namespace nedf {

// One-time kernel setup (attributes, occupancy queries) is cached per device: one
// process may drive several GPUs, each through its own context.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d >= 0 && d < kMaxDevices ? d : 0;
}

// STEP 1 pairs held back by front-first culling (setup_pixel): evaluated after
// the pixel's nearest-bound pair only if their depth lower bound can still win
struct DeferList {
  uint32_t* pix;                 // NULL: culling off
  uint32_t* obj;
  float* low;                    // fp32 lower bound of the pair's world depth
  int* count;
};

struct FrameJob {
  RayJob ray;                    // camera / light / object tables
  const NedfField* fields;       // device copy of the field nodes
  int n_objs;
  int n_pix;
  unsigned long long* key;       // per-pixel packed z-key (STEP 1 or STEP 3)
  double* depth;                 // per-pixel depth
  int* id;                       // per-pixel user id
  float* rgb;
  float* shadow;
  float* image;
  double* planes;                // optional [n_objs][n_pix]
  double eps;                    // shadow epsilon
  double beta;
  double sigma_threshold;        // < 0: per-field default
  int resample, resample_samples;
  double clear[3];
  unsigned long long* stats;     // [0] covered, [1] outliers, [2] evals, [3] guarded, [4] exact box tests,
                                 // [5] pairs culled
  DeferList defer;               // STEP 1 front-first culling (RAY_PRIMARY without a plane cache)
};

// exact = 1: every box test in float64 (no certified fp32 clip)
cudaError_t launch_setup(const FrameJob& fj, const GroupTable& gt, const ListSet& ls, int mode, int exact, int n_sms,
                         cudaStream_t st);
// fused STEP 1 resolve + STEP 2 + shadow := 1 + STEP 3 lists of the first light (smode < 0: none)
cudaError_t launch_resolve_shade(const FrameJob& fj, const GroupTable& gt, const ListSet& ls, const FrameJob& sj,
                                 int smode, int exact, int n_sms, cudaStream_t st);
// the deferred pairs whose lower bound does not exceed the pixel's z-key depth -> ls (counts reset by the caller)
cudaError_t launch_defer_filter(const FrameJob& fj, const ListSet& ls, int n_sms, cudaStream_t st);
cudaError_t launch_step1_resolve(const FrameJob& fj, const GroupTable& gt, int n_sms, cudaStream_t st);
cudaError_t launch_recombine(const FrameJob& fj, int n_sms, cudaStream_t st);
cudaError_t launch_shade(const FrameJob& fj, const GroupTable& gt, int n_sms, cudaStream_t st);
// image != NULL: also image = rgb * shadow (the frame's last light)
cudaError_t launch_shadow_resolve(const FrameJob& fj, const GroupTable& gt, int mode, float* image, int n_sms,
                                  cudaStream_t st);
cudaError_t launch_fill(float* buf, int64_t n, float v, int n_sms, cudaStream_t st);
cudaError_t launch_composite(const float* rgb, const float* shadow, float* image, int64_t n, int n_sms,
                             cudaStream_t st);
cudaError_t launch_explicit_setup(const RayJob& job, const GroupTable& gt, const ListSet& ls, const OutSpec& out,
                                  int64_t n, int n_sms, cudaStream_t st);
cudaError_t launch_iota_setup(const ListSet& ls, int64_t n, int n_sms, cudaStream_t st);

// network
size_t simt_smem_bytes();
cudaError_t launch_mlp_fp32(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                            int n_sms, cudaStream_t stream);

// fp32 network with streamed weights (mlp_fp32s.cu), paper-shaped models
cudaError_t launch_mlp_fp32_stream(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                   int n_sms, int rays_per_cta, cudaStream_t stream);
// cluster-split fp32 network (mlp_fp32c.cu) for the guard's small batches
// (cluster = 4 or 8 CTAs; the image must have been packed for the same cluster size)
cudaError_t launch_mlp_fp32_cluster(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                                    int n_sms, int cluster, cudaStream_t stream);
cudaError_t fp32_pack_cluster(const float* params_host, int d_in, int d_feat, int n_blocks, int n_coarse, int n_fine,
                              int cluster, float** dev);
cudaError_t fp32_pack_stream(const float* params_host, int d_in, int d_feat, int n_blocks, int n_coarse, int n_fine,
                             float** dev);

// tensor-core network (mlp_tc.cu): evaluates `ls`; with guard > 0, rays whose
// top-2 margins fall below guard * max|logit| are appended to `redo` instead
// of being written.
struct TcArgs {
  GroupTable gt;
  ListSet ls;
  ListSet redo;
  RayJob job;
  OutSpec out;
  float guard;
  int use_guard;
  int shadow_cert;               // STEP 3: finish flagged pairs whose shadow decision is certain (no guard)
  int* tile_counter;
};
// tcgen05 guard (guard_tc.cu): fp32-accurate re-evaluation of `ls` (the redo list) in 4-CTA clusters
bool guard_tc_available();
// max_tiles16 >= 0: return at once when the batch has more 16-ray tiles (mlp_precise takes it)
cudaError_t launch_guard_tc(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                            int n_sms, cudaStream_t stream, int max_tiles16 = -1);
cudaError_t guard_tc_pack(const float* params_host, int d_in, int d_feat, int n_blocks, int n_coarse, int n_fine,
                          void** dev);
// fp32-accurate split-tf32 tcgen05 GEMM (train_gemm.cu): C[M][N] (+)= op(A)[M][K] op(B)[N][K]^T,
// ta / tb: operand stored transposed; ws (optional) for split K over the CTAs; a fused
// elementwise epilogue on v = acc (+ beta C), all arrays [M][ldc]:
enum GemmEpiMode : int {
  GEMM_EPI_NONE = 0,        // C = v
  GEMM_EPI_BIAS = 1,        // C = v + bias[col]
  GEMM_EPI_BIAS_RELU = 2,   // C = a = v + bias[col]; aux = relu(a)
  GEMM_EPI_RESIDUAL = 3,    // C = a = v + bias[col]; aux = in + relu(a)
  GEMM_EPI_MASK = 4,        // C = in > 0 ? v : 0
  GEMM_EPI_MASK_AUX = 5     // C = v; aux = in > 0 ? v : 0
};
struct GemmEpi {
  int mode = GEMM_EPI_NONE;
  const float* bias = nullptr;
  const float* in = nullptr;
  float* aux = nullptr;
};
cudaError_t gemm_tf32x3(const float* A, int lda, int ta, const float* B, int ldb, int tb, float* C, int ldc, int M,
                        int N, int K, float beta, float* ws, size_t ws_floats, int n_sms, cudaStream_t st,
                        const GemmEpi& epi = GemmEpi());
// copy the 8 frame counters to mapped host memory and clear them (nedf_read_stats)
cudaError_t launch_stats_export(unsigned long long* stats, unsigned long long* host_mapped, cudaStream_t st);
bool tc_available();
// csize = CTAs per cluster sharing one multicast weight stream (1, 2 or 4)
cudaError_t launch_mlp_tc(const TcArgs& a, int n_ctas, int csize, cudaStream_t stream);
// one-time fp16 operand image of a paper-shaped model for the tensor-core kernel (part 0), or the
// low halves 4096 (w - fp16(w)) in the same layout (part 1, mlp_precise.cu); bias_dev may be NULL
cudaError_t tc_pack_weights(const float* params_host, int d_in, int d_feat, int n_blocks, int n_coarse, int n_fine,
                            __half** wpack_dev, float** bias_dev, size_t* bytes, int part = 0);
// fp32-accurate network for large guard batches (mlp_precise.cu): returns at once on the device
// when the batch has at most min_tiles16 16-ray tiles (guard_tc's one round)
cudaError_t launch_mlp_precise(const GroupTable& gt, const ListSet& ls, const RayJob& job, const OutSpec& out,
                               int n_sms, int min_tiles16, cudaStream_t stream);
// co-resident 4-CTA clusters of guard_tc (its one-round capacity in 16-ray tiles)
int guard_tc_capacity(int n_sms);

}  // namespace nedf
