// internal.h — launcher interfaces shared by the .cu files behind the C-ABI.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <utility>

namespace edl {

// Raise a kernel's dynamic shared-memory limit (and, for clusters wider than
// 8, allow non-portable sizes) once per (kernel, device): the attribute lives
// in the device context, so a process driving several GPUs (teacher workers
// on other devices) must set it on each.
cudaError_t ensure_kernel_attrs(const void* kern, int smem_bytes, bool nonportable_cluster = false);

// Launch with programmatic stream serialization (PDL) and an optional
// cluster shape; every kernel of the library calls griddep_wait() before its
// first global access, so early launch is always safe.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int n = 0;
  attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[n].val.programmaticStreamSerializationAllowed = 1;
  ++n;
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

enum EpiMode : int {
  EPI_TANH_BF16 = 0,   // out(bf16) = tanh(acc + bias)
  EPI_BIAS_F32 = 1,    // out(f32)  = acc + bias
  EPI_DTANH_BF16 = 2,  // out(bf16) = acc * (1 - aux^2)
  EPI_F32 = 3,         // out(f32)  = acc * scale
  EPI_SGD_F32 = 4,     // out(f32) -= scale * acc in place; out_bf16 = bf16(out)
  EPI_RELU_BF16 = 5,   // out(bf16) = relu(acc + bias [+ aux residual]) (conv layers, cfg4)
  EPI_BIAS_BF16 = 6,   // out(bf16) = acc + bias (cfg4 shortcut projections)
  EPI_DRELU_BF16 = 7,  // out(bf16) = (acc [+ aux]) * (aux2 > 0): a conv data gradient through a ReLU
};

// Implicit-GEMM convolution geometry (A = im2col of an NHWC tensor through a
// TMA im2col map; K index = (r, s, c) with 64-channel blocks). Q == 0: plain GEMM.
struct ConvGeom {
  int P = 0, Q = 0;       // output rows / cols per image
  int stride = 1, pad = 0;
  int S = 1;              // filter width (taps per filter row)
  int cblocks = 1;        // C / 64
  // weight gradient (MN-major operands, K = pixels): which operand is the
  // im2col matrix, read as [pixels][(r, s, c)] 64 x 64 boxes -- 0: A, 1: B
  int operand = 0;
};

struct EpiArgs {
  void* out;
  long long ld_out;
  const float* bias;
  const __nv_bfloat16* aux;
  long long ld_aux;
  float scale;
  unsigned* sched = nullptr;  // per-stream {next tile, CTAs done}; null -> static schedule
  __nv_bfloat16* out_bf16 = nullptr;  // EPI_SGD_F32: bf16 copy of `out` (same ld)
  // split-K (gemm_kernel only): work item t = (split, tile); split s reduces
  // k-blocks [s * kps, (s + 1) * kps) into out + s * split_stride
  int ksplit = 1;
  long long split_stride = 0;
  ConvGeom conv;          // A operand from an im2col map (gemm_kernel / gemm_pair_kernel, K-major A)
  const __nv_bfloat16* aux2 = nullptr;   // EPI_DRELU_BF16: the ReLU mask (the layer's output), ld_aux2
  long long ld_aux2 = 0;
  int raster = 0;         // tile raster group (m-tiles per group); 0: raster_group()'s heuristic
  int l2hint = 0;         // gemm_pair_kernel, K-major operands: 1 = A evict_last, B evict_first
};

struct HeadArgs {
  const float* bias;
  float inv_t;
  int k;
  float* vals;
  int* idx;
};

// student logit layer + KD loss + dlogits (kd_head_kernel)
struct KdArgs {
  const float* bias;
  const int64_t* labels;
  const float* qv;      // top-k soft labels [B][k] (k = 0 or beta = 0: none)
  const int* qi;
  int k;
  float alpha, beta, T, inv_t;
  int t2;               // T == 2: exp(d) = exp(d / 2)^2
  float* row_loss;
  int* status;
  int debug = 0;        // timing experiments only (EDL_KD_DEBUG): 1 skip pass 1, 2 skip pass 2, 4 skip both
};

enum class GemmKind { FwdTanh, FwdLinear, BwdData, BwdWeight, FwdRelu, FwdIdentBf16, BwdDataPlain, ConvDgrad };

constexpr int kMaxGroup = 4;
struct GroupMaps {
  CUtensorMap a[kMaxGroup];
  CUtensorMap b[kMaxGroup];
};
struct GroupArgs {
  int count;
  int M[kMaxGroup], N[kMaxGroup], K[kMaxGroup];
  int tile_start[kMaxGroup + 1];
  EpiArgs ep[kMaxGroup];
};
cudaError_t launch_gemm_grouped_bwd_weight(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                           cudaStream_t stream, bool fused_sgd = false);
int grouped_tile_bn();
// The same on 256 x 256 CTA-pair tiles; ga.tile_start counts pair tiles.
cudaError_t launch_gemm_grouped_pair_bwd_weight(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                                cudaStream_t stream, bool fused_sgd = false);

// ty: the output's TMA-store map (32 x 32 boxes; tensor_map_out) for the
// bias / tanh / (1-a^2) epilogues; ignored (any valid map) for BwdWeight.
// tr: FwdRelu with a residual (ep.aux) only -- the residual's 32 x 32 box map
// (tensor_map_out on ep.aux), streamed into shared memory by TMA.
cudaError_t launch_gemm(GemmKind kind, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                        const CUtensorMap& ty, int M, int N, int K, const EpiArgs& ep, int num_sms,
                        cudaStream_t stream, const CUtensorMap* tr = nullptr, bool w128 = false);
// Hidden-layer tanh of the GEMM epilogues on the current device: 1 = tanhf
// (default), 0 = tanh.approx.f32 (gemm_sm100.cu).
cudaError_t set_tanh_mode(int mode);
// Stream-ordered flag fallbacks (exchange.cu).
cudaError_t launch_flag_wait(const uint32_t* addr, uint32_t value, cudaStream_t stream);
cudaError_t launch_flag_write(uint32_t* addr, uint32_t value, cudaStream_t stream);
// Fused gradient exchange + SGD over NVSwitch multicast (exchange.cu).
int nvls_max_blocks(int world, long long pad_bytes);
cudaError_t launch_nvls_allreduce_sgd(float* mc_grad, float* mc_param, void* mc_bf16, const float* param,
                                      uint32_t* const* pads, uint32_t* counter, long long n, float scale,
                                      uint32_t epoch, int rank, int world, int blocks, cudaStream_t stream);
// 256 x bn tiles on CTA pairs (cta_group::2); bn in {128, 256}; B's tensor
// map box covers bn/2 rows (K-major) or bn/2 columns (MN-major).
cudaError_t launch_gemm_pair(GemmKind kind, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                             const CUtensorMap& ty, int M, int N, int K, const EpiArgs& ep, int num_sms,
                             cudaStream_t stream, const CUtensorMap* tr = nullptr, bool w128 = false);
// teacher head on CTA pairs, class chunks merged through `part`
// ([ceil(N/256)][2 + 2 kmax][M] floats) and `tickets` (ceil(M/128), zeroed once)
cudaError_t launch_teacher_head_pair(int kmax, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                                     const HeadArgs& hp, float* part, unsigned* tickets, cudaStream_t stream);
cudaError_t launch_kd_head(int kmax, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M,
                           int N, int Nw, int K, const KdArgs& kp, cudaStream_t stream);
cudaError_t launch_loss_mean(const float* row_loss, int B, float* loss_out, int* status, cudaStream_t stream);
cudaError_t launch_teacher_head(int bn, int kmax, const CUtensorMap& ta, const CUtensorMap& tb,
                                int M, int N, int K, const HeadArgs& hp, cudaStream_t stream);

// cfg4 data movement (conv.cu): NHWC bf16, C a multiple of 8
cudaError_t launch_im2col_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int c_used, int R, int S,
                               int stride, int pad, int P, int Q, __nv_bfloat16* out, long long ldo,
                               cudaStream_t stream);
cudaError_t launch_maxpool_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int k, int stride, int pad,
                                int P, int Q, __nv_bfloat16* out, uint32_t* argmax, bool relu_mask,
                                cudaStream_t stream);
cudaError_t launch_conv_flip_weights(const __nv_bfloat16* w, long long ldw, int K, int C, int R, int S,
                                     __nv_bfloat16* wf, long long ldf, cudaStream_t stream);
// training-mode BN + ReLU of the stem's raw conv output z fused into its 3x3 /
// 2 max pool with argmax (+ ReLU mask nibbles): y itself is never stored
cudaError_t launch_bn_relu_maxpool3s2_nhwc(const __nv_bfloat16* z, int N, int H, int W, int C, int pad, int P, int Q,
                                           const float* mean, const float* rstd, const float* gamma,
                                           const float* beta, __nv_bfloat16* out, uint32_t* argmax,
                                           cudaStream_t stream);
cudaError_t launch_maxpool_bwd_argmax_nhwc(const uint32_t* argmax, int N, int H, int W, int C, int k, int stride,
                                           int pad, int P, int Q, const __nv_bfloat16* dy, const __nv_bfloat16* mask,
                                           __nv_bfloat16* dx, cudaStream_t stream);
cudaError_t launch_avgpool_nhwc(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* out, long long ldo,
                                cudaStream_t stream);
cudaError_t launch_col2im_nhwc(const __nv_bfloat16* dcol, long long ldc, int N, int H, int W, int C, int R, int S,
                               int stride, int pad, int P, int Q, const __nv_bfloat16* add,
                               const __nv_bfloat16* mask, __nv_bfloat16* dx, cudaStream_t stream);
cudaError_t launch_avgpool_bwd_nhwc(const __nv_bfloat16* df, long long ldf, int N, int HW, int C,
                                    const __nv_bfloat16* mask, __nv_bfloat16* dx, cudaStream_t stream);
cudaError_t launch_maxpool_bwd_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int k, int stride, int pad,
                                    int P, int Q, const __nv_bfloat16* dy, const __nv_bfloat16* mask,
                                    __nv_bfloat16* dx, cudaStream_t stream);

// many layers' weight flips (conv.cu) in one launch
constexpr int kMaxFlips = 24;
struct FlipGroup {
  int count;
  int start[kMaxFlips + 1];                 // element offsets, start[count] = total
  int K[kMaxFlips], C[kMaxFlips], RS[kMaxFlips];
  long long ldw[kMaxFlips], ldf[kMaxFlips];
  const __nv_bfloat16* w[kMaxFlips];
  __nv_bfloat16* wf[kMaxFlips];
};
cudaError_t launch_conv_flip_weights_many(const FlipGroup& g, cudaStream_t stream);

// halo-tiled 3x3 convolution (halo.cu): C = K = 64, stride 1, pad 1, W + 2 <= 128;
// out = [relu](conv + bias [+ res]), then * (mask > 0) when mask is given
struct HaloArgs {
  int N, H, W, R;                   // R output rows per 128-row tile (128 / (W + 2))
  int tiles_per_image, tiles;
  const float* bias;
  const __nv_bfloat16* res;
  const __nv_bfloat16* mask;
  int relu;
  __nv_bfloat16* out;
  int debug;                        // timing experiments (EDL_HALO_DEBUG): 1 no epilogue math / stores, 2 one patch load
};
int halo_rows_per_tile(int W);
// halo weight gradient (same layers): dW[cout][(r, s, c)] = scale * sum dz x;
// partial: halo_wgrad_partial_floats(grid) floats
long long halo_wgrad_partial_floats(int sms);
cudaError_t launch_halo_wgrad(const CUtensorMap& tmX, const CUtensorMap& tmD, const HaloArgs& a, int grid,
                              float* partial, float scale, float* dW, long long lddw, cudaStream_t stream);
cudaError_t launch_halo_conv(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmY,
                             const CUtensorMap& tmR, const CUtensorMap& tmM, const HaloArgs& a, int grid,
                             cudaStream_t stream);
cudaError_t launch_halo_probe(const CUtensorMap& tmX, const CUtensorMap& tmW, int n, int h0, int W, int off, int mode,
                              int reps, int smem_kb, float* out, cudaStream_t stream);

// training-mode BatchNorm (bn.cu): z / g NHWC bf16 rows [M][C], C % 8 == 0, C <= 2048;
// partial: bn_partial_floats(M, C, sms) floats (fp64 per-cluster partials);
// ticket: a zeroed per-stream counter (left zeroed), or nullptr for a
// separate finishing launch
long long bn_partial_floats(int M, int C, int sms);
cudaError_t launch_bn_stats(const __nv_bfloat16* z, int M, int C, float* partial, unsigned* ticket, float* mean,
                            float* rstd, float eps, int sms, cudaStream_t stream);
cudaError_t launch_bn_bwd_reduce(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                 const float* rstd, float* partial, unsigned* ticket, float* dbeta, float* dgamma,
                                 int sms, cudaStream_t stream);
cudaError_t launch_bn_apply(const __nv_bfloat16* z, int M, int C, const float* mean, const float* rstd,
                            const float* gamma, const float* beta, const __nv_bfloat16* res, bool relu,
                            __nv_bfloat16* y, int sms, cudaStream_t stream);
cudaError_t launch_bn_bwd_apply(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                const float* rstd, const float* gamma, const float* dbeta, const float* dgamma,
                                __nv_bfloat16* dz, int sms, cudaStream_t stream);

// SIMT kernels (kernels.cu)
cudaError_t launch_kd_loss(const float* logits, long long ld_z, const int64_t* labels,
                           const float* q_vals, const int* q_idx, int B, int K, int k,
                           float alpha, float beta, float T, float* row_loss, float* loss_out,
                           unsigned* ticket, __nv_bfloat16* dlogits, long long ld_dz,
                           int* status, cudaStream_t stream);
cudaError_t launch_tempered_softmax(const float* logits, long long ld, float* probs,
                                    long long ld_p, int B, int K, float T, cudaStream_t stream);
cudaError_t launch_sgd(float* p, __nv_bfloat16* p_bf16, const float* g, long long n,
                       float scale, cudaStream_t stream);
cudaError_t launch_gather_rows(const __nv_bfloat16* src, long long ld_src, const int64_t* idx,
                               __nv_bfloat16* dst, long long ld_dst, int B, int D,
                               const int64_t* src_labels, int64_t* dst_labels, cudaStream_t stream);
cudaError_t launch_colsum(const __nv_bfloat16* x, long long ld, int M, int N, float* partial,
                          float* out, float scale, cudaStream_t stream);
struct ColsumGroup {
  int count;
  const __nv_bfloat16* x[kMaxGroup];
  long long ld[kMaxGroup];
  int M[kMaxGroup], N[kMaxGroup];
  float* out[kMaxGroup];
  __nv_bfloat16* out_bf16[kMaxGroup];  // sgd: bf16 copies of the updated biases
  float scale;
  int sgd;                             // 0: out = scale * colsum; 1: out -= scale * colsum
  float* partial;
  long long part_off[kMaxGroup];
  int blk_start[kMaxGroup + 1];
};
cudaError_t launch_colsum_group(ColsumGroup g, cudaStream_t stream);
// tall-skinny column sums (conv bias gradients): G = colsum_tall_blocks(M, sms)
// blocks, workspace G * N floats; N % 8 == 0, N <= 2048 (colsum_tall_ok)
int colsum_tall_blocks(int M, int sms);
bool colsum_tall_ok(int N);
cudaError_t launch_colsum_tall(const __nv_bfloat16* x, long long ld, int M, int N, float* partial, float* out,
                               float scale, int sms, cudaStream_t stream);
// split-K partial sums P[ksplit][GM][GN] -> out (transposed: out[GN][GM])
cudaError_t launch_splitk_reduce(const float* P, int ksplit, long long sstride, int GM, int GN, bool transposed,
                                 float* out, long long ldo, int sms, cudaStream_t stream);
long long colsum_workspace_floats(int count, const int* M, const int* N);
cudaError_t launch_topk_hits(const float* logits, long long ld, const int64_t* labels, int B,
                             int K, int k, unsigned* hits, cudaStream_t stream);
cudaError_t launch_cast_bf16(const float* src, long long ld_src, __nv_bfloat16* dst,
                             long long ld_dst, int rows, int cols, cudaStream_t stream);
cudaError_t launch_cast_bf16_f64(const double* src, long long ld_src, __nv_bfloat16* dst,
                                 long long ld_dst, int rows, int cols, cudaStream_t stream);
cudaError_t launch_stream_delay(unsigned long long ns, cudaStream_t stream);

}  // namespace edl
