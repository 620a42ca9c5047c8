/* edl_b200.h — C-ABI of the B200 (sm_100a) EDL-Dist distillation hot path.
 *
 * The reference (EDL-Dist, pkg/src/edl) is pure Python + numpy float64 and has
 * no FFI layer; its boundary is the Python API of edl.nnkit / edl.teacher_node /
 * edl.student_node. Each entry point below replaces the numpy arithmetic behind
 * one of those calls (cited per function); the Python mirror
 * paper_2207_06667_b200/nnkit.py binds them with ctypes, keeping the reference
 * names, argument meaning and error classes.
 *
 * Conventions
 *   - All pointers are device pointers owned by the caller; nothing allocates.
 *   - Matrices are row-major with an explicit leading dimension in ELEMENTS.
 *     bf16 operands of the tensor-core paths need a 16-byte aligned base and
 *     ld % 8 == 0 (TMA row pitch). Padding columns must hold zeros.
 *   - `stream` is a cudaStream_t (passed as void*); every call is asynchronous
 *     on it and reentrant per (device, stream).
 *   - Return 0 on success or a negative EDL_ERR_* code; edl_last_error() holds
 *     the message (thread-local). Device-detected errors (bad label / class id,
 *     non-finite loss) are reported through the `status` word of the loss call.
 */
#ifndef EDL_B200_H
#define EDL_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define EDL_B200_ABI_VERSION 2

/* status codes: mirror edl.nnkit's exception classes (edl/nnkit.py:31-40) */
#define EDL_OK 0
#define EDL_ERR_SHAPE (-1)   /* ShapeError(ValueError)                    */
#define EDL_ERR_NUMERIC (-2) /* NumericError: non-finite loss (nnkit:296) */
#define EDL_ERR_PARAM (-3)   /* ValueError: T <= 0, bad k / alpha / beta  */
#define EDL_ERR_CUDA (-4)    /* launch / driver failure                   */

#define EDL_ACT_NONE 0 /* z = x W^T + b, fp32 out (logit layer)           */
#define EDL_ACT_TANH 1 /* h = tanh(x W^T + b), bf16 out (hidden layers)   */
#define EDL_ACT_RELU 2 /* h = relu(x W^T + b), bf16 out (cfg4 conv layers) */
#define EDL_ACT_IDENT 3 /* h = x W^T + b, bf16 out (cfg4 shortcut projections) */

int edl_version(void);
const char* edl_last_error(void);
int edl_device_sms(void);

/* Cap the persistent tensor-core kernels launched on `stream` at `max_ctas`
 * CTAs (<= 0 removes the cap). A co-located teacher stream capped below the
 * SM count leaves SMs for the student's NCCL all-reduce, which would
 * otherwise queue behind teacher GEMMs that hold every SM. */
int edl_set_stream_max_ctas(void* stream, int max_ctas);

/* Hidden-layer tanh of the forward GEMM epilogues on the CURRENT device:
 * 0 = tanh.approx.f32, one MUFU op with ~2^-11 relative error (default);
 * 1 = tanhf, <= 2 ulp fp32 (+2.6% teacher batch, +6% student step at cfg3,
 * gradient error vs the bf16-storage oracle 1.38e-3 instead of 1.65e-3:
 * profiles/r02_parity_probe.json). Not stream
 * ordered: call while no forward GEMM is in flight on that device.
 *
 * Tile scheduling: every stream that launches the persistent GEMMs gets a
 * {next tile, CTAs done} counter pair from a static device pool on first
 * use (nothing is allocated, so the first use may be inside stream capture).
 * A graph captured on stream S reuses S's pair: do not replay it while eager
 * GEMMs run on S from another thread, or replay it on two streams at once. */
int edl_set_tanh_mode(int mode);

/* One dense layer of edl.nnkit.forward (edl/nnkit.py:223-234, `z = h @ w.T + b`
 * at :232, tanh at :233). X: bf16 [M][ldx] (K used), W: bf16 [N][ldw], bias:
 * fp32 [N]. act=EDL_ACT_TANH writes bf16 Y [M][ldy]; EDL_ACT_NONE writes fp32.
 * tcgen05 GEMM, TMA-fed, fused bias/activation epilogue, TMA-stored output:
 * every operand AND Y need a 16-byte aligned base and row pitch
 * (ld * element size % 16 == 0), else EDL_ERR_SHAPE. */
int edl_linear_fwd(const void* X, long long ldx, const void* W, long long ldw, const float* bias,
                   void* Y, long long ldy, int M, int N, int K, int act, void* stream);

/* ---- cfg4 (ResNet-style teacher, BASELINE.json configs[3]; the reference has
 * no convolutions). A convolution is edl_im2col_nhwc into a
 * caller workspace followed by edl_linear_fwd (act RELU) or
 * edl_linear_fwd_residual with the folded-BN weights W[K_out][R*S*C] and bias.
 * Activations: NHWC bf16, C a multiple of 8 (16 keeps TMA rows aligned). */

/* Y = relu(X W^T + b + R): a ResNet block's last convolution with its
 * shortcut R (bf16 [M][ldr], same shape as Y). Alignment as edl_linear_fwd. */
int edl_linear_fwd_residual(const void* X, long long ldx, const void* W, long long ldw, const float* bias,
                            const void* R, long long ldr, void* Y, long long ldy, int M, int N, int K,
                            void* stream);
/* out[(n,p,q)][(r,s,c)] = x[n][p*stride-pad+r][q*stride-pad+s][c] (0 outside),
 * P = (H + 2pad - R)/stride + 1, Q likewise. x has C channels (pitch);
 * c_used == C: row pitch ldo >= R*S*C; c_used < C (e.g. the RGB stem): only
 * channels < c_used are gathered, densely, K = R*S*c_used, the row zero-padded
 * to ldo. */
int edl_im2col_nhwc(const void* x, int N, int H, int W, int C, int c_used, int R, int S, int stride, int pad,
                    void* out, long long ldo, void* stream);
/* k x k max pool (stride, zero-extended window never wins: -inf padding). */
int edl_maxpool_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                     void* stream);
/* Global average pool: out[n][c] = mean over H*W of x[n][.][.][c] (bf16). */
int edl_avgpool_nhwc(const void* x, int N, int HW, int C, void* out, long long ldo, void* stream);

/* Implicit-GEMM convolution (cfg4), NHWC bf16 with
 * C % 64 == 0: y[n][p][q][k] = act(sum over (r, s, c) of
 * x[n][p*stride-pad+r][q*stride-pad+s][c] * w[k][(r*S+s)*C+c] + bias[k]
 * (+ residual[(n,p,q)][k])). The tcgen05 GEMM's producer loads its A tiles
 * straight from x with TMA im2col loads (one filter tap x 64 channels per
 * k-block): no column matrix in HBM. act: EDL_ACT_RELU or EDL_ACT_IDENT;
 * residual (optional) needs EDL_ACT_RELU. y: [N*P*Q][ldy], TMA-stored.
 * C == K == 64, 3x3, stride 1, pad 1, W <= 62 (the stage-1 layers) runs the
 * halo-tiled conv instead: one TMA patch per two output rows, the nine taps
 * as row-shifted views of it (bitwise equal; EDL_HALO=0 disables). */
int edl_conv_fwd_nhwc(const void* x, int N, int H, int W, int C, const void* w, long long ldw, const float* bias,
                      int K, int R, int S, int stride, int pad, const void* residual, long long ldr, void* y,
                      long long ldy, int act, void* stream);

/* Its weight gradient: dW[k][(r,s,c)] = scale * sum over output pixels of
 * dY[(n,p,q)][k] * x[n][p*stride-pad+r][q*stride-pad+s][c] (+ db = scale *
 * colsum dY), the split-K plan of edl_linear_bwd_weight_ws with the im2col
 * operand read through a TMA im2col map (64 pixels x 64 channels per box).
 * workspace: edl_bwd_weight_workspace_floats(N*P*Q, K, R*S*C) floats. */
int edl_conv_bwd_weight_nhwc(const void* x, int N, int H, int W, int C, int R, int S, int stride, int pad,
                             const void* dY, long long lddy, int K, float* dW, long long lddw, float* db,
                             float* workspace, long long workspace_floats, float scale, void* stream);

/* Data gradient of a stride-1 convolution as an implicit-GEMM convolution of
 * dZ [N][P][Q][K] (K % 64 == 0) with the flipped filter (edl_conv_flip_weights:
 * wf [C][(r, s, k)] from w [K][(r, s, c)]) at padding R-1-pad:
 *   dx[n][h][w][c] = (sum ... [+ add]) * (mask > 0 if mask)     (bf16, [N][H][W][C])
 * add: the residual branch's gradient; mask: the layer input's stored ReLU
 * output. Replaces edl_linear_bwd_data + edl_col2im_nhwc for stride 1. */
int edl_conv_flip_weights(const void* w, long long ldw, int K, int C, int R, int S, void* wf, long long ldf,
                          void* stream);
/* The same for `count` (<= 24) layers in one launch: arrays of the
 * per-layer arguments above (host memory). */
int edl_conv_flip_weights_many(int count, const void* const* w, const long long* ldw, const int* K, const int* C,
                               const int* R, const int* S, void* const* wf, const long long* ldf, void* stream);
/* Layout probe for the halo conv (diagnostics and tests only): the 128 x 64
 * product of one tap's row-shifted view of the staged patch of image n (rows
 * h0-1 .. h0+2) with w [64][64] (mode 3: [64][576], nine taps), into out
 * [128][64] fp32; mode 0: no-swizzle chunk-plane layout, 1: SWIZZLE_128B with
 * the descriptor base offset (wrong by design), 2: SWIZZLE_128B. reps > 0:
 * issue the 9-tap sequence reps % 1000 times (odd thousands digit: on 148
 * CTAs) and store the cycle count in out[128 * 64]; smem_kb > 0 sets the
 * dynamic shared memory. x: NHWC bf16 with C = 64. */
int edl_halo_probe(const void* x, int N, int H, int W, int n, int h0, int off, const void* w, int mode, int reps,
                   int smem_kb, float* out, void* stream);
int edl_conv_dgrad_nhwc(const void* dz, int N, int P, int Q, int K, const void* wf, long long ldf, int C, int R,
                        int S, int pad, const void* add, const void* mask, void* dx, void* stream);

/* cfg4 student backward (BN-free ResNet-18-style): the data gradient of a
 * convolution is edl_linear_bwd_data with H = NULL (dcol = dZ W, no tanh
 * factor) followed by this gather:
 *   dx[n][h][w][c] = (sum of dcol over the windows covering (h, w) [+ add])
 *                    * (mask > 0 if mask != NULL)
 * i.e. straight to the previous ReLU layer's pre-activation gradient, with the
 * block shortcut's gradient in `add`. Deterministic (gather, fixed order). */
int edl_col2im_nhwc(const void* dcol, long long ldc, int N, int H, int W, int C, int R, int S, int stride, int pad,
                    const void* add, const void* mask, void* dx, void* stream);
/* dx[n][i][c] = df[n][c] / HW (* (mask > 0)): global average pool backward. */
int edl_avgpool_bwd_nhwc(const void* df, long long ldf, int N, int HW, int C, const void* mask, void* dx,
                         void* stream);
/* Max pool backward: each input collects the gradients of the windows whose
 * first maximum it is (torch's tie rule) (* (mask > 0)). */
int edl_maxpool_bwd_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, const void* dy,
                         const void* mask, void* dx, void* stream);
/* Training pair: the forward max pool also records, per output window and
 * 8-channel vector, one 32-bit word of 4-bit first-maximum positions r*k+s
 * (argmax: unsigned [N][P][Q][C/8], k*k <= 15); the backward then gathers
 * from those words instead of re-scanning every window. Same results as
 * edl_maxpool_nhwc / edl_maxpool_bwd_nhwc. */
int edl_maxpool_argmax_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                            unsigned* argmax, void* stream);
/* Training-mode BN + ReLU fused into the 3x3 / 2 max pool with argmax (the
 * BN student's stem): out / argmax as edl_maxpool_argmax_relu_nhwc applied to
 * y = bf16(relu(gamma (z - mean) rstd + beta)) (edl_bn_apply_nhwc's
 * arithmetic), computed per tap from the raw conv output z; y is not stored. */
int edl_bn_relu_maxpool_argmax_nhwc(const void* z, int N, int H, int W, int C, const float* mean, const float* rstd,
                                    const float* gamma, const float* beta, int k, int stride, int pad, void* out,
                                    unsigned* argmax, void* stream);
int edl_maxpool_bwd_argmax_nhwc(const unsigned* argmax, int N, int H, int W, int C, int k, int stride, int pad,
                                const void* dy, const void* mask, void* dx, void* stream);
/* edl_maxpool_argmax_nhwc for a pool whose input is a ReLU output (the
 * stem): lanes whose window maximum is not > 0 get the no-match position 0xF,
 * so edl_maxpool_bwd_argmax_nhwc with mask = NULL equals the masked backward
 * (mask = the pool input) without reading the full-resolution mask. */
int edl_maxpool_argmax_relu_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                                 unsigned* argmax, void* stream);

/* Backprop through one tanh layer, edl/nnkit.py:308:
 *   dX[M][K] = (dY[M][N] @ W[N][K]) * (1 - H[M][K]^2)      (all bf16)
 * H = NULL: dX = dY @ W (the conv column gradient, cfg4).
 * Same alignment rule as edl_linear_fwd (dX is TMA-stored). */
int edl_linear_bwd_data(const void* dY, long long lddy, const void* W, long long ldw,
                        const void* H, long long ldh, void* dX, long long lddx, int M, int N,
                        int K, void* stream);

/* Weight/bias gradients, edl/nnkit.py:305-306:
 *   dW[N][K] = scale * dY[M][N]^T @ X[M][K]   (fp32 out)
 *   db[N]    = scale * sum_m dY[m][:]         (fp32, optional; needs workspace of
 *              edl_colsum_workspace_floats(M, N) floats)                        */
int edl_linear_bwd_weight(const void* dY, long long lddy, const void* X, long long ldx, float* dW,
                          long long lddw, float* db, float* workspace, int M, int N, int K,
                          float scale, void* stream);
long long edl_colsum_workspace_floats(int M, int N);

/* The same gradients for tall reductions (conv layers: M = B*H*W pixels, few
 * output tiles): split-K tcgen05 partials + a fixed-order reduce
 * (deterministic), operands swapped when N < 128 so the 128-row MMA is full,
 * and a tall column sum for db. workspace: workspace_floats >=
 * edl_bwd_weight_workspace_floats(M, N, K) for the planned split; a smaller
 * workspace only narrows the split. */
int edl_linear_bwd_weight_ws(const void* dY, long long lddy, const void* X, long long ldx, float* dW,
                             long long lddw, float* db, float* workspace, long long workspace_floats, int M, int N,
                             int K, float scale, void* stream);
long long edl_bwd_weight_workspace_floats(int M, int N, int K);

/* The same for up to 4 independent layers in ONE persistent tcgen05 launch
 * (host arrays of per-layer pointers / sizes). The backward pass issues every
 * dW of the student this way once the delta chain (edl_linear_bwd_data) is
 * done: each layer alone has too few output tiles to fill 148 SMs.
 * workspace: edl_colsum_group_workspace_floats(count, M, N) floats (all the
 * layers' column sums run as one deterministic two-pass launch pair). */
int edl_linear_bwd_weight_grouped(int count, const void* const* dY, const long long* lddy,
                                  const void* const* X, const long long* ldx, float* const* dW,
                                  const long long* lddw, float* const* db, float* workspace,
                                  const int* M, const int* N, const int* K, float scale, void* stream);
long long edl_colsum_group_workspace_floats(int count, const int* M, const int* N);

/* Single-student step fusion of the above with sgd_step (edl/nnkit.py:320-321):
 *   W[p] -= eta * dY[p]^T @ X[p];  b[p] -= eta * colsum(dY[p])
 * on the fp32 masters in place, refreshing the bf16 copies W_bf16 / b_bf16
 * (b_bf16 may be NULL). The gradients never reach HBM. Only valid when no
 * gradient all-reduce sits between backward and update (world_size 1). */
int edl_linear_bwd_weight_grouped_sgd(int count, const void* const* dY, const long long* lddy,
                                      const void* const* X, const long long* ldx, float* const* W,
                                      void* const* W_bf16, const long long* ldw, float* const* b,
                                      void* const* b_bf16, float* workspace, const int* M, const int* N,
                                      const int* K, float eta, void* stream);

/* Teacher head = soft_label_reply's math (edl/teacher_node.py:54:
 * tempered_softmax(forward(model, inputs), T), edl/nnkit.py:193-208,232) fused
 * with the top-k soft-label extraction EDL-Dist ships to students:
 *   p = softmax((H W^T + b) / T);  (vals[M][k], idx[M][k]) = top-k of p per row,
 *   ordered by probability desc, ties -> lower class index (edl/nnkit.py:333).
 * Logits stay on chip (TMEM -> registers -> DSMEM merge across a cluster).
 * N = number of classes (<= 2048), 1 <= k <= min(N, 32). */
int edl_teacher_head_softmax_topk(const void* H, long long ldh, const void* W, long long ldw,
                                  const float* bias, int M, int N, int K, float T, int k,
                                  float* vals, int* idx, void* stream);

/* edl_teacher_head_softmax_topk on CTA pairs (256-row tiles, cta_group::2):
 * the class chunks (256 classes each, any number) are merged through
 * `workspace` (edl_teacher_head_workspace_bytes(M, N, k) bytes, ZEROED once
 * by the caller at allocation; the kernel leaves its tickets at zero), so no
 * cluster has to span the class range. One workspace per stream. With
 * workspace == NULL (or EDL_HEAD_CLUSTER=1) the single-CTA cluster head runs
 * instead. Same outputs and tie rule. With an even number of 256-row blocks
 * two pairs share each weight tile through a 2-SM TMA multicast (4-CTA
 * clusters; bitwise equal, EDL_HEAD_MC=0 disables). */
long long edl_teacher_head_workspace_bytes(int M, int N, int k);
int edl_teacher_head_softmax_topk_ws(const void* H, long long ldh, const void* W, long long ldw, const float* bias,
                                     int M, int N, int K, float T, int k, float* vals, int* idx, void* workspace,
                                     long long ws_bytes, void* stream);

/* Dense tempered softmax, edl/nnkit.py:193-208 (fp32 logits -> fp32 probs). */
int edl_tempered_softmax(const float* logits, long long ld, float* probs, long long ldp, int B,
                         int K, float T, void* stream);

/* The student's logit layer fused with kd_loss (edl/nnkit.py:232 for the
 * last layer, :283-299 for the loss and dlogits): one launch computes
 * z = H W^T + b on the tensor cores, keeps the logit tile in TMEM, and writes
 * only the per-row loss and bf16 dlogits — the fp32 logits never reach HBM.
 * H: bf16 [B][ldh] (D used), W: bf16 [K][ldw], bias fp32 [K], labels int64
 * [B], top-k soft labels as for edl_kd_loss_fwd_bwd; dlogits bf16 [B][lddz]
 * (columns K .. pad16(K) written as 0). Followed by the same fixed-order
 * batch mean into loss_out. K <= 2048 and k <= 32 (else EDL_ERR_SHAPE: use
 * edl_linear_fwd + edl_kd_loss_fwd_bwd). */
int edl_linear_kd_loss_fwd_bwd(const void* H, long long ldh, const void* W, long long ldw, const float* bias,
                               const long long* labels, const float* q_vals, const int* q_idx, int B, int K, int D,
                               int k, float alpha, float beta, float T, float* row_loss, float* loss_out,
                               void* dlogits, long long lddz, int* status, void* stream);

/* Fused distillation loss forward + backward, edl/nnkit.py:283-295:
 *   loss = mean_rows[ alpha*CE(onehot(y), softmax z) + beta*T^2*CE(q, softmax(z/T)) ]
 *   dz   = alpha/B*(softmax z - onehot y) + beta*T/B*(softmax(z/T) - q)
 * q = (q_vals, q_idx)[B][k] renormalised to sum 1 per row (k = K: dense).
 * logits fp32 [B][ldz]; labels int64 [B]; dlogits bf16 [B][lddz] (padding
 * columns zeroed); row_loss fp32 [B] scratch; loss_out fp32 scalar (batch mean,
 * deterministic order); ticket: one zero-initialised uint (self-resetting);
 * status: int, set to EDL_ERR_SHAPE / EDL_ERR_NUMERIC by the device. */
int edl_kd_loss_fwd_bwd(const float* logits, long long ldz, const long long* labels,
                        const float* q_vals, const int* q_idx, int B, int K, int k, float alpha,
                        float beta, float T, float* row_loss, float* loss_out, unsigned* ticket,
                        void* dlogits, long long lddz, int* status, void* stream);

/* SGD, edl/nnkit.py:312-322 (`w - eta * gw`), on fp32 masters in place; the
 * optional bf16 copy (same element offsets) is refreshed in the same pass.
 * scale = eta / world_size folds the all-reduce mean (edl/allreduce.py:119). */
int edl_sgd_step(float* p, void* p_bf16, const float* g, long long n, float scale, void* stream);

/* Stream-ordered 32-bit flags for the teacher-pool -> student soft-label
 * handoff over NVLink (split placement; replaces the INFER_REPLY delivery of
 * edl/teacher_node.py:47-58 into DistilReader._accept_reply / consume,
 * edl/student_node.py:407-457). addr is device memory of this GPU or a peer's
 * (symmetric-memory signal pad). wait: later work on `stream` waits until
 * (int32)(*addr - value) >= 0. write: *addr = value once all earlier work on
 * `stream` (e.g. the peer copy of a soft-label batch) is complete and visible.
 * Neither holds an SM (cuStreamWaitValue32 / cuStreamWriteValue32; one-thread
 * kernels if the driver lacks stream memory operations). */
int edl_stream_wait_geq(unsigned* addr, unsigned value, void* stream);
int edl_stream_write_u32(unsigned* addr, unsigned value, void* stream);

/* Data-parallel gradient exchange fused with SGD, over NVSwitch multicast.
 * Replaces, at world > 1, the ring all-reduce to the mean
 * (edl/allreduce.py:77-120, called at edl/student_node.py:741) followed by
 * sgd_step (edl/nnkit.py:312-322, edl/student_node.py:745). Every rank calls
 * it on its stream after its gradient kernels; rank r sums shard r of the
 * gradient across ranks in the switch, applies p -= scale * sum and writes
 * the new fp32 and bf16 parameters into every rank's replica. When the
 * kernel completes on any rank, all replicas are updated and identical.
 *   mc_grad, mc_param, mc_param_bf16: multicast addresses of symmetric buffers
 *       of n elements (fp32, fp32, bf16); n a multiple of 8 * world.
 *   param: this rank's own fp32 replica (unicast address of mc_param's copy).
 *   pads: device array of `world` pointers to the ranks' uint32 signal pads of
 *       pad_bytes each (zero before the first call); counter: one device
 *       uint32, zero before the first call.
 *   scale: eta / world (the mean folded into the step).
 *   epoch: strictly increasing per call, identical on all ranks.
 * Errors: -1 bad shape, -3 bad rank/world/pad size, -4 CUDA. */
int edl_nvls_allreduce_sgd(float* mc_grad, float* mc_param, void* mc_param_bf16, const float* param,
                           unsigned* const* pads, long long pad_bytes, unsigned* counter, int rank, int world,
                           long long n, float scale, unsigned epoch, void* stream);

/* Batch gather from an HBM-resident shard, edl/student_node.py:150-151:
 * dst[b][:D] = src[idx[b]][:D] (bf16, idx int64) and, when both label
 * pointers are given, dst_labels[b] = src_labels[idx[b]] (int64). */
int edl_gather_rows(const void* src, long long ld_src, const long long* idx, void* dst,
                    long long ld_dst, int B, int D, const long long* src_labels,
                    long long* dst_labels, void* stream);

/* Top-k accuracy counter, edl/nnkit.py:325-335: hits += #rows whose label
 * ranks < k under (logit desc, class asc). */
int edl_topk_hits(const float* logits, long long ld, const long long* labels, int B, int K, int k,
                  unsigned* hits, void* stream);

/* fp32 -> bf16 matrix cast (parameter / input staging). */
int edl_cast_bf16(const float* src, long long ld_src, void* dst, long long ld_dst, int rows,
                  int cols, void* stream);

/* A reference caller's float64 batch (edl/nnkit.py:97-110 Batch.inputs,
 * B x D) uploaded as is and converted on the device: fp64 -> fp32 -> bf16,
 * the same double rounding as the host path (numpy astype(float32) then
 * round-to-nearest-even), into the padded bf16 batch layout. */
int edl_cast_bf16_f64(const double* src, long long ld_src, void* dst, long long ld_dst, int rows, int cols,
                      void* stream);

/* Training-mode BatchNorm for the cfg4 ResNet-18-style student (BASELINE.json
 * configs[3]; the reference has no convolutions). z / g / y / dz
 * are NHWC bf16 rows [M = N*H*W][C], C % 8 == 0 and <= 2048; per-channel
 * fp32 vectors [C]. Batch statistics are biased (nn.BatchNorm2d training
 * mode); reductions are deterministic (fixed row blocks, cluster partials
 * combined in rank order, fp64 final sums) and take one launch each: the last
 * block to arrive finishes, counted on a per-(device, stream) ticket from a
 * static pool (as the GEMM tile counters: a graph captured on stream S uses
 * S's ticket, so do not replay it while eager BN calls run on S).
 *   stats:  mean, rstd = 1 / sqrt(var + eps)
 *   apply:  y = [relu](gamma (z - mean) rstd + beta [+ residual])
 *   bwd:    dbeta = sum g, dgamma = sum g xhat (written, not accumulated),
 *           dz = gamma rstd (g - dbeta / M - xhat dgamma / M)
 * workspace: edl_bn_workspace_floats(M, C) floats. */
long long edl_bn_workspace_floats(int M, int C);
int edl_bn_stats_nhwc(const void* z, int M, int C, float* workspace, long long ws_floats, float* mean, float* rstd,
                      float eps, void* stream);
int edl_bn_apply_nhwc(const void* z, int M, int C, const float* mean, const float* rstd, const float* gamma,
                      const float* beta, const void* residual, int relu, void* y, void* stream);
int edl_bn_bwd_nhwc(const void* g, const void* z, int M, int C, const float* mean, const float* rstd,
                    const float* gamma, float* workspace, long long ws_floats, float* dgamma, float* dbeta, void* dz,
                    void* stream);

/* TeacherConfig.simulated_delay (edl/teacher_node.py:30-44, slept per batch
 * by TeacherServer._compute_loop :157-170): a single-thread device busy wait
 * of `ns` nanoseconds on `stream`, so a throttled teacher delays its own
 * stream and never the host thread. */
int edl_stream_delay_ns(long long ns, void* stream);

/* Soft-label handoff from a teacher GPU to its student's slot (the reply
 * leg of edl/student_node.py:407-423): cudaMemcpyPeerAsync on the TEACHER's
 * stream only. (torch's cross-device copy_ also orders the destination
 * device's current stream, i.e. the student's training stream, which
 * serialises teacher and student.) */
int edl_memcpy_peer_async(void* dst, int dst_device, const void* src, int src_device, long long bytes,
                          void* stream);

/* Elastic teacher pool across processes (pool.ElasticPool; replaces the
 * reference's INFER_REQUEST / INFER_REPLY socket path,
 * edl/student_node.py:369-423 and edl/teacher_node.py:157-170, and the
 * coordinator's registry, edl/coordinator.py:99-197, for teachers and
 * students on one box):
 *   edl_ipc_export / edl_ipc_open / edl_ipc_close: CUDA IPC of the student's
 *     soft-label slot ring (handle = 64 bytes; the export names the whole
 *     allocation, `offset` locates `ptr` in it). A teacher process opens it
 *     and its head kernel writes (prob, class) pairs straight into the slot,
 *     over NVLink when the student sits on another GPU.
 *   edl_host_register / edl_host_unregister: map the pool's shared-memory
 *     control block into the device address space, so a teacher's stream
 *     writes a slot's READY tag (edl_stream_write_u32) after its kernels and
 *     the student's host sees it with a plain load — no host waits on the
 *     teacher's side and no device waits on the student's side, so a dead
 *     teacher can never leave a student stream blocked.
 *   edl_memcpy_async: cudaMemcpyAsync(cudaMemcpyDefault) for UVA / IPC
 *     pointers. */
int edl_memcpy_async(void* dst, const void* src, long long bytes, void* stream);
int edl_host_register(void* ptr, long long bytes, void** dev_ptr);
int edl_host_unregister(void* ptr);
int edl_ipc_export(const void* ptr, void* handle, long long* offset);
int edl_ipc_open(const void* handle, void** base);
int edl_ipc_close(void* base);

#ifdef __cplusplus
}
#endif

#endif /* EDL_B200_H */
