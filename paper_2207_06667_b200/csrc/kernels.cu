// kernels.cu — the HBM-bound (SIMT) kernels of the EDL-Dist hot path.
//
//   kd_loss_kernel        edl/nnkit.py:283-295  fused hard+soft loss and dlogits,
//                         one warp per row, both log-sum-exps in one HBM pass
//   tempered_softmax      edl/nnkit.py:193-208  dense probabilities (reference API)
//   sgd_kernel            edl/nnkit.py:312-322  p -= scale * g on fp32 masters,
//                         refreshes the bf16 operand copy in the same pass
//   gather_rows           edl/student_node.py:145-151  batch = shard[rows]
//   colsum                edl/nnkit.py:306      db = sum over the batch of delta
//   topk_hits             edl/nnkit.py:325-335  top-k accuracy, lower-index ties
#include "internal.h"
#include "sm100.cuh"

#include <cfloat>

namespace edl {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ void set_status(int* status, int code) {
  if (status) atomicCAS(status, 0, code);
}

// ------------------------------------------------------------------ KD loss
// loss_row = alpha * (lse(z) - z_y) + beta * T^2 * (-sum_j q_j (z_{i_j}/T - lse(z/T)))
// dz       = alpha/B (softmax(z) - onehot(y)) + beta*T/B (softmax(z/T) - q)
// q is the teacher's top-k (prob, class) list renormalised to sum 1 (k = K is
// the dense reference case). One warp per row: the row is loaded into
// registers up front (KPL independent loads per lane -> full memory-level
// parallelism), both log-sum-exps come from registers, and only dz is staged
// in shared memory (fp32) so the k sparse corrections can land before the
// coalesced bf16 store. HBM sees one read of z and one write of dz.
constexpr int kKdWarps = 8;

template <int KPL>
__global__ void __launch_bounds__(kKdWarps * 32, (KPL >= 64) ? 1 : (KPL >= 32 ? 2 : 3))
    kd_loss_kernel(const float* __restrict__ z, long long ld_z, const int64_t* __restrict__ labels,
                   const float* __restrict__ qv, const int* __restrict__ qi, int B, int K,
                   int Kw, int k, float alpha, float beta, float T, float* __restrict__ row_loss,
                   float* __restrict__ loss_out, unsigned* __restrict__ ticket,
                   __nv_bfloat16* __restrict__ dz, long long ld_dz, int* __restrict__ status) {
  griddep_wait();
  extern __shared__ float sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float* ds = sm + warp * (32 * KPL);
  const float inv_t = 1.0f / T;
  const float ch = alpha / static_cast<float>(B);
  const float cs = beta * T / static_cast<float>(B);
  const bool use_soft = beta > 0.f && k > 0;

  for (int row = blockIdx.x * kKdWarps + warp; row < B; row += gridDim.x * kKdWarps) {
    const float* zr = z + static_cast<size_t>(row) * ld_z;
    float v[KPL];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      v[i] = c < K ? __ldg(zr + c) : -INFINITY;
    }
    const int64_t y = labels[row];
    float qsum = 0.f, qv_l = 0.f;
    int qi_l = -1;
    if (use_soft && lane < k) {
      qv_l = __ldg(qv + static_cast<size_t>(row) * k + lane);
      qi_l = __ldg(qi + static_cast<size_t>(row) * k + lane);
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) m = fmaxf(m, v[i]);
    m = warp_max(m);
    // the exponentials of both log-sum-exps are kept (v -> exp(z - m), et ->
    // exp((z - m) / T)) and reused for the softmaxes in dz: two MUFU.EX2 per
    // element instead of four (z itself is re-read from L2 only at the k soft
    // classes and at the label)
    float s1 = 0.f, st = 0.f;
    float et[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const float d = v[i] - m;
      v[i] = __expf(d);
      et[i] = __expf(d * inv_t);
      s1 += v[i];
      st += et[i];
    }
    s1 = warp_sum(s1);
    st = warp_sum(st);
    const float lse1 = m + __logf(s1);
    const float lset = m * inv_t + __logf(st);
    const float inv_s1 = 1.0f / s1, inv_st = 1.0f / st;
    const bool y_ok = (y >= 0 && y < K);
    if (!y_ok && lane == 0) set_status(status, -1);
    if (use_soft) {
      float part = qv_l;
      for (int j = lane + 32; j < k; j += 32) part += __ldg(qv + static_cast<size_t>(row) * k + j);
      qsum = warp_sum(part);
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int c = lane + 32 * i;
      float d = 0.f;
      if (alpha > 0.f) d += ch * (v[i] * inv_s1 - (c == y ? 1.f : 0.f));
      if (use_soft) d += cs * (et[i] * inv_st);
      ds[c] = d;
    }
    __syncwarp();
    float lsoft = 0.f;
    if (use_soft) {
      const float inv_q = 1.0f / qsum;
      for (int j = lane; j < k; j += 32) {
        const float q = (j == lane ? qv_l : __ldg(qv + static_cast<size_t>(row) * k + j)) * inv_q;
        const int id = (j == lane ? qi_l : __ldg(qi + static_cast<size_t>(row) * k + j));
        if (id < 0 || id >= K) { set_status(status, -1); continue; }
        ds[id] -= cs * q;
        lsoft += q * (__ldg(zr + id) * inv_t - lset);
      }
      lsoft = -warp_sum(lsoft);
    }
    __syncwarp();
    __nv_bfloat16* dr = dz + static_cast<size_t>(row) * ld_dz;
    for (int c = 2 * lane; c < Kw; c += 64) {
      const float a = c < K ? ds[c] : 0.f;
      const float b = c + 1 < K ? ds[c + 1] : 0.f;
      *reinterpret_cast<__nv_bfloat162*>(dr + c) = __floats2bfloat162_rn(a, b);
    }
    if (lane == 0) {
      float l = 0.f;
      if (alpha > 0.f) l += alpha * (y_ok ? (lse1 - __ldg(zr + y)) : 0.f);
      if (use_soft) l += beta * T * T * lsoft;
      row_loss[row] = l;
    }
    __syncwarp();
  }
}

// Deterministic batch mean of the row losses (fixed association order,
// independent of any grid), a separate tiny launch: a last-block ticket inside
// kd_loss_kernel needed a gpu-scope fence (membar + L1 invalidate) in every
// block, which cost more than this PDL-overlapped launch.
__global__ void __launch_bounds__(256) loss_mean_kernel(const float* __restrict__ row_loss, int B,
                                                         float* __restrict__ loss_out,
                                                         int* __restrict__ status) {
  griddep_wait();
  __shared__ double red[8];
  // 8 independent loads in flight per thread (a dependent strided loop would
  // serialise on L2 latency); fixed-order shuffle + 8-way tree, no grid
  // dependence, so the mean is bitwise reproducible
  double acc = 0.0;
  for (int r0 = threadIdx.x; r0 < B; r0 += 8 * blockDim.x) {
    float f[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int r = r0 + u * blockDim.x;
      f[u] = r < B ? __ldcg(row_loss + r) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += static_cast<double>(f[u]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    const float loss = static_cast<float>(tot / static_cast<double>(B));
    *loss_out = loss;
    if (!isfinite(loss)) set_status(status, -2);
  }
}

cudaError_t launch_loss_mean(const float* row_loss, int B, float* loss_out, int* status, cudaStream_t stream) {
  return launch_pdl(loss_mean_kernel, dim3(1), dim3(256), 0, stream, 1, row_loss, B, loss_out, status);
}

template <int KPL>
static cudaError_t launch_kd_t(const float* logits, long long ld_z, const int64_t* labels,
                               const float* q_vals, const int* q_idx, int B, int K, int Kw, int k,
                               float alpha, float beta, float T, float* row_loss, float* loss_out,
                               unsigned* ticket, __nv_bfloat16* dlogits, long long ld_dz, int* status,
                               cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(kKdWarps) * 32 * KPL * sizeof(float);
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kd_loss_kernel<KPL>), static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  int blocks = (B + kKdWarps - 1) / kKdWarps;
  if (blocks > 148 * 8) blocks = 148 * 8;
  e = launch_pdl(kd_loss_kernel<KPL>, dim3(blocks), dim3(kKdWarps * 32), smem, stream, 1, logits, ld_z,
                             labels, q_vals, q_idx, B, K, Kw, k, alpha, beta, T, row_loss, loss_out, ticket,
                             dlogits, ld_dz, status);
  if (e != cudaSuccess) return e;
  return launch_pdl(loss_mean_kernel, dim3(1), dim3(256), 0, stream, 1, static_cast<const float*>(row_loss), B,
                    loss_out, status);
}

cudaError_t launch_kd_loss(const float* logits, long long ld_z, const int64_t* labels,
                           const float* q_vals, const int* q_idx, int B, int K, int k,
                           float alpha, float beta, float T, float* row_loss, float* loss_out,
                           unsigned* ticket, __nv_bfloat16* dlogits, long long ld_dz,
                           int* status, cudaStream_t stream) {
  // columns written: the padded width (multiple of 16), capped by the row pitch
  const int Kp = ((K + 15) / 16) * 16;
  const int Kw = static_cast<int>(ld_dz < Kp ? ld_dz : Kp);
  const int need = (Kw + 31) / 32;  // columns per lane
#define EDL_KD(KPL)                                                                                  \
  return launch_kd_t<KPL>(logits, ld_z, labels, q_vals, q_idx, B, K, Kw, k, alpha, beta, T, row_loss, \
                          loss_out, ticket, dlogits, ld_dz, status, stream)
  if (need <= 1) EDL_KD(1);
  if (need <= 2) EDL_KD(2);
  if (need <= 4) EDL_KD(4);
  if (need <= 8) EDL_KD(8);
  if (need <= 16) EDL_KD(16);
  if (need <= 32) EDL_KD(32);
  if (need <= 64) EDL_KD(64);
#undef EDL_KD
  return cudaErrorInvalidValue;  // > 2048 classes
}

// ------------------------------------------------------------------ tempered softmax
__global__ void tempered_softmax_kernel(const float* __restrict__ z, long long ld,
                                        float* __restrict__ p, long long ld_p, int B, int K,
                                        float inv_t) {
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= B) return;
  const float* zr = z + static_cast<size_t>(warp) * ld;
  float m = -INFINITY;
  for (int c = lane; c < K; c += 32) m = fmaxf(m, zr[c]);
  m = warp_max(m);
  float s = 0.f;
  for (int c = lane; c < K; c += 32) s += __expf((zr[c] - m) * inv_t);
  s = warp_sum(s);
  const float inv_s = 1.0f / s;
  float* pr = p + static_cast<size_t>(warp) * ld_p;
  for (int c = lane; c < K; c += 32) pr[c] = __expf((zr[c] - m) * inv_t) * inv_s;
}

cudaError_t launch_tempered_softmax(const float* logits, long long ld, float* probs,
                                    long long ld_p, int B, int K, float T, cudaStream_t stream) {
  const int threads = 256;
  const int blocks = (B * 32 + threads - 1) / threads;
  return launch_pdl(tempered_softmax_kernel, dim3(blocks), dim3(threads), 0, stream, 1, logits, ld, probs, ld_p, B, K,
                    1.0f / T);
}

// ------------------------------------------------------------------ SGD
__global__ void sgd_kernel(float* __restrict__ p, __nv_bfloat16* __restrict__ pb,
                           const float* __restrict__ g, long long n, float scale) {
  griddep_wait();
  const long long n4 = n / 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 pv = reinterpret_cast<float4*>(p)[i];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    pv.x -= scale * gv.x; pv.y -= scale * gv.y; pv.z -= scale * gv.z; pv.w -= scale * gv.w;
    reinterpret_cast<float4*>(p)[i] = pv;
    if (pb) {
      uint2 q;
      __nv_bfloat162 a = __floats2bfloat162_rn(pv.x, pv.y), b = __floats2bfloat162_rn(pv.z, pv.w);
      q.x = *reinterpret_cast<uint32_t*>(&a);
      q.y = *reinterpret_cast<uint32_t*>(&b);
      reinterpret_cast<uint2*>(pb)[i] = q;
    }
  }
  for (long long i = n4 * 4 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    p[i] -= scale * g[i];
    if (pb) pb[i] = __float2bfloat16_rn(p[i]);
  }
}

cudaError_t launch_sgd(float* p, __nv_bfloat16* p_bf16, const float* g, long long n, float scale,
                       cudaStream_t stream) {
  const int threads = 256;
  long long blocks = (n / 4 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  return launch_pdl(sgd_kernel, dim3(static_cast<int>(blocks)), dim3(threads), 0, stream, 1, p, p_bf16, g, n, scale);
}

// ------------------------------------------------------------------ gather
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ src, long long ld_src,
                                   const int64_t* __restrict__ idx, __nv_bfloat16* __restrict__ dst,
                                   long long ld_dst, int B, int D, const int64_t* __restrict__ src_lab,
                                   int64_t* __restrict__ dst_lab) {
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= B) return;
  const int64_t r = idx[warp];
  if (dst_lab && lane == 0) dst_lab[warp] = src_lab[r];
  const __nv_bfloat16* s = src + static_cast<size_t>(r) * ld_src;
  __nv_bfloat16* d = dst + static_cast<size_t>(warp) * ld_dst;
  const int v = D / 8;
  // 4 independent 16-byte loads in flight per lane before the stores
  int c = lane;
  for (; c + 96 < v; c += 128) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = __ldg(reinterpret_cast<const uint4*>(s) + c + 32 * u);
#pragma unroll
    for (int u = 0; u < 4; ++u) reinterpret_cast<uint4*>(d)[c + 32 * u] = q[u];
  }
  for (; c < v; c += 32) reinterpret_cast<uint4*>(d)[c] = __ldg(reinterpret_cast<const uint4*>(s) + c);
  for (int e = v * 8 + lane; e < D; e += 32) d[e] = s[e];
}

cudaError_t launch_gather_rows(const __nv_bfloat16* src, long long ld_src, const int64_t* idx,
                               __nv_bfloat16* dst, long long ld_dst, int B, int D,
                               const int64_t* src_labels, int64_t* dst_labels, cudaStream_t stream) {
  const int threads = 256;
  const int blocks = (B * 32 + threads - 1) / threads;
  return launch_pdl(gather_rows_kernel, dim3(blocks), dim3(threads), 0, stream, 1, src, ld_src, idx, dst, ld_dst, B, D,
                    src_labels, dst_labels);
}

// ------------------------------------------------------------------ column sum
// db_l = scale * sum over the batch of delta_l, for up to kMaxGroup layers in
// ONE pair of launches. Pass 1: a block owns 64 rows x 256 columns of one
// layer; each warp issues its 8 rows' 16-byte loads (8 bf16 columns per lane)
// at once, the 8 warps combine in a fixed order -> partial[row chunk][n].
// Pass 2: row chunks summed in order. Deterministic, no atomics. (256-row
// chunks ran at 19% of HBM bandwidth: too few blocks, 4 dependent load rounds
// per warp — profiles/README.md.)
constexpr int kColRows = 64;
constexpr int kColCols = 256;
constexpr int kColRowsPerWarp = kColRows / 8;

__global__ void __launch_bounds__(256) colsum_partial_kernel(ColsumGroup g) {
  griddep_wait();
  __shared__ float red[8][kColCols];
  int p = 0;
  while (p + 1 < g.count && static_cast<int>(blockIdx.x) >= g.blk_start[p + 1]) ++p;
  const int local = blockIdx.x - g.blk_start[p];
  const int cgs = (g.N[p] + kColCols - 1) / kColCols;
  const int cg = local % cgs, rc = local / cgs;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = cg * kColCols + lane * 8;
  const int r0 = rc * kColRows + warp * kColRowsPerWarp;
  const int M = g.M[p], N = g.N[p];
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (n0 < N) {
    const __nv_bfloat16* base = g.x[p] + n0;
    uint4 q[kColRowsPerWarp];
#pragma unroll
    for (int u = 0; u < kColRowsPerWarp; ++u) {
      const int r = r0 + u;
      q[u] = r < M ? __ldg(reinterpret_cast<const uint4*>(base + static_cast<size_t>(r) * g.ld[p]))
                   : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < kColRowsPerWarp; ++u) {
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q[u]);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(h[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[warp][lane * 8 + j] = acc[j];
  __syncthreads();
  const int n = cg * kColCols + threadIdx.x;
  if (n < N) {
    float s = red[0][threadIdx.x];
#pragma unroll
    for (int w = 1; w < 8; ++w) s += red[w][threadIdx.x];
    g.partial[g.part_off[p] + static_cast<long long>(rc) * N + n] = s;
  }
}

// Pass 2: a block owns 32 columns; lane = column, the 8 warps stride the row
// chunks (all loads in flight at once) and combine in a fixed order. (One
// thread per column walking 64 chunks serially cost 12 us.)
__global__ void __launch_bounds__(256) colsum_final_kernel(ColsumGroup g) {
  griddep_wait();
  __shared__ float red[8][32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int t = blockIdx.x * 32 + lane;
  int p = 0;
  while (p < g.count && t >= g.N[p]) { t -= g.N[p]; ++p; }
  const bool valid = p < g.count;
  float s = 0.f;
  if (valid) {
    const int chunks = (g.M[p] + kColRows - 1) / kColRows;
    const float* part = g.partial + g.part_off[p];
    float f[8];
    for (int c0 = warp; c0 < chunks; c0 += 64) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + 8 * u;
        f[u] = c < chunks ? __ldcg(part + static_cast<long long>(c) * g.N[p] + t) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) s += f[u];
    }
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp != 0 || !valid) return;
#pragma unroll
  for (int w = 1; w < 8; ++w) s += red[w][lane];
  if (g.sgd) {   // fused SGD on the bias (edl/nnkit.py:321): b -= eta * db
    const float b = g.out[p][t] - g.scale * s;
    g.out[p][t] = b;
    if (g.out_bf16[p]) g.out_bf16[p][t] = __float2bfloat16_rn(b);
  } else {
    g.out[p][t] = s * g.scale;
  }
}

long long colsum_workspace_floats(int count, const int* M, const int* N) {
  long long w = 0;
  for (int p = 0; p < count; ++p) w += static_cast<long long>((M[p] + kColRows - 1) / kColRows) * N[p];
  return w;
}

cudaError_t launch_colsum_group(ColsumGroup g, cudaStream_t stream) {
  int blocks = 0, cols = 0;
  long long off = 0;
  for (int p = 0; p < g.count; ++p) {
    g.blk_start[p] = blocks;
    g.part_off[p] = off;
    const int chunks = (g.M[p] + kColRows - 1) / kColRows;
    blocks += ((g.N[p] + kColCols - 1) / kColCols) * chunks;
    off += static_cast<long long>(chunks) * g.N[p];
    cols += g.N[p];
  }
  g.blk_start[g.count] = blocks;
  cudaError_t e = launch_pdl(colsum_partial_kernel, dim3(blocks), dim3(256), 0, stream, 1, g);
  if (e != cudaSuccess) return e;
  return launch_pdl(colsum_final_kernel, dim3((cols + 31) / 32), dim3(256), 0, stream, 1, g);
}

cudaError_t launch_colsum(const __nv_bfloat16* x, long long ld, int M, int N, float* partial,
                          float* out, float scale, cudaStream_t stream) {
  ColsumGroup g = {};
  g.count = 1;
  g.x[0] = x;
  g.ld[0] = ld;
  g.M[0] = M;
  g.N[0] = N;
  g.out[0] = out;
  g.scale = scale;
  g.partial = partial;
  return launch_colsum_group(g, stream);
}

// ------------------------------------------------------------------ tall column sums
// Conv bias gradients: colsum over M = B*H*W rows (up to ~1.6M) of N <= 2048
// columns. Block b owns rows [b * rpb, (b + 1) * rpb) of every column: thread
// = (row lane, 8-column vector), eight independent 16-byte loads in flight per
// thread; row lanes combine through shared memory in a fixed order, and the
// final pass sums the per-block partials in block order (deterministic).
__global__ void __launch_bounds__(256) colsum_tall_partial_kernel(const __nv_bfloat16* __restrict__ x, long long ld,
                                                                  int M, int N, int rpb, float* __restrict__ partial) {
  griddep_wait();
  __shared__ float red[256 * 8];
  const int cv = N / 8;
  const int rpp = blockDim.x / cv;        // rows in flight per pass
  const int rl = threadIdx.x / cv, c8 = threadIdx.x % cv;
  const int r0 = blockIdx.x * rpb;
  const int r1 = r0 + rpb < M ? r0 + rpb : M;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  auto add = [&](const uint4& q) {
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(h[j]);
  };
  if (rl < rpp) {
    const __nv_bfloat16* base = x + 8 * c8;
    int r = r0 + rl;
    for (; r + 7 * rpp < r1; r += 8 * rpp) {
      uint4 q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        q[u] = __ldg(reinterpret_cast<const uint4*>(base + static_cast<long long>(r + u * rpp) * ld));
#pragma unroll
      for (int u = 0; u < 8; ++u) add(q[u]);
    }
    for (; r < r1; r += rpp) add(__ldg(reinterpret_cast<const uint4*>(base + static_cast<long long>(r) * ld)));
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) red[threadIdx.x * 8 + j] = acc[j];
  __syncthreads();
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < rpp; ++q) s += red[(q * cv + n / 8) * 8 + n % 8];
    partial[static_cast<long long>(blockIdx.x) * N + n] = s;
  }
}

// 32 columns per block, 32 warps striding the partial rows with 8 loads in
// flight each (a 2-block grid for N = 64, so the parallelism has to come from
// inside the block), combined in a fixed order.
__global__ void __launch_bounds__(1024) colsum_tall_final_kernel(const float* __restrict__ partial, int G, int N,
                                                                 float* __restrict__ out, float scale) {
  griddep_wait();
  __shared__ float red[32][33];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n = blockIdx.x * 32 + lane;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (n < N) {
    int b = warp;
    for (; b + 7 * 32 < G; b += 8 * 32) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += __ldcg(partial + static_cast<long long>(b + 32 * u) * N + n);
    }
    for (; b < G; b += 32) a[0] += __ldcg(partial + static_cast<long long>(b) * N + n);
  }
  red[warp][lane] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  if (warp != 0 || n >= N) return;
  float s = 0.f;
#pragma unroll
  for (int w = 0; w < 32; ++w) s += red[w][lane];
  out[n] = s * scale;
}

int colsum_tall_blocks(int M, int sms) {
  // 4 x 256 threads per SM with 8 16-byte loads in flight each keep HBM busy;
  // fewer partial rows keep the latency-bound final pass short (it ran
  // 7.6-12 us per launch over 8 * 148 partial rows)
  const int g = 4 * sms;
  const int by_rows = (M + 127) / 128;    // at least 128 rows per block
  return by_rows < g ? (by_rows < 1 ? 1 : by_rows) : g;
}

bool colsum_tall_ok(int N) { return N % 8 == 0 && N >= 8 && N <= 2048; }

cudaError_t launch_colsum_tall(const __nv_bfloat16* x, long long ld, int M, int N, float* partial, float* out,
                               float scale, int sms, cudaStream_t stream) {
  const int G = colsum_tall_blocks(M, sms);
  const int rpb = (M + G - 1) / G;
  cudaError_t e = launch_pdl(colsum_tall_partial_kernel, dim3(G), dim3(256), 0, stream, 1, x, ld, M, N, rpb, partial);
  if (e != cudaSuccess) return e;
  return launch_pdl(colsum_tall_final_kernel, dim3((N + 31) / 32), dim3(1024), 0, stream, 1,
                    static_cast<const float*>(partial), G, N, out, scale);
}

// ------------------------------------------------------------------ split-K reduce
// out = sum over s of P[s] (fixed order). P[s] is [GM][GN] fp32; transposed:
// out[r][c] = sum_s P[s][c][r] (the swapped-operand weight gradient, GEMM M =
// kdim, N = cout, back to the [cout][kdim] layout) through a 32 x 33 smem tile.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ P, int ksplit,
                                                            long long sstride, int GM, int GN,
                                                            float* __restrict__ out, long long ldo) {
  griddep_wait();
  const long long total = static_cast<long long>(GM) * GN;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int s = 0;
    for (; s + 7 < ksplit; s += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += __ldcg(P + (s + u) * sstride + i);
    }
    for (; s < ksplit; ++s) a[0] += __ldcg(P + s * sstride + i);
    const int r = static_cast<int>(i / GN), c = static_cast<int>(i % GN);
    out[r * ldo + c] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
}

// One thread per output (1024-thread blocks): the swapped-operand weight
// gradients have few 32 x 32 tiles (36 for a 3x3 64 -> 64 conv, 10 for the
// stem) and deep split-K stacks (29-75 partials), so 256-thread blocks with
// four outputs per thread were latency-bound (22-44 us). Same per-output
// summation order as before.
__global__ void __launch_bounds__(1024) splitk_reduce_t_kernel(const float* __restrict__ P, int ksplit,
                                                               long long sstride, int GM, int GN,
                                                               float* __restrict__ out, long long ldo) {
  griddep_wait();
  __shared__ float tile[32][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int r0 = blockIdx.x * 32;       // output rows = GEMM columns (GN)
  const int c0 = blockIdx.y * 32;       // output cols = GEMM rows (GM)
  {
    const int c = c0 + ty, r = r0 + tx;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (c < GM && r < GN) {
      const float* src = P + static_cast<long long>(c) * GN + r;
      int s = 0;
      for (; s + 7 < ksplit; s += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += __ldcg(src + (s + u) * sstride);
      }
      for (; s < ksplit; ++s) a[0] += __ldcg(src + s * sstride);
    }
    tile[ty][tx] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  }
  __syncthreads();
  const int r = r0 + ty, c = c0 + tx;
  if (r < GN && c < GM) out[r * ldo + c] = tile[tx][ty];
}

cudaError_t launch_splitk_reduce(const float* P, int ksplit, long long sstride, int GM, int GN, bool transposed,
                                 float* out, long long ldo, int sms, cudaStream_t stream) {
  if (transposed)
    return launch_pdl(splitk_reduce_t_kernel, dim3((GN + 31) / 32, (GM + 31) / 32), dim3(1024), 0, stream, 1, P,
                      ksplit, sstride, GM, GN, out, ldo);
  const long long total = static_cast<long long>(GM) * GN;
  long long blocks = (total + 255) / 256;
  if (blocks > 16LL * sms) blocks = 16LL * sms;
  return launch_pdl(splitk_reduce_kernel, dim3(static_cast<unsigned>(blocks)), dim3(256), 0, stream, 1, P, ksplit,
                    sstride, GM, GN, out, ldo);
}

// ------------------------------------------------------------------ top-k accuracy
__global__ void topk_hits_kernel(const float* __restrict__ z, long long ld,
                                 const int64_t* __restrict__ labels, int B, int K, int k,
                                 unsigned* __restrict__ hits) {
  griddep_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  if (warp >= B) return;
  const float* zr = z + static_cast<size_t>(warp) * ld;
  const int64_t y = labels[warp];
  const float zy = zr[y];
  int cnt = 0;
  for (int c = lane; c < K; c += 32) {
    const float v = zr[c];
    cnt += (v > zy || (v == zy && c < y)) ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0 && cnt < k) atomicAdd(hits, 1u);
}

cudaError_t launch_topk_hits(const float* logits, long long ld, const int64_t* labels, int B,
                             int K, int k, unsigned* hits, cudaStream_t stream) {
  const int threads = 256;
  topk_hits_kernel<<<(B * 32 + threads - 1) / threads, threads, 0, stream>>>(logits, ld, labels, B, K, k, hits);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fp32 -> bf16
// Row-blocked cast (refresh of the bf16 weight copy; host fp32 batches staged
// on the device, bench e2e): blockIdx.y strides rows, each thread converts 4
// consecutive columns per iteration (16-byte load, 8-byte store) when the
// row pitches and bases allow it, so there is no per-element division.
template <typename T>
__global__ void cast_bf16_kernel(const T* __restrict__ src, long long ld_src,
                                 __nv_bfloat16* __restrict__ dst, long long ld_dst, int rows,
                                 int cols, int vec) {
  griddep_wait();
  const long long step = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int r = blockIdx.y; r < rows; r += gridDim.y) {
    const T* sr = src + static_cast<size_t>(r) * ld_src;
    __nv_bfloat16* dr = dst + static_cast<size_t>(r) * ld_dst;
    if (vec) {
      const int c4 = cols / 4;
      for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < c4; i += step) {
        float v0, v1, v2, v3;
        if constexpr (sizeof(T) == 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(sr) + i);
          v0 = v.x; v1 = v.y; v2 = v.z; v3 = v.w;
        } else {
          // fp64 -> fp32 -> bf16: the reference's float64 batch through the
          // same double rounding as the host path (numpy astype(float32),
          // then round-to-nearest-even to bf16)
          const double2 a = __ldg(reinterpret_cast<const double2*>(sr) + 2 * i);
          const double2 b = __ldg(reinterpret_cast<const double2*>(sr) + 2 * i + 1);
          v0 = __double2float_rn(a.x); v1 = __double2float_rn(a.y);
          v2 = __double2float_rn(b.x); v3 = __double2float_rn(b.y);
        }
        uint2 o;
        o.x = pack_bf16x2(v0, v1);
        o.y = pack_bf16x2(v2, v3);
        reinterpret_cast<uint2*>(dr)[i] = o;
      }
    } else {
      for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < cols; c += step)
        dr[c] = __float2bfloat16_rn(static_cast<float>(sr[c]));
    }
  }
}

template <typename T>
static cudaError_t launch_cast_t(const T* src, long long ld_src, __nv_bfloat16* dst, long long ld_dst, int rows,
                                 int cols, cudaStream_t stream) {
  const bool vec = cols % 4 == 0 && ld_src % 4 == 0 && ld_dst % 4 == 0 &&
                   reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 8 == 0;
  const long long per_row = vec ? cols / 4 : cols;
  long long bx = (per_row + 255) / 256;
  int by = rows;
  // two 256-thread blocks per SM, each thread looping: the bf16 conversion of a
  // host batch runs beside the teacher's GEMMs and NCCL's kernels (e2e input
  // path) and must not flood the SMs with thousands of CTAs
  const long long target = 148LL * 2;
  if (by > target) by = static_cast<int>(target);
  if (bx * by > target) bx = (target + by - 1) / by;
  if (bx < 1) bx = 1;
  if (by < 1) by = 1;
  return launch_pdl(cast_bf16_kernel<T>, dim3(static_cast<unsigned>(bx), static_cast<unsigned>(by)), dim3(256), 0,
                    stream, 1, src, ld_src, dst, ld_dst, rows, cols, vec ? 1 : 0);
}

cudaError_t launch_cast_bf16(const float* src, long long ld_src, __nv_bfloat16* dst,
                             long long ld_dst, int rows, int cols, cudaStream_t stream) {
  return launch_cast_t(src, ld_src, dst, ld_dst, rows, cols, stream);
}

cudaError_t launch_cast_bf16_f64(const double* src, long long ld_src, __nv_bfloat16* dst,
                                 long long ld_dst, int rows, int cols, cudaStream_t stream) {
  return launch_cast_t(src, ld_src, dst, ld_dst, rows, cols, stream);
}

// ------------------------------------------------------------------ stream delay
// A device-side busy wait of `ns` nanoseconds on one thread (globaltimer):
// TeacherConfig.simulated_delay (edl/teacher_node.py:30-44) on the teacher's
// stream, so a throttled teacher slows its stream, not the host.
__global__ void stream_delay_kernel(unsigned long long ns) {
  griddep_wait();
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

cudaError_t launch_stream_delay(unsigned long long ns, cudaStream_t stream) {
  return launch_pdl(stream_delay_kernel, dim3(1), dim3(32), 0, stream, 1, ns);
}

}  // namespace edl
