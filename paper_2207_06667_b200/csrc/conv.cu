// conv.cu — the data-movement kernels of the cfg4 (ResNet-style) teacher
// path (BASELINE.json configs[3]). The reference has no
// convolutions; parity is against torch.nn.functional on the
// CPU. Activations are NHWC bf16 with C padded to a multiple of 16, so every
// row of the implicit GEMM is 16-byte aligned for TMA.
//
//   im2col_nhwc      conv as GEMM: A[(n,p,q)][(r,s,c)] (zero outside the image),
//                    multiplied by W[k][(r,s,c)] in the tcgen05 GEMM whose
//                    epilogue adds the folded-BN bias, the residual, and ReLU
//   maxpool_nhwc     k x k / stride window max (ResNet stem)
//   avgpool_nhwc     global average pool -> [N][C] (the head GEMM's input)
#include "internal.h"
#include "sm100.cuh"

namespace edl {

namespace {

// One thread per 16-byte (8-channel) vector of the im2col matrix.
__global__ void __launch_bounds__(256) im2col_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W,
                                                          int C, int R, int S, int stride, int pad, int P, int Q,
                                                          __nv_bfloat16* __restrict__ out, long long ldo) {
  griddep_wait();
  const int cv = C / 8;                       // 8-channel vectors per pixel
  const long long per_row = static_cast<long long>(R) * S * cv;
  const long long total = static_cast<long long>(N) * P * Q * per_row;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = i / per_row;
    const int j = static_cast<int>(i - m * per_row);
    const int c8 = j % cv;
    const int rs = j / cv;
    const int s = rs % S, r = rs / S;
    const int q = static_cast<int>(m % Q);
    const int p = static_cast<int>((m / Q) % P);
    const int n = static_cast<int>(m / (static_cast<long long>(P) * Q));
    const int h = p * stride - pad + r, w = q * stride - pad + s;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (h >= 0 && h < H && w >= 0 && w < W)
      v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * H + h) * W + w) * C) + c8);
    *reinterpret_cast<uint4*>(out + m * ldo + static_cast<long long>(rs) * C + 8 * c8) = v;
  }
}

// Packed variant for inputs with few used channels (the RGB stem): the K
// index runs over (r, s, c < c_used) densely, so a 7x7x3 stem has K = 147
// (padded to ldo) instead of 7x7x16. One thread per 16-byte output chunk.
__global__ void __launch_bounds__(256) im2col_nhwc_packed_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                                 int W, int C, int c_used, int R, int S, int stride,
                                                                 int pad, int P, int Q,
                                                                 __nv_bfloat16* __restrict__ out, long long ldo) {
  griddep_wait();
  const int kreal = R * S * c_used;
  const int chunks = static_cast<int>(ldo / 8);
  const long long total = static_cast<long long>(N) * P * Q * chunks;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = i / chunks;
    const int ch = static_cast<int>(i - m * chunks);
    const int q = static_cast<int>(m % Q);
    const int p = static_cast<int>((m / Q) % P);
    const int n = static_cast<int>(m / (static_cast<long long>(P) * Q));
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int kidx = 8 * ch + j;
      v[j] = 0.f;
      if (kidx < kreal) {
        const int c = kidx % c_used, rs = kidx / c_used;
        const int h = p * stride - pad + rs / S, w = q * stride - pad + rs % S;
        if (h >= 0 && h < H && w >= 0 && w < W)
          v[j] = __bfloat162float(x[((static_cast<long long>(n) * H + h) * W + w) * C + c]);
      }
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(out + m * ldo + 8 * ch) = o;
  }
}

__global__ void __launch_bounds__(256) maxpool_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W,
                                                           int C, int k, int stride, int pad, int P, int Q,
                                                           __nv_bfloat16* __restrict__ out) {
  griddep_wait();
  const int cv = C / 8;
  const long long total = static_cast<long long>(N) * P * Q * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    const long long m = i / cv;
    const int q = static_cast<int>(m % Q);
    const int p = static_cast<int>((m / Q) % P);
    const int n = static_cast<int>(m / (static_cast<long long>(P) * Q));
    float best[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) best[j] = -INFINITY;
    for (int r = 0; r < k; ++r) {
      const int h = p * stride - pad + r;
      if (h < 0 || h >= H) continue;
      for (int s = 0; s < k; ++s) {
        const int w = q * stride - pad + s;
        if (w < 0 || w >= W) continue;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * H + h) * W + w) * C) + c8);
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) best[j] = fmaxf(best[j], __bfloat162float(b[j]));
      }
    }
    uint4 o;
    o.x = pack_bf16x2(best[0], best[1]);
    o.y = pack_bf16x2(best[2], best[3]);
    o.z = pack_bf16x2(best[4], best[5]);
    o.w = pack_bf16x2(best[6], best[7]);
    *reinterpret_cast<uint4*>(out + m * C + 8 * c8) = o;
  }
}

// Global average pool: block = one image; threads over 8-channel vectors,
// each summing its channels over all H*W pixels (coalesced across threads).
__global__ void __launch_bounds__(256) avgpool_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int HW, int C,
                                                           __nv_bfloat16* __restrict__ out, long long ldo) {
  griddep_wait();
  const int n = blockIdx.x;
  const int cv = C / 8;
  const float inv = 1.0f / static_cast<float>(HW);
  for (int c8 = threadIdx.x; c8 < cv; c8 += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const __nv_bfloat16* base = x + static_cast<long long>(n) * HW * C + 8 * c8;
    for (int i = 0; i < HW; ++i) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + static_cast<long long>(i) * C));
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(b[j]);
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0] * inv, acc[1] * inv);
    o.y = pack_bf16x2(acc[2] * inv, acc[3] * inv);
    o.z = pack_bf16x2(acc[4] * inv, acc[5] * inv);
    o.w = pack_bf16x2(acc[6] * inv, acc[7] * inv);
    *reinterpret_cast<uint4*>(out + n * ldo + 8 * c8) = o;
  }
}

// ---- backward (cfg4 student)
// dx[n][h][w][c] = sum over (r, s) with h = p*stride - pad + r, w = q*stride -
// pad + s of dcol[(n,p,q)][(r,s,c)]  (+ add[n][h][w][c]), then times
// (mask[n][h][w][c] > 0) if mask is given: the gradient w.r.t. a ReLU
// layer's pre-activation straight from the next conv's column gradient. A
// gather (each output summed by one thread in a fixed order): deterministic.
__global__ void __launch_bounds__(256) col2im_nhwc_kernel(const __nv_bfloat16* __restrict__ dcol, long long ldc,
                                                          int N, int H, int W, int C, int R, int S, int stride,
                                                          int pad, int P, int Q, const __nv_bfloat16* __restrict__ add,
                                                          const __nv_bfloat16* __restrict__ mask,
                                                          __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int cv = C / 8;
  const long long total = static_cast<long long>(N) * H * W * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    const long long pix = i / cv;
    const int w = static_cast<int>(pix % W);
    const int h = static_cast<int>((pix / W) % H);
    const int n = static_cast<int>(pix / (static_cast<long long>(H) * W));
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < R; ++r) {
      const int ph = h + pad - r;
      if (ph < 0 || ph % stride) continue;
      const int p = ph / stride;
      if (p >= P) continue;
      for (int s = 0; s < S; ++s) {
        const int qw = w + pad - s;
        if (qw < 0 || qw % stride) continue;
        const int q = qw / stride;
        if (q >= Q) continue;
        const long long m = (static_cast<long long>(n) * P + p) * Q + q;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(dcol + m * ldc + (static_cast<long long>(r) * S + s) * C) + c8);
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(b[j]);
      }
    }
    const long long off = pix * C + 8 * c8;
    if (add != nullptr) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(add + off));
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(b[j]);
    }
    if (mask != nullptr) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(mask + off));
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __bfloat162float(b[j]) > 0.f ? acc[j] : 0.f;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(dx + off) = o;
  }
}

// Global average pool backward: dx[n][i][c] = df[n][c] / HW, times
// (mask[n][i][c] > 0) if given (the last block's output ReLU).
__global__ void __launch_bounds__(256) avgpool_bwd_nhwc_kernel(const __nv_bfloat16* __restrict__ df, long long ldf,
                                                               int N, int HW, int C,
                                                               const __nv_bfloat16* __restrict__ mask,
                                                               __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int cv = C / 8;
  const float inv = 1.0f / static_cast<float>(HW);
  const long long total = static_cast<long long>(N) * HW * cv;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    const long long pix = i / cv;
    const int n = static_cast<int>(pix / HW);
    const uint4 g = __ldg(reinterpret_cast<const uint4*>(df + n * ldf) + c8);
    const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&g);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(gb[j]) * inv;
    if (mask != nullptr) {
      const uint4 m = __ldg(reinterpret_cast<const uint4*>(mask + pix * C) + c8);
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(mb[j]) > 0.f ? v[j] : 0.f;
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(dx + pix * C + 8 * c8) = o;
  }
}

// Max pool backward as a gather: each input element collects the gradients of
// the windows whose FIRST maximum (scan order r, s) it is, as torch does;
// times (mask > 0) if given.
__global__ void __launch_bounds__(256) maxpool_bwd_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                               int W, int C, int k, int stride, int pad, int P,
                                                               int Q, const __nv_bfloat16* __restrict__ dy,
                                                               const __nv_bfloat16* __restrict__ mask,
                                                               __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const long long total = static_cast<long long>(N) * H * W * C;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const long long pix = i / C;
    const int w = static_cast<int>(pix % W);
    const int h = static_cast<int>((pix / W) % H);
    const int n = static_cast<int>(pix / (static_cast<long long>(H) * W));
    float acc = 0.f;
    for (int r = 0; r < k; ++r) {
      const int ph = h + pad - r;
      if (ph < 0 || ph % stride) continue;
      const int p = ph / stride;
      if (p >= P) continue;
      for (int s = 0; s < k; ++s) {
        const int qw = w + pad - s;
        if (qw < 0 || qw % stride) continue;
        const int q = qw / stride;
        if (q >= Q) continue;
        // the window (p, q): is (h, w) its first maximum?
        float best = -INFINITY;
        int bh = -1, bw = -1;
        for (int rr = 0; rr < k; ++rr) {
          const int hh = p * stride - pad + rr;
          if (hh < 0 || hh >= H) continue;
          for (int ss = 0; ss < k; ++ss) {
            const int ww = q * stride - pad + ss;
            if (ww < 0 || ww >= W) continue;
            const float v = __bfloat162float(x[((static_cast<long long>(n) * H + hh) * W + ww) * C + c]);
            if (v > best) { best = v; bh = hh; bw = ww; }
          }
        }
        if (bh == h && bw == w)
          acc += __bfloat162float(dy[((static_cast<long long>(n) * P + p) * Q + q) * C + c]);
      }
    }
    if (mask != nullptr && !(__bfloat162float(mask[i]) > 0.f)) acc = 0.f;
    dx[i] = __float2bfloat16_rn(acc);
  }
}

int grid_for(long long work) {
  long long b = (work + 255) / 256;
  return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t launch_im2col_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int c_used, int R, int S,
                               int stride, int pad, int P, int Q, __nv_bfloat16* out, long long ldo,
                               cudaStream_t stream) {
  if (c_used < C) {
    const long long work = static_cast<long long>(N) * P * Q * (ldo / 8);
    return launch_pdl(im2col_nhwc_packed_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, c_used,
                      R, S, stride, pad, P, Q, out, ldo);
  }
  const long long work = static_cast<long long>(N) * P * Q * R * S * (C / 8);
  return launch_pdl(im2col_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, R, S, stride,
                    pad, P, Q, out, ldo);
}

cudaError_t launch_maxpool_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int k, int stride, int pad,
                                int P, int Q, __nv_bfloat16* out, cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * P * Q * (C / 8);
  return launch_pdl(maxpool_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, k, stride, pad,
                    P, Q, out);
}

cudaError_t launch_avgpool_nhwc(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* out, long long ldo,
                                cudaStream_t stream) {
  return launch_pdl(avgpool_nhwc_kernel, dim3(N), dim3(256), 0, stream, 1, x, HW, C, out, ldo);
}

cudaError_t launch_col2im_nhwc(const __nv_bfloat16* dcol, long long ldc, int N, int H, int W, int C, int R, int S,
                               int stride, int pad, int P, int Q, const __nv_bfloat16* add,
                               const __nv_bfloat16* mask, __nv_bfloat16* dx, cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * H * W * (C / 8);
  return launch_pdl(col2im_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, dcol, ldc, N, H, W, C, R, S,
                    stride, pad, P, Q, add, mask, dx);
}

cudaError_t launch_avgpool_bwd_nhwc(const __nv_bfloat16* df, long long ldf, int N, int HW, int C,
                                    const __nv_bfloat16* mask, __nv_bfloat16* dx, cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * HW * (C / 8);
  return launch_pdl(avgpool_bwd_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, df, ldf, N, HW, C, mask,
                    dx);
}

cudaError_t launch_maxpool_bwd_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int k, int stride, int pad,
                                    int P, int Q, const __nv_bfloat16* dy, const __nv_bfloat16* mask,
                                    __nv_bfloat16* dx, cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * H * W * C;
  return launch_pdl(maxpool_bwd_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, k, stride,
                    pad, P, Q, dy, mask, dx);
}

}  // namespace edl
