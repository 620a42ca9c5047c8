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

// One thread per 16-byte (8-channel) vector of the im2col matrix. I is the
// element-index type: int whenever the element count fits (64-bit division
// and modulo in the index decomposition cost more than the copy itself).
template <typename I>
__global__ void __launch_bounds__(256) im2col_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W,
                                                          int C, int R, int S, int stride, int pad, int P, int Q,
                                                          __nv_bfloat16* __restrict__ out, long long ldo) {
  griddep_wait();
  const int cv = C / 8;                       // 8-channel vectors per pixel
  const int per_row = R * S * cv;
  const I total = static_cast<I>(N) * P * Q * per_row;
  for (I i = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<I>(gridDim.x) * blockDim.x) {
    const I m = i / per_row;
    const int j = static_cast<int>(i - m * per_row);
    const int c8 = j % cv;
    const int rs = j / cv;
    const int s = rs % S, r = rs / S;
    const int q = static_cast<int>(m % Q);
    const I nq = m / Q;
    const int p = static_cast<int>(nq % P);
    const int n = static_cast<int>(nq / P);
    const int h = p * stride - pad + r, w = q * stride - pad + s;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (h >= 0 && h < H && w >= 0 && w < W)
      v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * H + h) * W + w) * C) + c8);
    *reinterpret_cast<uint4*>(out + static_cast<long long>(m) * ldo + static_cast<long long>(rs) * C + 8 * c8) = v;
  }
}

// Packed variant for inputs with few used channels (the RGB stem): the K
// index runs over (r, s, c < c_used) densely, so a 7x7x3 stem has K = 147
// (padded to ldo) instead of 7x7x16. A block builds kPackQ consecutive output
// pixels of one output row: the R x Wt input patch they read is staged in
// shared memory with coalesced 16-byte loads (zeros outside the image), and
// the block's kPackQ * ldo outputs are one contiguous span written as
// coalesced 16-byte stores.
constexpr int kPackQ = 56;

// The patch is staged COMPACT (c_used channels per pixel, rows of Wt pixels),
// so the K run of one filter row (s, c) is contiguous in shared memory. With
// the C-padded pixel pitch (32 B) the 7 taps of a filter row fell on 4 bank
// groups and the 16-bit gathers ran ~8-way bank-conflicted (716 us at batch
// 256, ~1.6 TB/s). Each thread owns one 16-byte output column chunk `ch`
// (8 consecutive K indices) and walks the block's pixels with it, so its 8
// patch offsets are computed once; threads ch = 0..chunks-1 of one pixel
// write one contiguous output row.
// CU / RR / ST / LDO: compile-time c_used, R = S, stride and ldo (0: the
// runtime argument); the <3, 7, 2, 160> instance (the RGB stem) unrolls the
// staging and the gather (the runtime-shaped loops ran ~225 instructions per
// 16-byte output chunk, ALU-bound at 487 us per batch of 256).
template <int CU, int RR, int ST, int LDO>
__global__ void __launch_bounds__(256) im2col_nhwc_packed_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                                 int W, int C, int c_used_rt, int R_rt, int S_rt,
                                                                 int stride_rt, int pad, int P, int Q,
                                                                 __nv_bfloat16* __restrict__ out, long long ldo_rt) {
  griddep_wait();
  const int c_used = CU > 0 ? CU : c_used_rt;
  const int R = RR > 0 ? RR : R_rt, S = RR > 0 ? RR : S_rt;
  const int stride = ST > 0 ? ST : stride_rt;
  const long long ldo = LDO > 0 ? LDO : ldo_rt;
  extern __shared__ __align__(16) uint8_t psm[];
  unsigned short* patch = reinterpret_cast<unsigned short*>(psm);   // [R][Wt][c_used]
  const int qblocks = (Q + kPackQ - 1) / kPackQ;
  const int qb = blockIdx.x % qblocks;
  const long long np = blockIdx.x / qblocks;
  const int p = static_cast<int>(np % P), n = static_cast<int>(np / P);
  const int q0 = qb * kPackQ;
  const int nq = Q - q0 < kPackQ ? Q - q0 : kPackQ;
  const int Wt = (nq - 1) * stride + S;
  const int h0 = p * stride - pad, w0 = q0 * stride - pad;
  // stage the used channels of the R x Wt input patch (zeros outside the image)
  for (int i = threadIdx.x; i < R * Wt; i += blockDim.x) {
    const int r = i / Wt, wl = i - r * Wt;
    const int h = h0 + r, w = w0 + wl;
    const bool in = h >= 0 && h < H && w >= 0 && w < W;
    const __nv_bfloat16* px = x + ((static_cast<long long>(n) * H + (in ? h : 0)) * W + (in ? w : 0)) * C;
    if (c_used <= 8) {   // one 16-byte load covers the used channels
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (in) v = __ldg(reinterpret_cast<const uint4*>(px));
      const unsigned short* e = reinterpret_cast<const unsigned short*>(&v);
      for (int c = 0; c < c_used; ++c) patch[i * c_used + c] = e[c];
    } else {
      const unsigned short* e = reinterpret_cast<const unsigned short*>(px);
      for (int c = 0; c < c_used; ++c) patch[i * c_used + c] = in ? e[c] : static_cast<unsigned short>(0);
    }
  }
  const int chunks = static_cast<int>(ldo / 8);
  const int groups = blockDim.x / chunks;
  const int ch = threadIdx.x % chunks, qg = threadIdx.x / chunks;
  const int krow = S * c_used;            // K run of one filter row
  const int kreal = R * krow;
  const int rowpitch = Wt * c_used;
  int off[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = 8 * ch + j;
    const int r = k / krow;
    off[j] = k < kreal ? r * rowpitch + (k - r * krow) : 0;   // K padding: any in-patch element, masked below
  }
  uint32_t keep[4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
    keep[j] = (8 * ch + 2 * j < kreal ? 0xFFFFu : 0u) | (8 * ch + 2 * j + 1 < kreal ? 0xFFFF0000u : 0u);
  __syncthreads();
  if (qg >= groups) return;
  uint4* dst = reinterpret_cast<uint4*>(out + ((static_cast<long long>(n) * P + p) * Q + q0) * ldo) + ch;
  for (int ql = qg; ql < nq; ql += groups) {
    const int base = ql * stride * c_used;
    uint32_t v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v[j] = (static_cast<uint32_t>(patch[base + off[2 * j]]) | (static_cast<uint32_t>(patch[base + off[2 * j + 1]]) << 16)) &
             keep[j];
    }
    dst[static_cast<long long>(ql) * chunks] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

// argmax (training): per (window, 8-channel vector) one 32-bit word of 4-bit
// window positions r * k + s of the FIRST maximum in scan order (torch's
// rule), for maxpool_bwd_argmax_nhwc_kernel.
template <typename I>
__global__ void __launch_bounds__(256) maxpool_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H, int W,
                                                           int C, int k, int stride, int pad, int P, int Q,
                                                           __nv_bfloat16* __restrict__ out,
                                                           uint32_t* __restrict__ argmax, bool relu_mask) {
  griddep_wait();
  const int cv = C / 8;
  const I total = static_cast<I>(N) * P * Q * cv;
  for (I i = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<I>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    const I m = i / cv;
    const int q = static_cast<int>(m % Q);
    const I nq = m / Q;
    const int p = static_cast<int>(nq % P);
    const int n = static_cast<int>(nq / P);
    float best[8];
    uint32_t arg = 0xFFFFFFFFu;
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
        for (int j = 0; j < 8; ++j) {
          const float f = __bfloat162float(b[j]);
          if (f > best[j]) {
            best[j] = f;
            arg = (arg & ~(0xFu << (4 * j))) | (static_cast<uint32_t>(r * k + s) << (4 * j));
          }
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(best[0], best[1]);
    o.y = pack_bf16x2(best[2], best[3]);
    o.z = pack_bf16x2(best[4], best[5]);
    o.w = pack_bf16x2(best[6], best[7]);
    *reinterpret_cast<uint4*>(out + static_cast<long long>(m) * C + 8 * c8) = o;
    if (relu_mask) {   // a window whose maximum is not > 0 routes no gradient (see the 3x3 / 2 kernel)
      const __nv_bfloat16* ob = reinterpret_cast<const __nv_bfloat16*>(&o);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (!(__bfloat162float(ob[j]) > 0.f)) arg |= 0xFu << (4 * j);
    }
    if (argmax != nullptr) argmax[i] = arg;
  }
}

// 3x3 / stride 2 case of maxpool_nhwc_kernel (the stem pool): the nine
// window loads are issued unconditionally from clamped addresses (invalid
// taps masked to -inf afterwards), so each thread has all nine 16-byte loads
// in flight; the generic kernel's bounds branches serialised them (240 us at
// batch 256, ~2.2 TB/s). Same first-maximum scan order and argmax words.
// ARG: record argmax words (training); inference skips the nibble masks.
// BN: x is the stem conv's raw output z and every tap is first taken through
// training-mode BatchNorm + ReLU, y = bf16(relu(fma(z, gamma rstd, beta -
// mean gamma rstd))), the exact arithmetic of bn_apply_kernel: the stem's y
// (411 MB at batch 256) is never written nor re-read.
struct BnPoolArgs {
  const float* mean;
  const float* rstd;
  const float* gamma;
  const float* beta;
};

template <bool ARG, bool BN = false>
__global__ void __launch_bounds__(256) maxpool3s2_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                              int W, int C, int pad, int P, int Q,
                                                              __nv_bfloat16* __restrict__ out,
                                                              uint32_t* __restrict__ argmax, bool relu_mask,
                                                              BnPoolArgs bn = BnPoolArgs{}) {
  griddep_wait();
  const int cv = C / 8;
  const int total = N * P * Q * cv;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int c8 = i % cv;
    const int m = i / cv;
    const int q = m % Q;
    const int nq = m / Q;
    const int p = nq % P;
    const int n = nq / P;
    const int h0 = 2 * p - pad, w0 = 2 * q - pad;
    uint4 v[9];
    bool ok[9];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int h = h0 + r, w = w0 + s;
        ok[3 * r + s] = h >= 0 && h < H && w >= 0 && w < W;
        const int hc = h < 0 ? 0 : (h >= H ? H - 1 : h), wc = w < 0 ? 0 : (w >= W ? W - 1 : w);
        v[3 * r + s] = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * H + hc) * W + wc) * C) + c8);
      }
    }
    if constexpr (BN) {
      float sc[8], sh[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = 8 * c8 + j;
        sc[j] = __ldg(bn.gamma + c) * __ldg(bn.rstd + c);
        sh[j] = __ldg(bn.beta + c) - __ldg(bn.mean + c) * sc[j];
      }
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const __nv_bfloat16* hz = reinterpret_cast<const __nv_bfloat16*>(&v[t]);
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = fmaxf(fmaf(__bfloat162float(hz[j]), sc[j], sh[j]), 0.f);
        v[t].x = pack_bf16x2(f[0], f[1]);
        v[t].y = pack_bf16x2(f[2], f[3]);
        v[t].z = pack_bf16x2(f[4], f[5]);
        v[t].w = pack_bf16x2(f[6], f[7]);
      }
    }
    // Packed bf16x2 arithmetic (the per-lane float scan was ALU-bound, 362
    // instructions per output vector): invalid taps become -inf, the max is
    // four HMNMX2 per tap, and a scan from the last tap to the first writes
    // each tap's equal-to-max lanes into the output and argmax word, so the
    // FIRST maximum in scan order wins, value (incl. the sign of a zero) and
    // position, exactly as the strict '>' scan.
    uint32_t mx[4] = {0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u};   // -inf
#pragma unroll
    for (int t = 0; t < 9; ++t) {
      if (!ok[t]) v[t] = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
      const uint32_t* vt = reinterpret_cast<const uint32_t*>(&v[t]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const __nv_bfloat162 r = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&mx[k]),
                                         *reinterpret_cast<const __nv_bfloat162*>(&vt[k]));
        mx[k] = *reinterpret_cast<const uint32_t*>(&r);
      }
    }
    uint32_t o[4] = {mx[0], mx[1], mx[2], mx[3]};
    uint32_t arg = 0xFFFFFFFFu;
#pragma unroll
    for (int t = 8; t >= 0; --t) {
      const uint32_t* vt = reinterpret_cast<const uint32_t*>(&v[t]);
      uint32_t e[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        e[k] = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vt[k]),
                           *reinterpret_cast<const __nv_bfloat162*>(&mx[k]));
        o[k] = (vt[k] & e[k]) | (o[k] & ~e[k]);
      }
      // lane 2k <- low half of e[k], lane 2k + 1 <- high half: nibble masks
      if constexpr (ARG) {
        const uint32_t p01 = __byte_perm(e[0], e[1], 0x6420), p23 = __byte_perm(e[2], e[3], 0x6420);
        const uint32_t lo = __byte_perm(p01, p23, 0x6420), hi = __byte_perm(p01, p23, 0x7531);
        const uint32_t nm = (lo & 0x0F0F0F0Fu) | (hi & 0xF0F0F0F0u);
        arg = (arg & ~nm) | (nm & (static_cast<uint32_t>(t) * 0x11111111u));
      }
    }
    *reinterpret_cast<uint4*>(out + static_cast<long long>(m) * C + 8 * c8) = make_uint4(o[0], o[1], o[2], o[3]);
    if (ARG && relu_mask) {
      // training pair behind a ReLU: the pool input's ReLU mask at a window's
      // argmax is (window max > 0), so lanes whose max is not > 0 get the
      // no-match nibble 0xF and the backward needs no full-resolution mask
      uint32_t g[4];
#pragma unroll
      for (int k = 0; k < 4; ++k)
        g[k] = ~__hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&o[k]), __float2bfloat162_rn(0.f));
      const uint32_t p01 = __byte_perm(g[0], g[1], 0x6420), p23 = __byte_perm(g[2], g[3], 0x6420);
      const uint32_t lo = __byte_perm(p01, p23, 0x6420), hi = __byte_perm(p01, p23, 0x7531);
      arg |= (lo & 0x0F0F0F0Fu) | (hi & 0xF0F0F0F0u);
    }
    if (ARG) argmax[i] = arg;
  }
}

// Stride-2 col2im with R, S <= 4: an output row h receives taps r = r0 and
// r0 + 2 only (r0 = (h + pad) % 2), likewise s, so the <= 4 contributions
// are enumerated directly and their loads issued together from clamped
// addresses (masked afterwards), in the generic kernel's (r, s) order: the
// same fp32 sums. The generic kernel's parity / bounds branches serialised
// its loads (the student's stride-2 data gradients: 520 us per step).
__global__ void __launch_bounds__(256) col2im_s2_nhwc_kernel(const __nv_bfloat16* __restrict__ dcol, long long ldc,
                                                             int N, int H, int W, int C, int R, int S, int pad,
                                                             int P, int Q, const __nv_bfloat16* __restrict__ add,
                                                             const __nv_bfloat16* __restrict__ mask,
                                                             __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int cv = C / 8;
  // one block per input row (n, h): the row's tap parity r0 is block-uniform
  // and each item needs one division (by cv), not the four of a flat index
  const int n = blockIdx.x / H, h = blockIdx.x - n * H;
  const int r0 = (h + pad) & 1;
  for (int i = threadIdx.x; i < W * cv; i += blockDim.x) {
    const int w = i / cv, c8 = i - w * cv;
    const int pix = blockIdx.x * W + w;
    const int s0 = (w + pad) & 1;
    const long long off = static_cast<long long>(pix) * C + 8 * c8;
    // the add / mask vectors are loaded up front with the taps
    const uint4 a4 = add != nullptr ? __ldg(reinterpret_cast<const uint4*>(add + off)) : make_uint4(0u, 0u, 0u, 0u);
    const uint4 m4 = mask != nullptr ? __ldg(reinterpret_cast<const uint4*>(mask + off)) : make_uint4(0u, 0u, 0u, 0u);
    uint4 v[4];
    bool ok[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int r = r0 + 2 * a, s = s0 + 2 * b;
        const int p = (h + pad - r) >> 1, q = (w + pad - s) >> 1;   // exact: h + pad - r is even
        const bool valid = r < R && s < S && h + pad - r >= 0 && w + pad - s >= 0 && p < P && q < Q;
        ok[2 * a + b] = valid;
        const long long m = valid ? (static_cast<long long>(n) * P + p) * Q + q : 0;
        const int rs = valid ? r * S + s : 0;
        v[2 * a + b] = __ldg(reinterpret_cast<const uint4*>(dcol + m * ldc + static_cast<long long>(rs) * C) + c8);
      }
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!ok[t]) continue;
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v[t]);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(b[j]);
    }
    if (add != nullptr) {
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&a4);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(b[j]);
    }
    if (mask != nullptr) {
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&m4);
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
template <typename I>
__global__ void __launch_bounds__(256) col2im_nhwc_kernel(const __nv_bfloat16* __restrict__ dcol, long long ldc,
                                                          int N, int H, int W, int C, int R, int S, int stride,
                                                          int pad, int P, int Q, const __nv_bfloat16* __restrict__ add,
                                                          const __nv_bfloat16* __restrict__ mask,
                                                          __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int cv = C / 8;
  const I total = static_cast<I>(N) * H * W * cv;
  for (I i = blockIdx.x * static_cast<I>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<I>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % cv);
    const I pix = i / cv;
    const int w = static_cast<int>(pix % W);
    const I nh = pix / W;
    const int h = static_cast<int>(nh % H);
    const int n = static_cast<int>(nh / H);
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
    const long long off = static_cast<long long>(pix) * C + 8 * c8;
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
// times (mask > 0) if given. One thread per (pixel, 8-channel vector): each
// window's per-channel argmax comes from k*k 16-byte loads (L1-resident: the
// neighbouring threads read the same windows).
__global__ void __launch_bounds__(256) maxpool_bwd_nhwc_kernel(const __nv_bfloat16* __restrict__ x, int N, int H,
                                                               int W, int C, int k, int stride, int pad, int P,
                                                               int Q, const __nv_bfloat16* __restrict__ dy,
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
        // the window (p, q): which channels have (h, w) as their first maximum?
        float best[8];
        uint32_t arg = 0xFFFFFFFFu;           // 4-bit window positions (k * k <= 15)
#pragma unroll
        for (int j = 0; j < 8; ++j) best[j] = -INFINITY;
        for (int rr = 0; rr < k; ++rr) {
          const int hh = p * stride - pad + rr;
          if (hh < 0 || hh >= H) continue;
          for (int ss = 0; ss < k; ++ss) {
            const int ww = q * stride - pad + ss;
            if (ww < 0 || ww >= W) continue;
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((static_cast<long long>(n) * H + hh) * W + ww) * C) + c8);
            const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float f = __bfloat162float(b[j]);
              if (f > best[j]) {
                best[j] = f;
                arg = (arg & ~(0xFu << (4 * j))) | (static_cast<uint32_t>(rr * k + ss) << (4 * j));
              }
            }
          }
        }
        const int mine = r * k + s;
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(dy + ((static_cast<long long>(n) * P + p) * Q + q) * C) + c8);
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&g);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (((arg >> (4 * j)) & 0xFu) == static_cast<uint32_t>(mine)) acc[j] += __bfloat162float(gb[j]);
      }
    }
    const long long off = pix * C + 8 * c8;
    if (mask != nullptr) {
      const uint4 m = __ldg(reinterpret_cast<const uint4*>(mask + off));
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __bfloat162float(mb[j]) > 0.f ? acc[j] : 0.f;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(dx + off) = o;
  }
}

// Max pool backward from the forward's argmax words: each input element
// collects dy of the windows whose recorded first maximum it is (<= 4 windows
// for 3x3 / 2), times (mask > 0) if given. One block per input row (n, h),
// threads over (w, 8-channel vector): one 4-byte word + one 16-byte dy load
// per window. KK / ST: compile-time window / stride (0: runtime k, stride).
template <int KK, int ST>
__global__ void __launch_bounds__(256) maxpool_bwd_argmax_nhwc_kernel(const uint32_t* __restrict__ argmax, int N,
                                                                      int H, int W, int C, int k_rt, int stride_rt,
                                                                      int pad, int P, int Q,
                                                                      const __nv_bfloat16* __restrict__ dy,
                                                                      const __nv_bfloat16* __restrict__ mask,
                                                                      __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int k = KK > 0 ? KK : k_rt;
  const int stride = ST > 0 ? ST : stride_rt;
  const int n = blockIdx.x / H, h = blockIdx.x - (blockIdx.x / H) * H;
  const int cv = C / 8;
  for (int i = threadIdx.x; i < W * cv; i += blockDim.x) {
    const int w = i / cv, c8 = i - w * cv;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int r = 0; r < (KK > 0 ? KK : 16); ++r) {
      if (KK == 0 && r >= k) break;
      const int ph = h + pad - r;
      if (ph < 0 || ph % stride) continue;
      const int p = ph / stride;
      if (p >= P) continue;
#pragma unroll
      for (int s = 0; s < (KK > 0 ? KK : 16); ++s) {
        if (KK == 0 && s >= k) break;
        const int qw = w + pad - s;
        if (qw < 0 || qw % stride) continue;
        const int q = qw / stride;
        if (q >= Q) continue;
        const long long win = (static_cast<long long>(n) * P + p) * Q + q;
        const uint32_t arg = __ldg(argmax + win * cv + c8);
        const uint32_t mine = static_cast<uint32_t>(r * k + s);
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(dy + win * C) + c8);
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&g);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (((arg >> (4 * j)) & 0xFu) == mine) acc[j] += __bfloat162float(gb[j]);
      }
    }
    const long long off = ((static_cast<long long>(n) * H + h) * W + w) * C + 8 * c8;
    if (mask != nullptr) {
      const uint4 m = __ldg(reinterpret_cast<const uint4*>(mask + off));
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __bfloat162float(mb[j]) > 0.f ? acc[j] : 0.f;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(dx + off) = o;
  }
}

// 3x3 / stride 2 case of maxpool_bwd_argmax_nhwc_kernel (the stem pool's
// backward): input row h lies in windows p with 2p - pad + r = h, i.e. taps
// r = r0, r0 + 2 (r0 = (h + pad) & 1), likewise s: <= 4 windows, whose argmax
// words, dy vectors and the mask are all loaded up front from clamped
// addresses (invalid windows masked afterwards). Same (r, s) summation
// order as the generic kernel, whose branches serialised the loads.
// CV > 0: the channel vectors per pixel at compile time (8 for the 64-channel
// stem): the per-item (w, c8) split becomes a shift and a mask (ncu: the
// runtime divisions kept the issue slots 84% busy at 1.8 TB/s).
template <int CV>
__global__ void __launch_bounds__(256) maxpool3s2_bwd_nhwc_kernel(const uint32_t* __restrict__ argmax, int N,
                                                                  int H, int W, int C, int pad, int P, int Q,
                                                                  const __nv_bfloat16* __restrict__ dy,
                                                                  const __nv_bfloat16* __restrict__ mask,
                                                                  __nv_bfloat16* __restrict__ dx) {
  griddep_wait();
  const int cv = CV > 0 ? CV : C / 8;
  const int n = blockIdx.x / H, h = blockIdx.x - n * H;   // one block per input row (n, h)
  const int r0 = (h + pad) & 1;
  bool rok[2];
  long long prow[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int r = r0 + 2 * u, p = (h + pad - r) >> 1;
    rok[u] = r < 3 && h + pad - r >= 0 && p < P;
    prow[u] = rok[u] ? (static_cast<long long>(n) * P + p) * Q : 0;
  }
  for (int i = threadIdx.x; i < W * cv; i += blockDim.x) {
    const int w = i / cv, c8 = i - w * cv;
    const int s0 = (w + pad) & 1;
    const long long off = ((static_cast<long long>(n) * H + h) * W + w) * C + 8 * c8;
    uint4 m4 = make_uint4(0u, 0u, 0u, 0u);
    if (mask != nullptr) m4 = __ldg(reinterpret_cast<const uint4*>(mask + off));
    // per window: the lanes whose argmax nibble is this window's tap, as a
    // zero-nibble test of a ^ (tap * 0x11111111), turned into bf16x2 masks
    // that zero the other lanes' dy (acc starts at +0 and so is never -0:
    // adding a masked +0 leaves it bitwise unchanged, as skipping would)
    uint4 g[4];
    uint32_t z[4];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int r = r0 + 2 * u, s = s0 + 2 * v, q = (w + pad - s) >> 1;
        const bool valid = rok[u] && s < 3 && w + pad - s >= 0 && q < Q;
        const long long win = valid ? prow[u] + q : 0;
        const uint32_t x = __ldg(argmax + win * cv + c8) ^ (static_cast<uint32_t>(r * 3 + s) * 0x11111111u);
        g[2 * u + v] = __ldg(reinterpret_cast<const uint4*>(dy + win * C) + c8);
        const uint32_t zz = ~(((x & 0x77777777u) + 0x77777777u) | x | 0x77777777u);   // bit 4j+3: nibble j == 0
        z[2 * u + v] = valid ? zz : 0u;
      }
    }
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t* gt = reinterpret_cast<const uint32_t*>(&g[t]);
      // byte k of z carries lane 2k's flag in bit 3 and lane 2k + 1's in bit
      // 7; prmt's sign-replicate selectors (bit 3 of a selector nibble; the
      // __byte_perm intrinsic masks it off, hence the asm) broadcast a byte's
      // msb, so one PRMT builds word k's two lane masks
      const uint32_t zl = z[t] << 4;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t lm;
        asm("prmt.b32 %0, %1, %2, %3;" : "=r"(lm) : "r"(zl), "r"(z[t]),
            "r"((8u | k) | ((8u | k) << 4) | ((12u | k) << 8) | ((12u | k) << 12)));
        const uint32_t gm = gt[k] & lm;
        acc[2 * k] += __uint_as_float(gm << 16);
        acc[2 * k + 1] += __uint_as_float(gm & 0xFFFF0000u);
      }
    }
    if (mask != nullptr) {
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m4);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __bfloat162float(mb[j]) > 0.f ? acc[j] : 0.f;
    }
    uint4 o;
    o.x = pack_bf16x2(acc[0], acc[1]);
    o.y = pack_bf16x2(acc[2], acc[3]);
    o.z = pack_bf16x2(acc[4], acc[5]);
    o.w = pack_bf16x2(acc[6], acc[7]);
    *reinterpret_cast<uint4*>(dx + off) = o;
  }
}

bool fits32(long long n) { return n < (1LL << 31) - (1LL << 24); }

int grid_for(long long work) {
  long long b = (work + 255) / 256;
  return static_cast<int>(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

}  // namespace

cudaError_t launch_im2col_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int c_used, int R, int S,
                               int stride, int pad, int P, int Q, __nv_bfloat16* out, long long ldo,
                               cudaStream_t stream) {
  if (c_used < C) {
    if (ldo > 8 * 256 || ldo % 8) return cudaErrorInvalidValue;
    const int Wt = (kPackQ - 1) * stride + S;
    const int smem = R * Wt * c_used * 2;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    const bool stem = c_used == 3 && R == 7 && S == 7 && stride == 2 && ldo == 160;
    const void* kern = stem ? reinterpret_cast<const void*>(im2col_nhwc_packed_kernel<3, 7, 2, 160>)
                            : reinterpret_cast<const void*>(im2col_nhwc_packed_kernel<0, 0, 0, 0>);
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_kernel_attrs(kern, smem);
      if (e != cudaSuccess) return e;
    }
    const long long blocks = static_cast<long long>(N) * P * ((Q + kPackQ - 1) / kPackQ);
    if (stem)
      return launch_pdl(im2col_nhwc_packed_kernel<3, 7, 2, 160>, dim3(static_cast<unsigned>(blocks)), dim3(256), smem,
                        stream, 1, x, N, H, W, C, c_used, R, S, stride, pad, P, Q, out, ldo);
    return launch_pdl(im2col_nhwc_packed_kernel<0, 0, 0, 0>, dim3(static_cast<unsigned>(blocks)), dim3(256), smem,
                      stream, 1, x, N, H, W, C, c_used, R, S, stride, pad, P, Q, out, ldo);
  }
  const long long work = static_cast<long long>(N) * P * Q * R * S * (C / 8);
  if (fits32(work))
    return launch_pdl(im2col_nhwc_kernel<int>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, R, S,
                      stride, pad, P, Q, out, ldo);
  return launch_pdl(im2col_nhwc_kernel<long long>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, R,
                    S, stride, pad, P, Q, out, ldo);
}

cudaError_t launch_maxpool_nhwc(const __nv_bfloat16* x, int N, int H, int W, int C, int k, int stride, int pad,
                                int P, int Q, __nv_bfloat16* out, uint32_t* argmax, bool relu_mask,
                                cudaStream_t stream) {
  if (argmax != nullptr && k * k > 15) return cudaErrorInvalidValue;
  const long long work = static_cast<long long>(N) * P * Q * (C / 8);
  if (k == 3 && stride == 2 && fits32(work) && fits32(static_cast<long long>(N) * H * W * C))
    return argmax != nullptr
               ? launch_pdl(maxpool3s2_nhwc_kernel<true>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W,
                            C, pad, P, Q, out, argmax, relu_mask, BnPoolArgs{})
               : launch_pdl(maxpool3s2_nhwc_kernel<false>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W,
                            C, pad, P, Q, out, argmax, relu_mask, BnPoolArgs{});
  if (fits32(work))
    return launch_pdl(maxpool_nhwc_kernel<int>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, k,
                      stride, pad, P, Q, out, argmax, relu_mask);
  return launch_pdl(maxpool_nhwc_kernel<long long>, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, k,
                    stride, pad, P, Q, out, argmax, relu_mask);
}

cudaError_t launch_bn_relu_maxpool3s2_nhwc(const __nv_bfloat16* z, int N, int H, int W, int C, int pad, int P, int Q,
                                           const float* mean, const float* rstd, const float* gamma,
                                           const float* beta, __nv_bfloat16* out, uint32_t* argmax,
                                           cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * P * Q * (C / 8);
  if (!fits32(work) || !fits32(static_cast<long long>(N) * H * W * C)) return cudaErrorInvalidValue;
  return launch_pdl(maxpool3s2_nhwc_kernel<true, true>, dim3(grid_for(work)), dim3(256), 0, stream, 1, z, N, H, W, C,
                    pad, P, Q, out, argmax, true, BnPoolArgs{mean, rstd, gamma, beta});
}

cudaError_t launch_avgpool_nhwc(const __nv_bfloat16* x, int N, int HW, int C, __nv_bfloat16* out, long long ldo,
                                cudaStream_t stream) {
  return launch_pdl(avgpool_nhwc_kernel, dim3(N), dim3(256), 0, stream, 1, x, HW, C, out, ldo);
}

cudaError_t launch_col2im_nhwc(const __nv_bfloat16* dcol, long long ldc, int N, int H, int W, int C, int R, int S,
                               int stride, int pad, int P, int Q, const __nv_bfloat16* add,
                               const __nv_bfloat16* mask, __nv_bfloat16* dx, cudaStream_t stream) {
  const long long work = static_cast<long long>(N) * H * W * (C / 8);
  if (stride == 2 && R <= 4 && S <= 4 && fits32(static_cast<long long>(N) * H * W * C)) {
    const int threads = W * (C / 8) >= 256 ? 256 : ((W * (C / 8) + 31) / 32) * 32;
    return launch_pdl(col2im_s2_nhwc_kernel, dim3(static_cast<unsigned>(N * H)), dim3(threads), 0, stream, 1, dcol,
                      ldc, N, H, W, C, R, S, pad, P, Q, add, mask, dx);
  }
  if (fits32(work))
    return launch_pdl(col2im_nhwc_kernel<int>, dim3(grid_for(work)), dim3(256), 0, stream, 1, dcol, ldc, N, H, W, C,
                      R, S, stride, pad, P, Q, add, mask, dx);
  return launch_pdl(col2im_nhwc_kernel<long long>, dim3(grid_for(work)), dim3(256), 0, stream, 1, dcol, ldc, N, H, W,
                    C, R, S, stride, pad, P, Q, add, mask, dx);
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
  if (k * k > 15) return cudaErrorInvalidValue;
  const long long work = static_cast<long long>(N) * H * W * (C / 8);
  return launch_pdl(maxpool_bwd_nhwc_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, x, N, H, W, C, k, stride,
                    pad, P, Q, dy, mask, dx);
}

cudaError_t launch_maxpool_bwd_argmax_nhwc(const uint32_t* argmax, int N, int H, int W, int C, int k, int stride,
                                           int pad, int P, int Q, const __nv_bfloat16* dy, const __nv_bfloat16* mask,
                                           __nv_bfloat16* dx, cudaStream_t stream) {
  if (k * k > 15 || k > 16) return cudaErrorInvalidValue;
  const long long rows = static_cast<long long>(N) * H;
  if (rows > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int threads = W * (C / 8) >= 256 ? 256 : ((W * (C / 8) + 31) / 32) * 32;
  if (k == 3 && stride == 2)
    return C == 64 ? launch_pdl(maxpool3s2_bwd_nhwc_kernel<8>, dim3(static_cast<unsigned>(rows)), dim3(threads), 0,
                                stream, 1, argmax, N, H, W, C, pad, P, Q, dy, mask, dx)
                   : launch_pdl(maxpool3s2_bwd_nhwc_kernel<0>, dim3(static_cast<unsigned>(rows)), dim3(threads), 0,
                                stream, 1, argmax, N, H, W, C, pad, P, Q, dy, mask, dx);
  return launch_pdl(maxpool_bwd_argmax_nhwc_kernel<0, 0>, dim3(static_cast<unsigned>(rows)), dim3(threads), 0, stream,
                    1, argmax, N, H, W, C, k, stride, pad, P, Q, dy, mask, dx);
}

// Data-gradient weights of a stride-1 convolution: the transposed, spatially
// flipped filter wf[c][(r', s', k)] = w[k][((R-1-r') * S + (S-1-s')) * C + c],
// so dX = conv(dZ, wf, pad' = R - 1 - pad) runs through the forward
// implicit-GEMM kernel. One thread per output element (weights are small).
__global__ void __launch_bounds__(256) conv_flip_weights_kernel(const __nv_bfloat16* __restrict__ w, long long ldw,
                                                                int K, int C, int RS,
                                                                __nv_bfloat16* __restrict__ wf, long long ldf) {
  griddep_wait();
  const long long total = static_cast<long long>(C) * RS * K;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(o % K);
    const long long t = o / K;
    const int rs = static_cast<int>(t % RS), c = static_cast<int>(t / RS);
    wf[c * ldf + static_cast<long long>(rs) * K + k] = w[k * ldw + static_cast<long long>(RS - 1 - rs) * C + c];
  }
}

// Every layer's flip in one launch (the student's 13 stride-1 layers cost 13
// small launches, ~106 us): a grid-stride walk over the concatenated element
// ranges, each element finding its layer by the prefix offsets.
__global__ void __launch_bounds__(256) conv_flip_weights_many_kernel(FlipGroup g) {
  griddep_wait();
  const int total = g.start[g.count];
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
    int l = 0;
    while (o >= g.start[l + 1]) ++l;
    const int r = o - g.start[l];
    const int K = g.K[l], C = g.C[l], RS = g.RS[l];
    const int k = r % K, t = r / K;
    const int rs = t % RS, c = t / RS;
    g.wf[l][c * g.ldf[l] + static_cast<long long>(rs) * K + k] =
        g.w[l][k * g.ldw[l] + static_cast<long long>(RS - 1 - rs) * C + c];
  }
}

cudaError_t launch_conv_flip_weights_many(const FlipGroup& g, cudaStream_t stream) {
  const int total = g.start[g.count];
  if (total <= 0) return cudaSuccess;
  return launch_pdl(conv_flip_weights_many_kernel, dim3(grid_for(total)), dim3(256), 0, stream, 1, g);
}

cudaError_t launch_conv_flip_weights(const __nv_bfloat16* w, long long ldw, int K, int C, int R, int S,
                                     __nv_bfloat16* wf, long long ldf, cudaStream_t stream) {
  const long long work = static_cast<long long>(C) * R * S * K;
  return launch_pdl(conv_flip_weights_kernel, dim3(grid_for(work)), dim3(256), 0, stream, 1, w, ldw, K, C, R * S, wf,
                    ldf);
}

}  // namespace edl
