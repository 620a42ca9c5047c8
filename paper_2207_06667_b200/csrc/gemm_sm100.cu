// gemm_sm100.cu — the tensor-core kernels of the EDL-Dist hot path (sm_100a).
//
//   C[M,N] = sum_k A[m,k] * B[n,k]      bf16 x bf16 -> fp32 accumulate in TMEM
//
// One warp-specialised, persistent kernel template covers every dense layer the
// reference runs through numpy `@` (edl/nnkit.py:232,243,305,308):
//   forward hidden  h = tanh(x W^T + b)        A=x  (K-major)  B=W (K-major)   EPI_TANH_BF16
//   student logits  z = h W^T + b              A=h  (K-major)  B=W (K-major)   EPI_BIAS_F32
//   backprop data   d = (dY W) * (1 - a^2)     A=dY (K-major)  B=W (MN-major)  EPI_DTANH_BF16
//   backprop weight dW = dY^T a                A=dY (MN-major) B=a (MN-major)  EPI_F32
// and a cluster kernel for the teacher head (edl/nnkit.py:193-208 + top-k, see
// teacher_head_kernel below) whose epilogue never writes logits to HBM.
//
// Roles (256 threads, 1 CTA/SM): warp0 lane0 = TMA producer, warp1 lane0 =
// tcgen05.mma issuer, warp2 = TMEM allocator, warps4-7 = epilogue (each owns the
// 32 TMEM lanes = 32 accumulator rows its warp-in-warpgroup index selects).
// Pipelines: STAGES-deep smem ring (full/empty mbarriers) and a 2-deep TMEM
// accumulator ring (tmem_full/tmem_empty) so tile i's epilogue overlaps tile
// i+1's MMAs. Operand tiles are 128-byte-swizzled TMA boxes of 64 bf16 along
// the contiguous dimension.
#include "internal.h"
#include "sm100.cuh"

namespace edl {

__device__ int g_tanh_mode = 0;

cudaError_t set_tanh_mode(int mode) {
  return cudaMemcpyToSymbol(g_tanh_mode, &mode, sizeof(int));
}

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kThreads = 256;

__host__ __device__ constexpr uint32_t tmem_cols_for(int cols) {
  return cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
}

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN >= 256 ? 4 : BN >= 128 ? 6 : 8;
  static constexpr int kAcc = BN <= 64 ? 4 : 2;          // TMEM accumulator ring (gemm_kernel)
  static constexpr uint32_t kABytes = kBM * kBK * 2;
  static constexpr uint32_t kBBytes = BN * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kEpiBytes = BN * 4;          // the tile's bias slice
  static constexpr uint32_t kStoreBytes = 4 * 2 * 4096;  // TMA-store staging: two 32x32 fp32 tiles per epilogue warp
  static constexpr uint32_t kSmem =
      kStages * kStageBytes + kStoreBytes + kEpiBytes + 1024 /*align*/ + 352 /*barriers*/;
  static_assert(kSmem <= 227 * 1024, "exceeds the sm_100 per-CTA shared memory limit");
};

// Issue the TMA loads of one (A,B) k-block into stage buffers, with per-operand
// L2 eviction policies (pa, pb).
template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ void load_kblock(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                            uint8_t* sa, uint8_t* sb, uint64_t* bar, int m0,
                                            int n0, int k0, uint64_t pa, uint64_t pb) {
  mbar_arrive_expect_tx(bar, GemmCfg<BN>::kStageBytes);
  if constexpr (!A_MN) {
    tma_load_2d_hint(sa, tmA, bar, k0, m0, pa);
  } else {
#pragma unroll
    for (int j = 0; j < kBM / 64; ++j) tma_load_2d_hint(sa + j * 8192, tmA, bar, m0 + 64 * j, k0, pa);
  }
  if constexpr (!B_MN) {
    tma_load_2d_hint(sb, tmB, bar, k0, n0, pb);
  } else {
#pragma unroll
    for (int j = 0; j < BN / 64; ++j) tma_load_2d_hint(sb + j * 8192, tmB, bar, n0 + 64 * j, k0, pb);
  }
}

// Implicit-GEMM convolution: the output tile's first pixel m0 -> its window
// corner (wb, hb) in image nb; k-block kb -> filter tap (r, s) and 64-channel
// block cb (K = (r, s, c), c fastest, C a multiple of 64).
struct ConvTile {
  int wb, hb, nb;
};
__device__ __forceinline__ ConvTile conv_tile(const ConvGeom& cv, int m0) {
  const int pq = cv.P * cv.Q;
  const int nb = m0 / pq, rem = m0 - nb * pq;
  const int p = rem / cv.Q, q = rem - p * cv.Q;
  return ConvTile{q * cv.stride - cv.pad, p * cv.stride - cv.pad, nb};
}
__device__ __forceinline__ void conv_tap(const ConvGeom& cv, int kb, int& cb, int& r, int& s) {
  const int rs = kb / cv.cblocks;
  cb = kb - rs * cv.cblocks;
  r = rs / cv.S;
  s = rs - r * cv.S;
}

// The producer walks k-blocks in order, so it advances (cb, s, r) and the
// pixel cursor incrementally: a single thread issues every TMA of the CTA,
// and two integer divisions per k-block (~60 dependent instructions) made
// it the bottleneck of the 64- and 128-wide conv GEMMs (ncu source view:
// ~130 producer instructions per k-block against 128-256 MMA cycles).
struct TapCursor {
  int cb, r, s;
  TapCursor() = default;
  __device__ __forceinline__ TapCursor(const ConvGeom& cv, int kb) { conv_tap(cv, kb, cb, r, s); }
  __device__ __forceinline__ void next(const ConvGeom& cv) {
    if (++cb == cv.cblocks) {
      cb = 0;
      if (++s == cv.S) { s = 0; ++r; }
    }
  }
};
// Window corner of output pixel m, advanced by 64 pixels per step (weight
// gradient k-blocks).
struct PixelCursor {
  int q, p, nb;
  __device__ __forceinline__ PixelCursor(const ConvGeom& cv, int m) {
    const int pq = cv.P * cv.Q;
    nb = m / pq;
    const int rem = m - nb * pq;
    p = rem / cv.Q;
    q = rem - p * cv.Q;
  }
  __device__ __forceinline__ ConvTile tile(const ConvGeom& cv) const {
    return ConvTile{q * cv.stride - cv.pad, p * cv.stride - cv.pad, nb};
  }
  __device__ __forceinline__ void advance64(const ConvGeom& cv) {
    q += 64;
    while (q >= cv.Q) {
      q -= cv.Q;
      if (++p == cv.P) { p = 0; ++nb; }
    }
  }
};

template <int BN>
__device__ __forceinline__ void load_kblock_conv(const CUtensorMap* tmA, const CUtensorMap* tmB, uint8_t* sa,
                                                 uint8_t* sb, uint64_t* bar, const ConvTile& ct,
                                                 int n0, int kb, const TapCursor& tap, uint64_t pb) {
  mbar_arrive_expect_tx(bar, GemmCfg<BN>::kStageBytes);
  tma_load_im2col_4d(sa, tmA, bar, tap.cb * 64, ct.wb, ct.hb, ct.nb, static_cast<uint16_t>(tap.s),
                     static_cast<uint16_t>(tap.r));
  tma_load_2d_hint(sb, tmB, bar, kb * kBK, n0, pb);
}

// Weight gradient of a convolution: the reduction runs over output pixels
// (k-block kb = pixels [64 kb, 64 kb + 64)), the im2col operand is MN-major
// with MN index (r, s, c): each 64-wide MN chunk is one im2col box of 64
// pixels x 64 channels at one filter tap. Chunks past the real K (r >= R)
// load in-range garbage that only feeds discarded output rows.
template <int BN>
__device__ __forceinline__ void load_kblock_conv_wgrad(const CUtensorMap* tmA, const CUtensorMap* tmB, uint8_t* sa,
                                                       uint8_t* sb, uint64_t* bar, const ConvGeom& cv, int m0,
                                                       int n0, int kb, const ConvTile& ct, const TapCursor* taps,
                                                       uint64_t pa, uint64_t pb) {
  mbar_arrive_expect_tx(bar, GemmCfg<BN>::kStageBytes);
  const int k0 = kb * kBK;
  if (cv.operand == 0) {
#pragma unroll
    for (int j = 0; j < kBM / 64; ++j)
      tma_load_im2col_4d(sa + j * 8192, tmA, bar, taps[j].cb * 64, ct.wb, ct.hb, ct.nb,
                         static_cast<uint16_t>(taps[j].s), static_cast<uint16_t>(taps[j].r));
#pragma unroll
    for (int j = 0; j < BN / 64; ++j) tma_load_2d_hint(sb + j * 8192, tmB, bar, n0 + 64 * j, k0, pb);
  } else {
#pragma unroll
    for (int j = 0; j < kBM / 64; ++j) tma_load_2d_hint(sa + j * 8192, tmA, bar, m0 + 64 * j, k0, pa);
#pragma unroll
    for (int j = 0; j < BN / 64; ++j)
      tma_load_im2col_4d(sb + j * 8192, tmB, bar, taps[j].cb * 64, ct.wb, ct.hb, ct.nb,
                         static_cast<uint16_t>(taps[j].s), static_cast<uint16_t>(taps[j].r));
  }
}

// L2 policy per operand. Measured on B200 (profiles/): evict_last on the
// re-read activations + evict_first on the streamed weights RAISED teacher
// layer-2 DRAM reads (619 -> 683 MB/launch) and lowered tensor-pipe activity,
// so every operand uses the normal policy.
template <int EPI>
__device__ __forceinline__ void gemm_policies(uint64_t& pa, uint64_t& pb) {
  pa = l2_policy_evict_normal();
  pb = l2_policy_evict_normal();
}

// Four 128xBNx16 MMAs consume one 64-deep k-block.
template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_kblock(uint32_t d_tmem, uint32_t a_base, uint32_t b_base,
                                           bool first) {
  constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN, A_MN, B_MN);
  // K-major: a 16-element K slice is 32 bytes further along each swizzled row.
  // MN-major: a 16-row K slice is 16 * 128 bytes further; LBO = one 64-wide box.
  // The descriptors are built once per k-block and stepped in their address
  // field (addr >> 4 stays below 2^14 inside shared memory, so no carry).
  const uint64_t ad0 = A_MN ? smem_desc_sw128(a_base, 8192, 1024) : smem_desc_sw128(a_base, 16, 1024);
  const uint64_t bd0 = B_MN ? smem_desc_sw128(b_base, 8192, 1024) : smem_desc_sw128(b_base, 16, 1024);
#pragma unroll
  for (int k = 0; k < kBK / 16; ++k) {
    const uint64_t ad = ad0 + static_cast<uint64_t>(A_MN ? k * (2048 >> 4) : k * (32 >> 4));
    const uint64_t bd = bd0 + static_cast<uint64_t>(B_MN ? k * (2048 >> 4) : k * (32 >> 4));
    umma_bf16(d_tmem, ad, bd, idesc, (first && k == 0) ? 0u : 1u);
  }
}

// ------------------------------------------------------------------ epilogues
template <int EPI>
__host__ __device__ constexpr bool epi_has_bias() {
  return EPI == EPI_TANH_BF16 || EPI == EPI_BIAS_F32 || EPI == EPI_RELU_BF16 || EPI == EPI_BIAS_BF16;
}

// sb: this chunk's 32 bias values staged in shared memory (stage_bias), or
// null to read ep.bias from global memory.
template <int EPI>
__device__ __forceinline__ void epilogue_store(const EpiArgs& ep, int row, int M, int col0,
                                               int N, float (&v)[32], const float* sb = nullptr,
                                               const uint4* hpre = nullptr, float* out_f32 = nullptr) {
  if (row >= M) return;
  const bool full = (col0 + 32 <= N);
  if constexpr (EPI == EPI_TANH_BF16 || EPI == EPI_BIAS_F32) {
    if (sb != nullptr) {
      const float4* b4 = reinterpret_cast<const float4*>(sb);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 b = b4[i];
        v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
      }
    } else if (ep.bias != nullptr) {
      if (full) {
        const float4* b4 = reinterpret_cast<const float4*>(ep.bias + col0);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float4 b = __ldg(b4 + i);
          v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < N) v[i] += __ldg(ep.bias + col0 + i);
      }
    }
  }
  if constexpr (EPI == EPI_TANH_BF16) {
    const int tm = g_tanh_mode;
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = tanh_act(v[i], tm);
  }
  if constexpr (EPI == EPI_DTANH_BF16) {
    const __nv_bfloat16* h = ep.aux + static_cast<size_t>(row) * ep.ld_aux + col0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q = hpre != nullptr ? hpre[i] : __ldg(reinterpret_cast<const uint4*>(h) + i);
        const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float a = __bfloat162float(hb[j]);
          v[8 * i + j] *= (1.0f - a * a);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) {
          float a = __bfloat162float(h[i]);
          v[i] *= (1.0f - a * a);
        }
    }
  }
  if constexpr (EPI == EPI_F32) {
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= ep.scale;
  }
  if constexpr (EPI == EPI_SGD_F32) {
    // fused SGD (edl/nnkit.py:320): the fp32 master row slice is updated in
    // place, p -= eta * dW, and its bf16 operand copy refreshed; the gradient
    // itself never reaches HBM
    float* o = reinterpret_cast<float*>(ep.out) + static_cast<size_t>(row) * ep.ld_out + col0;
    __nv_bfloat16* ob = ep.out_bf16 + static_cast<size_t>(row) * ep.ld_out + col0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 p = reinterpret_cast<float4*>(o)[i];
        p.x -= ep.scale * v[4 * i]; p.y -= ep.scale * v[4 * i + 1];
        p.z -= ep.scale * v[4 * i + 2]; p.w -= ep.scale * v[4 * i + 3];
        reinterpret_cast<float4*>(o)[i] = p;
        v[4 * i] = p.x; v[4 * i + 1] = p.y; v[4 * i + 2] = p.z; v[4 * i + 3] = p.w;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q;
        q.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
        q.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
        q.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
        q.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
        reinterpret_cast<uint4*>(ob)[i] = q;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) {
          const float p = o[i] - ep.scale * v[i];
          o[i] = p;
          ob[i] = __float2bfloat16_rn(p);
        }
    }
    return;
  }
  if constexpr (EPI == EPI_TANH_BF16 || EPI == EPI_DTANH_BF16) {
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(ep.out) + static_cast<size_t>(row) * ep.ld_out + col0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q;
        q.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
        q.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
        q.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
        q.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
        reinterpret_cast<uint4*>(o)[i] = q;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) o[i] = __float2bfloat16_rn(v[i]);
    }
  } else {
    float* o = (out_f32 != nullptr ? out_f32 : reinterpret_cast<float*>(ep.out)) + static_cast<size_t>(row) * ep.ld_out + col0;
    if (full) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        reinterpret_cast<float4*>(o)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) o[i] = v[i];
    }
  }
}

// Stage the tile's bias slice [n0, n0 + BN) in shared memory; `et` is the
// thread's index among the 128 epilogue threads. Done before waiting for the
// accumulator, so the chunk loop's bias adds never wait on L2.
template <int BN, int EPI>
__device__ __forceinline__ void stage_bias(const EpiArgs& ep, float* sb, int n0, int N, int et) {
  if constexpr (epi_has_bias<EPI>()) {
    for (int j = et; j < BN; j += 128)
      sb[j] = (ep.bias != nullptr && n0 + j < N) ? __ldg(ep.bias + n0 + j) : 0.f;
  }
}

// One accumulator tile (this warp's 32 rows x BN columns at TMEM address
// taddr) through the epilogue, the TMEM load of chunk c+1 in flight while
// chunk c is processed and stored. In one-wave GEMMs nothing hides the
// epilogue, so its serial load latencies were the kernel's critical path.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(const EpiArgs& ep, uint32_t taddr, int row, int M, int n0,
                                              int N, const float* sb, float* out_f32 = nullptr) {
  // EPI_DTANH_BF16 reads the layer's activations: the next chunk's 64 bytes
  // are loaded together with the next TMEM chunk
  constexpr bool kAux = EPI == EPI_DTANH_BF16;
  const bool row_ok = row < M;
  auto aux_ptr = [&](int c) {
    return reinterpret_cast<const uint4*>(ep.aux + static_cast<size_t>(row) * ep.ld_aux + n0 + c);
  };
  uint4 h[4];
  if constexpr (kAux) {
    if (row_ok && n0 + 32 <= N) {
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __ldg(aux_ptr(0) + i);
    }
  }
  uint32_t r[32];
  tmem_ld32_issue(taddr, r);
  tmem_ld_wait(r);
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    uint4 hc[4];
    if constexpr (kAux) {
#pragma unroll
      for (int i = 0; i < 4; ++i) hc[i] = h[i];
      if (row_ok && c + 32 < BN && n0 + c + 64 <= N) {
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __ldg(aux_ptr(c + 32) + i);
      }
    }
    if (c + 32 < BN) tmem_ld32_issue(taddr + c + 32, r);
    if (n0 + c < N)
      epilogue_store<EPI>(ep, row, M, n0 + c, N, v, sb != nullptr ? sb + c : nullptr,
                          (kAux && n0 + c + 32 <= N) ? hc : nullptr, out_f32);
    if (c + 32 < BN) tmem_ld_wait(r);
  }
}

// ---- TMA-store epilogue (bias / tanh / (1-a^2) outputs)
// A thread-per-row store pattern sends every warp store instruction to 32
// different rows (16 B each): measured ~1.5-2 TB/s, the fixed cost that
// dominated the one-wave GEMMs (scripts/gemm_scaling.py: ~11 us at K=64 for
// a 4096 x 1008 fp32 output). Instead each epilogue warp writes its 32 x 32
// chunk into a swizzled shared-memory tile and one TMA store moves it out in
// full lines; ragged M / N edges are clipped by the tensor map.
template <int EPI>
__host__ __device__ constexpr bool epi_tma_store() {
  return EPI == EPI_TANH_BF16 || EPI == EPI_BIAS_F32 || EPI == EPI_DTANH_BF16 || EPI == EPI_RELU_BF16 ||
         EPI == EPI_BIAS_BF16 || EPI == EPI_DRELU_BF16;
}

// 32 bf16 of row `row` at col0 (+ ld), 16-byte loads when the chunk is full.
__device__ __forceinline__ void load_row32(const __nv_bfloat16* base, long long ld, int row, int col0, int N,
                                           float (&o)[32]) {
  const __nv_bfloat16* h = base + static_cast<size_t>(row) * ld + col0;
  if (col0 + 32 <= N) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(h) + i);
      const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
      for (int j = 0; j < 8; ++j) o[8 * i + j] = __bfloat162float(hb[j]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = col0 + i < N ? __bfloat162float(h[i]) : 0.f;
  }
}

// The epilogue math of epilogue_store without its global stores (v in place).
template <int EPI>
__device__ __forceinline__ void epi_math(const EpiArgs& ep, int row, int M, int col0, int N, float (&v)[32],
                                         const float* sb, const uint4* hpre) {
  if constexpr (EPI == EPI_TANH_BF16 || EPI == EPI_BIAS_F32 || EPI == EPI_RELU_BF16 || EPI == EPI_BIAS_BF16) {
    if (sb != nullptr) {
      const float4* b4 = reinterpret_cast<const float4*>(sb);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 b = b4[i];
        v[4 * i] += b.x; v[4 * i + 1] += b.y; v[4 * i + 2] += b.z; v[4 * i + 3] += b.w;
      }
    } else if (ep.bias != nullptr) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) v[i] += __ldg(ep.bias + col0 + i);
    }
  }
  if constexpr (EPI == EPI_TANH_BF16) {
    const int tm = g_tanh_mode;
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = tanh_act(v[i], tm);
  }
  if constexpr (EPI == EPI_RELU_BF16) {
    // residual (ResNet shortcut, bf16, same shape as the output), then ReLU
    if (ep.aux != nullptr && row < M) {
      if (hpre != nullptr) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hpre[i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) v[8 * i + j] += __bfloat162float(hb[j]);
        }
      } else {
        const __nv_bfloat16* h = ep.aux + static_cast<size_t>(row) * ep.ld_aux + col0;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < N) v[i] += __bfloat162float(h[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
  }
  if constexpr (EPI == EPI_DRELU_BF16) {
    // conv data gradient: + the shortcut branch's gradient, then the ReLU
    // derivative of the layer input (its stored post-ReLU activation > 0)
    if (row >= M) return;
    float t[32];
    if (ep.aux != nullptr) {
      load_row32(ep.aux, ep.ld_aux, row, col0, N, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += t[i];
    }
    if (ep.aux2 != nullptr) {
      load_row32(ep.aux2, ep.ld_aux2, row, col0, N, t);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = t[i] > 0.f ? v[i] : 0.f;
    }
  }
  if constexpr (EPI == EPI_DTANH_BF16) {
    if (row >= M) return;
    if (hpre != nullptr) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&hpre[i]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float a = __bfloat162float(hb[j]);
          v[8 * i + j] *= (1.0f - a * a);
        }
      }
    } else {
      const __nv_bfloat16* h = ep.aux + static_cast<size_t>(row) * ep.ld_aux + col0;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) {
          const float a = __bfloat162float(h[i]);
          v[i] *= (1.0f - a * a);
        }
    }
  }
}

// Thread `lane` writes its row's 32 values into the warp's staging tile in the
// tensor map's swizzle: fp32 rows of 128 B (SWIZZLE_128B: 16-byte chunk i at
// i ^ (row % 8)), bf16 rows of 64 B (SWIZZLE_64B: chunk i at i ^ ((row / 2) % 4)).
// Both orders make the eight rows of each 128-bit store phase hit distinct banks.
template <bool kF32>
__device__ __forceinline__ void stage_chunk(uint8_t* stg, int lane, const float (&v)[32]) {
  if constexpr (kF32) {
    float4* base = reinterpret_cast<float4*>(stg + lane * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) base[i ^ (lane & 7)] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
    uint4* base = reinterpret_cast<uint4*>(stg + lane * 64);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 q;
      q.x = pack_bf16x2(v[8 * i + 0], v[8 * i + 1]);
      q.y = pack_bf16x2(v[8 * i + 2], v[8 * i + 3]);
      q.z = pack_bf16x2(v[8 * i + 4], v[8 * i + 5]);
      q.w = pack_bf16x2(v[8 * i + 6], v[8 * i + 7]);
      base[i ^ ((lane >> 1) & 3)] = q;
    }
  }
}

// epilogue_tile with the TMA-store path; row0 = first of this warp's 32 rows.
// stg: this warp's two 4 KB staging tiles, used alternately by store count
// (`stores`, per warp, carried across tiles) so a chunk is written while the
// previous chunk's store is still reading the other tile.
// Residual stream for EPI_RELU_BF16 (conv layers with a shortcut): the
// residual's 32 x 32 bf16 chunks arrive by TMA in the upper 2 KB of the
// warp's two 4 KB store-staging tiles (a bf16 output chunk uses the lower
// 2 KB), two chunks ahead, on two per-warp mbarriers. Per-thread 16-byte
// __ldg's of 32 different rows, one chunk ahead, left the epilogue waiting on
// DRAM: ~1/3 of its stall samples in the 1x1 expansion convs (finding 30).
// ri / rc count issued / consumed chunks per warp (warp-uniform), buffer
// (count & 1), phase (count >> 1) & 1.
struct ResStream {
  const CUtensorMap* map;
  uint8_t* rbuf;      // slot b at rbuf + b * stride
  uint32_t stride;
  uint64_t* bar;      // this warp's `depth` barriers
  uint32_t depth;     // boxes in flight
  uint32_t bytes;     // box bytes: 2048 (32 x 32, SWIZZLE_64B) or 4096 (64 x 32, SWIZZLE_128B)
  uint32_t ri, rc;
  __device__ __forceinline__ void issue(int lane, int col, int row0) {
    const uint32_t b = ri % depth;
    if (lane == 0) {
      mbar_arrive_expect_tx(&bar[b], bytes);
      tma_load_2d(rbuf + b * stride, map, &bar[b], col, row0);
    }
    ++ri;
  }
  // the first `depth` boxes of a tile (cols = the box width)
  __device__ __forceinline__ void prime(int lane, int n0, int N, int BN, int cols, int row0) {
    for (uint32_t j = 0; j < depth; ++j)
      if (static_cast<int>(cols * j) < BN && n0 + static_cast<int>(cols * j) < N) issue(lane, n0 + cols * j, row0);
  }
  // this lane's row of the next 32 x 32 box (bf16 SWIZZLE_64B: 16-byte unit i at i ^ ((row / 2) % 4))
  __device__ __forceinline__ void take(int lane, uint4 (&h)[4]) {
    const uint32_t b = rc % depth;
    mbar_wait(&bar[b], (rc / depth) & 1);
    const uint4* src = reinterpret_cast<const uint4*>(rbuf + b * stride + lane * 64);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = src[i ^ ((lane >> 1) & 3)];
    ++rc;
    __syncwarp();   // every lane has read the buffer before it is refilled
  }
  // this lane's row of the next 64 x 32 box (bf16 SWIZZLE_128B: unit i at i ^ (row % 8))
  __device__ __forceinline__ void take8(int lane, uint4 (&h)[8]) {
    const uint32_t b = rc % depth;
    mbar_wait(&bar[b], (rc / depth) & 1);
    const uint4* src = reinterpret_cast<const uint4*>(rbuf + b * stride + lane * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = src[i ^ (lane & 7)];
    ++rc;
    __syncwarp();
  }
};

// bf16 epilogue on 64-column steps with 128-byte TMA boxes (64 x 32,
// SWIZZLE_128B) for the output stores and the residual loads: half the box
// rows of the 32-column path per byte. The TMA walks a box row by row, and
// with 64-byte rows its row rate bounded the K = 64 residual convs (the
// teacher's 1x1 expansions; profiles/README.md finding 41). stg: 2 x 4 KB.
template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile_tma128(const EpiArgs& ep, uint32_t taddr, int row0, int lane, int M,
                                                     int n0, int N, const float* sb, const CUtensorMap* tmY,
                                                     uint8_t* stg, uint32_t& stores, ResStream* rs) {
  static_assert(EPI == EPI_RELU_BF16 || EPI == EPI_BIAS_BF16 || EPI == EPI_TANH_BF16 || EPI == EPI_DRELU_BF16 ||
                    EPI == EPI_DTANH_BF16,
                "bf16 epilogues only");
  const int row = row0 + lane;
  uint32_t ra[32], rb[32];
  tmem_ld32_issue(taddr, ra);
  tmem_ld32_issue(taddr + 32, rb);
  tmem_ld_wait(ra);
  tmem_ld_wait(rb);
#pragma unroll 1
  for (int c = 0; c < BN; c += 64) {
    float v0[32], v1[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) { v0[i] = __uint_as_float(ra[i]); v1[i] = __uint_as_float(rb[i]); }
    if (c + 64 < BN) {
      tmem_ld32_issue(taddr + c + 64, ra);
      tmem_ld32_issue(taddr + c + 96, rb);
    }
    const bool live = n0 + c < N;   // warp-uniform
    if (live) {
      if (EPI == EPI_RELU_BF16 && rs != nullptr) {
        uint4 h[8];
        rs->take8(lane, h);
        const int cn = c + 64 * static_cast<int>(rs->depth);
        if (cn < BN && n0 + cn < N) rs->issue(lane, n0 + cn, row0);
        uint4 h0[4] = {h[0], h[1], h[2], h[3]}, h1[4] = {h[4], h[5], h[6], h[7]};
        epi_math<EPI>(ep, row, M, n0 + c, N, v0, sb != nullptr ? sb + c : nullptr, h0);
        epi_math<EPI>(ep, row, M, n0 + c + 32, N, v1, sb != nullptr ? sb + c + 32 : nullptr, h1);
      } else {
        epi_math<EPI>(ep, row, M, n0 + c, N, v0, sb != nullptr ? sb + c : nullptr, nullptr);
        epi_math<EPI>(ep, row, M, n0 + c + 32, N, v1, sb != nullptr ? sb + c + 32 : nullptr, nullptr);
      }
      uint8_t* buf = stg + (stores & 1) * 4096;
      if (lane == 0) bulk_wait_read1();        // only the newest store may still be reading
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(buf + lane * 128);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 q;
        q.x = pack_bf16x2(v0[8 * i + 0], v0[8 * i + 1]);
        q.y = pack_bf16x2(v0[8 * i + 2], v0[8 * i + 3]);
        q.z = pack_bf16x2(v0[8 * i + 4], v0[8 * i + 5]);
        q.w = pack_bf16x2(v0[8 * i + 6], v0[8 * i + 7]);
        dst[i ^ (lane & 7)] = q;
        q.x = pack_bf16x2(v1[8 * i + 0], v1[8 * i + 1]);
        q.y = pack_bf16x2(v1[8 * i + 2], v1[8 * i + 3]);
        q.z = pack_bf16x2(v1[8 * i + 4], v1[8 * i + 5]);
        q.w = pack_bf16x2(v1[8 * i + 6], v1[8 * i + 7]);
        dst[(4 + i) ^ (lane & 7)] = q;
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmY, buf, n0 + c, row0);
        bulk_commit();
      }
      ++stores;
    }
    if (c + 64 < BN) {
      tmem_ld_wait(ra);
      tmem_ld_wait(rb);
    }
  }
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile_tma(const EpiArgs& ep, uint32_t taddr, int row0, int lane, int M,
                                                  int n0, int N, const float* sb, const CUtensorMap* tmY,
                                                  uint8_t* stg, uint32_t& stores, ResStream* rs = nullptr) {
  // the (1 - a^2) factor or the residual: a bf16 row segment per chunk
  constexpr bool kAux = EPI == EPI_DTANH_BF16 || EPI == EPI_RELU_BF16;
  const int row = row0 + lane;
  const bool row_ok = row < M && (EPI != EPI_RELU_BF16 || (ep.aux != nullptr && rs == nullptr));
  auto aux_ptr = [&](int c) {
    return reinterpret_cast<const uint4*>(ep.aux + static_cast<size_t>(row) * ep.ld_aux + n0 + c);
  };
  uint4 h[4];
  if constexpr (kAux) {
    if (row_ok && n0 + 32 <= N) {
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __ldg(aux_ptr(0) + i);
    }
  }
  uint32_t r[32];
  tmem_ld32_issue(taddr, r);
  tmem_ld_wait(r);
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
    uint4 hc[4];
    if constexpr (kAux) {
#pragma unroll
      for (int i = 0; i < 4; ++i) hc[i] = h[i];
      if (row_ok && c + 32 < BN && n0 + c + 64 <= N) {
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __ldg(aux_ptr(c + 32) + i);
      }
    }
    if (c + 32 < BN) tmem_ld32_issue(taddr + c + 32, r);
    const bool live = n0 + c < N;   // warp-uniform
    if (EPI == EPI_RELU_BF16 && rs != nullptr && live) {
      rs->take(lane, hc);
      const int cn = c + 32 * static_cast<int>(rs->depth);
      if (cn < BN && n0 + cn < N) rs->issue(lane, n0 + cn, row0);
      epi_math<EPI>(ep, row, M, n0 + c, N, v, sb != nullptr ? sb + c : nullptr, hc);
    } else if (live) {
      epi_math<EPI>(ep, row, M, n0 + c, N, v, sb != nullptr ? sb + c : nullptr,
                    (kAux && n0 + c + 32 <= N) ? hc : nullptr);
    }
    if (live) {
      uint8_t* buf = stg + (stores & 1) * 4096;
      if (lane == 0) bulk_wait_read1();        // only the newest store (other tile) may still be reading
      __syncwarp();
      stage_chunk<EPI == EPI_BIAS_F32>(buf, lane, v);   // bf16 tile unless the fp32 logits
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmY, buf, n0 + c, row0);
        bulk_commit();
      }
      ++stores;
    }
    if (c + 32 < BN) tmem_ld_wait(r);
  }
}

// Tile raster: groups of kRasterGroup m-tiles, m fastest inside a group,
// then n, then the next group. A wave of ~148 tiles then covers a
// kRasterGroup x ~(148 / kRasterGroup) block, and the group's A panels stay
// L2-resident across the waves that sweep its n range. With plain m-fastest
// order every wave re-read the whole A operand from DRAM (teacher layer 2:
// 676 MB per launch against 256 MB algorithmic, profiles/).
// Only when A is too big to stay resident anyway: with a 25 MB A (teacher
// layer 1) m-fastest already reads it once, and grouping would re-read B.
constexpr int kRasterGroup = 8;
__device__ __forceinline__ int raster_group(int num_m, int M, int K) {
  return static_cast<long long>(M) * K * 2 > (32ll << 20) ? kRasterGroup : num_m;
}
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int group, int& mt, int& nt) {
  const int per_group = group * num_n;
  const int g = t / per_group;
  const int r = t - g * per_group;
  const int gm = num_m - g * group < group ? num_m - g * group : group;
  mt = g * group + r % gm;
  nt = r / gm;
}

// ------------------------------------------------------------------ GEMM
// W128: bf16 outputs without a residual in 64 x 32 SWIZZLE_128B boxes
// (epilogue_tile_tma128), as in the pair kernel.
template <int BN, bool A_MN, bool B_MN, int EPI, bool W128 = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR, int M, int N,
                int K, EpiArgs ep) {
  using Cfg = GemmCfg<BN>;
  unsigned* const sched = ep.sched;
  constexpr int S = Cfg::kStages;
  // TMEM accumulator ring depth: 4 for BN = 64 (short-K conv tiles: the
  // epilogue and the TMA latency alternate as the stall; 2 deep left both
  // the MMA and the producer waiting), 2 otherwise
  constexpr int kAcc = Cfg::kAcc;
  constexpr uint32_t kTmemCols = tmem_cols_for(kAcc * BN);
  constexpr bool kW128 = W128;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* stg = sB + S * Cfg::kBBytes;                              // [4 warps][2][4 KB] TMA-store staging
  float* sbias = reinterpret_cast<float*>(stg + Cfg::kStoreBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + kAcc;
  uint64_t* tile_full = tempty + kAcc;    // [4] tile-index ring
  uint64_t* tile_empty = tile_full + 4;   // [4]
  int* tile_ring = reinterpret_cast<int*>(tile_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + 4);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);   // [4 warps][2] residual stream
  // the residual of EPI_RELU_BF16 arrives by TMA (ResStream)
  const bool tma_res = EPI == EPI_RELU_BF16 && ep.aux != nullptr;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < kAcc; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4); }
    // tile ring consumers: the MMA thread, the second producer, 4 epilogue warps
    for (int s = 0; s < 4; ++s) { mbar_init(&tile_full[s], 1); mbar_init(&tile_empty[s], 2 + 4); }
    if (tma_res) {
      prefetch_tmap(&tmR);
      for (int s = 0; s < 8; ++s) mbar_init(&rbar[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // PDL: everything above overlapped the previous kernel's tail

  const int num_m = (M + kBM - 1) / kBM;
  const int num_n = (N + BN - 1) / BN;
  const int mn_tiles = num_m * num_n;
  const int tiles = mn_tiles * ep.ksplit;
  const int nk_all = (K + kBK - 1) / kBK;
  const int kps = (nk_all + ep.ksplit - 1) / ep.ksplit;   // k-blocks per split
  const int rgroup = raster_group(num_m, M, K);
  // work item t -> (split, output tile, k-block range)
  auto decode = [&](int t, int& mt, int& nt, int& kb0, int& kb1) -> int {
    const int split = t / mn_tiles;
    tile_coords(t - split * mn_tiles, num_m, num_n, rgroup, mt, nt);
    kb0 = split * kps;
    kb1 = kb0 + kps < nk_all ? kb0 + kps : nk_all;
    return split;
  };

  // Dynamic tile scheduler: the producer claims tiles from a per-stream
  // global counter and publishes them to the MMA and epilogue roles through a
  // 4-deep smem ring. A CTA that starts late (its SM was busy with another
  // stream's kernel) simply claims fewer tiles, so concurrent teacher and
  // student kernels share the SMs without a tail; the last CTA to exit
  // resets the counter for the next launch on the stream (PDL orders it).
  auto next_tile = [&](int i) -> int {
    return sched ? static_cast<int>(atomicAdd(sched, 1u)) : static_cast<int>(blockIdx.x + i * gridDim.x);
  };

  if ((warp == 0 || warp == 3) && lane == 0) {
    // Two producer threads split the k-blocks by parity (warp 0: even, warp 3:
    // odd; S is even, so each owns every other stage). One thread's issue
    // chain (barrier wait, expect_tx, two TMA issues, cursor update: ~50
    // instructions at several cycles each) is longer than a 64- or 128-wide
    // k-block's 128-256 MMA cycles (ncu, finding 32). Warp 0 claims tiles
    // and publishes them; warp 3 reads them from the ring like the MMA role.
    static_assert(S % 2 == 0, "the producer split needs an even stage count");
    const uint32_t par = warp == 0 ? 0u : 1u;
    uint64_t pa, pb;
    gemm_policies<EPI>(pa, pb);
    uint32_t g = 0;
    for (int i = 0;; ++i) {
      const int slot = i & 3;
      int t;
      if (par == 0) {
        mbar_wait(&tile_empty[slot], ((i >> 2) & 1) ^ 1);
        t = next_tile(i);
        tile_ring[slot] = t;
        mbar_arrive(&tile_full[slot]);
      } else {
        mbar_wait(&tile_full[slot], (i >> 2) & 1);
        t = tile_ring[slot];
        mbar_arrive(&tile_empty[slot]);
      }
      if (t >= tiles) break;
      int mt, nt, kb0, kb1;
      decode(t, mt, nt, kb0, kb1);
      const int m0 = mt * kBM, n0 = nt * BN;
      if constexpr (!A_MN && !B_MN) {
        if (ep.conv.Q > 0) {   // implicit-GEMM convolution: A tiles from the im2col map
          const ConvTile ct = conv_tile(ep.conv, m0);
          TapCursor tap(ep.conv, kb0);
          for (int kb = kb0; kb < kb1; ++kb, ++g, tap.next(ep.conv)) {
            if ((g & 1u) != par) continue;
            const int s = g % S;
            mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
            load_kblock_conv<BN>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes, &full[s], ct, n0, kb,
                                 tap, pb);
          }
          continue;
        }
      }
      if constexpr (A_MN && B_MN) {
        if (ep.conv.Q > 0) {   // convolution weight gradient: the im2col operand from its map
          constexpr int kTaps = (kBM > BN ? kBM : BN) / 64;
          TapCursor taps[kTaps] = {};
          const int mn0 = (ep.conv.operand == 0 ? m0 : n0) / 64;
#pragma unroll
          for (int j = 0; j < kTaps; ++j) taps[j] = TapCursor(ep.conv, mn0 + j);
          PixelCursor px(ep.conv, kb0 * kBK);
          for (int kb = kb0; kb < kb1; ++kb, ++g, px.advance64(ep.conv)) {
            if ((g & 1u) != par) continue;
            const int s = g % S;
            mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
            load_kblock_conv_wgrad<BN>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes, &full[s],
                                       ep.conv, m0, n0, kb, px.tile(ep.conv), taps, pa, pb);
          }
          continue;
        }
      }
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        if ((g & 1u) != par) continue;
        const int s = g % S;
        mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
        load_kblock<BN, A_MN, B_MN>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                    &full[s], m0, n0, kb * kBK, pa, pb);
      }
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t g = 0;
    for (uint32_t i = 0;; ++i) {
      const int slot = i & 3;
      mbar_wait(&tile_full[slot], (i >> 2) & 1);
      const int t = tile_ring[slot];
      mbar_arrive(&tile_empty[slot]);
      if (t >= tiles) break;
      int mt, nt, kb0, kb1;
      decode(t, mt, nt, kb0, kb1);
      const uint32_t as = i % kAcc;
      mbar_wait(&tempty[as], ((i / kAcc) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * BN;
      for (int kb = kb0; kb < kb1; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&full[s], (g / S) & 1);
        tc_fence_after();
        mma_kblock<BN, A_MN, B_MN>(d, smem_u32(sA + s * Cfg::kABytes),
                                   smem_u32(sB + s * Cfg::kBBytes), kb == kb0);
        umma_commit(&empty[s]);
      }
      umma_commit(&tfull[as]);
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    uint32_t stores = 0;
    ResStream rs{&tmR, stg + e * 8192 + 2048, 4096u, rbar + 2 * e, 2u, 2048u, 0u, 0u};
    int staged_n0 = -1;
    for (uint32_t i = 0;; ++i) {
      const int slot = i & 3;
      mbar_wait(&tile_full[slot], (i >> 2) & 1);
      const int t = tile_ring[slot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&tile_empty[slot]);
      if (t >= tiles) break;
      int mt, nt, kb0, kb1;
      const int split = decode(t, mt, nt, kb0, kb1);
      const int m0 = mt * kBM, n0 = nt * BN;
      // split-K partials: split s writes its slice of the fp32 workspace. (A
      // by-value copy of `ep` with a patched `out` here broke the split-K
      // results once EpiArgs outgrew 128 bytes; the slice pointer is passed
      // down instead.)
      float* const split_out = split ? static_cast<float*>(ep.out) + split * ep.split_stride : nullptr;
      float* sb = sbias;
      if (tma_res) rs.prime(lane, n0, N, BN, kW128 ? 64 : 32, m0 + 32 * e);   // behind this tile's MMAs
      // the bias slice only changes with n0 (one n-tile: staged once per CTA);
      // the first barrier keeps a re-stage behind every warp's previous tile
      if (epi_has_bias<EPI>() && n0 != staged_n0) {
        if (staged_n0 >= 0) epi_bar_sync();
        stage_bias<BN, EPI>(ep, sb, n0, N, static_cast<int>(threadIdx.x) - 128);
        epi_bar_sync();
        staged_n0 = n0;
      }
      const uint32_t as = i % kAcc;
      mbar_wait(&tfull[as], (i / kAcc) & 1);
      tc_fence_after();
      if constexpr (kW128)
        epilogue_tile_tma128<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e,
                                      lane, M, n0, N, epi_has_bias<EPI>() ? sb : nullptr, &tmY, stg + e * 8192, stores,
                                      nullptr);
      else if constexpr (epi_tma_store<EPI>())
        epilogue_tile_tma<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e,
                                   lane, M, n0, N, epi_has_bias<EPI>() ? sb : nullptr, &tmY, stg + e * 8192, stores,
                                   tma_res ? &rs : nullptr);
      else
        epilogue_tile<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e + lane,
                               M, n0, N, epi_has_bias<EPI>() ? sb : nullptr, split_out);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
    if constexpr (epi_tma_store<EPI>()) {   // this warp's TMA stores are complete before smem goes away
      if (lane == 0) bulk_wait0();
      __syncwarp();
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
  if (sched && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1u) == gridDim.x - 1) {   // last CTA out: reset for the next launch
      atomicExch(sched, 0u);
      atomicExch(sched + 1, 0u);
    }
  }
}

// ------------------------------------------------------------------ CTA-pair GEMM
// The same contract as gemm_kernel on 256 x BN tiles computed by a CTA pair
// (cluster of 2, cta_group::2): rank r stages A rows [m0+128r, +128) and B
// rows [n0 + r*BN/2, +BN/2); rank 0's single MMA thread issues 256 x BN x 16
// MMAs that read both CTAs' halves, so each SM pulls 2/3 of the operand bytes
// per FLOP that a 128 x BN single-CTA tile needs (the L2 -> SM TMA stream is
// what limits the single-CTA kernel on the teacher's big layers).
// Pipelines: the smem ring's full barriers live in rank 0 (both CTAs' TMA
// loads complete there); empty / tmem-full barriers are multicast-committed
// to both CTAs; tmem-empty (rank 0) collects all 8 epilogue warps. Tiles come
// from the per-stream counter through rank 0's producer, which publishes each
// tile index into both CTAs' rings.
template <int BN>
struct PairCfg {
  static constexpr int kHalfN = BN / 2;
  static constexpr uint32_t kABytes = kBM * kBK * 2;
  static constexpr uint32_t kBBytes = kHalfN * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
  static constexpr uint32_t kEpiBytes = BN * 4;
  static constexpr uint32_t kStoreBytes = 4 * 2 * 4096;
  static constexpr uint32_t kSmem = kStages * kStageBytes + kStoreBytes + kEpiBytes + 1024 + 320;
  static_assert(kSmem <= 227 * 1024, "exceeds the sm_100 per-CTA shared memory limit");
};

template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ void load_kblock_pair(const CUtensorMap* tmA, const CUtensorMap* tmB,
                                                 uint8_t* sa, uint8_t* sb, uint32_t bar, int m0,
                                                 int n0, int k0) {
  if constexpr (!A_MN) {
    tma_load_2d_pair(sa, tmA, bar, k0, m0);
  } else {
#pragma unroll
    for (int j = 0; j < kBM / 64; ++j) tma_load_2d_pair(sa + j * 8192, tmA, bar, m0 + 64 * j, k0);
  }
  if constexpr (!B_MN) {
    tma_load_2d_pair(sb, tmB, bar, k0, n0);
  } else {
#pragma unroll
    for (int j = 0; j < PairCfg<BN>::kHalfN / 64; ++j)
      tma_load_2d_pair(sb + j * 8192, tmB, bar, n0 + 64 * j, k0);
  }
}

template <int BN, bool A_MN, bool B_MN>
__device__ __forceinline__ void mma_kblock_pair(uint32_t d_tmem, uint32_t a_base, uint32_t b_base,
                                                bool first) {
  constexpr uint32_t idesc = idesc_bf16_f32(2 * kBM, BN, A_MN, B_MN);
  const uint64_t ad0 = A_MN ? smem_desc_sw128(a_base, 8192, 1024) : smem_desc_sw128(a_base, 16, 1024);
  const uint64_t bd0 = B_MN ? smem_desc_sw128(b_base, 8192, 1024) : smem_desc_sw128(b_base, 16, 1024);
#pragma unroll
  for (int k = 0; k < kBK / 16; ++k) {
    const uint64_t ad = ad0 + static_cast<uint64_t>(A_MN ? k * (2048 >> 4) : k * (32 >> 4));
    const uint64_t bd = bd0 + static_cast<uint64_t>(B_MN ? k * (2048 >> 4) : k * (32 >> 4));
    umma_bf16_pair(d_tmem, ad, bd, idesc, (first && k == 0) ? 0u : 1u);
  }
}

// W128 (bf16 conv epilogues, edl_conv_fwd_nhwc): outputs and residual in
// 64 x 32 SWIZZLE_128B boxes (epilogue_tile_tma128). With a residual
// (EPI_RELU_BF16) the operand ring gives up two stages for a 4-deep 4 KB
// residual ring per epilogue warp.
template <int BN, bool A_MN, bool B_MN, int EPI, bool W128 = false>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR, int M, int N,
                     int K, EpiArgs ep) {
  using Cfg = PairCfg<BN>;
  unsigned* const sched = ep.sched;
  constexpr bool kW128 = W128;
  constexpr bool kResRing = W128 && EPI == EPI_RELU_BF16;
  constexpr int kRD = 4;                                   // residual boxes in flight (kResRing)
  constexpr int S = Cfg::kStages - (kResRing ? 2 : 0);
  static_assert(!kResRing || (2 * kRD * 4096 <= 2 * Cfg::kABytes && 2 * kRD * 4096 <= 2 * Cfg::kBBytes),
                "the residual ring must fit the two freed stages");
  constexpr uint32_t kTmemCols = tmem_cols_for(2 * BN);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cfg::kStages * Cfg::kABytes;
  uint8_t* stg = sB + Cfg::kStages * Cfg::kBBytes;                   // [4 warps][2][4 KB] TMA-store staging
  float* sbias = reinterpret_cast<float*>(stg + Cfg::kStoreBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* tile_full = tempty + 2;       // [4] tile-index ring
  uint64_t* tile_empty = tile_full + 4;   // [4] (rank 0's is the one used)
  int* tile_ring = reinterpret_cast<int*>(tile_empty + 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + 4);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(tmem_slot + 2);   // [4 warps][2 or kRD] residual stream
  // the residual of EPI_RELU_BF16 arrives by TMA (ResStream)
  const bool tma_res = EPI == EPI_RELU_BF16 && ep.aux != nullptr;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 8); }
    // tile ring: rank 0's MMA + 4 epilogue warps, rank 1's producer + 4 epilogue warps
    for (int s = 0; s < 4; ++s) { mbar_init(&tile_full[s], 1); mbar_init(&tile_empty[s], 10); }
    if (tma_res) {
      prefetch_tmap(&tmR);
      for (int s = 0; s < 4 * (kResRing ? kRD : 2); ++s) mbar_init(&rbar[s], 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();      // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();

  const int num_m = (M + 2 * kBM - 1) / (2 * kBM);
  const int num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int nk = (K + kBK - 1) / kBK;
  const int rgroup = ep.raster > 0 ? (ep.raster < num_m ? ep.raster : num_m) : raster_group(num_m, M, K);
  const int pair = static_cast<int>(blockIdx.x) / 2;
  const int npairs = static_cast<int>(gridDim.x) / 2;
  const uint32_t full0 = mapa(smem_u32(full), 0);           // rank 0's full[0]
  const uint32_t tile_empty0 = mapa(smem_u32(tile_empty), 0);
  const uint32_t tempty0 = mapa(smem_u32(tempty), 0);

  // every role but rank 0's producer reads tile i from its own ring and
  // releases the slot on rank 0's tile_empty
  auto take_tile = [&](uint32_t i) -> int {
    const int slot = i & 3;
    mbar_wait_cluster(&tile_full[slot], (i >> 2) & 1);
    return tile_ring[slot];
  };
  auto release_tile = [&](uint32_t i) { mbar_arrive_cluster_relaxed(tile_empty0 + 8 * (i & 3)); };

  if (warp == 0 && lane == 0) {
    uint32_t g = 0;
    for (uint32_t i = 0;; ++i) {
      int t;
      if (rank == 0) {
        const int slot = i & 3;
        mbar_wait_cluster(&tile_empty[slot], ((i >> 2) & 1) ^ 1);
        t = sched ? static_cast<int>(atomicAdd(sched, 1u)) : pair + static_cast<int>(i) * npairs;
        tile_ring[slot] = t;
        st_dsmem_s32(mapa(smem_u32(&tile_ring[slot]), 1), t);
        mbar_arrive(&tile_full[slot]);
        mbar_arrive_cluster(mapa(smem_u32(&tile_full[slot]), 1));
      } else {
        t = take_tile(i);
        release_tile(i);
      }
      if (t >= tiles) break;
      int mt, nt;
      tile_coords(t, num_m, num_n, rgroup, mt, nt);
      const int m0 = mt * 2 * kBM + static_cast<int>(rank) * kBM;
      const int n0 = nt * BN + static_cast<int>(rank) * Cfg::kHalfN;
      if constexpr (!A_MN && !B_MN) {
        if (ep.conv.Q > 0) {   // implicit-GEMM convolution: this CTA's 128 A rows from the im2col map
          const ConvTile ct = conv_tile(ep.conv, m0);
          TapCursor tap(ep.conv, 0);
          for (int kb = 0; kb < nk; ++kb, ++g, tap.next(ep.conv)) {
            const int s = g % S;
            mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
            tma_load_im2col_4d_pair(sA + s * Cfg::kABytes, &tmA, full0 + 8 * s, tap.cb * 64, ct.wb, ct.hb, ct.nb,
                                    static_cast<uint16_t>(tap.s), static_cast<uint16_t>(tap.r));
            tma_load_2d_pair(sB + s * Cfg::kBBytes, &tmB, full0 + 8 * s, kb * kBK, n0);
          }
          continue;
        }
      }
      if constexpr (!A_MN && !B_MN) {
        if (ep.l2hint == 1) {   // keep the A panel resident, stream B through L2
          const uint64_t pa = l2_policy_evict_last(), pb = l2_policy_evict_first();
          for (int kb = 0; kb < nk; ++kb, ++g) {
            const int s = g % S;
            mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
            tma_load_2d_pair_hint(sA + s * Cfg::kABytes, &tmA, full0 + 8 * s, kb * kBK, m0, pa);
            tma_load_2d_pair_hint(sB + s * Cfg::kBBytes, &tmB, full0 + 8 * s, kb * kBK, n0, pb);
          }
          continue;
        }
      }
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
        load_kblock_pair<BN, A_MN, B_MN>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                         full0 + 8 * s, m0, n0, kb * kBK);
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    uint32_t g = 0;
    for (uint32_t i = 0;; ++i) {
      const int t = take_tile(i);
      release_tile(i);
      if (t >= tiles) break;
      const uint32_t as = i & 1;
      mbar_wait_cluster(&tempty[as], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * BN;
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&full[s], (g / S) & 1);
        tc_fence_after();
        mma_kblock_pair<BN, A_MN, B_MN>(d, smem_u32(sA + s * Cfg::kABytes),
                                        smem_u32(sB + s * Cfg::kBBytes), kb == 0);
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(&tfull[as]);
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    uint32_t stores = 0;
    uint8_t* const rring = !kResRing ? stg + e * 8192 + 2048
                                     : (e < 2 ? sA + S * Cfg::kABytes + e * kRD * 4096
                                              : sB + S * Cfg::kBBytes + (e - 2) * kRD * 4096);
    ResStream rs{&tmR, rring, kResRing ? 4096u : 4096u, rbar + (kResRing ? kRD : 2) * e,
                 kResRing ? static_cast<uint32_t>(kRD) : 2u, kW128 ? 4096u : 2048u, 0u, 0u};
    int staged_n0 = -1;
    for (uint32_t i = 0;; ++i) {
      const int t = take_tile(i);
      __syncwarp();
      if (lane == 0) release_tile(i);
      if (t >= tiles) break;
      int mt, nt;
      tile_coords(t, num_m, num_n, rgroup, mt, nt);
      const int m0 = mt * 2 * kBM + static_cast<int>(rank) * kBM;
      const int n0 = nt * BN;
      float* sb = sbias;
      if (tma_res) rs.prime(lane, n0, N, BN, kW128 ? 64 : 32, m0 + 32 * e);   // behind this tile's MMAs
      // the bias slice only changes with n0 (one n-tile: staged once per CTA);
      // the first barrier keeps a re-stage behind every warp's previous tile
      if (epi_has_bias<EPI>() && n0 != staged_n0) {
        if (staged_n0 >= 0) epi_bar_sync();
        stage_bias<BN, EPI>(ep, sb, n0, N, static_cast<int>(threadIdx.x) - 128);
        epi_bar_sync();
        staged_n0 = n0;
      }
      const uint32_t as = i & 1;
      mbar_wait(&tfull[as], (i >> 1) & 1);
      tc_fence_after();
      if constexpr (kW128)
        epilogue_tile_tma128<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e,
                                      lane, M, n0, N, epi_has_bias<EPI>() ? sb : nullptr, &tmY, stg + e * 8192, stores,
                                      tma_res ? &rs : nullptr);
      else if constexpr (epi_tma_store<EPI>())
        epilogue_tile_tma<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e,
                                   lane, M, n0, N, epi_has_bias<EPI>() ? sb : nullptr, &tmY, stg + e * 8192, stores,
                                   tma_res ? &rs : nullptr);
      else
        epilogue_tile<BN, EPI>(ep, tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, m0 + 32 * e + lane,
                               M, n0, N, epi_has_bias<EPI>() ? sb : nullptr);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(tempty0 + 8 * as);
    }
    if constexpr (epi_tma_store<EPI>()) {
      if (lane == 0) bulk_wait0();
      __syncwarp();
    }
  }
  tc_fence_before();
  cluster_sync();      // the peer's TMEM / smem stay live until rank 0's MMAs are done
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
  if (sched && threadIdx.x == 0 && rank == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1u) == gridDim.x / 2 - 1) {   // last pair out: reset for the next launch
      atomicExch(sched, 0u);
      atomicExch(sched + 1, 0u);
    }
  }
}

// ------------------------------------------------------------------ grouped CTA-pair GEMM
// The grouped dW launch (below) on 256 x 256 pair tiles: the pair kernel's
// roles and barriers with a static pair schedule (tile t -> (problem, m0, n0)
// through ga.tile_start, counted in pair tiles). Both operands MN-major.
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_grouped_pair_kernel(const __grid_constant__ GroupMaps maps, GroupArgs ga) {
  using Cfg = PairCfg<BN>;
  constexpr int S = Cfg::kStages;
  constexpr uint32_t kTmemCols = tmem_cols_for(2 * BN);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * Cfg::kBBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < ga.count; ++p) { prefetch_tmap(&maps.a[p]); prefetch_tmap(&maps.b[p]); }
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 8); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();

  const int tiles = ga.tile_start[ga.count];
  const int pair = static_cast<int>(blockIdx.x) / 2;
  const int npairs = static_cast<int>(gridDim.x) / 2;
  auto locate = [&](int t, int& p, int& m0, int& n0) {
    p = 0;
    while (p + 1 < ga.count && t >= ga.tile_start[p + 1]) ++p;
    const int local = t - ga.tile_start[p];
    const int num_m = (ga.M[p] + 2 * kBM - 1) / (2 * kBM);
    m0 = (local % num_m) * 2 * kBM + static_cast<int>(rank) * kBM;
    n0 = (local / num_m) * BN;
  };
  const uint32_t full0 = mapa(smem_u32(full), 0);
  const uint32_t tempty0 = mapa(smem_u32(tempty), 0);

  if (warp == 0 && lane == 0) {
    uint32_t g = 0;
    for (int t = pair; t < tiles; t += npairs) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const int nk = (ga.K[p] + kBK - 1) / kBK;
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
        load_kblock_pair<BN, A_MN, B_MN>(&maps.a[p], &maps.b[p], sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                         full0 + 8 * s, m0, n0 + static_cast<int>(rank) * Cfg::kHalfN, kb * kBK);
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    uint32_t g = 0, i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const int nk = (ga.K[p] + kBK - 1) / kBK;
      const uint32_t as = i & 1;
      mbar_wait_cluster(&tempty[as], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * BN;
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&full[s], (g / S) & 1);
        tc_fence_after();
        mma_kblock_pair<BN, A_MN, B_MN>(d, smem_u32(sA + s * Cfg::kABytes), smem_u32(sB + s * Cfg::kBBytes),
                                        kb == 0);
        umma_commit_pair(&empty[s]);
      }
      umma_commit_pair(&tfull[as]);
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    uint32_t i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const uint32_t as = i & 1;
      mbar_wait(&tfull[as], (i >> 1) & 1);
      tc_fence_after();
      epilogue_tile<BN, EPI>(ga.ep[p], tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN,
                             m0 + 32 * e + lane, ga.M[p], n0, ga.N[p], nullptr);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_relaxed(tempty0 + 8 * as);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
}

// ------------------------------------------------------------------ grouped GEMM
// Several independent problems in ONE persistent launch (the student's dW_l
// for every layer: each alone has 32-192 output tiles, too few for 148 SMs;
// together they fill ~2 waves). Tile t maps to (problem, m-block, n-block)
// through the prefix sums in GroupArgs; the pipelines are the same as above.
template <int BN, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_grouped_kernel(const __grid_constant__ GroupMaps maps, GroupArgs ga) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  constexpr uint32_t kTmemCols = tmem_cols_for(2 * BN);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* stg = sB + S * Cfg::kBBytes;                              // [4 warps][2][4 KB] TMA-store staging
  float* sbias = reinterpret_cast<float*>(stg + Cfg::kStoreBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int p = 0; p < ga.count; ++p) { prefetch_tmap(&maps.a[p]); prefetch_tmap(&maps.b[p]); }
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // PDL: everything above overlapped the previous kernel's tail
  const int tiles = ga.tile_start[ga.count];

  // tile -> (problem, m0, n0)
  auto locate = [&](int t, int& p, int& m0, int& n0) {
    p = 0;
    while (p + 1 < ga.count && t >= ga.tile_start[p + 1]) ++p;
    const int local = t - ga.tile_start[p];
    const int num_m = (ga.M[p] + kBM - 1) / kBM;
    m0 = (local % num_m) * kBM;
    n0 = (local / num_m) * BN;
  };

  if (warp == 0 && lane == 0) {
    uint64_t pa, pb;
    gemm_policies<EPI>(pa, pb);
    uint32_t g = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const int nk = (ga.K[p] + kBK - 1) / kBK;
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&empty[s], ((g / S) & 1) ^ 1);
        load_kblock<BN, A_MN, B_MN>(&maps.a[p], &maps.b[p], sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                    &full[s], m0, n0, kb * kBK, pa, pb);
      }
    }
  } else if (warp == 1 && lane == 0) {
    uint32_t g = 0, i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const int nk = (ga.K[p] + kBK - 1) / kBK;
      const uint32_t as = i & 1;
      mbar_wait(&tempty[as], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + as * BN;
      for (int kb = 0; kb < nk; ++kb, ++g) {
        const int s = g % S;
        mbar_wait(&full[s], (g / S) & 1);
        tc_fence_after();
        mma_kblock<BN, A_MN, B_MN>(d, smem_u32(sA + s * Cfg::kABytes), smem_u32(sB + s * Cfg::kBBytes), kb == 0);
        umma_commit(&empty[s]);
      }
      umma_commit(&tfull[as]);
    }
  } else if (warp >= 4) {
    const int e = warp - 4;
    uint32_t i = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      int p, m0, n0;
      locate(t, p, m0, n0);
      const uint32_t as = i & 1;
      mbar_wait(&tfull[as], (i >> 1) & 1);
      tc_fence_after();
      const int row = m0 + 32 * e + lane;
      const int M = ga.M[p], N = ga.N[p];
      epilogue_tile<BN, EPI>(ga.ep[p], tmem_base + (static_cast<uint32_t>(32 * e) << 16) + as * BN, row, M, n0,
                             N, nullptr);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[as]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ teacher head
// Logits z = H W^T + b for a 128-row block, scaled s = z / T, and per row: the
// running max / rescaled sum of exp(s) (online softmax) plus a register top-k
// list kept SORTED by (value desc, class index asc) — the tie rule of
// edl/nnkit.py:333. The class dimension is split across a cluster of CS CTAs
// (BN classes each); rank 0 merges the CS partial states through distributed
// shared memory and writes only (prob, class) pairs: logits never reach HBM.
//
// Selection is built from data-independent sorting networks (no divergence,
// all-static register indexing, high ILP): the first 32-column chunk is
// bitonic-sorted and its best KMAX kept; later chunks only insert the rare
// columns that beat the current k-th entry; partial lists (the two warp halves,
// then the cluster ranks) are combined with a bitonic merge-split + clean.
// Everything below is written branch-free (non-short-circuit predicates +
// selects): lanes of a warp hold different rows, so a data-dependent branch
// per compare-exchange diverges and serialises both paths (the first version
// compiled to 262 reconvergence blocks and ran the epilogue ~3x slower).
struct Key {
  __device__ __forceinline__ static bool better(float a, int ia, float b, int ib) {
    return (a > b) | ((a == b) & (ia < ib));
  }
};

__device__ __forceinline__ float sel(bool p, float a, float b) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}"
      : "=f"(r) : "f"(a), "f"(b), "r"(static_cast<int>(p)));
  return r;
}
__device__ __forceinline__ int sel(bool p, int a, int b) {
  int r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
      : "=r"(r) : "r"(a), "r"(b), "r"(static_cast<int>(p)));
  return r;
}

// compare-exchange so that slot a holds the better entry
__device__ __forceinline__ void cex(float& va, int& ia, float& vb, int& ib) {
  const bool s = Key::better(vb, ib, va, ia);
  const float x = va, y = vb;
  const int p = ia, q = ib;
  va = sel(s, y, x);
  vb = sel(s, x, y);
  ia = sel(s, q, p);
  ib = sel(s, p, q);
}

// bitonic sort of N entries, descending by Key
template <int N>
__device__ __forceinline__ void bitonic_sort(float (&v)[N], int (&ix)[N]) {
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size / 2; stride > 0; stride >>= 1) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        const int p = j ^ stride;
        if (p > j) {
          if ((j & size) == 0) cex(v[j], ix[j], v[p], ix[p]);
          else cex(v[p], ix[p], v[j], ix[j]);
        }
      }
    }
  }
}

// sort a bitonic sequence of N entries descending (the "clean" half of a merge)
template <int N>
__device__ __forceinline__ void bitonic_clean(float (&v)[N], int (&ix)[N]) {
#pragma unroll
  for (int stride = N / 2; stride > 0; stride >>= 1) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int p = j ^ stride;
      if (p > j) cex(v[j], ix[j], v[p], ix[p]);
    }
  }
}

template <int KMAX>
struct TopK {
  float v[KMAX];  // sorted: v[0] best
  int i[KMAX];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int j = 0; j < KMAX; ++j) { v[j] = -INFINITY; i[j] = 0x7fffffff; }
  }
  // keep the best KMAX of (this) U (o), both sorted
  __device__ __forceinline__ void merge(const float (&ov)[KMAX], const int (&oi)[KMAX]) {
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      const float bv = ov[KMAX - 1 - j];
      const int bi = oi[KMAX - 1 - j];
      const bool s = Key::better(bv, bi, v[j], i[j]);
      v[j] = sel(s, bv, v[j]);
      i[j] = sel(s, bi, i[j]);
    }
    bitonic_clean<KMAX>(v, i);
  }
  // insert a candidate that beats the current last entry (branch-free shift);
  // its index exceeds every listed one (columns scanned in increasing order),
  // so a tie keeps the listed entry and the order test is a plain v[j] >= x
  __device__ __forceinline__ void insert_later(float x, int ix) {
    bool b[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) b[j] = v[j] >= x;
#pragma unroll
    for (int j = KMAX - 1; j > 0; --j) {
      const float nv = sel(b[j - 1], x, v[j - 1]);
      const int ni = sel(b[j - 1], ix, i[j - 1]);
      v[j] = sel(b[j], v[j], nv);
      i[j] = sel(b[j], i[j], ni);
    }
    v[0] = sel(b[0], v[0], x);
    i[0] = sel(b[0], i[0], ix);
  }
};

// The head epilogue's per-row pass over this CTA's 128 x BN logit tile in
// TMEM (teacher_head_kernel / teacher_head_pair_kernel): bias + 1/T, online
// max / sum of exp, and the top-KMAX list; the two warp halves (interleaved
// 32-column chunks) merge through `hx`. On return the half-0 threads hold the
// row's state; all 256 threads must call it.
template <int BN, int KMAX>
__device__ __forceinline__ void head_rows(uint32_t tmem_base, uint64_t* tfull, int n0, int N, const float* bias,
                                          float inv_t, float* sbias, float* stage, float* hx, float& run_m,
                                          float& run_l, TopK<KMAX>& top) {
  constexpr int kState = 2 + 2 * KMAX;
  (void)kState;
  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int q = warp & 3;       // TMEM lane quarter == row block of this warp
  const int half = warp >> 2;   // which interleaved 32-column chunks this warp takes
  const int rl = 32 * q + lane; // local row
  const int tid = threadIdx.x;
  top.init();
  run_m = -INFINITY;
  run_l = 0.f;
  // the class chunk's bias, staged by warps 2-7 while the MMAs run; warps 0/1
  // join the barrier when their producer / MMA loops are done
  if (warp >= 2) {
    for (int j = tid - 64; j < BN; j += kThreads - 64)
      sbias[j] = (n0 + j < N) ? __ldg(bias + n0 + j) : 0.f;
  }
  asm volatile("bar.sync 2, 256;" ::: "memory");
  mbar_wait(&tfull[0], 0);
  tc_fence_after();
  bool first = true;
  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
  uint32_t r[32];
  tmem_ld32_issue(taddr + 32 * half, r);
  tmem_ld_wait(r);
#pragma unroll 1
  for (int c = 32 * half; c < BN; c += 64) {
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    const bool more = c + 64 < BN;
    if (more) tmem_ld32_issue(taddr + c + 64, r);   // next chunk's load overlaps this one's work
    const int col0 = n0 + c;
    if (col0 >= N) {
      if (more) tmem_ld_wait(r);
      continue;
    }
    float cmax = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int n = col0 + j;
      const float s = (n < N) ? (v[j] + sbias[c + j]) * inv_t : -INFINITY;
      v[j] = s;
      cmax = fmaxf(cmax, s);
    }
    const float nm = fmaxf(run_m, cmax);
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += __expf(v[j] - nm);
    run_l = run_l * __expf(run_m - nm) + acc;
    run_m = nm;
    if (first) {
      // the first chunk seeds the list: bitonic-sort all 32, keep the best KMAX
      first = false;
      int ix[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) ix[j] = (col0 + j < N) ? col0 + j : 0x7fffffff;
      bitonic_sort<32>(v, ix);
#pragma unroll
      for (int j = 0; j < KMAX; ++j) { top.v[j] = v[j]; top.i[j] = ix[j]; }
      if (more) tmem_ld_wait(r);
      continue;
    }
    // later chunks: only columns beating the current k-th entry (rare), each
    // inserted by a branch-free shift; the values are staged in smem so the
    // rolled loop can address them. Every listed index is below col0 (the
    // chunks are scanned in increasing column order), so a tie never beats a
    // listed entry and the tests are plain float compares.
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) mask |= (v[j] > top.v[KMAX - 1] ? 1u : 0u) << j;
    if (mask) {
#pragma unroll
      for (int j = 0; j < 32; ++j) stage[j * kThreads + tid] = v[j];
      while (mask) {
        const int j = __ffs(mask) - 1;
        mask &= mask - 1;
        const float x = stage[j * kThreads + tid];
        if (x > top.v[KMAX - 1]) top.insert_later(x, col0 + j);
      }
    }
    __syncwarp();   // the insertions above diverge; tcgen05.wait::ld is .sync.aligned
    if (more) tmem_ld_wait(r);
  }
  tc_fence_before();
  // halves -> one state per row (half 1 hands over through shared memory)
  if (half == 1) {
    hx[0 * kBM + rl] = run_m;
    hx[1 * kBM + rl] = run_l;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      hx[(2 + j) * kBM + rl] = top.v[j];
      hx[(2 + KMAX + j) * kBM + rl] = __int_as_float(top.i[j]);
    }
  }
  __syncthreads();
  if (half == 0) {
    const float om = hx[0 * kBM + rl], ol = hx[1 * kBM + rl];
    const float nm = fmaxf(run_m, om);
    run_l = (run_l > 0.f ? run_l * __expf(run_m - nm) : 0.f) + (ol > 0.f ? ol * __expf(om - nm) : 0.f);
    run_m = nm;
    float ov[KMAX];
    int oi[KMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      ov[j] = hx[(2 + j) * kBM + rl];
      oi[j] = __float_as_int(hx[(2 + KMAX + j) * kBM + rl]);
    }
    top.merge(ov, oi);
  }
}

template <int BN, int KMAX>
__global__ void __launch_bounds__(kThreads, 1)
    teacher_head_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                        HeadArgs hp) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  constexpr uint32_t kTmemCols = tmem_cols_for(BN);
  constexpr int kState = 2 + 2 * KMAX;  // words per row: m, l, v[KMAX], i[KMAX]
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* stg = sB + S * Cfg::kBBytes;                              // [4 warps][2][4 KB] TMA-store staging
  float* sbias = reinterpret_cast<float*>(stg + Cfg::kStoreBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  // Epilogue scratch reuses the drained operand ring (word-interleaved by
  // thread / row so every access is bank-conflict free):
  float* stage = reinterpret_cast<float*>(smem);                    // [32][256] candidates
  float* hx = stage + 32 * kThreads;                                 // [kState][128] half merge
  float* st = hx + kState * kBM;                                     // [kState][128] cluster merge

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int cs = static_cast<int>(gridDim.x);            // cluster spans the class chunks
  const int rank = static_cast<int>(blockIdx.x);         // == %cluster_ctarank
  const int m0 = blockIdx.y * kBM;
  const int n0 = rank * BN;
  const int nk = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull[0], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();  // PDL: everything above overlapped the previous kernel's tail

  if (warp == 0 && lane == 0) {
    const uint64_t pa = l2_policy_evict_normal(), pb = l2_policy_evict_normal();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&empty[s], ((kb / S) & 1) ^ 1);
      load_kblock<BN, false, false>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                    &full[s], m0, n0, kb * kBK, pa, pb);
    }
  } else if (warp == 1 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      tc_fence_after();
      mma_kblock<BN, false, false>(tmem_base, smem_u32(sA + s * Cfg::kABytes),
                                   smem_u32(sB + s * Cfg::kBBytes), kb == 0);
      umma_commit(&empty[s]);
    }
    umma_commit(&tfull[0]);
  }
  __syncwarp();

  const int q = warp & 3;
  const int half = warp >> 2;
  const int rl = 32 * q + lane;
  TopK<KMAX> top;
  float run_m, run_l;
  head_rows<BN, KMAX>(tmem_base, tfull, n0, N, hp.bias, hp.inv_t, sbias, stage, hx, run_m, run_l, top);
  (void)q;
  if (half == 0) {
    st[0 * kBM + rl] = run_m;
    st[1 * kBM + rl] = run_l;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      st[(2 + j) * kBM + rl] = top.v[j];
      st[(2 + KMAX + j) * kBM + rl] = __int_as_float(top.i[j]);
    }
  }
  if (cs > 1) cluster_sync(); else __syncthreads();
  if (rank == 0 && half == 0) {
#pragma unroll 1
    for (int r = 1; r < cs; ++r) {
      // all remote words in flight at once, then a register bitonic merge
      float rv[kState];
#pragma unroll
      for (int w = 0; w < kState; ++w) rv[w] = ld_dsmem_f32(mapa(smem_u32(st + w * kBM + rl), r));
      const float nm = fmaxf(run_m, rv[0]);
      run_l = run_l * __expf(run_m - nm) + rv[1] * __expf(rv[0] - nm);
      run_m = nm;
      float ov[KMAX];
      int oi[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) { ov[j] = rv[2 + j]; oi[j] = __float_as_int(rv[2 + KMAX + j]); }
      top.merge(ov, oi);
    }
    const int row = m0 + rl;
    if (row < M) {
      const float inv_l = 1.0f / run_l;
      float* ov = hp.vals + static_cast<size_t>(row) * hp.k;
      int* oi = hp.idx + static_cast<size_t>(row) * hp.k;
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < hp.k) { ov[j] = __expf(top.v[j] - run_m) * inv_l; oi[j] = top.i[j]; }
    }
  }
  if (cs > 1) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---- teacher head on CTA pairs (cta_group::2, 256-row tiles) with the
// class-chunk merge through global memory. The cluster head above needs the
// whole class range of a row block in one cluster (4 CTAs, 128 x 256 each);
// on pairs that is 8 CTAs, and clusters of 8 CTAs of ~200 KB do not fit in a
// GPC often enough (finding 21). Here a cluster is one pair: the pair's two
// CTAs stage their 128 A rows and half of the 256 B rows per k-block, rank 0
// issues 256 x 256 x 16 MMAs over both (2/3 of the single-CTA kernel's
// operand bytes per FLOP — the head's mainloop is operand-delivery bound),
// and each CTA's epilogue (head_rows) reduces its 128 rows x 256 classes to
// a per-row state (max, sum, top-KMAX) in global scratch. The last of the
// ceil(K / 256) class chunks of a 128-row block (atomic ticket) merges the
// states in chunk order — deterministic — and writes the (prob, class)
// pairs.
//
// CL == 4: a cluster is two pairs on the same class chunk and adjacent row
// blocks. Pair 0's CTAs multicast the chunk's B halves into both pairs
// (tma_load_2d_pair_mc), so L2 delivers each B tile once per cluster (3/4 of
// the pair kernel's operand bytes); each stage's empty barrier then waits for
// both pairs' MMA commits (count 2, commits multicast to all four CTAs).
template <int KMAX, int CL>
__global__ void __launch_bounds__(kThreads, 1)
    teacher_head_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             int M, int N, int K, HeadArgs hp, float* part, unsigned* tickets) {
  constexpr int BN = 256;
  using Cfg = PairCfg<BN>;
  constexpr int S = 6;
  constexpr uint32_t kTmemCols = tmem_cols_for(BN);
  constexpr int kState = 2 + 2 * KMAX;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  float* sbias = reinterpret_cast<float*>(sB + S * Cfg::kBBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(sbias + BN);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  int* merger = reinterpret_cast<int*>(tmem_slot + 2);
  // epilogue scratch in the drained operand ring
  float* stage = reinterpret_cast<float*>(smem);                     // [32][256]
  float* hx = stage + 32 * kThreads;                                  // [kState][128]

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  static_assert(CL == 2 || CL == 4, "head pair cluster");
  const uint32_t crank = cluster_ctarank();
  const uint32_t rank = crank & 1;                    // rank within the pair
  const int pr = static_cast<int>(crank >> 1);        // pair within the cluster
  const int num_n = (N + BN - 1) / BN;
  const int cl = static_cast<int>(blockIdx.x) / CL;
  // class chunks of a row block adjacent: A reuse in L2
  const int mt = (cl / num_n) * (CL / 2) + pr, nt = cl % num_n;
  const int m0 = mt * 2 * kBM + static_cast<int>(rank) * kBM;
  const int nk = (K + kBK - 1) / kBK;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL / 2); }
    mbar_init(&tfull[0], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();
  const uint32_t full0 = mapa(smem_u32(full), crank & ~1u);   // this pair's leader

  if (warp == 0 && lane == 0) {
    const int nb0 = nt * BN + static_cast<int>(rank) * Cfg::kHalfN;
    const uint16_t bmask = static_cast<uint16_t>((1u << rank) | (1u << (rank + 2)));
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&empty[s], ((kb / S) & 1) ^ 1);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
      if constexpr (CL == 2) {
        load_kblock_pair<BN, false, false>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                           full0 + 8 * s, m0, nb0, kb * kBK);
      } else {
        tma_load_2d_pair(sA + s * Cfg::kABytes, &tmA, full0 + 8 * s, kb * kBK, m0);
        if (pr == 0) tma_load_2d_pair_mc(sB + s * Cfg::kBBytes, &tmB, full0 + 8 * s, kb * kBK, nb0, bmask);
      }
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    const uint16_t all = CL == 2 ? 3 : 15, own = static_cast<uint16_t>(3u << (crank & 2));
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      tc_fence_after();
      mma_kblock_pair<BN, false, false>(tmem_base, smem_u32(sA + s * Cfg::kABytes),
                                        smem_u32(sB + s * Cfg::kBBytes), kb == 0);
      umma_commit_pair_mask(&empty[s], all);
    }
    umma_commit_pair_mask(&tfull[0], own);
  }
  __syncwarp();

  const int half = warp >> 2;
  const int rl = 32 * (warp & 3) + lane;
  const int row = m0 + rl;
  TopK<KMAX> top;
  float run_m, run_l;
  head_rows<BN, KMAX>(tmem_base, tfull, nt * BN, N, hp.bias, hp.inv_t, sbias, stage, hx, run_m, run_l, top);
  if (half == 0 && row < M) {
    float* pp = part + static_cast<size_t>(nt) * kState * M + row;
    pp[0] = run_m;
    pp[static_cast<size_t>(M)] = run_l;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      pp[static_cast<size_t>(2 + j) * M] = top.v[j];
      pp[static_cast<size_t>(2 + KMAX + j) * M] = __int_as_float(top.i[j]);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* t = tickets + m0 / kBM;
    const bool last = atomicAdd(t, 1u) == static_cast<unsigned>(num_n - 1);
    if (last) atomicExch(t, 0u);        // every chunk has arrived: reset for the next launch
    *merger = last ? 1 : 0;
  }
  __syncthreads();
  if (*merger && half == 0 && row < M) {
    __threadfence();
    // chunk c + 1's state is loaded while chunk c merges (one L2 round trip
    // per chunk otherwise sits on the critical path)
    float nx[kState];
#pragma unroll
    for (int w = 0; w < kState; ++w) nx[w] = __ldcg(part + static_cast<size_t>(w) * M + row);
#pragma unroll 1
    for (int c = 0; c < num_n; ++c) {
      float rv[kState];
#pragma unroll
      for (int w = 0; w < kState; ++w) rv[w] = nx[w];
      if (c + 1 < num_n) {
        const float* pn = part + static_cast<size_t>(c + 1) * kState * M + row;
#pragma unroll
        for (int w = 0; w < kState; ++w) nx[w] = __ldcg(pn + static_cast<size_t>(w) * M);
      }
      float ov[KMAX];
      int oi[KMAX];
#pragma unroll
      for (int j = 0; j < KMAX; ++j) { ov[j] = rv[2 + j]; oi[j] = __float_as_int(rv[2 + KMAX + j]); }
      if (c == 0) {
        run_m = rv[0];
        run_l = rv[1];
#pragma unroll
        for (int j = 0; j < KMAX; ++j) { top.v[j] = ov[j]; top.i[j] = oi[j]; }
      } else {
        const float nm = fmaxf(run_m, rv[0]);
        run_l = run_l * __expf(run_m - nm) + rv[1] * __expf(rv[0] - nm);
        run_m = nm;
        top.merge(ov, oi);
      }
    }
    const float inv_l = 1.0f / run_l;
    float* ov = hp.vals + static_cast<size_t>(row) * hp.k;
    int* oi = hp.idx + static_cast<size_t>(row) * hp.k;
#pragma unroll
    for (int j = 0; j < KMAX; ++j)
      if (j < hp.k) { ov[j] = __expf(top.v[j] - run_m) * inv_l; oi[j] = top.i[j]; }
  }
  tc_fence_before();
  cluster_sync();      // the peer's TMEM / smem stay live until rank 0's MMAs are done
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair<kTmemCols>(tmem_base);
}

// ---- student KD head: the logit GEMM with the distillation loss and its
// gradient in the epilogue (edl/nnkit.py:283-299), so the fp32 logits never
// reach HBM. A cluster of ceil(K / BN) CTAs splits the classes of a 128-row
// block; each CTA keeps its 128 x BN logit tile in TMEM for two passes:
//   pass 1: per row, running max m and the sums l1 = sum exp(z - m),
//           lT = sum exp((z - m) / T), plus z at the label and the q-weighted
//           sum of z at the soft classes (gathered through a per-thread
//           shared-memory spill only for the ~1 in 2 chunks that hold one);
//   merge:  halves through shared memory, then every CTA reads all the
//           cluster's row states over DSMEM in rank order (identical results
//           in every CTA); rank 0 writes the row loss
//           alpha (lse1 - z_y) + beta T^2 (lseT - sum_j q_j z_j / T);
//   pass 2: dz = alpha/B (softmax(z) - onehot(y)) + beta T/B (softmax(z/T) - q)
//           from the same TMEM tile, sparse terms applied through the spill,
//           bf16 through the TMA-store staging tiles (columns >= K are 0).
// With T == 2 one MUFU per element and pass: exp(d) = exp(d / 2)^2.
// The batch mean stays a separate fixed-order launch (loss_mean_kernel).
template <int BN, int KMAX, bool T2>
__global__ void __launch_bounds__(kThreads, 1)
    kd_head_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmY, int M, int N, int Nw, int K, KdArgs kp) {
  using Cfg = GemmCfg<BN>;
  constexpr int S = Cfg::kStages;
  // T2: columns BN..2BN-1 keep pass 1's exponentials for pass 2
  constexpr uint32_t kTmemCols = tmem_cols_for(T2 ? 2 * BN : BN);
  constexpr int kChunks = BN / 64;            // chunks per thread and pass
  constexpr float kL2E = 1.4426950408889634f;
  constexpr int kSt = 5;                      // row state: m, l1, lT, z_y, sum q z
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kABytes;
  uint8_t* stg = sB + S * Cfg::kBBytes;                              // [8 warps][2][2 KB] bf16 store tiles
  float* sbias = reinterpret_cast<float*>(stg + Cfg::kStoreBytes);   // [BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(stg + Cfg::kStoreBytes + Cfg::kEpiBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);
  // epilogue scratch in the drained operand ring (word-interleaved by thread)
  float* spill = reinterpret_cast<float*>(smem);                    // [32][256]
  float* hx = spill + 32 * kThreads;                                 // [kSt][128] half handover
  float* st = hx + kSt * kBM;                                        // [kSt][128] this CTA's row states

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int cs = static_cast<int>(gridDim.x);
  const int rank = static_cast<int>(blockIdx.x);
  const int m0 = blockIdx.y * kBM;
  const int n0 = rank * BN;
  const int nk = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmY);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&tfull[0], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_wait();

  if (warp == 0 && lane == 0) {
    const uint64_t pa = l2_policy_evict_normal(), pb = l2_policy_evict_normal();
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&empty[s], ((kb / S) & 1) ^ 1);
      load_kblock<BN, false, false>(&tmA, &tmB, sA + s * Cfg::kABytes, sB + s * Cfg::kBBytes,
                                    &full[s], m0, n0, kb * kBK, pa, pb);
    }
  } else if (warp == 1 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % S;
      mbar_wait(&full[s], (kb / S) & 1);
      tc_fence_after();
      mma_kblock<BN, false, false>(tmem_base, smem_u32(sA + s * Cfg::kABytes),
                                   smem_u32(sB + s * Cfg::kBBytes), kb == 0);
      umma_commit(&empty[s]);
    }
    umma_commit(&tfull[0]);
  }
  __syncwarp();

  const int q = warp & 3;
  const int half = warp >> 2;
  const int rl = 32 * q + lane;
  const int row = m0 + rl;
  const int tid = threadIdx.x;
  const bool row_ok = row < M;
  const bool soft = kp.beta > 0.f && kp.k > 0;
  // this row's sparse entries (label, renormalised top-k), loaded while the MMAs run
  int y = -1;
  int qc[KMAX];
  float qn[KMAX];
  bool bad = false;
  if (row_ok) {
    const int64_t yy = __ldg(kp.labels + row);
    bad = yy < 0 || yy >= N;
    y = bad ? -1 : static_cast<int>(yy);
  }
  float qsum = 0.f;
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    qc[j] = -1;
    qn[j] = 0.f;
    if (soft && row_ok && j < kp.k) {
      qn[j] = __ldg(kp.qv + static_cast<size_t>(row) * kp.k + j);
      const int c = __ldg(kp.qi + static_cast<size_t>(row) * kp.k + j);
      qsum += qn[j];
      if (c >= 0 && c < N) qc[j] = c;
      else bad = true;
    }
  }
  if (soft) {
    const float inv_q = qsum > 0.f ? 1.0f / qsum : 0.f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) qn[j] *= inv_q;
  }
  if (bad && rank == 0 && half == 0 && kp.status) atomicCAS(kp.status, 0, -1);
  // Everything below works in base-2 units of the tempered logit:
  // t = z log2(e) / T = fma(acc, kT, bias kT). Columns >= N get bias -inf,
  // so their t and every exponential of them vanish without a predicate.
  const float kT = kL2E * kp.inv_t;
  const float Tt = kp.T;
  if (warp >= 2) {
    for (int j = tid - 64; j < BN; j += kThreads - 64)
      sbias[j] = (n0 + j < N) ? __ldg(kp.bias + n0 + j) * kT : -INFINITY;
  }
  asm volatile("bar.sync 2, 256;" ::: "memory");
  mbar_wait(&tfull[0], 0);
  tc_fence_after();

  const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16);
  auto hit_of = [&](int col0) {
    bool h = static_cast<unsigned>(y - col0) < 32u;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) h |= static_cast<unsigned>(qc[j] - col0) < 32u;
    return h;
  };
  // t for the 32 columns of a chunk (bias pre-scaled, float4 smem broadcast)
  auto tvals = [&](const uint32_t (&rr)[32], int c, float (&t)[32]) {
    const float4* b4 = reinterpret_cast<const float4*>(sbias + c);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 b = b4[i];
      t[4 * i + 0] = fmaf(__uint_as_float(rr[4 * i + 0]), kT, b.x);
      t[4 * i + 1] = fmaf(__uint_as_float(rr[4 * i + 1]), kT, b.y);
      t[4 * i + 2] = fmaf(__uint_as_float(rr[4 * i + 2]), kT, b.z);
      t[4 * i + 3] = fmaf(__uint_as_float(rr[4 * i + 3]), kT, b.w);
    }
  };
  // scale factors of a running state when its max moves from m to nm
  // (both 0 when the state is empty)
  auto rescale = [&](float m, float nm, float& sT, float& s1) {
    const bool live = m != -INFINITY;
    const float e = live ? exp2f_approx(m - nm) : 0.f;
    sT = e;
    if constexpr (T2) s1 = e * e;
    else s1 = live ? exp2f_approx((m - nm) * Tt) : 0.f;
  };

  // ---- pass 1: row statistics (tm = max t, lT = sum 2^(t - tm),
  //      l1 = sum 2^((t - tm) T), ty = t at the label, tq = sum q t)
  float tm = -INFINITY, l1 = 0.f, lT = 0.f, ty = 0.f, tq = 0.f;
  float cmv[kChunks];            // T2: each chunk's max (pass 2 rescales its stored exponentials)
  uint32_t r[32];
  tmem_ld32_issue(taddr + 32 * half, r);
  tmem_ld_wait(r);
#pragma unroll
  for (int i = 0; i < kChunks; ++i) {
    const int c = 32 * half + 64 * i;
    float t[32];
    tvals(r, c, t);
    const bool more = i + 1 < kChunks;
    if (more) tmem_ld32_issue(taddr + c + 64, r);
    const int col0 = n0 + c;
    cmv[i] = -INFINITY;
    if (col0 < N && !(kp.debug & 5)) {
      // tree max and 4-way partial sums: no 32-long dependency chains
      float mx[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) mx[j] = fmaxf(t[j], t[j + 16]);
#pragma unroll
      for (int w = 8; w > 0; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) mx[j] = fmaxf(mx[j], mx[j + w]);
      const float cm = mx[0];
      float aT[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
      if constexpr (T2) {
        // exponentials relative to the chunk's own max, kept in TMEM
        float e[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          e[j] = exp2f_approx(t[j] - cm);
          aT[j & 3] += e[j];
          a1[j & 3] = fmaf(e[j], e[j], a1[j & 3]);
        }
        tmem_st32(taddr + BN + c, e);
        cmv[i] = cm;
        const float nm = fmaxf(tm, cm);
        float sa, sa1;
        rescale(tm, nm, sa, sa1);
        const float sb = exp2f_approx(cm - nm);
        lT = lT * sa + ((aT[0] + aT[1]) + (aT[2] + aT[3])) * sb;
        l1 = l1 * sa1 + ((a1[0] + a1[1]) + (a1[2] + a1[3])) * (sb * sb);
        tm = nm;
      } else {
        if (cm > tm) {
          float sT, s1;
          rescale(tm, cm, sT, s1);
          lT *= sT;
          l1 *= s1;
          tm = cm;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = exp2f_approx(t[j] - tm);
          aT[j & 3] += e;
          a1[j & 3] += exp2f_approx((t[j] - tm) * Tt);
        }
        lT += (aT[0] + aT[1]) + (aT[2] + aT[3]);
        l1 += (a1[0] + a1[1]) + (a1[2] + a1[3]);
      }
      if (hit_of(col0)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) spill[j * kThreads + tid] = t[j];
        if (static_cast<unsigned>(y - col0) < 32u) ty += spill[(y - col0) * kThreads + tid];
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (static_cast<unsigned>(qc[j] - col0) < 32u) tq += qn[j] * spill[(qc[j] - col0) * kThreads + tid];
      }
    }
    __syncwarp();
    if (more) tmem_ld_wait(r);
  }
  if constexpr (T2) tmem_st_wait();
  // ---- merge: halves, then the cluster (every CTA, rank order)
  auto combine = [&](float om, float ol1, float olT) {
    const float nm = fmaxf(tm, om);
    float sa, sa1, sb, sb1;
    rescale(tm, nm, sa, sa1);
    rescale(om, nm, sb, sb1);
    l1 = l1 * sa1 + ol1 * sb1;
    lT = lT * sa + olT * sb;
    tm = nm;
  };
  if (half == 1) {
    hx[0 * kBM + rl] = tm;
    hx[1 * kBM + rl] = l1;
    hx[2 * kBM + rl] = lT;
    hx[3 * kBM + rl] = ty;
    hx[4 * kBM + rl] = tq;
  }
  __syncthreads();
  if (half == 0) {
    combine(hx[0 * kBM + rl], hx[1 * kBM + rl], hx[2 * kBM + rl]);
    st[0 * kBM + rl] = tm;
    st[1 * kBM + rl] = l1;
    st[2 * kBM + rl] = lT;
    st[3 * kBM + rl] = ty + hx[3 * kBM + rl];
    st[4 * kBM + rl] = tq + hx[4 * kBM + rl];
  }
  if (cs > 1) cluster_sync(); else __syncthreads();
  {
    float rv[kSt];
#pragma unroll
    for (int w = 0; w < kSt; ++w) rv[w] = ld_dsmem_f32(mapa(smem_u32(st + w * kBM + rl), 0));
    tm = rv[0]; l1 = rv[1]; lT = rv[2]; ty = rv[3]; tq = rv[4];
#pragma unroll 1
    for (int rr = 1; rr < cs; ++rr) {
#pragma unroll
      for (int w = 0; w < kSt; ++w) rv[w] = ld_dsmem_f32(mapa(smem_u32(st + w * kBM + rl), rr));
      combine(rv[0], rv[1], rv[2]);
      ty += rv[3];
      tq += rv[4];
    }
  }
  const float ch = kp.alpha / static_cast<float>(M);
  const float csoft = soft ? kp.beta * kp.T / static_cast<float>(M) : 0.f;
  if (rank == 0 && half == 0 && row_ok) {
    // ln 2 [alpha (T (tm - t_y) + log2 l1) + beta T^2 (tm - sum q t + log2 lT)]
    constexpr float kLn2 = 0.6931471805599453f;
    float loss = 0.f;
    if (kp.alpha > 0.f && y >= 0) loss += kp.alpha * (Tt * (tm - ty) + __log2f(l1));
    if (soft) loss += kp.beta * Tt * Tt * (tm - tq + __log2f(lT));
    kp.row_loss[row] = loss * kLn2;
  }
  // ---- pass 2: dz = c1 2^((t - tm) T) + cT 2^(t - tm), sparse terms, bf16 TMA store
  const float c1 = kp.alpha > 0.f ? ch / l1 : 0.f;
  const float cT = csoft / lT;
  uint32_t stores = 0;
  uint8_t* wstg = stg + warp * 4096;
  const uint32_t src = T2 ? BN : 0;   // T2: the stored exponentials; else the accumulator
  tmem_ld32_issue(taddr + src + 32 * half, r);
  tmem_ld_wait(r);
#pragma unroll
  for (int i = 0; i < kChunks; ++i) {
    const int c = 32 * half + 64 * i;
    float v[32];
    if constexpr (T2) {
      // e' = e 2^(cm - tm) = 2^(t - tm); dz = e' (cT + c1 e')
      const float sg = cmv[i] == -INFINITY ? 0.f : exp2f_approx(cmv[i] - tm);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float e = __uint_as_float(r[j]) * sg;
        v[j] = e * fmaf(c1, e, cT);
      }
    } else {
      tvals(r, c, v);
    }
    const bool more = i + 1 < kChunks;
    if (more) tmem_ld32_issue(taddr + src + c + 64, r);
    const int col0 = n0 + c;
    if (col0 < Nw && !(kp.debug & 6)) {
      if constexpr (!T2) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = v[j] - tm;
          v[j] = fmaf(c1, exp2f_approx(x * Tt), cT * exp2f_approx(x));
        }
      } else if (col0 >= N) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;   // no exponentials were stored for this chunk
      }
      if (hit_of(col0)) {
#pragma unroll
        for (int j = 0; j < 32; ++j) spill[j * kThreads + tid] = v[j];
        if (kp.alpha > 0.f && static_cast<unsigned>(y - col0) < 32u) spill[(y - col0) * kThreads + tid] -= ch;
#pragma unroll
        for (int j = 0; j < KMAX; ++j)
          if (static_cast<unsigned>(qc[j] - col0) < 32u) spill[(qc[j] - col0) * kThreads + tid] -= csoft * qn[j];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = spill[j * kThreads + tid];
      }
      uint8_t* buf = wstg + (stores & 1) * 2048;
      if (lane == 0) bulk_wait_read1();
      __syncwarp();
      stage_chunk<false>(buf, lane, v);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tmY, buf, col0, m0 + 32 * q);
        bulk_commit();
      }
      ++stores;
    }
    __syncwarp();
    if (more) tmem_ld_wait(r);
  }
  if (lane == 0) bulk_wait0();
  tc_fence_before();
  if (cs > 1) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ------------------------------------------------------------------ launchers
template <int BN, bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M, int N,
                                 int K, const EpiArgs& ep, int num_sms, cudaStream_t stream,
                                 const CUtensorMap* tr, bool w128 = false) {
  if (EPI == EPI_RELU_BF16 && ep.aux != nullptr && tr == nullptr) return cudaErrorInvalidValue;
  constexpr bool kCanW128 = BN % 64 == 0 && !A_MN &&
                            (EPI == EPI_RELU_BF16 || EPI == EPI_BIAS_BF16 || EPI == EPI_TANH_BF16 ||
                             EPI == EPI_DRELU_BF16 || EPI == EPI_DTANH_BF16);
  if (w128 && (!kCanW128 || tr != nullptr || ep.ksplit > 1)) return cudaErrorInvalidValue;
  auto kern = (kCanW128 && w128) ? gemm_kernel<BN, A_MN, B_MN, EPI, kCanW128> : gemm_kernel<BN, A_MN, B_MN, EPI>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), GemmCfg<BN>::kSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ((M + kBM - 1) / kBM) * ((N + BN - 1) / BN) * ep.ksplit;
  const int grid = tiles < num_sms ? tiles : num_sms;
  return launch_pdl(kern, dim3(grid), dim3(kThreads), GemmCfg<BN>::kSmem, stream, 1, ta, tb, ty, tr ? *tr : ty, M, N,
                    K, ep);
}

template <bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_gemm_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty,
                                  int M, int N, int K, const EpiArgs& ep, int num_sms, cudaStream_t stream,
                                  const CUtensorMap* tr = nullptr, bool w128 = false) {
  switch (bn) {
    case 64: return launch_gemm_t<64, A_MN, B_MN, EPI>(ta, tb, ty, M, N, K, ep, num_sms, stream, tr, w128);
    case 128: return launch_gemm_t<128, A_MN, B_MN, EPI>(ta, tb, ty, M, N, K, ep, num_sms, stream, tr, w128);
    case 256: return launch_gemm_t<256, A_MN, B_MN, EPI>(ta, tb, ty, M, N, K, ep, num_sms, stream, tr, w128);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm(GemmKind kind, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                        const CUtensorMap& ty, int M, int N, int K, const EpiArgs& ep, int num_sms,
                        cudaStream_t stream, const CUtensorMap* tr, bool w128) {
  if (w128) {   // 64 x 32 SWIZZLE_128B output maps, no residual
    if (tr != nullptr) return cudaErrorInvalidValue;
    if (kind == GemmKind::FwdRelu)
      return launch_gemm_bn<false, false, EPI_RELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::FwdIdentBf16)
      return launch_gemm_bn<false, false, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::FwdTanh)
      return launch_gemm_bn<false, false, EPI_TANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::BwdData)
      return launch_gemm_bn<false, true, EPI_DTANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::BwdDataPlain)
      return launch_gemm_bn<false, true, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::ConvDgrad)
      return launch_gemm_bn<false, false, EPI_DRELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr,
                                                          true);
    return cudaErrorInvalidValue;
  }
  switch (kind) {
    case GemmKind::FwdTanh:
      return launch_gemm_bn<false, false, EPI_TANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::FwdLinear:
      return launch_gemm_bn<false, false, EPI_BIAS_F32>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::BwdData:
      return launch_gemm_bn<false, true, EPI_DTANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::BwdWeight:
      return launch_gemm_bn<true, true, EPI_F32>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::FwdRelu:
      return launch_gemm_bn<false, false, EPI_RELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, tr);
    case GemmKind::FwdIdentBf16:
      return launch_gemm_bn<false, false, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::BwdDataPlain:
      return launch_gemm_bn<false, true, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::ConvDgrad:
      return launch_gemm_bn<false, false, EPI_DRELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
  }
  return cudaErrorInvalidValue;
}

template <int BN, bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_pair_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M, int N,
                                 int K, const EpiArgs& ep, int num_sms, cudaStream_t stream,
                                 const CUtensorMap* tr, bool w128 = false) {
  if (EPI == EPI_RELU_BF16 && ep.aux != nullptr && tr == nullptr) return cudaErrorInvalidValue;
  constexpr bool kCanW128 = BN == 256 && !A_MN &&
                            (EPI == EPI_RELU_BF16 || EPI == EPI_BIAS_BF16 || EPI == EPI_TANH_BF16 ||
                             EPI == EPI_DRELU_BF16 || EPI == EPI_DTANH_BF16);
  auto kern = (kCanW128 && w128) ? gemm_pair_kernel<BN, A_MN, B_MN, EPI, kCanW128>
                                 : gemm_pair_kernel<BN, A_MN, B_MN, EPI>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), PairCfg<BN>::kSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ((M + 2 * kBM - 1) / (2 * kBM)) * ((N + BN - 1) / BN);
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  if (pairs < 1) return cudaErrorInvalidValue;
  return launch_pdl(kern, dim3(2 * pairs), dim3(kThreads), PairCfg<BN>::kSmem, stream, 2, ta, tb, ty, tr ? *tr : ty,
                    M, N, K, ep);
}

template <bool A_MN, bool B_MN, int EPI>
static cudaError_t launch_pair_bn(int bn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M,
                                  int N, int K, const EpiArgs& ep, int num_sms, cudaStream_t stream,
                                  const CUtensorMap* tr = nullptr, bool w128 = false) {
  switch (bn) {
    case 128: return launch_pair_t<128, A_MN, B_MN, EPI>(ta, tb, ty, M, N, K, ep, num_sms, stream, tr);
    case 256: return launch_pair_t<256, A_MN, B_MN, EPI>(ta, tb, ty, M, N, K, ep, num_sms, stream, tr, w128);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_gemm_pair(GemmKind kind, int bn, const CUtensorMap& ta, const CUtensorMap& tb,
                             const CUtensorMap& ty, int M, int N, int K, const EpiArgs& ep, int num_sms,
                             cudaStream_t stream, const CUtensorMap* tr, bool w128) {
  if (w128) {   // 64 x 32 SWIZZLE_128B output / residual maps (edl_conv_fwd_nhwc, bn == 256)
    if (bn != 256) return cudaErrorInvalidValue;
    if (kind == GemmKind::FwdRelu)
      return launch_pair_bn<false, false, EPI_RELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, tr, true);
    if (kind == GemmKind::FwdIdentBf16)
      return launch_pair_bn<false, false, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::FwdTanh)
      return launch_pair_bn<false, false, EPI_TANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::BwdData)
      return launch_pair_bn<false, true, EPI_DTANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::BwdDataPlain)
      return launch_pair_bn<false, true, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr, true);
    if (kind == GemmKind::ConvDgrad)
      return launch_pair_bn<false, false, EPI_DRELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, nullptr,
                                                          true);
    return cudaErrorInvalidValue;
  }
  switch (kind) {
    case GemmKind::FwdTanh:
      return launch_pair_bn<false, false, EPI_TANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::FwdLinear:
      return launch_pair_bn<false, false, EPI_BIAS_F32>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::BwdData:
      return launch_pair_bn<false, true, EPI_DTANH_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::FwdRelu:
      return launch_pair_bn<false, false, EPI_RELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream, tr);
    case GemmKind::FwdIdentBf16:
      return launch_pair_bn<false, false, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::BwdDataPlain:
      return launch_pair_bn<false, true, EPI_BIAS_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    case GemmKind::ConvDgrad:
      return launch_pair_bn<false, false, EPI_DRELU_BF16>(bn, ta, tb, ty, M, N, K, ep, num_sms, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

template <int EPI>
static cudaError_t launch_grouped_t(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                    cudaStream_t stream) {
  constexpr int BN = 256;
  auto kern = gemm_grouped_kernel<BN, true, true, EPI>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), GemmCfg<BN>::kSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ga.tile_start[ga.count];
  const int grid = tiles < num_sms ? tiles : num_sms;
  return launch_pdl(kern, dim3(grid), dim3(kThreads), GemmCfg<BN>::kSmem, stream, 1, maps, ga);
}

cudaError_t launch_gemm_grouped_bwd_weight(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                           cudaStream_t stream, bool fused_sgd) {
  return fused_sgd ? launch_grouped_t<EPI_SGD_F32>(maps, ga, num_sms, stream)
                   : launch_grouped_t<EPI_F32>(maps, ga, num_sms, stream);
}

template <int EPI>
static cudaError_t launch_grouped_pair_t(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                         cudaStream_t stream) {
  constexpr int BN = 256;
  auto kern = gemm_grouped_pair_kernel<BN, true, true, EPI>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), PairCfg<BN>::kSmem);
  if (e != cudaSuccess) return e;
  const int tiles = ga.tile_start[ga.count];
  const int pairs = tiles < num_sms / 2 ? tiles : num_sms / 2;
  if (pairs < 1) return cudaErrorInvalidValue;
  return launch_pdl(kern, dim3(2 * pairs), dim3(kThreads), PairCfg<BN>::kSmem, stream, 2, maps, ga);
}

cudaError_t launch_gemm_grouped_pair_bwd_weight(const GroupMaps& maps, const GroupArgs& ga, int num_sms,
                                                cudaStream_t stream, bool fused_sgd) {
  return fused_sgd ? launch_grouped_pair_t<EPI_SGD_F32>(maps, ga, num_sms, stream)
                   : launch_grouped_pair_t<EPI_F32>(maps, ga, num_sms, stream);
}

int grouped_tile_bn() { return 256; }

template <int BN, int KMAX>
static cudaError_t launch_head_t(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N,
                                 int K, const HeadArgs& hp, cudaStream_t stream) {
  auto kern = teacher_head_kernel<BN, KMAX>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), GemmCfg<BN>::kSmem, true);
  if (e != cudaSuccess) return e;
  const int cs = (N + BN - 1) / BN;
  return launch_pdl(kern, dim3(cs, (M + kBM - 1) / kBM, 1), dim3(kThreads), GemmCfg<BN>::kSmem, stream, cs,
                    ta, tb, M, N, K, hp);
}

template <int BN>
static cudaError_t launch_head_k(int kmax, const CUtensorMap& ta, const CUtensorMap& tb, int M,
                                 int N, int K, const HeadArgs& hp, cudaStream_t stream) {
  switch (kmax) {
    case 4: return launch_head_t<BN, 4>(ta, tb, M, N, K, hp, stream);
    case 8: return launch_head_t<BN, 8>(ta, tb, M, N, K, hp, stream);
    case 16: return launch_head_t<BN, 16>(ta, tb, M, N, K, hp, stream);
    case 32: return launch_head_t<BN, 32>(ta, tb, M, N, K, hp, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int KMAX>
static cudaError_t launch_kd_head_t(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M,
                                   int N, int Nw, int K, const KdArgs& kp, cudaStream_t stream) {
  constexpr int BN = 256;
  auto kern = kp.t2 ? kd_head_kernel<BN, KMAX, true> : kd_head_kernel<BN, KMAX, false>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), GemmCfg<BN>::kSmem);
  if (e != cudaSuccess) return e;
  const int cs = (Nw + BN - 1) / BN;
  if (cs > 8) return cudaErrorInvalidValue;
  return launch_pdl(kern, dim3(cs, (M + kBM - 1) / kBM, 1), dim3(kThreads), GemmCfg<BN>::kSmem, stream, cs,
                    ta, tb, ty, M, N, Nw, K, kp);
}

cudaError_t launch_kd_head(int kmax, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, int M,
                           int N, int Nw, int K, const KdArgs& kp, cudaStream_t stream) {
  switch (kmax) {
    case 4: return launch_kd_head_t<4>(ta, tb, ty, M, N, Nw, K, kp, stream);
    case 8: return launch_kd_head_t<8>(ta, tb, ty, M, N, Nw, K, kp, stream);
    case 16: return launch_kd_head_t<16>(ta, tb, ty, M, N, Nw, K, kp, stream);
    case 32: return launch_kd_head_t<32>(ta, tb, ty, M, N, Nw, K, kp, stream);
    default: return cudaErrorInvalidValue;
  }
}

template <int KMAX>
static cudaError_t launch_head_pair_t(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                                     const HeadArgs& hp, float* part, unsigned* tickets, cudaStream_t stream) {
  constexpr int BN = 256, S = 6;
  constexpr int smem = S * PairCfg<BN>::kStageBytes + BN * 4 + 1024 + 256;
  static_assert(smem <= 227 * 1024, "head pair smem");
  static const bool mc = [] {
    const char* v = getenv("EDL_HEAD_MC");       // A/B switch: 0 = pairs without the B multicast
    return !(v && v[0] == '0');
  }();
  const int mpairs = (M + 2 * kBM - 1) / (2 * kBM);
  const int pairs = mpairs * ((N + BN - 1) / BN);
  const bool cl4 = mc && mpairs % 2 == 0;
  auto kern = cl4 ? teacher_head_pair_kernel<KMAX, 4> : teacher_head_pair_kernel<KMAX, 2>;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(kern, dim3(2 * pairs), dim3(kThreads), smem, stream, cl4 ? 4 : 2, ta, tb, M, N, K, hp, part,
                    tickets);
}

cudaError_t launch_teacher_head_pair(int kmax, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                                     const HeadArgs& hp, float* part, unsigned* tickets, cudaStream_t stream) {
  switch (kmax) {
    case 4: return launch_head_pair_t<4>(ta, tb, M, N, K, hp, part, tickets, stream);
    case 8: return launch_head_pair_t<8>(ta, tb, M, N, K, hp, part, tickets, stream);
    case 16: return launch_head_pair_t<16>(ta, tb, M, N, K, hp, part, tickets, stream);
    case 32: return launch_head_pair_t<32>(ta, tb, M, N, K, hp, part, tickets, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_teacher_head(int bn, int kmax, const CUtensorMap& ta, const CUtensorMap& tb,
                                int M, int N, int K, const HeadArgs& hp, cudaStream_t stream) {
  switch (bn) {
    case 64: return launch_head_k<64>(kmax, ta, tb, M, N, K, hp, stream);
    case 128: return launch_head_k<128>(kmax, ta, tb, M, N, K, hp, stream);
    case 256: return launch_head_k<256>(kmax, ta, tb, M, N, K, hp, stream);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace edl
