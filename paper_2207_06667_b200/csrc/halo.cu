// halo.cu — halo-tiled implicit-GEMM 3x3 convolution for the 64-channel
// stage-1 layers of the cfg4 ResNets (BASELINE.json configs[3]).
//
// The TMA im2col path (gemm_sm100.cu, ConvGeom) loads one 128-pixel x
// 64-channel A box per filter tap, so every input pixel crosses L2 -> SM nine
// times. Here a CTA stages the zero-padded input PATCH of a tile once —
// rows h0-1 .. h0+R of one image, columns -1 .. W, all 64 channels — and each
// tap's A operand is a row-shifted view of that patch:
//
//   tile rows m = i * (W + 2) + j   (i < R output rows, j < W + 2; j >= W are
//                                    discarded), tap (r, s) reads patch row
//                                    m + r * (W + 2) + s.
//
// The patch is staged by one 4-D tiled TMA box {64 channels, W + 2, R + 2, 1}
// with SWIZZLE_128B: pixel rows of 128 B, the K-major operand layout of a
// 2-D box. The tensor core applies the 128-byte swizzle to absolute shared
// addresses, as the TMA does, so a descriptor that starts ANY whole number of
// rows into a 1024-byte-aligned patch (base-offset field 0) reads the shifted
// view correctly (`edl_halo_probe` checks every layout claim here). Out-of-
// image rows and columns are the TMA's zero fill. A no-swizzle chunk-plane
// layout (5-D box with a 16-byte chunk stride) also works, but its 16-byte
// box rows make the TMA ~2.4x slower than the MMAs.
#include "internal.h"
#include "sm100.cuh"

namespace edl {

namespace {

// UMMA shared-memory descriptor, no swizzle (canonical K-major interleave).
__device__ __forceinline__ uint64_t smem_desc_noswz(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                              // layout type 0: SWIZZLE_NONE
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* m, uint32_t dst, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void tma_load_5d(const CUtensorMap* m, uint32_t dst, uint32_t bar, int c0, int c1, int c2,
                                            int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

// Probe (tests / layout experiments): one tap's product out[128][64] =
// patch[m + off][:] . w[n][:] with the patch of image n, rows h0-1 .. h0+2
// (R = 2 output rows). mode 0: no-swizzle chunk-plane layout (5-D map);
// mode 1: SWIZZLE_128B pixel rows (4-D map) with the descriptor's base-offset
// field = start row % 8; mode 2: the same without the base offset. reps > 0
// re-issues the 9-tap x 4 MMA sequence `reps` times and stores the cycle
// count in out[128 * 64] (throughput of the layout's operand reads).
__global__ void __launch_bounds__(128, 1) halo_probe_kernel(const __grid_constant__ CUtensorMap tmX,
                                                            const __grid_constant__ CUtensorMap tmW, int n, int h0,
                                                            int W, int off, int mode, int reps,
                                                            float* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sw = smem;                     // 64 x 64 bf16 per tap, SWIZZLE_128B (8 KB; mode 3: 9 taps)
  uint8_t* sp = smem + (mode == 3 ? 9 * 8192 : 8192);   // the patch
  __shared__ uint64_t bar, done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rows = 4 * (W + 2);
  const uint32_t plane = static_cast<uint32_t>(rows) * 16u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  const bool big_tmem = (reps / 2000) & 1;   // experiment switches in reps' thousands
  if (warp == 0) {
    if (big_tmem) tmem_alloc<128>(&tslot); else tmem_alloc<64>(&tslot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, (mode == 3 ? 9 : 1) * 8192 + 8 * plane);
    for (int t = 0; t < (mode == 3 ? 9 : 1); ++t) tma_load_2d(sw + t * 8192, &tmW, &bar, t * 64, 0);
    if (mode == 0) tma_load_5d(&tmX, smem_u32(sp), smem_u32(&bar), 0, -1, h0 - 1, n, 0);
    else tma_load_4d(&tmX, smem_u32(sp), smem_u32(&bar), 0, -1, h0 - 1, n);
    mbar_wait(&bar, 0);
    tc_fence_after();
    constexpr uint32_t idesc = idesc_bf16_f32(128, 64, false, false);
    auto issue = [&](int o, bool first, int tap, uint32_t d) {
      for (int k = 0; k < 4; ++k) {
        uint64_t ad;
        if (mode == 0) {
          ad = smem_desc_noswz(smem_u32(sp) + static_cast<uint32_t>(o) * 16u + 2u * k * plane, plane, 128);
        } else {
          const uint32_t a = smem_u32(sp) + static_cast<uint32_t>(o) * 128u + 32u * k;
          ad = smem_desc_sw128(a, 16, 1024);
          if (mode == 1) ad |= static_cast<uint64_t>((a >> 7) & 7) << 49;
        }
        const uint64_t bd = smem_desc_sw128(smem_u32(sw) + (mode == 3 ? tap * 8192u : 0u) + 32u * k, 16, 1024);
        umma_bf16(d, ad, bd, idesc, (first && k == 0) ? 0u : 1u);
      }
    };
    long long t0 = clock64();
    if (mode == 4) {
      // MN-major A of two stacked 64-wide views (rows off and off + reps) via
      // LBO = reps rows; B = the weight tile read MN-major (K = its rows)
      constexpr uint32_t idesc_mn = idesc_bf16_f32(128, 64, true, true);
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = smem_desc_sw128(smem_u32(sp) + static_cast<uint32_t>(off) * 128u + 2048u * k,
                                            static_cast<uint32_t>(reps) * 128u, 1024);
        const uint64_t bd = smem_desc_sw128(smem_u32(sw) + 2048u * k, 8192, 1024);
        umma_bf16(tmem, ad, bd, idesc_mn, k ? 1u : 0u);
      }
    } else if (reps == 0) {
      issue(off, true, 0, tmem);
    } else {
      for (int r = 0; r < reps % 1000; ++r) {  // NOLINT
        const uint32_t d = (mode == 3 && big_tmem) ? tmem + 64u * (r & 1) : tmem;
        for (int tap = 0; tap < 9; ++tap)
          issue((tap / 3) * (W + 2) + tap % 3, (mode == 3 || r == 0) && tap == 0, tap, d);
      }
    }
    umma_commit(&done);
    mbar_wait(&done, 0);
    if (mode != 4 && reps > 0 && blockIdx.x == 0) out[128 * 64] = static_cast<float>(clock64() - t0);
    if (mode != 4 && reps > 0 && blockIdx.x == 0) out[128 * 64 + 1] = static_cast<float>(smem_u32(sp));
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  const int row = 32 * warp + lane;
  for (int c = 0; c < 64 && blockIdx.x == 0; c += 32) {
    float v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c, v);
#pragma unroll
    for (int j = 0; j < 32; ++j) out[row * 64 + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    if (big_tmem) tmem_dealloc<128>(tmem); else tmem_dealloc<64>(tmem);
  }
}

constexpr int kHaloThreads = 256;     // warp 0 TMA, warps 1 / 3 MMA, warp 2 TMEM, warps 4-7 epilogue
constexpr int kHaloMaxStages = 3;
constexpr int kTapBytes = 64 * 64 * 2;   // one tap's 64 x 64 bf16 weights (SWIZZLE_128B, K-major)

struct HaloGeom {
  uint32_t patch_bytes, stage_bytes;     // TMA patch bytes / stage stride
  uint32_t tile_bytes, out_bytes;        // an R x W x 128 B output-shaped tile / its 1 KB-aligned stride
  int stages, n_aux;                     // patch stages; aux tiles per tile (residual / add, mask)
};

// Persistent: CTA b takes tiles b, b + grid, ... (static, deterministic). Per
// tile: one TMA patch load (+ the residual / mask tiles the epilogue needs),
// 9 taps x 4 UMMAs (128 x 64 x 16) into one of two TMEM accumulators, and the
// epilogue of the previous tile under them: TMEM -> registers, + bias
// (shared memory), + residual, ReLU, x mask (shared memory tiles), bf16 into
// a SWIZZLE_128B staging tile, one TMA store of the R x W output rows.
__global__ void __launch_bounds__(kHaloThreads, 1)
    halo_conv_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                     const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                     const __grid_constant__ CUtensorMap tmM, HaloArgs a, HaloGeom g) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sW = smem;                                    // 9 taps
  uint8_t* sP = smem + 9 * kTapBytes;                     // patch stages
  uint8_t* sA = sP + g.stages * g.stage_bytes;            // 2 aux slots (one per TMEM accumulator): [residual][mask]
  uint8_t* sO = sA + 2 * g.n_aux * g.out_bytes;           // 2 output staging tiles [R][W][128 B], SWIZZLE_128B
  float* sbias = reinterpret_cast<float*>(sO + 2 * g.out_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbias + 64);
  uint64_t* wbar = bars;
  uint64_t* full = bars + 1;
  uint64_t* empty = full + kHaloMaxStages;
  uint64_t* afull = empty + kHaloMaxStages;
  uint64_t* aempty = afull + 2;
  uint64_t* tfull = aempty + 2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int Wp = a.W + 2;
  const int S = g.stages;
  const bool has_res = a.res != nullptr, has_mask = a.mask != nullptr;
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmY);
    mbar_init(wbar, 1);
    for (int i = 0; i < kHaloMaxStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 4);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<128>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_wait();

  if (warp == 0 && lane == 0) {
    mbar_arrive_expect_tx(wbar, 9 * kTapBytes);
    for (int t = 0; t < 9; ++t) tma_load_2d(sW + t * kTapBytes, &tmW, wbar, t * 64, 0);
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int s = it % S, u = it / S;
      mbar_wait(&empty[s], (u & 1) ^ 1);
      const int n = tile / a.tiles_per_image, h0 = (tile % a.tiles_per_image) * a.R;
      if (a.debug == 2 && it >= S) {
        mbar_arrive(&full[s]);
      } else {
        mbar_arrive_expect_tx(&full[s], g.patch_bytes);
        tma_load_4d(&tmX, smem_u32(sP + s * g.stage_bytes), smem_u32(&full[s]), 0, -1, h0 - 1, n);
      }
      if (g.n_aux) {
        // the epilogue's tiles, in a 2-slot ring paced like the TMEM accumulators
        const int sa = it & 1, ua = it >> 1;
        mbar_wait(&aempty[sa], (ua & 1) ^ 1);
        mbar_arrive_expect_tx(&afull[sa], g.n_aux * g.tile_bytes);
        uint8_t* aux = sA + sa * g.n_aux * g.out_bytes;
        if (has_res) {
          tma_load_4d(&tmR, smem_u32(aux), smem_u32(&afull[sa]), 0, 0, h0, n);
          aux += g.out_bytes;
        }
        if (has_mask) tma_load_4d(&tmM, smem_u32(aux), smem_u32(&afull[sa]), 0, 0, h0, n);
      }
    }
  } else if ((warp == 1 || warp == 3) && lane == 0) {
    // two issuing warps, one per TMEM accumulator (warp 1: even tiles, warp 3:
    // odd): a 128 x 64 x 16 UMMA retires in ~49 cycles, about what one
    // thread's issue sequence takes, so one issuer left the tensor core idle
    const int parity = warp == 1 ? 0 : 1;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 64, false, false);
    // Descriptors are built once and stepped in their 14-bit address field
    // (addr >> 4 < 2^14 in shared memory, so the adds never carry into LBO):
    // the issue loop is 36 UTCHMMAs with one add each. Descriptor arithmetic
    // per MMA made the ISSUE the limit for these N = 64 MMAs (97 -> 74 us).
    const uint64_t bd0 = smem_desc_sw128(smem_u32(sW), 16, 1024);
    const uint64_t ad0 = smem_desc_sw128(smem_u32(sP), 16, 1024);
    mbar_wait(wbar, 0);
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      if ((it & 1) != parity) continue;
      const int s = it % S, u = it / S;
      const int acc = it & 1, ua = it >> 1;
      mbar_wait(&tempty[acc], (ua & 1) ^ 1);
      mbar_wait(&full[s], u & 1);
      tc_fence_after();
      const uint32_t d = tmem + 64u * acc;
      const uint64_t as = ad0 + static_cast<uint64_t>((s * g.stage_bytes) >> 4);
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const uint64_t at = as + static_cast<uint64_t>(((tap / 3) * Wp + tap % 3) * 8);   // rows of 128 B
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(d, at + 2 * kk, bd0 + static_cast<uint64_t>(tap * (kTapBytes >> 4) + 2 * kk), idesc,
                    (tap | kk) ? 1u : 0u);
      }
      umma_commit(&empty[s]);
      umma_commit(&tfull[acc]);
    }
  } else if (warp >= 4) {
    const int q = warp - 4;
    const int m = 32 * q + lane;
    const int i = m / Wp, j = m % Wp;
    const int srow = i * a.W + j;
    const bool in_tile = i < a.R && j < a.W;
    if (threadIdx.x - 128 < 64) sbias[threadIdx.x - 128] = a.bias != nullptr ? __ldg(a.bias + threadIdx.x - 128) : 0.f;
    epi_bar_sync();
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int s = it % S, u = it / S;
      const int acc = it & 1, ua = it >> 1;
      mbar_wait(&tfull[acc], ua & 1);
      tc_fence_after();
      float v[64];
      uint32_t r0[32], r1[32];
      const uint32_t ta = tmem + (static_cast<uint32_t>(32 * q) << 16) + 64u * acc;
      tmem_ld32_issue(ta, r0);
      tmem_ld32_issue(ta + 32, r1);
      tmem_ld_wait(r0);
      tmem_ld_wait(r1);
#pragma unroll
      for (int c = 0; c < 32; ++c) { v[c] = __uint_as_float(r0[c]); v[32 + c] = __uint_as_float(r1[c]); }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (a.debug == 1) {
        if (g.n_aux) {
          mbar_wait(&afull[acc], ua & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&aempty[acc]);
        }
        continue;
      }
      const int n = tile / a.tiles_per_image, h0 = (tile % a.tiles_per_image) * a.R;
      // the staging tile written two tiles ago has been read by its TMA store
      if (threadIdx.x == 128) bulk_wait_read1();
      epi_bar_sync();
      uint8_t* stg = sO + (it & 1) * g.out_bytes;
      if (g.n_aux) mbar_wait(&afull[acc], ua & 1);
      if (in_tile) {
        const float4* b4 = reinterpret_cast<const float4*>(sbias);
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 b = b4[c4];
          v[4 * c4] += b.x; v[4 * c4 + 1] += b.y; v[4 * c4 + 2] += b.z; v[4 * c4 + 3] += b.w;
        }
        const uint8_t* aux = sA + acc * g.n_aux * g.out_bytes;
        if (has_res) {
          const uint4* rp = reinterpret_cast<const uint4*>(aux + srow * 128);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint4 qr = rp[c8 ^ (srow & 7)];
            const __nv_bfloat16* hr = reinterpret_cast<const __nv_bfloat16*>(&qr);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[8 * c8 + e] += __bfloat162float(hr[e]);
          }
          aux += g.out_bytes;
        }
        if (a.relu) {
#pragma unroll
          for (int c = 0; c < 64; ++c) v[c] = fmaxf(v[c], 0.f);
        }
        if (has_mask) {
          const uint4* mp = reinterpret_cast<const uint4*>(aux + srow * 128);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint4 qm = mp[c8 ^ (srow & 7)];
            const __nv_bfloat16* hm = reinterpret_cast<const __nv_bfloat16*>(&qm);
#pragma unroll
            for (int e = 0; e < 8; ++e) v[8 * c8 + e] = __bfloat162float(hm[e]) > 0.f ? v[8 * c8 + e] : 0.f;
          }
        }
        uint4* op = reinterpret_cast<uint4*>(stg + srow * 128);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          uint4 o;
          o.x = pack_bf16x2(v[8 * c8 + 0], v[8 * c8 + 1]);
          o.y = pack_bf16x2(v[8 * c8 + 2], v[8 * c8 + 3]);
          o.z = pack_bf16x2(v[8 * c8 + 4], v[8 * c8 + 5]);
          o.w = pack_bf16x2(v[8 * c8 + 6], v[8 * c8 + 7]);
          op[c8 ^ (srow & 7)] = o;           // SWIZZLE_128B: 16-byte chunk c at c ^ (row % 8)
        }
      }
      __syncwarp();
      if (g.n_aux && lane == 0) mbar_arrive(&aempty[acc]);
      fence_proxy_async_smem();
      epi_bar_sync();
      if (threadIdx.x == 128) {
        tma_store_4d(&tmY, stg, 0, 0, h0, n);   // rows past the image are clipped by the TMA
        bulk_commit();
      }
    }
    if (threadIdx.x == 128) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// ---- halo weight gradient: dW[cout][tap][cin] = sum over pixels of
// dz[p][cout] x[p + off(tap)][cin], for the same 64 -> 64 3x3 stride-1 layers.
// Per tile (two output rows): the zero-padded x patch (as in the forward) and
// the dz tile in the same padded row space (a {64, W + 2, R, 1} box: the two
// columns past the image are the TMA's zero fill, rows 116..127 stay zero).
// The UMMA's M = 128 rows are two taps' 64 input channels: an MN-major A
// whose two 64-wide halves are the patch viewed at both taps' row offsets
// (LBO = the offset difference; `edl_halo_probe` mode 4), K = 16 pixel rows
// per instruction, B = dz MN-major (N = cout 64). Five tap pairs (the ninth
// tap pairs with itself) accumulate in five TMEM accumulators over all of a
// CTA's tiles; the CTA writes its partial [tap][cin][cout] once and
// halo_wgrad_reduce_kernel adds the CTAs' partials in CTA order
// (deterministic). Three warps issue the MMAs (an N = 64 UMMA retires about
// as fast as one thread issues it).
constexpr int kWgStages = 3;
constexpr int kWgThreads = 256;

struct WgGeom {
  uint32_t patch_bytes, dz_bytes, stage_bytes, dz_off;   // per stage: patch (padded), then dz tile
};

__global__ void __launch_bounds__(kWgThreads, 1)
    halo_wgrad_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmD, HaloArgs a,
                      WgGeom g, float* __restrict__ partial) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint8_t* sS = smem;                                        // stages: [patch | dz]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sS + kWgStages * g.stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = full + kWgStages;
  uint64_t* done = empty + kWgStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int Wp = a.W + 2;
  // zero the stages once: dz rows past R (W + 2) and patch rows past (R + 2) (W + 2)
  // are never written by the TMA and must read as 0 (0 x garbage could be NaN)
  for (uint32_t i = threadIdx.x; i < kWgStages * g.stage_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sS)[i] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmD);
    for (int i = 0; i < kWgStages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 3); }
    mbar_init(done, 3);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  griddep_wait();

  if (warp == 0 && lane == 0) {
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int s = it % kWgStages, u = it / kWgStages;
      mbar_wait(&empty[s], (u & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], g.patch_bytes + g.dz_bytes);
      const int n = tile / a.tiles_per_image, h0 = (tile % a.tiles_per_image) * a.R;
      uint8_t* st = sS + s * g.stage_bytes;
      tma_load_4d(&tmX, smem_u32(st), smem_u32(&full[s]), 0, -1, h0 - 1, n);
      tma_load_4d(&tmD, smem_u32(st + g.dz_off), smem_u32(&full[s]), 0, 0, h0, n);
    }
  } else if (warp >= 1 && warp <= 3 && lane == 0) {
    // three issuers: tap pairs {0, 1}, {2, 3}, {4} (16 / 16 / 8 UMMAs per tile)
    constexpr uint32_t idesc = idesc_bf16_f32(128, 64, true, true);
    const int p_lo = warp == 1 ? 0 : warp == 2 ? 2 : 4, p_hi = warp == 1 ? 2 : warp == 2 ? 4 : 5;
    const uint64_t a0 = smem_desc_sw128(smem_u32(sS), 16, 1024);
    const uint64_t b0 = smem_desc_sw128(smem_u32(sS + g.dz_off), 8192, 1024);
    int it = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++it) {
      const int s = it % kWgStages, u = it / kWgStages;
      mbar_wait(&full[s], u & 1);
      tc_fence_after();
      const uint64_t so = static_cast<uint64_t>((s * g.stage_bytes) >> 4);
      for (int pr = p_lo; pr < p_hi; ++pr) {
        const int ta = 2 * pr, tb = pr == 4 ? 8 : 2 * pr + 1;
        const int oa = (ta / 3) * Wp + ta % 3, ob = (tb / 3) * Wp + tb % 3;
        // LBO (bits 16-29) = the second tap's view, (ob - oa) rows of 128 B further
        const uint64_t ad = (a0 & ~(static_cast<uint64_t>(0x3FFF) << 16)) |
                            (static_cast<uint64_t>(((ob - oa) * 128) >> 4) << 16);
        const uint32_t d = tmem + 64u * pr;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)          // 16 pixel rows per UMMA
          umma_bf16(d, ad + so + static_cast<uint64_t>(oa * 8 + kk * 128), b0 + so + static_cast<uint64_t>(kk * 128),
                    idesc, (it == 0 && kk == 0) ? 0u : 1u);
      }
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();
  if (warp >= 4) {
    mbar_wait(done, 0);
    tc_fence_after();
    const int q = warp - 4;
    const int lane_row = 32 * q + lane;                 // M row: tap half, input channel
    const int half = lane_row / 64, cin = lane_row % 64;
    float* dst = partial + static_cast<long long>(blockIdx.x) * 9 * 64 * 64;
    for (int pr = 0; pr < 5; ++pr) {
      const int tap = pr == 4 ? 8 : 2 * pr + half;
      const bool keep = !(pr == 4 && half == 1);
      for (int c = 0; c < 64; c += 32) {
        float v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(32 * q) << 16) + 64u * pr + c, v);
        if (keep) {
          float4* o = reinterpret_cast<float4*>(dst + (static_cast<long long>(tap) * 64 + cin) * 64 + c);
#pragma unroll
          for (int j = 0; j < 8; ++j) __stcg(o + j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    __syncwarp();   // lane 0 ran an MMA role: dealloc is .sync.aligned
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// dW[cout][tap * 64 + cin] = scale * sum over CTAs (in order) of partial[cta][tap][cin][cout]
__global__ void __launch_bounds__(256) halo_wgrad_reduce_kernel(const float* __restrict__ partial, int ctas,
                                                                 float scale, float* __restrict__ dW, long long lddw) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;   // (tap, cin, cout), cout fastest
  if (i >= 9 * 64 * 64) return;
  float acc = 0.f;
  for (int c = 0; c < ctas; ++c) acc += __ldg(partial + static_cast<long long>(c) * 9 * 64 * 64 + i);
  const int cout = i % 64, tc = i / 64;                  // tc = tap * 64 + cin
  dW[static_cast<long long>(cout) * lddw + tc] = scale * acc;
}

}  // namespace

cudaError_t launch_halo_probe(const CUtensorMap& tmX, const CUtensorMap& tmW, int n, int h0, int W, int off, int mode,
                              int reps, int smem_kb, float* out, cudaStream_t stream) {
  // room for either reading of the LBO / SBO fields (mode 3: 9 weight taps); smem_kb > 0 overrides
  const int smem = smem_kb > 0 ? smem_kb * 1024 : (mode == 3 ? 1024 + 9 * 8192 + 96 * 1024 : 1024 + 8192 + 96 * 1024);
  cudaError_t e = cudaFuncSetAttribute(halo_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  halo_probe_kernel<<<(mode != 4 && ((reps / 1000) & 1)) ? 148 : 1, 128, smem, stream>>>(tmX, tmW, n, h0, W, off, mode, reps, out);
  return cudaGetLastError();
}

}  // namespace edl

namespace edl {

int halo_rows_per_tile(int W) { return 128 / (W + 2); }

cudaError_t launch_halo_conv(const CUtensorMap& tmX, const CUtensorMap& tmW, const CUtensorMap& tmY,
                             const CUtensorMap& tmR, const CUtensorMap& tmM, const HaloArgs& a, int grid,
                             cudaStream_t stream) {
  HaloGeom g{};
  g.patch_bytes = static_cast<uint32_t>((a.R + 2) * (a.W + 2)) * 128u;
  // the last tap's view reaches 2 (W + 2) + 2 + 127 rows into the patch (past it only for discarded rows)
  const uint32_t view = static_cast<uint32_t>(2 * (a.W + 2) + 2 + 128) * 128u;
  g.stage_bytes = ((g.patch_bytes > view ? g.patch_bytes : view) + 1023) & ~1023u;
  g.tile_bytes = static_cast<uint32_t>(a.R * a.W) * 128u;
  g.out_bytes = (g.tile_bytes + 1023) & ~1023u;
  g.n_aux = (a.res != nullptr ? 1 : 0) + (a.mask != nullptr ? 1 : 0);
  auto bytes = [&](int stages) {
    return 1024 + 9 * kTapBytes + stages * static_cast<int>(g.stage_bytes) +
           2 * static_cast<int>((1 + g.n_aux) * g.out_bytes) + 64 * 4 + 256;
  };
  g.stages = bytes(3) <= 232448 ? 3 : 2;
  const int smem = bytes(g.stages);
  if (smem > 232448) return cudaErrorInvalidValue;
  // the attribute is set once per kernel: the largest request any W can make
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(halo_conv_kernel), 232448);
  if (e != cudaSuccess) return e;
  return launch_pdl(halo_conv_kernel, dim3(grid), dim3(kHaloThreads), smem, stream, 1, tmX, tmW, tmY, tmR, tmM, a, g);
}

}  // namespace edl

namespace edl {

long long halo_wgrad_partial_floats(int sms) { return static_cast<long long>(sms) * 9 * 64 * 64; }

cudaError_t launch_halo_wgrad(const CUtensorMap& tmX, const CUtensorMap& tmD, const HaloArgs& a, int grid,
                              float* partial, float scale, float* dW, long long lddw, cudaStream_t stream) {
  WgGeom g{};
  g.patch_bytes = static_cast<uint32_t>((a.R + 2) * (a.W + 2)) * 128u;
  // A views reach 2 (W + 2) + 2 + 127 rows into the patch (the rows past it read the zeroed tail)
  const uint32_t view = static_cast<uint32_t>(2 * (a.W + 2) + 2 + 128) * 128u;
  const uint32_t pbytes = ((g.patch_bytes > view ? g.patch_bytes : view) + 1023) & ~1023u;
  g.dz_bytes = static_cast<uint32_t>(a.R * (a.W + 2)) * 128u;
  g.dz_off = pbytes;
  g.stage_bytes = pbytes + 128u * 128u;                  // dz: 128 pixel rows of 128 B (tail zero)
  const int smem = 1024 + kWgStages * static_cast<int>(g.stage_bytes) + 256;
  if (smem > 232448 || a.R * (a.W + 2) > 128) return cudaErrorInvalidValue;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(halo_wgrad_kernel), 232448);
  if (e != cudaSuccess) return e;
  e = launch_pdl(halo_wgrad_kernel, dim3(grid), dim3(kWgThreads), smem, stream, 1, tmX, tmD, a, g, partial);
  if (e != cudaSuccess) return e;
  return launch_pdl(halo_wgrad_reduce_kernel, dim3((9 * 64 * 64 + 255) / 256), dim3(256), 0, stream, 1,
                    static_cast<const float*>(partial), grid, scale, dW, lddw);
}

}  // namespace edl
