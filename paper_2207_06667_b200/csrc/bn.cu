// bn.cu — training-mode BatchNorm for the cfg4 ResNet-18-style student
// (BASELINE.json configs[3]; the reference has no convolutions).
// Activations are NHWC bf16 rows: z [M = N*H*W][C], C a multiple of 8.
//
//   forward   mean_c, var_c over the M rows (biased, as nn.BatchNorm2d in
//             training mode); y = gamma (z - mean) rstd + beta [+ residual], ReLU
//   backward  dbeta = sum g, dgamma = sum g xhat (xhat = (z - mean) rstd),
//             dz = gamma rstd (g - dbeta / M - xhat dgamma / M)
//
// The two per-channel reductions run as a fixed grid of row-range blocks
// (fp32 partials per block, 8 channels per thread, row lanes combined in a
// fixed order through shared memory) and a final pass that adds the block
// partials in block order in fp64: deterministic, independent of timing.
#include "internal.h"
#include "sm100.cuh"

namespace edl {

namespace {

constexpr int kBnThreads = 256;

// MODE 0: (sum z, sum z^2); MODE 1: (sum g, sum g * xhat)
template <int MODE>
__global__ void __launch_bounds__(kBnThreads) bn_partial_kernel(const __nv_bfloat16* __restrict__ a,
                                                                const __nv_bfloat16* __restrict__ z, int M,
                                                                int C, int rpb, const float* __restrict__ mean,
                                                                const float* __restrict__ rstd,
                                                                float* __restrict__ partial) {
  griddep_wait();
  __shared__ float red[kBnThreads * 16];
  const int cv = C / 8;
  const int rpp = kBnThreads / cv;          // rows in flight per pass (C <= 2048)
  const int rl = threadIdx.x / cv, c8 = threadIdx.x % cv;
  const int r0 = blockIdx.x * rpb;
  const int r1 = r0 + rpb < M ? r0 + rpb : M;
  float s1[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float s2[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float mu[8], rs[8];
  if (MODE == 1 && rl < rpp) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { mu[j] = __ldg(mean + 8 * c8 + j); rs[j] = __ldg(rstd + 8 * c8 + j); }
  }
  if (rl < rpp) {
    for (int r = r0 + rl; r < r1; r += rpp) {
      const uint4 qa = __ldg(reinterpret_cast<const uint4*>(a + static_cast<long long>(r) * C + 8 * c8));
      const __nv_bfloat16* ha = reinterpret_cast<const __nv_bfloat16*>(&qa);
      if constexpr (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float v = __bfloat162float(ha[j]);
          s1[j] += v;
          s2[j] = fmaf(v, v, s2[j]);
        }
      } else {
        const uint4 qz = __ldg(reinterpret_cast<const uint4*>(z + static_cast<long long>(r) * C + 8 * c8));
        const __nv_bfloat16* hz = reinterpret_cast<const __nv_bfloat16*>(&qz);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float g = __bfloat162float(ha[j]);
          const float xh = (__bfloat162float(hz[j]) - mu[j]) * rs[j];
          s1[j] += g;
          s2[j] = fmaf(g, xh, s2[j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[threadIdx.x * 16 + j] = s1[j];
    red[threadIdx.x * 16 + 8 + j] = s2[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float t1 = 0.f, t2 = 0.f;
    for (int q = 0; q < rpp; ++q) {
      const int t = q * cv + c / 8;
      t1 += red[t * 16 + c % 8];
      t2 += red[t * 16 + 8 + c % 8];
    }
    partial[(static_cast<long long>(blockIdx.x) * 2) * C + c] = t1;
    partial[(static_cast<long long>(blockIdx.x) * 2 + 1) * C + c] = t2;
  }
}

// MODE 0: out1 = mean, out2 = rstd = 1 / sqrt(var + eps); MODE 1: out1 = dbeta, out2 = dgamma
template <int MODE>
__global__ void bn_final_kernel(const float* __restrict__ partial, int G, int C, int M, float eps,
                                float* __restrict__ out1, float* __restrict__ out2) {
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double t1 = 0.0, t2 = 0.0;
  for (int b = 0; b < G; ++b) {
    t1 += static_cast<double>(__ldcg(partial + (2ll * b) * C + c));
    t2 += static_cast<double>(__ldcg(partial + (2ll * b + 1) * C + c));
  }
  if constexpr (MODE == 0) {
    const double m = t1 / M;
    double var = t2 / M - m * m;
    if (var < 0.0) var = 0.0;
    out1[c] = static_cast<float>(m);
    out2[c] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
  } else {
    out1[c] = static_cast<float>(t1);
    out2[c] = static_cast<float>(t2);
  }
}

// y = act(gamma (z - mean) rstd + beta [+ res])
__global__ void __launch_bounds__(kBnThreads) bn_apply_kernel(const __nv_bfloat16* __restrict__ z, long long n8,
                                                              int C, const float* __restrict__ mean,
                                                              const float* __restrict__ rstd,
                                                              const float* __restrict__ gamma,
                                                              const float* __restrict__ beta,
                                                              const __nv_bfloat16* __restrict__ res, int relu,
                                                              __nv_bfloat16* __restrict__ y) {
  griddep_wait();
  extern __shared__ float sp[];            // [C] scale, [C] shift
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float sc = gamma[c] * rstd[c];
    sp[c] = sc;
    sp[C + c] = beta[c] - mean[c] * sc;
  }
  __syncthreads();
  const int cv = C / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % cv) * 8;
    const uint4 qz = __ldg(reinterpret_cast<const uint4*>(z) + i);
    const __nv_bfloat16* hz = reinterpret_cast<const __nv_bfloat16*>(&qz);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fmaf(__bfloat162float(hz[j]), sp[c0 + j], sp[C + c0 + j]);
    if (res != nullptr) {
      const uint4 qr = __ldg(reinterpret_cast<const uint4*>(res) + i);
      const __nv_bfloat16* hr = reinterpret_cast<const __nv_bfloat16*>(&qr);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += __bfloat162float(hr[j]);
    }
    if (relu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    reinterpret_cast<uint4*>(y)[i] = o;
  }
}

// dz = gamma rstd (g - dbeta / M - xhat dgamma / M)
__global__ void __launch_bounds__(kBnThreads) bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ g,
                                                                  const __nv_bfloat16* __restrict__ z, long long n8,
                                                                  int C, int M, const float* __restrict__ mean,
                                                                  const float* __restrict__ rstd,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ dbeta,
                                                                  const float* __restrict__ dgamma,
                                                                  __nv_bfloat16* __restrict__ dz) {
  griddep_wait();
  extern __shared__ float sp[];            // [C] k = gamma rstd, [C] dbeta / M, [C] dgamma / M, [C] mean, [C] rstd
  const float inv_m = 1.0f / static_cast<float>(M);
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    sp[c] = gamma[c] * rstd[c];
    sp[C + c] = dbeta[c] * inv_m;
    sp[2 * C + c] = dgamma[c] * inv_m;
    sp[3 * C + c] = mean[c];
    sp[4 * C + c] = rstd[c];
  }
  __syncthreads();
  const int cv = C / 8;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c0 = static_cast<int>(i % cv) * 8;
    const uint4 qg = __ldg(reinterpret_cast<const uint4*>(g) + i);
    const uint4 qz = __ldg(reinterpret_cast<const uint4*>(z) + i);
    const __nv_bfloat16* hg = reinterpret_cast<const __nv_bfloat16*>(&qg);
    const __nv_bfloat16* hz = reinterpret_cast<const __nv_bfloat16*>(&qz);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = c0 + j;
      const float xh = (__bfloat162float(hz[j]) - sp[3 * C + c]) * sp[4 * C + c];
      v[j] = sp[c] * (__bfloat162float(hg[j]) - sp[C + c] - xh * sp[2 * C + c]);
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    reinterpret_cast<uint4*>(dz)[i] = o;
  }
}

int blocks_for(long long n8, int sms) {
  long long b = (n8 + kBnThreads - 1) / kBnThreads;
  const long long cap = 8LL * sms;
  return static_cast<int>(b < cap ? (b < 1 ? 1 : b) : cap);
}

}  // namespace

int bn_partial_blocks(int M, int sms) {
  int g = 2 * sms;
  const int min_rows = 64;                 // keep each block's row range meaningful for tiny M
  if (g > (M + min_rows - 1) / min_rows) g = (M + min_rows - 1) / min_rows;
  return g < 1 ? 1 : g;
}

cudaError_t launch_bn_stats(const __nv_bfloat16* z, int M, int C, float* partial, float* mean, float* rstd,
                            float eps, int sms, cudaStream_t stream) {
  const int G = bn_partial_blocks(M, sms);
  const int rpb = (M + G - 1) / G;
  cudaError_t e = launch_pdl(bn_partial_kernel<0>, dim3(G), dim3(kBnThreads), 0, stream, 1, z, z, M, C, rpb,
                             static_cast<const float*>(nullptr), static_cast<const float*>(nullptr), partial);
  if (e != cudaSuccess) return e;
  return launch_pdl(bn_final_kernel<0>, dim3((C + 127) / 128), dim3(128), 0, stream, 1,
                    static_cast<const float*>(partial), G, C, M, eps, mean, rstd);
}

cudaError_t launch_bn_bwd_reduce(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                 const float* rstd, float* partial, float* dbeta, float* dgamma, int sms,
                                 cudaStream_t stream) {
  const int G = bn_partial_blocks(M, sms);
  const int rpb = (M + G - 1) / G;
  cudaError_t e = launch_pdl(bn_partial_kernel<1>, dim3(G), dim3(kBnThreads), 0, stream, 1, g, z, M, C, rpb, mean,
                             rstd, partial);
  if (e != cudaSuccess) return e;
  return launch_pdl(bn_final_kernel<1>, dim3((C + 127) / 128), dim3(128), 0, stream, 1,
                    static_cast<const float*>(partial), G, C, M, 0.f, dbeta, dgamma);
}

cudaError_t launch_bn_apply(const __nv_bfloat16* z, int M, int C, const float* mean, const float* rstd,
                            const float* gamma, const float* beta, const __nv_bfloat16* res, bool relu,
                            __nv_bfloat16* y, int sms, cudaStream_t stream) {
  const long long n8 = static_cast<long long>(M) * C / 8;
  return launch_pdl(bn_apply_kernel, dim3(blocks_for(n8, sms)), dim3(kBnThreads), 2 * C * sizeof(float), stream, 1,
                    z, n8, C, mean, rstd, gamma, beta, res, relu ? 1 : 0, y);
}

cudaError_t launch_bn_bwd_apply(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                const float* rstd, const float* gamma, const float* dbeta, const float* dgamma,
                                __nv_bfloat16* dz, int sms, cudaStream_t stream) {
  const long long n8 = static_cast<long long>(M) * C / 8;
  return launch_pdl(bn_bwd_apply_kernel, dim3(blocks_for(n8, sms)), dim3(kBnThreads), 5 * C * sizeof(float), stream,
                    1, g, z, n8, C, M, mean, rstd, gamma, dbeta, dgamma, dz);
}

}  // namespace edl
