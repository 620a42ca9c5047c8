// bn.cu — training-mode BatchNorm for the cfg4 ResNet-18-style student
// (BASELINE.json configs[3]; the reference has no convolutions).
// Activations are NHWC bf16 rows: z [M = N*H*W][C], C a multiple of 8.
//
//   forward   mean_c, var_c over the M rows (biased, as nn.BatchNorm2d in
//             training mode); y = gamma (z - mean) rstd + beta [+ residual], ReLU
//   backward  dbeta = sum g, dgamma = sum g xhat (xhat = (z - mean) rstd),
//             dz = gamma rstd (g - dbeta / M - xhat dgamma / M)
//
// The two per-channel reductions run in ONE launch each: 8-CTA clusters of
// row-range blocks (8 channels per thread, 16 loads in flight per thread, row
// lanes combined in a fixed order through shared memory), the cluster's 8
// block sums added in rank order over DSMEM into one fp64 partial per
// cluster (each rank one eighth of the channels), and the last cluster to
// arrive (a per-stream ticket; its 8 CTAs one eighth of the channels each) adds the
// cluster partials in cluster order: deterministic, independent of timing.
// The elementwise passes keep each thread on one 8-channel group (its
// per-channel constants in registers) and walk the rows back to front, so
// the rows the reduction read last (still in L2) are read first.
#include "internal.h"
#include "sm100.cuh"

namespace edl {

namespace {

constexpr int kBnThreads = 256;
constexpr int kBnCluster = 8;
constexpr int kBnUnroll = 8;

// Reduction grid: 4 blocks per SM, at least 64 rows each, and few enough
// clusters that the finishing block's read (clusters x 2C doubles) stays small.
int bn_stats_blocks(int M, int C, int sms) {
  int g = 4 * sms;
  const int min_rows = 64;
  if (g > (M + min_rows - 1) / min_rows) g = (M + min_rows - 1) / min_rows;
  const int max_clusters = 65536 / C > 1 ? 65536 / C : 1;   // finish: clusters x C / 8 per CTA
  if (g > max_clusters * kBnCluster) g = max_clusters * kBnCluster;
  g = (g + kBnCluster - 1) / kBnCluster * kBnCluster;
  return g < kBnCluster ? kBnCluster : g;
}

// Elementwise grid: 4 blocks per SM, fewer when each block would get < 1 pass.
int bn_apply_blocks(int M, int C, int sms) {
  const int rpp = kBnThreads / (C / 8);
  long long g = (static_cast<long long>(M) + rpp - 1) / rpp;
  if (g > 4LL * sms) g = 4LL * sms;
  return g < 1 ? 1 : static_cast<int>(g);
}

// DSMEM load the compiler may batch (the data is fixed after a cluster barrier)
__device__ __forceinline__ float ld_dsmem_f32_nv(uint32_t addr) {
  float v;
  asm("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ void bf16x8(const uint4& q, float* v) {
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&q);
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __bfloat162float(h[j]);
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 o;
  o.x = pack_bf16x2(v[0], v[1]);
  o.y = pack_bf16x2(v[2], v[3]);
  o.z = pack_bf16x2(v[4], v[5]);
  o.w = pack_bf16x2(v[6], v[7]);
  return o;
}

// The clusters' fp64 partials [Gc][2][C] -> the two per-channel outputs, by
// one block: L = 256 / C lanes per channel (C < 256), each adding a strided
// subset of the clusters in order, then the lanes in order.
// MODE 0: out1 = mean, out2 = rstd = 1 / sqrt(var + eps); MODE 1: out1 = dbeta, out2 = dgamma
template <int MODE>
__device__ void bn_finish(const double* partial, int Gc, int C, int M, float eps, float* out1, float* out2,
                          double* scratch, int cb, int ce) {
  const int span = ce - cb;
  const int L = span < kBnThreads ? kBnThreads / span : 1;
  for (int c0 = cb; c0 < ce; c0 += kBnThreads) {
    const int nc = ce - c0 < kBnThreads ? ce - c0 : kBnThreads;
    const int t = threadIdx.x;
    const int c = t % nc, lane = t / nc;
    double t1 = 0.0, t2 = 0.0;
    if (lane < L) {
      int g = lane;
      for (; g + 7 * L < Gc; g += 8 * L) {     // 16 loads in flight, added in cluster order
        double v1[8], v2[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v1[u] = __ldcg(partial + (2ll * (g + u * L)) * C + c0 + c);
          v2[u] = __ldcg(partial + (2ll * (g + u * L) + 1) * C + c0 + c);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          t1 += v1[u];
          t2 += v2[u];
        }
      }
      for (; g < Gc; g += L) {
        t1 += __ldcg(partial + (2ll * g) * C + c0 + c);
        t2 += __ldcg(partial + (2ll * g + 1) * C + c0 + c);
      }
      scratch[2 * t] = t1;
      scratch[2 * t + 1] = t2;
    }
    __syncthreads();
    if (t < nc) {
      t1 = 0.0;
      t2 = 0.0;
      for (int l = 0; l < L; ++l) {
        t1 += scratch[2 * (l * nc + t)];
        t2 += scratch[2 * (l * nc + t) + 1];
      }
      if constexpr (MODE == 0) {
        const double m = t1 / M;
        double var = t2 / M - m * m;
        if (var < 0.0) var = 0.0;
        out1[c0 + t] = static_cast<float>(m);
        out2[c0 + t] = static_cast<float>(1.0 / sqrt(var + static_cast<double>(eps)));
      } else {
        out1[c0 + t] = static_cast<float>(t1);
        out2[c0 + t] = static_cast<float>(t2);
      }
    }
    __syncthreads();
  }
}

// MODE 0: (sum z, sum z^2); MODE 1: (sum g, sum g * xhat). Launched in 8-CTA clusters.
template <int MODE>
__global__ void __launch_bounds__(kBnThreads) bn_reduce_kernel(const __nv_bfloat16* __restrict__ a,
                                                               const __nv_bfloat16* __restrict__ z, int M, int C,
                                                               int rpb, const float* __restrict__ mean,
                                                               const float* __restrict__ rstd,
                                                               double* __restrict__ partial, unsigned* ticket,
                                                               float eps, float* __restrict__ out1,
                                                               float* __restrict__ out2) {
  griddep_wait();
  __shared__ __align__(16) float red[kBnThreads * 16];
  __shared__ float csum[2 * 2048];
  __shared__ int s_last;
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
  auto add_row = [&](const uint4& qa, const uint4& qz) {
    float va[8];
    bf16x8(qa, va);
    if constexpr (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s1[j] += va[j];
        s2[j] = fmaf(va[j], va[j], s2[j]);
      }
    } else {
      float vz[8];
      bf16x8(qz, vz);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        s1[j] += va[j];
        s2[j] = fmaf(va[j], (vz[j] - mu[j]) * rs[j], s2[j]);
      }
    }
  };
  if (rl < rpp) {
    const long long col = 8 * c8;
    constexpr int U = MODE == 0 ? 2 * kBnUnroll : kBnUnroll;   // 16 x 16 B loads in flight per thread
    int r = r0 + rl;
    for (; r + (U - 1) * rpp < r1; r += U * rpp) {
      uint4 qa[U], qz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long off = static_cast<long long>(r + u * rpp) * C + col;
        qa[u] = __ldg(reinterpret_cast<const uint4*>(a + off));
        if constexpr (MODE == 1) qz[u] = __ldg(reinterpret_cast<const uint4*>(z + off));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) add_row(qa[u], qz[u]);
    }
    for (; r < r1; r += rpp) {
      const long long off = static_cast<long long>(r) * C + col;
      const uint4 qa = __ldg(reinterpret_cast<const uint4*>(a + off));
      uint4 qz = qa;
      if constexpr (MODE == 1) qz = __ldg(reinterpret_cast<const uint4*>(z + off));
      add_row(qa, qz);
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
    csum[c] = t1;
    csum[C + c] = t2;
  }
  cluster_sync();
  // each rank adds one eighth of the 2C sums over the cluster's 8 ranks (rank order) into the fp64 partial
  const uint32_t rank = cluster_ctarank();
  const int gc = blockIdx.x / kBnCluster;
  const int per_rank = 2 * C / kBnCluster;
  const uint32_t base = smem_u32(csum);
  for (int i = threadIdx.x; i < per_rank; i += blockDim.x) {
    const int v = static_cast<int>(rank) * per_rank + i;
    float w[kBnCluster];
#pragma unroll
    for (int k = 0; k < kBnCluster; ++k) w[k] = ld_dsmem_f32_nv(mapa(base + 4u * v, k));
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < kBnCluster; ++k) t += static_cast<double>(w[k]);
    partial[static_cast<long long>(gc) * 2 * C + v] = t;
  }
  cluster_sync();                            // every rank's csum stays alive until the cluster has read it
  if (ticket == nullptr) return;
  __threadfence();
  cluster_sync();                            // the cluster's partial is written before it is counted
  if (rank == 0 && threadIdx.x == 0) {
    const unsigned t = atomicAdd(ticket, 1u);
    const int last = t == static_cast<unsigned>(gridDim.x / kBnCluster - 1);
    if (last) *ticket = 0u;                  // every cluster has arrived: leave the counter zeroed
#pragma unroll
    for (int k = 0; k < kBnCluster; ++k) st_dsmem_s32(mapa(smem_u32(&s_last), k), last);
  }
  cluster_sync();
  if (!s_last) return;
  __threadfence();
  // the last cluster finishes: each rank one eighth of the channels
  const int per = C / kBnCluster;
  bn_finish<MODE>(partial, gridDim.x / kBnCluster, C, M, eps, out1, out2, reinterpret_cast<double*>(red),
                  static_cast<int>(rank) * per, static_cast<int>(rank + 1) * per);
}

// Without a ticket counter: the finishing pass as its own launch.
template <int MODE>
__global__ void __launch_bounds__(kBnThreads) bn_finish_kernel(const double* __restrict__ partial, int Gc, int C,
                                                               int M, float eps, float* __restrict__ out1,
                                                               float* __restrict__ out2) {
  griddep_wait();
  __shared__ double scratch[2 * kBnThreads];
  bn_finish<MODE>(partial, Gc, C, M, eps, out1, out2, scratch, 0, C);
}

// y = act(gamma (z - mean) rstd + beta [+ res])
__global__ void __launch_bounds__(kBnThreads) bn_apply_kernel(const __nv_bfloat16* __restrict__ z, int M, int C,
                                                              int rpb, const float* __restrict__ mean,
                                                              const float* __restrict__ rstd,
                                                              const float* __restrict__ gamma,
                                                              const float* __restrict__ beta,
                                                              const __nv_bfloat16* __restrict__ res, int relu,
                                                              __nv_bfloat16* __restrict__ y) {
  griddep_wait();
  const int cv = C / 8;
  const int rpp = kBnThreads / cv;
  const int rl = threadIdx.x / cv, c8 = threadIdx.x % cv;
  if (rl >= rpp) return;
  float sc[8], sh[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 8 * c8 + j;
    sc[j] = __ldg(gamma + c) * __ldg(rstd + c);
    sh[j] = __ldg(beta + c) - __ldg(mean + c) * sc[j];
  }
  const int blk = gridDim.x - 1 - blockIdx.x;
  const int r0 = blk * rpb;
  const int r1 = r0 + rpb < M ? r0 + rpb : M;
  const long long col = 8 * c8;
  auto row = [&](const uint4& qz, const uint4& qr, long long off) {
    float v[8], w[8];
    bf16x8(qz, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fmaf(v[j], sc[j], sh[j]);
    if (res != nullptr) {
      bf16x8(qr, w);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += w[j];
    }
    if (relu) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j], 0.f);
    }
    *reinterpret_cast<uint4*>(y + off) = pack8(v);
  };
  int r = r1 - 1 - rl;
  for (; r - (kBnUnroll - 1) * rpp >= r0; r -= kBnUnroll * rpp) {
    uint4 qz[kBnUnroll], qr[kBnUnroll];
#pragma unroll
    for (int u = 0; u < kBnUnroll; ++u) {
      const long long off = static_cast<long long>(r - u * rpp) * C + col;
      qz[u] = __ldg(reinterpret_cast<const uint4*>(z + off));
      if (res != nullptr) qr[u] = __ldg(reinterpret_cast<const uint4*>(res + off));
    }
#pragma unroll
    for (int u = 0; u < kBnUnroll; ++u) row(qz[u], qr[u], static_cast<long long>(r - u * rpp) * C + col);
  }
  for (; r >= r0; r -= rpp) {
    const long long off = static_cast<long long>(r) * C + col;
    const uint4 qz = __ldg(reinterpret_cast<const uint4*>(z + off));
    uint4 qr = qz;
    if (res != nullptr) qr = __ldg(reinterpret_cast<const uint4*>(res + off));
    row(qz, qr, off);
  }
}

// dz = gamma rstd (g - dbeta / M - xhat dgamma / M)
__global__ void __launch_bounds__(kBnThreads) bn_bwd_apply_kernel(const __nv_bfloat16* __restrict__ g,
                                                                  const __nv_bfloat16* __restrict__ z, int M, int C,
                                                                  int rpb, const float* __restrict__ mean,
                                                                  const float* __restrict__ rstd,
                                                                  const float* __restrict__ gamma,
                                                                  const float* __restrict__ dbeta,
                                                                  const float* __restrict__ dgamma,
                                                                  __nv_bfloat16* __restrict__ dz) {
  griddep_wait();
  const int cv = C / 8;
  const int rpp = kBnThreads / cv;
  const int rl = threadIdx.x / cv, c8 = threadIdx.x % cv;
  if (rl >= rpp) return;
  const float inv_m = 1.0f / static_cast<float>(M);
  // dz = k g - k dbeta / M - k rstd dgamma / M (z - mean), k = gamma rstd
  float k[8], kb[8], kr[8], mu[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 8 * c8 + j;
    const float rs = __ldg(rstd + c);
    mu[j] = __ldg(mean + c);
    k[j] = __ldg(gamma + c) * rs;
    kb[j] = k[j] * (__ldg(dbeta + c) * inv_m);
    kr[j] = k[j] * rs * (__ldg(dgamma + c) * inv_m);
  }
  const int blk = gridDim.x - 1 - blockIdx.x;
  const int r0 = blk * rpb;
  const int r1 = r0 + rpb < M ? r0 + rpb : M;
  const long long col = 8 * c8;
  auto row = [&](const uint4& qg, const uint4& qz, long long off) {
    float vg[8], vz[8], v[8];
    bf16x8(qg, vg);
    bf16x8(qz, vz);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fmaf(k[j], vg[j], -kb[j]) - kr[j] * (vz[j] - mu[j]);
    *reinterpret_cast<uint4*>(dz + off) = pack8(v);
  };
  int r = r1 - 1 - rl;
  for (; r - (kBnUnroll - 1) * rpp >= r0; r -= kBnUnroll * rpp) {
    uint4 qg[kBnUnroll], qz[kBnUnroll];
#pragma unroll
    for (int u = 0; u < kBnUnroll; ++u) {
      const long long off = static_cast<long long>(r - u * rpp) * C + col;
      qg[u] = __ldg(reinterpret_cast<const uint4*>(g + off));
      qz[u] = __ldg(reinterpret_cast<const uint4*>(z + off));
    }
#pragma unroll
    for (int u = 0; u < kBnUnroll; ++u) row(qg[u], qz[u], static_cast<long long>(r - u * rpp) * C + col);
  }
  for (; r >= r0; r -= rpp) {
    const long long off = static_cast<long long>(r) * C + col;
    row(__ldg(reinterpret_cast<const uint4*>(g + off)), __ldg(reinterpret_cast<const uint4*>(z + off)), off);
  }
}

template <int MODE>
cudaError_t launch_reduce(const __nv_bfloat16* a, const __nv_bfloat16* z, int M, int C, const float* mean,
                          const float* rstd, float* partial, unsigned* ticket, float eps, float* out1, float* out2,
                          int sms, cudaStream_t stream) {
  // one wave: no more clusters than fit on the GPU at once (8-CTA clusters
  // pack per GPC, so 2 CTAs / SM x 148 SMs is NOT 37 co-resident clusters)
  static const int wave = [] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kBnCluster);
    cfg.blockDim = dim3(kBnThreads);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = kBnCluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, bn_reduce_kernel<MODE>, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = 0;
    }
    return n;
  }();
  int G = bn_stats_blocks(M, C, sms);
  if (wave > 0 && G > wave * kBnCluster) G = wave * kBnCluster;
  const int rpb = (M + G - 1) / G;
  double* part = reinterpret_cast<double*>(partial);
  cudaError_t e = launch_pdl(bn_reduce_kernel<MODE>, dim3(G), dim3(kBnThreads), 0, stream, kBnCluster, a, z, M, C,
                             rpb, mean, rstd, part, ticket, eps, out1, out2);
  if (e != cudaSuccess || ticket != nullptr) return e;
  return launch_pdl(bn_finish_kernel<MODE>, dim3(1), dim3(kBnThreads), 0, stream, 1,
                    static_cast<const double*>(part), G / kBnCluster, C, M, eps, out1, out2);
}

}  // namespace

long long bn_partial_floats(int M, int C, int sms) {
  return 2LL * (bn_stats_blocks(M, C, sms) / kBnCluster) * 2 * C;   // fp64 [clusters][2][C]
}

cudaError_t launch_bn_stats(const __nv_bfloat16* z, int M, int C, float* partial, unsigned* ticket, float* mean,
                            float* rstd, float eps, int sms, cudaStream_t stream) {
  return launch_reduce<0>(z, z, M, C, nullptr, nullptr, partial, ticket, eps, mean, rstd, sms, stream);
}

cudaError_t launch_bn_bwd_reduce(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                 const float* rstd, float* partial, unsigned* ticket, float* dbeta, float* dgamma,
                                 int sms, cudaStream_t stream) {
  return launch_reduce<1>(g, z, M, C, mean, rstd, partial, ticket, 0.f, dbeta, dgamma, sms, stream);
}

cudaError_t launch_bn_apply(const __nv_bfloat16* z, int M, int C, const float* mean, const float* rstd,
                            const float* gamma, const float* beta, const __nv_bfloat16* res, bool relu,
                            __nv_bfloat16* y, int sms, cudaStream_t stream) {
  const int G = bn_apply_blocks(M, C, sms);
  return launch_pdl(bn_apply_kernel, dim3(G), dim3(kBnThreads), 0, stream, 1, z, M, C, (M + G - 1) / G, mean, rstd,
                    gamma, beta, res, relu ? 1 : 0, y);
}

cudaError_t launch_bn_bwd_apply(const __nv_bfloat16* g, const __nv_bfloat16* z, int M, int C, const float* mean,
                                const float* rstd, const float* gamma, const float* dbeta, const float* dgamma,
                                __nv_bfloat16* dz, int sms, cudaStream_t stream) {
  const int G = bn_apply_blocks(M, C, sms);
  return launch_pdl(bn_bwd_apply_kernel, dim3(G), dim3(kBnThreads), 0, stream, 1, g, z, M, C, (M + G - 1) / G,
                    mean, rstd, gamma, dbeta, dgamma, dz);
}

}  // namespace edl
