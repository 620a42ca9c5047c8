// exchange.cu — the student's data-parallel gradient exchange fused with SGD,
// over NVSwitch multicast (NVLS) instead of a ring.
//
// Reference (edl/student_node.py:738-745): every rank ring-all-reduces its
// flat gradient to the element-wise mean (edl/allreduce.py:77-120) and then
// applies p <- p - eta * g (edl/nnkit.py:312-322) on its own replica. Here one kernel
// per rank does both for a 1/world shard of the parameters:
//
//   g_sum = multimem.ld_reduce.add(grad[shard])     the switch sums all ranks' copies
//   p     = p[shard] - (eta / world) * g_sum         fp32 master, this rank's copy
//   multimem.st(param[shard], p); multimem.st(param_bf16[shard], bf16(p))
//                                                    written into EVERY rank's replica
//
// so each GPU moves 4n/world bytes in and 6n/world bytes out over NVLink and
// the separate all-reduce + SGD launches (and their HBM passes) disappear.
// Every rank ends with bit-identical parameters: each shard is updated once,
// by its owner, from one switch-side sum.
//
// Ordering: (0) a per-block start barrier over the ranks' signal pads. Block b
// of rank r arrives only after griddepcontrol.wait, so rank r's gradient is
// complete, and no rank reads a peer's gradient before then. (1) the shard
// loop. (2) the last block of each rank (grid-wide counter) signals every
// peer after a system-scope fence and waits for all of them, so when the
// kernel completes on any rank, every replica holds the new parameters.
// Barrier values are the per-call epoch (strictly increasing, the same on all
// ranks), so pads never need resetting.
#include "../../include/edl_b200.h"
#include "internal.h"
#include "sm100.cuh"

namespace edl {

namespace {

constexpr int kXThreads = 512;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ void wait_ge(const uint32_t* p, uint32_t epoch) {
  uint32_t spins = 0;
  // signed distance: epochs wrap after 2^32 calls
  while (static_cast<int32_t>(ld_acquire_sys(p) - epoch) < 0) {
    if (++spins > (1u << 26)) __trap();   // a rank that never arrives: fail loudly
    __nanosleep(64);
  }
}

__device__ __forceinline__ float4 mm_ld_reduce_add(const float* mc) {
  float4 v;
  asm volatile("multimem.ld_reduce.weak.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(mc)
               : "memory");
  return v;
}
__device__ __forceinline__ void mm_st_f32x4(float* mc, float4 v) {
  asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mm_st_bf16x8(uint32_t* mc, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("multimem.st.weak.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(a), "r"(b), "r"(c),
               "r"(d)
               : "memory");
}

struct XArgs {
  float* mc_grad;
  float* mc_param;
  uint32_t* mc_bf16;          // bf16 pairs
  const float* param;         // this rank's replica (unicast)
  uint32_t* const* pads;      // [world] signal pads (device pointers, own included)
  uint32_t* counter;          // grid-wide arrival counter (device, starts 0)
  long long groups;           // n / 8
  float scale;                // eta / world
  uint32_t epoch;
  int rank, world;
};

__global__ void __launch_bounds__(kXThreads) nvls_allreduce_sgd_kernel(XArgs a) {
  griddep_wait();   // this rank's gradient (previous kernels on the stream) is complete
  const int b = static_cast<int>(blockIdx.x);
  const int t = static_cast<int>(threadIdx.x);
  uint32_t* own = a.pads[a.rank];
  // (0) start barrier, one pad row per block (row 0 is the end barrier)
  if (t < a.world) {
    st_release_sys(a.pads[t] + static_cast<size_t>(1 + b) * a.world + a.rank, a.epoch);
    wait_ge(own + static_cast<size_t>(1 + b) * a.world + t, a.epoch);
  }
  __syncthreads();

  // (1) this rank's shard, 8 elements per item, kUnroll items per thread in
  // flight: the grid is small (it must fit beside the teacher's persistent
  // GEMMs), so each thread keeps several switch round trips outstanding
  const long long per = (a.groups + a.world - 1) / a.world;
  const long long lo = per * a.rank;
  const long long hi = lo + per < a.groups ? lo + per : a.groups;
  const long long stride = static_cast<long long>(gridDim.x) * kXThreads;
  constexpr int kUnroll = 4;
  auto update = [&](long long g, float4 g0, float4 g1) {
    float4 p0 = __ldg(reinterpret_cast<const float4*>(a.param + 8 * g));
    float4 p1 = __ldg(reinterpret_cast<const float4*>(a.param + 8 * g + 4));
    p0.x -= a.scale * g0.x; p0.y -= a.scale * g0.y; p0.z -= a.scale * g0.z; p0.w -= a.scale * g0.w;
    p1.x -= a.scale * g1.x; p1.y -= a.scale * g1.y; p1.z -= a.scale * g1.z; p1.w -= a.scale * g1.w;
    mm_st_f32x4(a.mc_param + 8 * g, p0);
    mm_st_f32x4(a.mc_param + 8 * g + 4, p1);
    mm_st_bf16x8(a.mc_bf16 + 4 * g, pack_bf16x2(p0.x, p0.y), pack_bf16x2(p0.z, p0.w), pack_bf16x2(p1.x, p1.y),
                 pack_bf16x2(p1.z, p1.w));
  };
  long long g = lo + static_cast<long long>(b) * kXThreads + t;
  for (; g + (kUnroll - 1) * stride < hi; g += kUnroll * stride) {
    float4 s[2 * kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      s[2 * u] = mm_ld_reduce_add(a.mc_grad + 8 * (g + u * stride));
      s[2 * u + 1] = mm_ld_reduce_add(a.mc_grad + 8 * (g + u * stride) + 4);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) update(g + u * stride, s[2 * u], s[2 * u + 1]);
  }
  for (; g < hi; g += stride) update(g, mm_ld_reduce_add(a.mc_grad + 8 * g), mm_ld_reduce_add(a.mc_grad + 8 * g + 4));

  // (2) end barrier: the last block of this rank publishes "all my stores are
  // done" to every peer and waits until every rank has done the same
  fence_sys();
  __syncthreads();
  __shared__ int last;
  if (t == 0) {
    const unsigned prev = atomicAdd(a.counter, 1u);
    last = (prev == gridDim.x - 1);
    if (last) atomicExch(a.counter, 0u);   // next launch on this stream starts from 0
  }
  __syncthreads();
  if (last && t < a.world) {
    fence_sys();
    st_release_sys(a.pads[t] + a.rank, a.epoch);
    wait_ge(own + t, a.epoch);
  }
}

}  // namespace

namespace {
// Fallbacks for edl_stream_wait_geq / edl_stream_write_u32 when the driver
// has no stream memory operations: one thread spins / stores at system scope.
__global__ void flag_wait_kernel(const uint32_t* addr, uint32_t value) {
  griddep_wait();
  wait_ge(addr, value);
}
__global__ void flag_write_kernel(uint32_t* addr, uint32_t value) {
  griddep_wait();
  fence_sys();
  st_release_sys(addr, value);
}
}  // namespace

cudaError_t launch_flag_wait(const uint32_t* addr, uint32_t value, cudaStream_t stream) {
  return launch_pdl(flag_wait_kernel, dim3(1), dim3(1), 0, stream, 1, addr, value);
}
cudaError_t launch_flag_write(uint32_t* addr, uint32_t value, cudaStream_t stream) {
  return launch_pdl(flag_write_kernel, dim3(1), dim3(1), 0, stream, 1, addr, value);
}

int nvls_max_blocks(int world, long long pad_bytes) {
  const long long slots = pad_bytes / 4;
  const long long rows = slots / world;   // row 0 + one per block
  return rows - 1 > 0 ? static_cast<int>(rows - 1) : 0;
}

cudaError_t launch_nvls_allreduce_sgd(float* mc_grad, float* mc_param, void* mc_bf16, const float* param,
                                      uint32_t* const* pads, uint32_t* counter, long long n, float scale,
                                      uint32_t epoch, int rank, int world, int blocks, cudaStream_t stream) {
  XArgs a{mc_grad, mc_param, reinterpret_cast<uint32_t*>(mc_bf16), param, pads, counter, n / 8, scale, epoch,
          rank, world};
  return launch_pdl(nvls_allreduce_sgd_kernel, dim3(blocks), dim3(kXThreads), 0, stream, 1, a);
}

}  // namespace edl
