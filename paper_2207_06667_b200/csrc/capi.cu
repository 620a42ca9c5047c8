// capi.cu — the C-ABI boundary (include/edl_b200.h). Plain pointers, sizes and
// a cudaStream_t; the caller owns all device memory and nothing here allocates
// on the step path. TMA tensor maps are encoded on first use and cached by
// (pointer, shape, box), so steady-state calls are a cache lookup + launch.
#include "../../include/edl_b200.h"
#include "internal.h"

#include <cudaTypedefs.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

using namespace edl;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(EDL_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  long long rows, cols, ld;
  int box0, box1, kind;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box0 == o.box0 &&
           box1 == o.box1 && kind == o.kind;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    h ^= std::hash<long long>()(k.rows * 1000003LL + k.cols) + 0x9e3779b9 + (h << 6) + (h >> 2);
    h ^= std::hash<long long>()(k.ld * 131 + k.box0 * 7 + k.box1 * 3 + k.kind) + 0x9e3779b9 + (h << 6) + (h >> 2);
    return h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2-D row-major matrix [rows][cols] with leading dimension ld (elements),
// box {box0 along cols, box1 along rows}, zero OOB fill. kind 0: bf16 GEMM
// operand, 128-byte swizzle; 1: fp32 TMA-store output, 128-byte swizzle;
// 2: bf16 TMA-store output, 64-byte swizzle (the epilogue's staging layouts).
enum MapKind { kOperandBf16 = 0, kOutF32 = 1, kOutBf16 = 2 };
int tensor_map_ex(const void* ptr, long long rows, long long cols, long long ld, int box0, int box1, int kind,
                  CUtensorMap* out) {
  MapKey key{ptr, rows, cols, ld, box0, box1, kind};
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) { *out = it->second; return 0; }
  }
  auto fn = encode_fn();
  if (!fn) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const long long esize = kind == kOutF32 ? 4 : 2;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * esize) % 16)
    return fail(EDL_ERR_SHAPE, "TMA operand needs 16-byte aligned base and row pitch (ld=%lld)", ld);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * esize)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = fn(&m, kind == kOutF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  kind == kOutBf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  {
    std::lock_guard<std::mutex> g(g_map_mu);
    if (g_maps.size() > 4096) g_maps.clear();
    g_maps.emplace(key, m);
  }
  *out = m;
  return 0;
}

// 4-D NHWC im2col map for implicit-GEMM convolution: dims {C, W, H, N},
// bounding box corners {-pad, pad - (S-1)} per spatial dim (W, H order), the
// conv stride as the traversal stride, `pixels` output pixels x 64 channels
// per load, 128-byte swizzle (the same smem layout as a K-major 2-D operand
// box). Drivers up to 13.1 mis-handle im2col maps of tensors under 128 KB
// unless descriptor bit 21 of word 1 is cleared (the workaround CUTLASS applies).
int conv_map(const void* x, int N, int H, int W, int C, int R, int S, int stride, int pad, int pixels,
             CUtensorMap* out) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  static int drv = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(p);
    cudaDriverGetVersion(&drv);
  });
  if (!fn) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || C % 64)
    return fail(EDL_ERR_SHAPE, "conv: x must be 16-byte aligned with C %% 64 == 0 (C=%d)", C);
  const int lo = -pad, hi_w = pad - (S - 1), hi_h = pad - (R - 1);
  if (lo < -128 || hi_w < -128 || hi_h < -128 || pad > 127) return fail(EDL_ERR_SHAPE, "conv: padding out of range");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W) * C * 2,
                           static_cast<cuuint64_t>(H) * W * C * 2};
  int lower[2] = {lo, lo};
  int upper[2] = {hi_w, hi_h};
  cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(stride), static_cast<cuuint32_t>(stride), 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower, upper, 64,
                  static_cast<cuuint32_t>(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeIm2col failed (%d)", static_cast<int>(r));
  if (drv <= 13010 && static_cast<long long>(N) * H * W * C * 2 < 131072)
    reinterpret_cast<uint64_t*>(out)[1] &= ~(1ull << 21);
  return 0;
}

// 5-D tiled map of an NHWC bf16 tensor with C = 64 for the halo conv
// (halo.cu): dims {8 channels, W, H, N, C/8 chunks}, the chunk dimension at a
// 16-byte stride, so a box {8, W + 2, rows, 1, 8} lands in shared memory as
// [chunk][row][pixel][8 channels] — the no-swizzle K-major core-matrix layout.
// Boxes starting at w = -1 / h = -1 read the TMA's zero fill.
int halo_map(const void* x, int N, int H, int W, int C, int box_rows, CUtensorMap* out) {
  auto fn = encode_fn();
  if (!fn) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || C != 64 || W + 2 > 256 || box_rows > 256)
    return fail(EDL_ERR_SHAPE, "halo map: C must be 64 and W + 2 <= 256 (C=%d W=%d)", C, W);
  cuuint64_t dims[5] = {8, static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(N),
                        static_cast<cuuint64_t>(C / 8)};
  cuuint64_t strides[4] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W) * C * 2,
                           static_cast<cuuint64_t>(H) * W * C * 2, 16};
  cuuint32_t box[5] = {8, static_cast<cuuint32_t>(W + 2), static_cast<cuuint32_t>(box_rows), 1,
                       static_cast<cuuint32_t>(C / 8)};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(x), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EDL_ERR_CUDA, "halo map: cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

// 4-D tiled map of an NHWC bf16 tensor with C = 64: box {64, box_w, rows, 1},
// SWIZZLE_128B — pixel rows of 128 B in the K-major operand layout.
int halo_map_sw128(const void* x, int N, int H, int W, int C, int box_w, int box_rows, CUtensorMap* out) {
  auto fn = encode_fn();
  if (!fn) return fail(EDL_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(x) & 15) || C != 64 || W + 2 > 256 || box_rows > 256)
    return fail(EDL_ERR_SHAPE, "halo map: C must be 64 and W + 2 <= 256 (C=%d W=%d)", C, W);
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C) * 2, static_cast<cuuint64_t>(W) * C * 2,
                           static_cast<cuuint64_t>(H) * W * C * 2};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(C), static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EDL_ERR_CUDA, "halo map: cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return 0;
}

int tensor_map(const void* ptr, long long rows, long long cols, long long ld, int box0, int box1,
               CUtensorMap* out) {
  return tensor_map_ex(ptr, rows, cols, ld, box0, box1, kOperandBf16, out);
}
// The TMA-store map of a GEMM output (32 x 32 boxes, one per epilogue warp chunk).
int tensor_map_out(const void* ptr, long long rows, long long cols, long long ld, bool f32, CUtensorMap* out) {
  return tensor_map_ex(ptr, rows, cols, ld, 32, 32, f32 ? kOutF32 : kOutBf16, out);
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

// Pick the N tile for `cap` CTAs: fewest waves x tile time (one tile's time
// ~ bn + 48 fixed cost), widest tile on ties (best operand reuse).
int pick_bn_cap(int M, int N, int cap) {
  static const int forced = [] {
    const char* v = getenv("EDL_FORCE_BN");   // tuning runs only: 64 / 128 / 256
    return v ? atoi(v) : 0;
  }();
  if (forced == 64 || forced == 128 || forced == 256) return forced;
  int best = 256;
  long long best_cost = -1;
  for (int bn : {256, 128, 64}) {
    if (bn > 64 && N <= bn / 2) continue;
    const long long tiles = static_cast<long long>((M + 127) / 128) * ((N + bn - 1) / bn);
    const long long cost = ((tiles + cap - 1) / cap) * (bn + 48);
    if (best_cost < 0 || cost < best_cost) { best_cost = cost; best = bn; }
  }
  return best;
}
int pick_bn(int M, int N) { return pick_bn_cap(M, N, num_sms()); }

// CTA-pair 256 x 256 tiles (cta_group::2) do the same per-SM MMA work per
// tile as a single-CTA 128 x 256 tile with 2/3 of the L2 -> SM operand bytes
// (measured on B200: teacher layers 437 -> 380 us, student layer 1 49.6 ->
// 42.5 us), so they win whenever their wave count is no worse. Returns 0 to
// use the single-CTA kernel. EDL_GEMM_PAIR=0 forces single-CTA (A/B runs).
bool pair_mode_enabled() {
  static const int mode = [] {
    const char* v = getenv("EDL_GEMM_PAIR");
    return v ? atoi(v) : 1;
  }();
  return mode != 0;
}

int pick_pair_bn(int M, int N, int cap) {
  if (!pair_mode_enabled() || cap < 2 || N <= 128) return 0;
  const int bn = pick_bn_cap(M, N, cap);
  const long long single = ((static_cast<long long>((M + 127) / 128) * ((N + bn - 1) / bn) + cap - 1) / cap) *
                           (bn + 48);
  const long long pair_tiles = static_cast<long long>((M + 255) / 256) * ((N + 255) / 256);
  const long long pair_waves = (pair_tiles + cap / 2 - 1) / (cap / 2);
  const long long pair = pair_waves * (256 + 48);
  // a single wave gains little operand traffic and pays the cluster's
  // setup (~0.5 us measured on the student's 1-wave layers): ties go single
  return (pair < single || (pair == single && pair_waves >= 2)) ? 256 : 0;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Weight-gradient plan for tall reductions (conv layers: dW[N][K] reduced over
// M = B*H*W pixels, as few as 5 output tiles). Split-K gives the SMs work:
// split s reduces k-blocks [s*kps, (s+1)*kps) into its own fp32 partial, and a
// fixed-order reduce kernel sums them (deterministic). With N < 128 output
// rows the operands swap (GEMM M = K, N = N) so the 128-row MMA is not half
// empty; the reduce then transposes back to [N][K]. Cost model (us): waves x
// max(k-blocks per item x 0.069 x bn/64 [one 128 x 64 x 64 k-block at the
// per-SM tensor peak], the item's fp32 epilogue at ~50 GB/s per SM) + 0.5 per
// wave, plus the reduce: the partials' HBM round trip at 5 TB/s, its chain of
// ks loads per thread (8 in flight, ~0.35 us per round) and ~2 us of launch.
struct WgradPlan {
  bool swap = false;
  int bn = 64;
  int ksplit = 1;
  int gm = 0, gn = 0;
  bool reduce() const { return swap || ksplit > 1; }
  long long partial_floats() const { return reduce() ? static_cast<long long>(ksplit) * gm * gn : 0; }
};

WgradPlan plan_wgrad(int M, int N, int K, int cap, long long max_partial_floats) {
  WgradPlan p;
  p.swap = N < 128 && K > N;
  p.gm = p.swap ? K : N;
  p.gn = p.swap ? N : K;
  if (p.swap && static_cast<long long>(p.gm) * p.gn > max_partial_floats) {
    p.swap = false;
    p.gm = N;
    p.gn = K;
  }
  p.bn = p.gn <= 64 ? 64 : (p.gn <= 128 ? 128 : 256);
  const long long tiles = static_cast<long long>((p.gm + 127) / 128) * ((p.gn + p.bn - 1) / p.bn);
  const int nk = (M + 63) / 64;
  const double t_kb = 0.069 * p.bn / 64.0;
  const double t_epi = 128.0 * p.bn * 4 / 5e4;
  const double gmn = static_cast<double>(p.gm) * p.gn;
  double best = -1.0;
  const int kmax = nk < 1024 ? nk : 1024;
  for (int ks = 1; ks <= kmax; ++ks) {
    const int kps = (nk + ks - 1) / ks;
    if ((nk + kps - 1) / kps != ks) continue;          // only splits with no empty tail
    if (ks > 1 && static_cast<double>(ks) * gmn > static_cast<double>(max_partial_floats)) break;
    const long long waves = (tiles * ks + cap - 1) / cap;
    const double item = kps * t_kb > t_epi ? kps * t_kb : t_epi;
    double cost = waves * (item + 0.5);
    // the reduce: partials' HBM round trip + its per-thread chain of ks loads
    // (8 in flight, ~0.35 us L2 latency each round) + launch
    if (ks > 1 || p.swap) cost += 2.0 * ks * gmn * 4 / 5e6 + 0.35 * ((ks + 7) / 8) + 2.0;
    if (best < 0 || cost < best) { best = cost; p.ksplit = ks; }
  }
  return p;
}

long long wgrad_workspace_floats(int M, int N, int K, int cap) {
  const WgradPlan p = plan_wgrad(M, N, K, cap, 1LL << 40);
  long long w = p.partial_floats();
  const long long cs = colsum_tall_ok(N) ? static_cast<long long>(colsum_tall_blocks(M, cap)) * N
                                         : colsum_workspace_floats(1, &M, &N);
  return w > cs ? w : cs;
}

std::mutex g_attr_mu;
std::unordered_map<const void*, unsigned long long> g_attr_done;  // kernel -> device bitmask

}  // namespace

cudaError_t edl::ensure_kernel_attrs(const void* kern, int smem_bytes, bool nonportable_cluster) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> g(g_attr_mu);
  unsigned long long& mask = g_attr_done[kern];
  if (mask & bit) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (smem_bytes > 48 * 1024)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e == cudaSuccess && nonportable_cluster)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) mask |= bit;
  return e;
}

namespace {

// Per-(device, stream) tile-scheduler counters for the persistent GEMM
// ({next tile, CTAs done}, reset by each launch's last CTA). They come from
// a static device pool (no allocation on any call, so a stream's first GEMM
// may be inside graph capture); a stream keeps its pair for the process
// lifetime. Launches on one stream are ordered (PDL waits); launches on
// different streams never share a pair. Past kSchedSlots streams per device
// the GEMMs fall back to the static tile schedule.
constexpr int kSchedSlots = 256;
__device__ unsigned g_sched_pool[2 * kSchedSlots];
std::mutex g_sched_mu;
std::unordered_map<std::string, unsigned*> g_sched;
std::unordered_map<int, int> g_sched_used;

// Per-stream cap on the persistent GEMM grid (edl_set_stream_max_ctas): a
// teacher stream capped below the SM count leaves SMs free, so the student's
// NCCL all-reduce kernels are not blocked behind teacher CTAs that hold
// every SM for a whole (hundreds of microseconds) GEMM.
std::mutex g_cap_mu;
std::unordered_map<cudaStream_t, int> g_cap;

int grid_cap(cudaStream_t s) {
  const int n = num_sms();
  std::lock_guard<std::mutex> g(g_cap_mu);
  auto it = g_cap.find(s);
  return (it == g_cap.end() || it->second <= 0 || it->second > n) ? n : it->second;
}

unsigned* stream_sched(cudaStream_t s) {
  static const bool disabled = [] {
    const char* v = getenv("EDL_STATIC_SCHED");
    return v && v[0] == '1';
  }();
  if (disabled) return nullptr;   // A/B switch: static tile schedule
  int dev = 0;
  cudaGetDevice(&dev);
  char key[64];
  snprintf(key, sizeof(key), "%d:%p", dev, static_cast<void*>(s));
  std::lock_guard<std::mutex> g(g_sched_mu);
  auto it = g_sched.find(key);
  if (it != g_sched.end()) return it->second;
  int& used = g_sched_used[dev];
  if (used >= kSchedSlots) return nullptr;   // static schedule
  void* base = nullptr;
  if (cudaGetSymbolAddress(&base, g_sched_pool) != cudaSuccess) return nullptr;
  unsigned* p = static_cast<unsigned*>(base) + 2 * used++;
  g_sched.emplace(key, p);
  return p;
}

// Per-(device, stream) arrival tickets for the one-launch BatchNorm
// reductions (bn.cu): zero at rest, reset by each launch's last cluster.
__device__ unsigned g_ticket_pool[kSchedSlots];
std::mutex g_ticket_mu;
std::unordered_map<std::string, unsigned*> g_ticket;
std::unordered_map<int, int> g_ticket_used;

unsigned* stream_ticket(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  char key[64];
  snprintf(key, sizeof(key), "%d:%p", dev, static_cast<void*>(s));
  std::lock_guard<std::mutex> g(g_ticket_mu);
  auto it = g_ticket.find(key);
  if (it != g_ticket.end()) return it->second;
  int& used = g_ticket_used[dev];
  if (used >= kSchedSlots) return nullptr;   // a separate finishing launch
  void* base = nullptr;
  if (cudaGetSymbolAddress(&base, g_ticket_pool) != cudaSuccess) return nullptr;
  unsigned* p = static_cast<unsigned*>(base) + used++;
  g_ticket.emplace(key, p);
  return p;
}

}  // namespace

extern "C" {

int edl_version(void) { return EDL_B200_ABI_VERSION; }

const char* edl_last_error(void) { return g_err.c_str(); }

int edl_device_sms(void) { return num_sms(); }

int edl_set_tanh_mode(int mode) {
  if (mode != 0 && mode != 1) return fail(EDL_ERR_PARAM, "set_tanh_mode: mode must be 0 or 1");
  const cudaError_t e = edl::set_tanh_mode(mode);
  return e == cudaSuccess ? 0 : cuda_fail(e, "set_tanh_mode");
}

int edl_set_stream_max_ctas(void* stream, int max_ctas) {
  std::lock_guard<std::mutex> g(g_cap_mu);
  if (max_ctas <= 0) g_cap.erase(as_stream(stream));
  else g_cap[as_stream(stream)] = max_ctas;
  return 0;
}

// bf16 conv-layer epilogues on 256-wide pair tiles store (and read their
// residual) in 64 x 32 SWIZZLE_128B boxes: 128-byte box rows, half the TMA
// row walk of 32 x 32 boxes (profiles/README.md finding 41). EDL_W128=0
// keeps the 32 x 32 path for A/B runs.
static bool w128_enabled() {
  static const bool on = [] {
    const char* v = getenv("EDL_W128");
    return !(v && v[0] == '0');
  }();
  return on;
}

// the MLP layers' tanh / dtanh epilogues too (EDL_W128_TANH=0: not)
static bool w128_tanh() {
  static const bool on = [] {
    const char* v = getenv("EDL_W128_TANH");
    return !(v && v[0] == '0');
  }();
  return on;
}

int edl_linear_fwd(const void* X, long long ldx, const void* W, long long ldw, const float* bias,
                   void* Y, long long ldy, int M, int N, int K, int act, void* stream) {
  if (M < 1 || N < 1 || K < 1 || ldx < K || ldw < K || ldy < N)
    return fail(EDL_ERR_SHAPE, "linear_fwd: bad shape M=%d N=%d K=%d", M, N, K);
  if (act != EDL_ACT_TANH && act != EDL_ACT_NONE && act != EDL_ACT_RELU && act != EDL_ACT_IDENT)
    return fail(EDL_ERR_SHAPE, "linear_fwd: bad act %d", act);
  const GemmKind kind = act == EDL_ACT_TANH    ? GemmKind::FwdTanh
                        : act == EDL_ACT_RELU  ? GemmKind::FwdRelu
                        : act == EDL_ACT_IDENT ? GemmKind::FwdIdentBf16
                                               : GemmKind::FwdLinear;
  const int cap = grid_cap(as_stream(stream));
  CUtensorMap ta, tb;
  int rc;
  if ((rc = tensor_map(X, M, K, ldx, 64, 128, &ta))) return rc;
  EpiArgs ep{Y, ldy, bias, nullptr, 0, 1.0f, stream_sched(as_stream(stream))};
  // raster / L2-policy experiments on the pair GEMM (EDL_RASTER = m-tiles per
  // raster group, EDL_L2HINT = 1: A evict_last + B evict_first)
  static const int raster_env = [] { const char* v = getenv("EDL_RASTER"); return v ? atoi(v) : 0; }();
  static const int l2hint_env = [] { const char* v = getenv("EDL_L2HINT"); return v ? atoi(v) : -1; }();
  ep.raster = raster_env;
  // default: when A is too big to sit in L2 beside the streaming B (the
  // grouped-raster case, raster_group), load A evict_last and B evict_first
  // -- teacher layer 2: DRAM 515 -> 419 MB per launch, 356 -> 351 us alone
  // (profiles/r02_layer2_raster.txt)
  ep.l2hint = l2hint_env >= 0 ? l2hint_env : (static_cast<long long>(M) * K * 2 > (32ll << 20) ? 1 : 0);
  CUtensorMap ty;
  const int pbn = pick_pair_bn(M, N, cap);
  const int bn = pbn > 0 ? pbn : pick_bn_cap(M, N, cap);
  const bool w128 = (pbn > 0 ? pbn == 256 : bn % 64 == 0) && w128_enabled() &&
                    (act == EDL_ACT_RELU || act == EDL_ACT_IDENT || (act == EDL_ACT_TANH && w128_tanh()));
  if ((rc = w128 ? tensor_map(Y, M, N, ldy, 64, 32, &ty) : tensor_map_out(Y, M, N, ldy, act == EDL_ACT_NONE, &ty)))
    return rc;
  cudaError_t e;
  if (pbn > 0) {
    if ((rc = tensor_map(W, N, K, ldw, 64, pbn / 2, &tb))) return rc;
    e = launch_gemm_pair(kind, pbn, ta, tb, ty, M, N, K, ep, cap, as_stream(stream), nullptr, w128);
  } else {
    if ((rc = tensor_map(W, N, K, ldw, 64, bn, &tb))) return rc;
    e = launch_gemm(kind, bn, ta, tb, ty, M, N, K, ep, cap, as_stream(stream), nullptr, w128);
  }
  return e == cudaSuccess ? 0 : cuda_fail(e, "linear_fwd");
}

// The halo-tiled conv (halo.cu) for 3x3 / stride 1 / pad 1 convolutions with
// 64 input and 64 output channels and W <= 62 (>= 2 output rows per tile; the
// cfg4 stage-1 layers and their data gradients); EDL_HALO=0 keeps them on the
// TMA im2col GEMM (A/B runs).
bool halo_enabled() {
  static const bool on = [] {
    const char* v = getenv("EDL_HALO");
    return !(v && v[0] == '0');
  }();
  return on;
}

int halo_conv(const void* x, int N, int H, int W, const void* w, long long ldw, const float* bias, const void* res,
              const void* mask, bool relu, void* out, cudaStream_t st) {
  CUtensorMap mx, mw, my, mr{}, mm{};
  const int R = halo_rows_per_tile(W);
  if (int rc = halo_map_sw128(x, N, H, W, 64, W + 2, R + 2, &mx)) return rc;
  if (int rc = halo_map_sw128(out, N, H, W, 64, W, R, &my)) return rc;
  if (res != nullptr)
    if (int rc = halo_map_sw128(res, N, H, W, 64, W, R, &mr)) return rc;
  if (mask != nullptr)
    if (int rc = halo_map_sw128(mask, N, H, W, 64, W, R, &mm)) return rc;
  if (int rc = tensor_map(w, 64, 9 * 64, ldw, 64, 64, &mw)) return rc;
  HaloArgs a{};
  a.N = N; a.H = H; a.W = W; a.R = R;
  a.tiles_per_image = (H + R - 1) / R;
  a.tiles = N * a.tiles_per_image;
  a.bias = bias;
  a.res = static_cast<const __nv_bfloat16*>(res);
  a.mask = static_cast<const __nv_bfloat16*>(mask);
  a.relu = relu ? 1 : 0;
  a.out = static_cast<__nv_bfloat16*>(out);
  static const int dbg = [] {
    const char* v = getenv("EDL_HALO_DEBUG");
    return v ? atoi(v) : 0;
  }();
  a.debug = dbg;
  const int cap = grid_cap(st);
  const int grid = a.tiles < cap ? a.tiles : cap;
  cudaError_t e = launch_halo_conv(mx, mw, my, mr, mm, a, grid, st);
  return e == cudaSuccess ? 0 : cuda_fail(e, "halo_conv");
}

// Layout probe for the halo conv (tests only): one tap's 128 x 64 product
// from the staged patch of image n, rows h0-1 .. h0+2, shifted by `off` rows.
int edl_halo_probe(const void* x, int N, int H, int W, int n, int h0, int off, const void* w, int mode, int reps,
                   int smem_kb, float* out, void* stream) {
  if (off < 0 || off + 128 > 256 || n < 0 || n >= N || mode < 0 || mode > 4 || reps < 0)
    return fail(EDL_ERR_SHAPE, "halo_probe: bad arguments");
  CUtensorMap mx, mw;
  if (mode == 0) {
    if (int rc = halo_map(x, N, H, W, 64, 4, &mx)) return rc;
  } else {
    if (int rc = halo_map_sw128(x, N, H, W, 64, W + 2, 4, &mx)) return rc;
  }
  if (int rc = tensor_map(w, 64, mode == 3 ? 576 : 64, mode == 3 ? 576 : 64, 64, 64, &mw)) return rc;
  if (smem_kb < 0 || smem_kb > 227) return fail(EDL_ERR_SHAPE, "halo_probe: smem_kb");
  cudaError_t e = launch_halo_probe(mx, mw, n, h0, W, off, mode, reps, smem_kb, out, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "halo_probe");
}

int edl_conv_fwd_nhwc(const void* x, int N, int H, int W, int C, const void* w, long long ldw, const float* bias,
                      int K, int R, int S, int stride, int pad, const void* residual, long long ldr, void* y,
                      long long ldy, int act, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 64 || C % 64 || K < 1 || R < 1 || S < 1 || stride < 1 || stride > 8 ||
      pad < 0 || R > 16 || S > 16)
    return fail(EDL_ERR_SHAPE, "conv_fwd_nhwc: bad shape");
  if (act != EDL_ACT_RELU && act != EDL_ACT_IDENT) return fail(EDL_ERR_SHAPE, "conv_fwd_nhwc: act must be RELU/IDENT");
  if (residual && act != EDL_ACT_RELU) return fail(EDL_ERR_SHAPE, "conv_fwd_nhwc: residual needs act RELU");
  const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "conv_fwd_nhwc: empty output");
  const long long Ml = static_cast<long long>(N) * P * Q;
  const int Kd = R * S * C;
  if (Ml > (1LL << 31) - 256 || ldw < Kd || ldy < K || (residual && ldr < K))
    return fail(EDL_ERR_SHAPE, "conv_fwd_nhwc: bad leading dimension");
  const int M = static_cast<int>(Ml);
  cudaStream_t st = as_stream(stream);
  if (C == 64 && K == 64 && R == 3 && S == 3 && stride == 1 && pad == 1 && W + 2 <= 64 && ldy == 64 &&
      (!residual || ldr == 64) && halo_enabled())
    return halo_conv(x, N, H, W, w, ldw, bias, residual, nullptr, act == EDL_ACT_RELU, y, st);
  const int cap = grid_cap(st);
  CUtensorMap ta, tb, ty;
  int rc;
  if ((rc = conv_map(x, N, H, W, C, R, S, stride, pad, 128, &ta))) return rc;
  if ((rc = tensor_map_out(y, M, K, ldy, false, &ty))) return rc;
  EpiArgs ep{y, ldy, bias, reinterpret_cast<const __nv_bfloat16*>(residual), residual ? ldr : 0, 1.0f,
             stream_sched(st)};
  ep.conv = ConvGeom{P, Q, stride, pad, S, C / 64};
  const GemmKind kind = act == EDL_ACT_RELU ? GemmKind::FwdRelu : GemmKind::FwdIdentBf16;
  CUtensorMap tr;   // the residual, streamed by TMA in the epilogue
  if (residual && (rc = tensor_map_out(residual, M, K, ldr, false, &tr))) return rc;
  const int pbn = pick_pair_bn(M, K, cap);
  cudaError_t e;
  if (pbn == 256 && w128_enabled()) {
    CUtensorMap ty2, tr2;
    if ((rc = tensor_map(y, M, K, ldy, 64, 32, &ty2))) return rc;
    if (residual && (rc = tensor_map(residual, M, K, ldr, 64, 32, &tr2))) return rc;
    if ((rc = tensor_map(w, K, Kd, ldw, 64, pbn / 2, &tb))) return rc;
    e = launch_gemm_pair(kind, pbn, ta, tb, ty2, M, K, Kd, ep, cap, st, residual ? &tr2 : nullptr, true);
  } else if (pbn > 0) {
    if ((rc = tensor_map(w, K, Kd, ldw, 64, pbn / 2, &tb))) return rc;
    e = launch_gemm_pair(kind, pbn, ta, tb, ty, M, K, Kd, ep, cap, st, residual ? &tr : nullptr);
  } else {
    const int bn = pick_bn_cap(M, K, cap);
    if ((rc = tensor_map(w, K, Kd, ldw, 64, bn, &tb))) return rc;
    if (!residual && bn % 64 == 0 && w128_enabled()) {   // 64 x 32 SWIZZLE_128B output boxes
      CUtensorMap ty2;
      if ((rc = tensor_map(y, M, K, ldy, 64, 32, &ty2))) return rc;
      e = launch_gemm(kind, bn, ta, tb, ty2, M, K, Kd, ep, cap, st, nullptr, true);
    } else {
      e = launch_gemm(kind, bn, ta, tb, ty, M, K, Kd, ep, cap, st, residual ? &tr : nullptr);
    }
  }
  return e == cudaSuccess ? 0 : cuda_fail(e, "conv_fwd_nhwc");
}

int edl_conv_flip_weights_many(int count, const void* const* w, const long long* ldw, const int* K, const int* C,
                               const int* R, const int* S, void* const* wf, const long long* ldf, void* stream) {
  if (count < 0 || count > kMaxFlips) return fail(EDL_ERR_SHAPE, "conv_flip_weights_many: count %d (0..%d)", count,
                                                  kMaxFlips);
  FlipGroup g{};
  g.count = count;
  long long total = 0;
  for (int l = 0; l < count; ++l) {
    if (K[l] < 1 || C[l] < 1 || R[l] < 1 || S[l] < 1 || ldw[l] < static_cast<long long>(R[l]) * S[l] * C[l] ||
        ldf[l] < static_cast<long long>(R[l]) * S[l] * K[l] || !w[l] || !wf[l])
      return fail(EDL_ERR_SHAPE, "conv_flip_weights_many: bad layer %d", l);
    g.start[l] = static_cast<int>(total);
    g.K[l] = K[l];
    g.C[l] = C[l];
    g.RS[l] = R[l] * S[l];
    g.ldw[l] = ldw[l];
    g.ldf[l] = ldf[l];
    g.w[l] = static_cast<const __nv_bfloat16*>(w[l]);
    g.wf[l] = static_cast<__nv_bfloat16*>(wf[l]);
    total += static_cast<long long>(C[l]) * R[l] * S[l] * K[l];
    if (total > (1LL << 31) - 1) return fail(EDL_ERR_SHAPE, "conv_flip_weights_many: too many elements");
  }
  g.start[count] = static_cast<int>(total);
  cudaError_t e = launch_conv_flip_weights_many(g, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "conv_flip_weights_many");
}

int edl_conv_flip_weights(const void* w, long long ldw, int K, int C, int R, int S, void* wf, long long ldf,
                          void* stream) {
  if (K < 1 || C < 1 || R < 1 || S < 1 || ldw < static_cast<long long>(R) * S * C ||
      ldf < static_cast<long long>(R) * S * K || !w || !wf)
    return fail(EDL_ERR_SHAPE, "conv_flip_weights: bad shape");
  cudaError_t e = launch_conv_flip_weights(reinterpret_cast<const __nv_bfloat16*>(w), ldw, K, C, R, S,
                                           reinterpret_cast<__nv_bfloat16*>(wf), ldf, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "conv_flip_weights");
}

int edl_conv_dgrad_nhwc(const void* dz, int N, int P, int Q, int K, const void* wf, long long ldf, int C, int R,
                        int S, int pad, const void* add, const void* mask, void* dx, void* stream) {
  const int pd = R - 1 - pad;
  if (N < 1 || P < 1 || Q < 1 || K < 64 || K % 64 || C < 1 || R < 1 || S < 1 || R > 16 || S > 16 || pad < 0 ||
      pd < 0 || R - 1 - pad != S - 1 - pad || ldf < static_cast<long long>(R) * S * K)
    return fail(EDL_ERR_SHAPE, "conv_dgrad_nhwc: bad shape");
  const int H = P + 2 * pd - R + 1, W = Q + 2 * pd - S + 1;
  if (H < 1 || W < 1) return fail(EDL_ERR_SHAPE, "conv_dgrad_nhwc: empty output");
  const long long Ml = static_cast<long long>(N) * H * W;
  if (Ml > (1LL << 31) - 256) return fail(EDL_ERR_SHAPE, "conv_dgrad_nhwc: too many pixels");
  const int M = static_cast<int>(Ml), Kd = R * S * K;
  cudaStream_t st = as_stream(stream);
  if (C == 64 && K == 64 && R == 3 && S == 3 && pd == 1 && Q + 2 <= 64 && halo_enabled())
    return halo_conv(dz, N, P, Q, wf, ldf, nullptr, add, mask, false, dx, st);
  const int cap = grid_cap(st);
  CUtensorMap ta, tb, ty;
  int rc;
  if ((rc = conv_map(dz, N, P, Q, K, R, S, 1, pd, 128, &ta))) return rc;
  const int pbn_d = pick_pair_bn(M, C, cap);
  const bool w128 = (pbn_d > 0 ? pbn_d == 256 : pick_bn_cap(M, C, cap) % 64 == 0) && w128_enabled();
  if ((rc = w128 ? tensor_map(dx, M, C, C, 64, 32, &ty) : tensor_map_out(dx, M, C, C, false, &ty))) return rc;
  EpiArgs ep{dx, C, nullptr, reinterpret_cast<const __nv_bfloat16*>(add), add ? C : 0, 1.0f, stream_sched(st)};
  ep.aux2 = reinterpret_cast<const __nv_bfloat16*>(mask);
  ep.ld_aux2 = mask ? C : 0;
  ep.conv = ConvGeom{H, W, 1, pd, S, K / 64};
  const int pbn = pbn_d;
  cudaError_t e;
  if (pbn > 0) {
    if ((rc = tensor_map(wf, C, Kd, ldf, 64, pbn / 2, &tb))) return rc;
    e = launch_gemm_pair(GemmKind::ConvDgrad, pbn, ta, tb, ty, M, C, Kd, ep, cap, st, nullptr, w128);
  } else {
    const int bn = pick_bn_cap(M, C, cap);
    if ((rc = tensor_map(wf, C, Kd, ldf, 64, bn, &tb))) return rc;
    e = launch_gemm(GemmKind::ConvDgrad, bn, ta, tb, ty, M, C, Kd, ep, cap, st, nullptr, w128);
  }
  return e == cudaSuccess ? 0 : cuda_fail(e, "conv_dgrad_nhwc");
}

int edl_linear_fwd_residual(const void* X, long long ldx, const void* W, long long ldw, const float* bias,
                            const void* R, long long ldr, void* Y, long long ldy, int M, int N, int K,
                            void* stream) {
  if (M < 1 || N < 1 || K < 1 || ldx < K || ldw < K || ldy < N || ldr < N || !R)
    return fail(EDL_ERR_SHAPE, "linear_fwd_residual: bad shape M=%d N=%d K=%d", M, N, K);
  const int cap = grid_cap(as_stream(stream));
  CUtensorMap ta, tb, ty;
  int rc;
  if ((rc = tensor_map(X, M, K, ldx, 64, 128, &ta))) return rc;
  const int pbn = pick_pair_bn(M, N, cap);
  const bool w128 = pbn == 256 && w128_enabled();
  if ((rc = w128 ? tensor_map(Y, M, N, ldy, 64, 32, &ty) : tensor_map_out(Y, M, N, ldy, false, &ty))) return rc;
  EpiArgs ep{Y, ldy, bias, reinterpret_cast<const __nv_bfloat16*>(R), ldr, 1.0f, stream_sched(as_stream(stream))};
  CUtensorMap tr;
  if ((rc = w128 ? tensor_map(R, M, N, ldr, 64, 32, &tr) : tensor_map_out(R, M, N, ldr, false, &tr))) return rc;
  cudaError_t e;
  if (pbn > 0) {
    if ((rc = tensor_map(W, N, K, ldw, 64, pbn / 2, &tb))) return rc;
    e = launch_gemm_pair(GemmKind::FwdRelu, pbn, ta, tb, ty, M, N, K, ep, cap, as_stream(stream), &tr, w128);
  } else {
    const int bn = pick_bn_cap(M, N, cap);
    if ((rc = tensor_map(W, N, K, ldw, 64, bn, &tb))) return rc;
    e = launch_gemm(GemmKind::FwdRelu, bn, ta, tb, ty, M, N, K, ep, cap, as_stream(stream), &tr);
  }
  return e == cudaSuccess ? 0 : cuda_fail(e, "linear_fwd_residual");
}

int edl_im2col_nhwc(const void* x, int N, int H, int W, int C, int c_used, int R, int S, int stride, int pad,
                    void* out, long long ldo, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || c_used < 1 || c_used > C || R < 1 || S < 1 || stride < 1 ||
      pad < 0 || ldo < static_cast<long long>(R) * S * (c_used < C ? c_used : C) || ldo % 8)
    return fail(EDL_ERR_SHAPE, "im2col_nhwc: bad shape N=%d H=%d W=%d C=%d R=%d S=%d ldo=%lld", N, H, W, C, R, S, ldo);
  const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "im2col_nhwc: empty output");
  cudaError_t e = launch_im2col_nhwc(reinterpret_cast<const __nv_bfloat16*>(x), N, H, W, C, c_used, R, S, stride, pad,
                                     P, Q, reinterpret_cast<__nv_bfloat16*>(out), ldo, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "im2col_nhwc");
}

int edl_maxpool_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                     void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || k < 1 || stride < 1 || pad < 0 || pad >= k)
    return fail(EDL_ERR_SHAPE, "maxpool_nhwc: bad shape");
  const int P = (H + 2 * pad - k) / stride + 1, Q = (W + 2 * pad - k) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "maxpool_nhwc: empty output");
  cudaError_t e = launch_maxpool_nhwc(reinterpret_cast<const __nv_bfloat16*>(x), N, H, W, C, k, stride, pad, P, Q,
                                      reinterpret_cast<__nv_bfloat16*>(out), nullptr, false, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "maxpool_nhwc");
}

namespace {
int maxpool_argmax_impl(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                        unsigned* argmax, bool relu_mask, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || k < 1 || k * k > 15 || stride < 1 || pad < 0 || pad >= k ||
      !argmax)
    return fail(EDL_ERR_SHAPE, "maxpool_argmax_nhwc: bad shape");
  const int P = (H + 2 * pad - k) / stride + 1, Q = (W + 2 * pad - k) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "maxpool_argmax_nhwc: empty output");
  cudaError_t e = launch_maxpool_nhwc(reinterpret_cast<const __nv_bfloat16*>(x), N, H, W, C, k, stride, pad, P, Q,
                                      reinterpret_cast<__nv_bfloat16*>(out), argmax, relu_mask, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "maxpool_argmax_nhwc");
}
}  // namespace

int edl_maxpool_argmax_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                            unsigned* argmax, void* stream) {
  return maxpool_argmax_impl(x, N, H, W, C, k, stride, pad, out, argmax, false, stream);
}

int edl_maxpool_argmax_relu_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, void* out,
                                 unsigned* argmax, void* stream) {
  return maxpool_argmax_impl(x, N, H, W, C, k, stride, pad, out, argmax, true, stream);
}

int edl_bn_relu_maxpool_argmax_nhwc(const void* z, int N, int H, int W, int C, const float* mean, const float* rstd,
                                    const float* gamma, const float* beta, int k, int stride, int pad, void* out,
                                    unsigned* argmax, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || k != 3 || stride != 2 || pad < 0 || pad >= k || !argmax || !mean ||
      !rstd || !gamma || !beta)
    return fail(EDL_ERR_SHAPE, "bn_relu_maxpool_argmax_nhwc: 3x3 / 2 pools with C %% 8 == 0 only");
  const int P = (H + 2 * pad - k) / stride + 1, Q = (W + 2 * pad - k) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "bn_relu_maxpool_argmax_nhwc: empty output");
  cudaError_t e = launch_bn_relu_maxpool3s2_nhwc(static_cast<const __nv_bfloat16*>(z), N, H, W, C, pad, P, Q, mean,
                                                 rstd, gamma, beta, static_cast<__nv_bfloat16*>(out),
                                                 reinterpret_cast<uint32_t*>(argmax), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "bn_relu_maxpool_argmax_nhwc");
}

int edl_maxpool_bwd_argmax_nhwc(const unsigned* argmax, int N, int H, int W, int C, int k, int stride, int pad,
                                const void* dy, const void* mask, void* dx, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || k < 1 || k * k > 15 || stride < 1 || pad < 0 || pad >= k ||
      !argmax)
    return fail(EDL_ERR_SHAPE, "maxpool_bwd_argmax_nhwc: bad shape");
  const int P = (H + 2 * pad - k) / stride + 1, Q = (W + 2 * pad - k) / stride + 1;
  cudaError_t e = launch_maxpool_bwd_argmax_nhwc(argmax, N, H, W, C, k, stride, pad, P, Q,
                                                 reinterpret_cast<const __nv_bfloat16*>(dy),
                                                 reinterpret_cast<const __nv_bfloat16*>(mask),
                                                 reinterpret_cast<__nv_bfloat16*>(dx), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "maxpool_bwd_argmax_nhwc");
}

int edl_avgpool_nhwc(const void* x, int N, int HW, int C, void* out, long long ldo, void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8 || ldo < C || ldo % 8) return fail(EDL_ERR_SHAPE, "avgpool_nhwc: bad shape");
  cudaError_t e = launch_avgpool_nhwc(reinterpret_cast<const __nv_bfloat16*>(x), N, HW, C,
                                      reinterpret_cast<__nv_bfloat16*>(out), ldo, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "avgpool_nhwc");
}

int edl_linear_bwd_data(const void* dY, long long lddy, const void* W, long long ldw,
                        const void* H, long long ldh, void* dX, long long lddx, int M, int N,
                        int K, void* stream) {
  if (M < 1 || N < 1 || K < 1 || lddy < N || ldw < K || (H && ldh < K) || lddx < K)
    return fail(EDL_ERR_SHAPE, "linear_bwd_data: bad shape M=%d N=%d K=%d", M, N, K);
  const GemmKind kind = H ? GemmKind::BwdData : GemmKind::BwdDataPlain;   // H null: no (1 - a^2)
  const int cap = grid_cap(as_stream(stream));
  CUtensorMap ta, tb;
  int rc;
  // A = dY [M][N] (reduction N contiguous: K-major); B = W [N][K] read as [red][MN].
  if ((rc = tensor_map(dY, M, N, lddy, 64, 128, &ta))) return rc;
  if ((rc = tensor_map(W, N, K, ldw, 64, 64, &tb))) return rc;
  EpiArgs ep{dX, lddx, nullptr, reinterpret_cast<const __nv_bfloat16*>(H), ldh, 1.0f,
             stream_sched(as_stream(stream))};
  CUtensorMap ty;
  const int pbn = pick_pair_bn(M, K, cap);
  const int bn = pbn > 0 ? pbn : pick_bn_cap(M, K, cap);
  // not with H (the (1 - a^2) epilogue): its per-element row reads of H made
  // the cfg3 student step 208 -> 256 us on 128-byte boxes
  const bool w128 = (pbn > 0 ? pbn == 256 : bn % 64 == 0) && w128_enabled() && H == nullptr;
  if ((rc = w128 ? tensor_map(dX, M, K, lddx, 64, 32, &ty) : tensor_map_out(dX, M, K, lddx, false, &ty))) return rc;
  cudaError_t e = pbn > 0 ? launch_gemm_pair(kind, pbn, ta, tb, ty, M, K, N, ep, cap, as_stream(stream), nullptr, w128)
                          : launch_gemm(kind, bn, ta, tb, ty, M, K, N, ep, cap, as_stream(stream), nullptr, w128);
  return e == cudaSuccess ? 0 : cuda_fail(e, "linear_bwd_data");
}

int edl_col2im_nhwc(const void* dcol, long long ldc, int N, int H, int W, int C, int R, int S, int stride, int pad,
                    const void* add, const void* mask, void* dx, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || R < 1 || S < 1 || stride < 1 || pad < 0 ||
      ldc < static_cast<long long>(R) * S * C || ldc % 8)
    return fail(EDL_ERR_SHAPE, "col2im_nhwc: bad shape");
  const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "col2im_nhwc: empty output");
  cudaError_t e = launch_col2im_nhwc(reinterpret_cast<const __nv_bfloat16*>(dcol), ldc, N, H, W, C, R, S, stride, pad,
                                     P, Q, reinterpret_cast<const __nv_bfloat16*>(add),
                                     reinterpret_cast<const __nv_bfloat16*>(mask),
                                     reinterpret_cast<__nv_bfloat16*>(dx), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "col2im_nhwc");
}

int edl_avgpool_bwd_nhwc(const void* df, long long ldf, int N, int HW, int C, const void* mask, void* dx,
                         void* stream) {
  if (N < 1 || HW < 1 || C < 8 || C % 8 || ldf < C || ldf % 8) return fail(EDL_ERR_SHAPE, "avgpool_bwd_nhwc: bad shape");
  cudaError_t e = launch_avgpool_bwd_nhwc(reinterpret_cast<const __nv_bfloat16*>(df), ldf, N, HW, C,
                                          reinterpret_cast<const __nv_bfloat16*>(mask),
                                          reinterpret_cast<__nv_bfloat16*>(dx), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "avgpool_bwd_nhwc");
}

int edl_maxpool_bwd_nhwc(const void* x, int N, int H, int W, int C, int k, int stride, int pad, const void* dy,
                         const void* mask, void* dx, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 8 || C % 8 || k < 1 || k * k > 15 || stride < 1 || pad < 0 || pad >= k)
    return fail(EDL_ERR_SHAPE, "maxpool_bwd_nhwc: bad shape");
  const int P = (H + 2 * pad - k) / stride + 1, Q = (W + 2 * pad - k) / stride + 1;
  cudaError_t e = launch_maxpool_bwd_nhwc(reinterpret_cast<const __nv_bfloat16*>(x), N, H, W, C, k, stride, pad, P, Q,
                                          reinterpret_cast<const __nv_bfloat16*>(dy),
                                          reinterpret_cast<const __nv_bfloat16*>(mask),
                                          reinterpret_cast<__nv_bfloat16*>(dx), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "maxpool_bwd_nhwc");
}

int edl_linear_bwd_weight(const void* dY, long long lddy, const void* X, long long ldx, float* dW,
                          long long lddw, float* db, float* workspace, int M, int N, int K,
                          float scale, void* stream) {
  if (M < 1 || N < 1 || K < 1 || lddy < N || ldx < K || lddw < K)
    return fail(EDL_ERR_SHAPE, "linear_bwd_weight: bad shape M=%d N=%d K=%d", M, N, K);
  const int bn = pick_bn(N, K);
  CUtensorMap ta, tb;
  int rc;
  // A = dY^T: dY [M][N] read as [red=M][MN=N]; B = X^T: X [M][K] read as [red=M][MN=K].
  if ((rc = tensor_map(dY, M, N, lddy, 64, 64, &ta))) return rc;
  if ((rc = tensor_map(X, M, K, ldx, 64, 64, &tb))) return rc;
  EpiArgs ep{dW, lddw, nullptr, nullptr, 0, scale, stream_sched(as_stream(stream))};
  cudaError_t e = launch_gemm(GemmKind::BwdWeight, bn, ta, tb, ta /*unused: plain-store epilogue*/, N, K, M, ep,
                              grid_cap(as_stream(stream)),
                              as_stream(stream));
  if (e != cudaSuccess) return cuda_fail(e, "linear_bwd_weight");
  if (db) {
    if (!workspace) return fail(EDL_ERR_SHAPE, "linear_bwd_weight: db needs a workspace");
    e = launch_colsum(reinterpret_cast<const __nv_bfloat16*>(dY), lddy, M, N, workspace, db, scale,
                      as_stream(stream));
    if (e != cudaSuccess) return cuda_fail(e, "colsum");
  }
  return 0;
}

}  // extern "C"

namespace {
// dW_p = scale * dY_p^T X_p (+ db_p = scale * colsum dY_p) for every p, or with
// `sgd` the fused update W_p -= scale * dY_p^T X_p, b_p -= scale * colsum dY_p
// (bf16 copies W16 / b16 refreshed) where the gradients never reach HBM.
int bwd_weight_grouped_impl(int count, const void* const* dY, const long long* lddy,
                            const void* const* X, const long long* ldx, float* const* dW,
                            const long long* lddw, float* const* db, void* const* W16,
                            void* const* b16, float* workspace, const int* M, const int* N,
                            const int* K, float scale, void* stream, bool sgd) {
  if (count < 1 || count > kMaxGroup)
    return fail(EDL_ERR_SHAPE, "linear_bwd_weight_grouped: count=%d (1..%d)", count, kMaxGroup);
  GroupMaps maps;
  GroupArgs ga;
  std::memset(&ga, 0, sizeof(ga));
  ga.count = count;
  const int bn = grouped_tile_bn();
  const int cap = grid_cap(as_stream(stream));
  // CTA-pair tiles when their wave-quantised cost is no worse (pick_pair_bn's
  // rule on the summed tile counts)
  long long single_tiles = 0, pair_tiles = 0;
  for (int p = 0; p < count; ++p) {
    single_tiles += static_cast<long long>((N[p] + 127) / 128) * ((K[p] + bn - 1) / bn);
    pair_tiles += static_cast<long long>((N[p] + 255) / 256) * ((K[p] + 255) / 256);
  }
  const long long single_waves = (single_tiles + cap - 1) / cap;
  const long long pair_waves = cap >= 2 ? (pair_tiles + cap / 2 - 1) / (cap / 2) : 0;
  const bool use_pair = cap >= 2 && pair_mode_enabled() &&
                        (pair_waves < single_waves || (pair_waves == single_waves && pair_waves >= 2));
  int tiles = 0;
  for (int p = 0; p < count; ++p) {
    if (M[p] < 1 || N[p] < 1 || K[p] < 1 || lddy[p] < N[p] || ldx[p] < K[p] || lddw[p] < K[p])
      return fail(EDL_ERR_SHAPE, "linear_bwd_weight_grouped[%d]: bad shape M=%d N=%d K=%d", p, M[p], N[p], K[p]);
    int rc;
    // same operand views as edl_linear_bwd_weight: GEMM M=N[p], N=K[p], K=M[p]
    if ((rc = tensor_map(dY[p], M[p], N[p], lddy[p], 64, 64, &maps.a[p]))) return rc;
    if ((rc = tensor_map(X[p], M[p], K[p], ldx[p], 64, 64, &maps.b[p]))) return rc;
    ga.M[p] = N[p];
    ga.N[p] = K[p];
    ga.K[p] = M[p];
    ga.ep[p] = EpiArgs{dW[p], lddw[p], nullptr, nullptr, 0, scale, nullptr,
                       sgd ? reinterpret_cast<__nv_bfloat16*>(W16[p]) : nullptr};
    if (sgd && !W16[p]) return fail(EDL_ERR_SHAPE, "linear_bwd_weight_grouped_sgd[%d]: missing bf16 copy", p);
    ga.tile_start[p] = tiles;
    tiles += use_pair ? ((N[p] + 255) / 256) * ((K[p] + 255) / 256) : ((N[p] + 127) / 128) * ((K[p] + bn - 1) / bn);
  }
  ga.tile_start[count] = tiles;
  cudaError_t e = use_pair ? launch_gemm_grouped_pair_bwd_weight(maps, ga, cap, as_stream(stream), sgd)
                           : launch_gemm_grouped_bwd_weight(maps, ga, cap, as_stream(stream), sgd);
  if (e != cudaSuccess) return cuda_fail(e, "linear_bwd_weight_grouped");
  if (db) {
    ColsumGroup g = {};
    for (int p = 0; p < count; ++p) {
      if (!db[p]) continue;
      g.x[g.count] = reinterpret_cast<const __nv_bfloat16*>(dY[p]);
      g.ld[g.count] = lddy[p];
      g.M[g.count] = M[p];
      g.N[g.count] = N[p];
      g.out[g.count] = db[p];
      g.out_bf16[g.count] = (sgd && b16) ? reinterpret_cast<__nv_bfloat16*>(b16[p]) : nullptr;
      ++g.count;
    }
    if (g.count > 0) {
      if (!workspace) return fail(EDL_ERR_SHAPE, "linear_bwd_weight_grouped: db needs a workspace");
      g.scale = scale;
      g.sgd = sgd ? 1 : 0;
      g.partial = workspace;
      e = launch_colsum_group(g, as_stream(stream));
      if (e != cudaSuccess) return cuda_fail(e, "colsum");
    }
  }
  return 0;
}
}  // namespace

extern "C" {

int edl_linear_bwd_weight_grouped(int count, const void* const* dY, const long long* lddy,
                                  const void* const* X, const long long* ldx, float* const* dW,
                                  const long long* lddw, float* const* db, float* workspace,
                                  const int* M, const int* N, const int* K, float scale, void* stream) {
  return bwd_weight_grouped_impl(count, dY, lddy, X, ldx, dW, lddw, db, nullptr, nullptr, workspace, M, N, K,
                                 scale, stream, false);
}

int edl_linear_bwd_weight_grouped_sgd(int count, const void* const* dY, const long long* lddy,
                                      const void* const* X, const long long* ldx, float* const* W,
                                      void* const* W_bf16, const long long* ldw, float* const* b,
                                      void* const* b_bf16, float* workspace, const int* M, const int* N,
                                      const int* K, float eta, void* stream) {
  return bwd_weight_grouped_impl(count, dY, lddy, X, ldx, W, ldw, b, W_bf16, b_bf16, workspace, M, N, K, eta,
                                 stream, true);
}

long long edl_colsum_workspace_floats(int M, int N) { return colsum_workspace_floats(1, &M, &N); }

long long edl_bwd_weight_workspace_floats(int M, int N, int K) {
  if (M < 1 || N < 1 || K < 1) return -1;
  const long long ws = wgrad_workspace_floats(M, N, K, num_sms());
  // a 64 -> 64 3x3 conv may run the halo weight gradient: its per-CTA partials
  const long long halo = (N == 64 && K == 576) ? halo_wgrad_partial_floats(num_sms()) : 0;
  return ws > halo ? ws : halo;
}

}  // extern "C"

namespace {
// dW = scale dY^T X over M rows (+ db), split-K planned; conv != nullptr: X is
// the im2col matrix of an NHWC tensor, read through a TMA im2col map (`xmap`).
int bwd_weight_ws_impl(const void* dY, long long lddy, const void* X, long long ldx, const CUtensorMap* xmap,
                       const ConvGeom* conv, float* dW, long long lddw, float* db, float* workspace,
                       long long workspace_floats, int M, int N, int K, float scale, void* stream) {
  if (!workspace || workspace_floats < 0)
    return fail(EDL_ERR_SHAPE, "linear_bwd_weight_ws: workspace required");
  cudaStream_t st = as_stream(stream);
  const int cap = grid_cap(st);
  const WgradPlan p = plan_wgrad(M, N, K, cap, workspace_floats);
  CUtensorMap ta, tb;
  int rc;
  // dY [M][N] and X [M][K] both read as [red=M][MN]; swapped: A = X^T, B = dY^T
  if (p.swap) {
    if (xmap) ta = *xmap;
    else if ((rc = tensor_map(X, M, K, ldx, 64, 64, &ta))) return rc;
    if ((rc = tensor_map(dY, M, N, lddy, 64, 64, &tb))) return rc;
  } else {
    if ((rc = tensor_map(dY, M, N, lddy, 64, 64, &ta))) return rc;
    if (xmap) tb = *xmap;
    else if ((rc = tensor_map(X, M, K, ldx, 64, 64, &tb))) return rc;
  }
  EpiArgs ep{p.reduce() ? static_cast<void*>(workspace) : static_cast<void*>(dW), p.reduce() ? p.gn : lddw,
             nullptr, nullptr, 0, scale, stream_sched(st)};
  if (conv) {
    ep.conv = *conv;
    ep.conv.operand = p.swap ? 0 : 1;
  }
  ep.ksplit = p.ksplit;
  ep.split_stride = static_cast<long long>(p.gm) * p.gn;
  cudaError_t e = launch_gemm(GemmKind::BwdWeight, p.bn, ta, tb, ta, p.gm, p.gn, M, ep, cap, st);
  if (e != cudaSuccess) return cuda_fail(e, "linear_bwd_weight_ws");
  if (p.reduce()) {
    e = launch_splitk_reduce(workspace, p.ksplit, ep.split_stride, p.gm, p.gn, p.swap, dW, lddw, cap, st);
    if (e != cudaSuccess) return cuda_fail(e, "splitk_reduce");
  }
  if (db) {   // the workspace is free again (stream order)
    const long long need = colsum_tall_ok(N) ? static_cast<long long>(colsum_tall_blocks(M, cap)) * N
                                             : colsum_workspace_floats(1, &M, &N);
    if (need > workspace_floats)
      return fail(EDL_ERR_SHAPE, "linear_bwd_weight_ws: workspace %lld < %lld floats", workspace_floats, need);
    e = colsum_tall_ok(N) ? launch_colsum_tall(reinterpret_cast<const __nv_bfloat16*>(dY), lddy, M, N, workspace,
                                               db, scale, cap, st)
                          : launch_colsum(reinterpret_cast<const __nv_bfloat16*>(dY), lddy, M, N, workspace, db,
                                          scale, st);
    if (e != cudaSuccess) return cuda_fail(e, "colsum");
  }
  return 0;
}
}  // namespace

extern "C" {

int edl_linear_bwd_weight_ws(const void* dY, long long lddy, const void* X, long long ldx, float* dW,
                             long long lddw, float* db, float* workspace, long long workspace_floats, int M, int N,
                             int K, float scale, void* stream) {
  if (M < 1 || N < 1 || K < 1 || lddy < N || ldx < K || lddw < K)
    return fail(EDL_ERR_SHAPE, "linear_bwd_weight_ws: bad shape M=%d N=%d K=%d", M, N, K);
  return bwd_weight_ws_impl(dY, lddy, X, ldx, nullptr, nullptr, dW, lddw, db, workspace, workspace_floats, M, N, K,
                            scale, stream);
}

int edl_conv_bwd_weight_nhwc(const void* x, int N, int H, int W, int C, int R, int S, int stride, int pad,
                             const void* dY, long long lddy, int K, float* dW, long long lddw, float* db,
                             float* workspace, long long workspace_floats, float scale, void* stream) {
  if (N < 1 || H < 1 || W < 1 || C < 64 || C % 64 || K < 1 || R < 1 || S < 1 || stride < 1 || stride > 8 ||
      pad < 0 || R > 16 || S > 16)
    return fail(EDL_ERR_SHAPE, "conv_bwd_weight_nhwc: bad shape");
  const int P = (H + 2 * pad - R) / stride + 1, Q = (W + 2 * pad - S) / stride + 1;
  if (P < 1 || Q < 1) return fail(EDL_ERR_SHAPE, "conv_bwd_weight_nhwc: empty output");
  const long long Ml = static_cast<long long>(N) * P * Q;
  const int Kd = R * S * C;
  if (Ml > (1LL << 31) - 256 || lddy < K || lddw < Kd)
    return fail(EDL_ERR_SHAPE, "conv_bwd_weight_nhwc: bad leading dimension");
  CUtensorMap xm;
  int rc;
  if (C == 64 && K == 64 && R == 3 && S == 3 && stride == 1 && pad == 1 && W + 2 <= 64 && lddy == 64 &&
      db == nullptr && halo_enabled()) {
    // the halo weight gradient (halo.cu): patch views as MN-major operands
    cudaStream_t st = as_stream(stream);
    const int Rt = halo_rows_per_tile(W);
    HaloArgs a{};
    a.N = N; a.H = H; a.W = W; a.R = Rt;
    a.tiles_per_image = (H + Rt - 1) / Rt;
    a.tiles = N * a.tiles_per_image;
    const int cap = grid_cap(st);
    const int grid = a.tiles < cap ? a.tiles : cap;
    if (workspace_floats >= halo_wgrad_partial_floats(grid)) {
      CUtensorMap mx, md;
      if ((rc = halo_map_sw128(x, N, H, W, 64, W + 2, Rt + 2, &mx))) return rc;
      if ((rc = halo_map_sw128(dY, N, H, W, 64, W + 2, Rt, &md))) return rc;
      cudaError_t e = launch_halo_wgrad(mx, md, a, grid, workspace, scale, dW, lddw, st);
      return e == cudaSuccess ? 0 : cuda_fail(e, "halo_wgrad");
    }
  }
  if ((rc = conv_map(x, N, H, W, C, R, S, stride, pad, 64, &xm))) return rc;
  const ConvGeom g{P, Q, stride, pad, S, C / 64};
  return bwd_weight_ws_impl(dY, lddy, nullptr, 0, &xm, &g, dW, lddw, db, workspace, workspace_floats,
                            static_cast<int>(Ml), K, Kd, scale, stream);
}

long long edl_colsum_group_workspace_floats(int count, const int* M, const int* N) {
  if (count < 1 || count > kMaxGroup) return -1;
  return colsum_workspace_floats(count, M, N);
}

int edl_teacher_head_softmax_topk(const void* H, long long ldh, const void* W, long long ldw,
                                  const float* bias, int M, int N, int K, float T, int k,
                                  float* vals, int* idx, void* stream) {
  if (M < 1 || N < 1 || K < 1 || ldh < K || ldw < K)
    return fail(EDL_ERR_SHAPE, "teacher_head: bad shape M=%d N=%d K=%d", M, N, K);
  if (!(T > 0.f) || !std::isfinite(T)) return fail(EDL_ERR_PARAM, "teacher_head: temperature %g", T);
  if (k < 1 || k > N || k > 32) return fail(EDL_ERR_PARAM, "teacher_head: k=%d (1..min(N,32))", k);
  const int kmax = k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
  const int bn = N <= 64 ? 64 : N <= 128 ? 128 : 256;
  if ((N + bn - 1) / bn > 8) return fail(EDL_ERR_SHAPE, "teacher_head: N=%d exceeds 8 x 256 classes", N);
  CUtensorMap ta, tb;
  int rc;
  if ((rc = tensor_map(H, M, K, ldh, 64, 128, &ta))) return rc;
  if ((rc = tensor_map(W, N, K, ldw, 64, bn, &tb))) return rc;
  HeadArgs hp{bias, 1.0f / T, k, vals, idx};
  cudaError_t e = launch_teacher_head(bn, kmax, ta, tb, M, N, K, hp, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "teacher_head");
}

long long edl_teacher_head_workspace_bytes(int M, int N, int k) {
  if (M < 1 || N < 1 || k < 1 || k > 32) return 0;
  const int kmax = k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
  const long long part = static_cast<long long>((N + 255) / 256) * (2 + 2 * kmax) * M * 4;
  const long long tickets = static_cast<long long>((M + 127) / 128 + 1) * 4;
  return (part + 255) / 256 * 256 + tickets;
}

int edl_teacher_head_softmax_topk_ws(const void* H, long long ldh, const void* W, long long ldw, const float* bias,
                                     int M, int N, int K, float T, int k, float* vals, int* idx, void* workspace,
                                     long long ws_bytes, void* stream) {
  static const bool cluster_head = [] {
    const char* v = getenv("EDL_HEAD_CLUSTER");   // A/B switch: the single-CTA cluster head
    return v && v[0] == '1';
  }();
  if (cluster_head || workspace == nullptr)
    return edl_teacher_head_softmax_topk(H, ldh, W, ldw, bias, M, N, K, T, k, vals, idx, stream);
  if (M < 1 || N < 1 || K < 1 || ldh < K || ldw < K)
    return fail(EDL_ERR_SHAPE, "teacher_head: bad shape M=%d N=%d K=%d", M, N, K);
  if (!(T > 0.f) || !std::isfinite(T)) return fail(EDL_ERR_PARAM, "teacher_head: temperature %g", T);
  if (k < 1 || k > N || k > 32) return fail(EDL_ERR_PARAM, "teacher_head: k=%d (1..min(N,32))", k);
  if (ws_bytes < edl_teacher_head_workspace_bytes(M, N, k))
    return fail(EDL_ERR_SHAPE, "teacher_head: workspace of %lld bytes < %lld", ws_bytes,
                edl_teacher_head_workspace_bytes(M, N, k));
  const int kmax = k <= 4 ? 4 : k <= 8 ? 8 : k <= 16 ? 16 : 32;
  CUtensorMap ta, tb;
  int rc;
  if ((rc = tensor_map(H, M, K, ldh, 64, 128, &ta))) return rc;
  if ((rc = tensor_map(W, N, K, ldw, 64, 128, &tb))) return rc;
  HeadArgs hp{bias, 1.0f / T, k, vals, idx};
  const long long part = static_cast<long long>((N + 255) / 256) * (2 + 2 * kmax) * M * 4;
  float* pw = static_cast<float*>(workspace);
  unsigned* tickets = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + (part + 255) / 256 * 256);
  cudaError_t e = launch_teacher_head_pair(kmax, ta, tb, M, N, K, hp, pw, tickets, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "teacher_head_pair");
}

int edl_tempered_softmax(const float* logits, long long ld, float* probs, long long ldp, int B,
                         int K, float T, void* stream) {
  if (B < 1 || K < 1 || ld < K || ldp < K) return fail(EDL_ERR_SHAPE, "tempered_softmax: bad shape");
  if (!(T > 0.f) || !std::isfinite(T)) return fail(EDL_ERR_PARAM, "tempered_softmax: temperature %g", T);
  cudaError_t e = launch_tempered_softmax(logits, ld, probs, ldp, B, K, T, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "tempered_softmax");
}

int edl_linear_kd_loss_fwd_bwd(const void* H, long long ldh, const void* W, long long ldw, const float* bias,
                               const long long* labels, const float* q_vals, const int* q_idx, int B, int K, int D,
                               int k, float alpha, float beta, float T, float* row_loss, float* loss_out,
                               void* dlogits, long long lddz, int* status, void* stream) {
  if (B < 1 || K < 1 || D < 1 || ldh < D || ldw < D || lddz < K)
    return fail(EDL_ERR_SHAPE, "linear_kd_loss: bad shape B=%d K=%d D=%d", B, K, D);
  if (!(T > 0.f) || !std::isfinite(T)) return fail(EDL_ERR_PARAM, "linear_kd_loss: temperature %g", T);
  if (alpha < 0.f || beta < 0.f || !(alpha + beta > 0.f)) return fail(EDL_ERR_PARAM, "linear_kd_loss: alpha/beta");
  if (beta > 0.f && (k < 1 || k > K || k > 32 || !q_vals || !q_idx))
    return fail(EDL_ERR_SHAPE, "linear_kd_loss: beta > 0 requires 1..32 soft labels (k=%d)", k);
  const long long kp16 = (K + 15) / 16 * 16;
  const int Nw = static_cast<int>(lddz < kp16 ? lddz : kp16);
  if (Nw > 8 * 256) return fail(EDL_ERR_SHAPE, "linear_kd_loss: %d classes exceed 8 x 256", K);
  const int ks = beta > 0.f ? k : 0;
  const int kmax = ks <= 4 ? 4 : ks <= 8 ? 8 : ks <= 16 ? 16 : 32;
  CUtensorMap ta, tb, ty;
  int rc;
  if ((rc = tensor_map(H, B, D, ldh, 64, 128, &ta))) return rc;
  if ((rc = tensor_map(W, K, D, ldw, 64, 256, &tb))) return rc;
  if ((rc = tensor_map_out(dlogits, B, Nw, lddz, false, &ty))) return rc;
  KdArgs kp{bias, reinterpret_cast<const int64_t*>(labels), q_vals, q_idx, ks, alpha, beta, T, 1.0f / T,
            T == 2.0f ? 1 : 0, row_loss, status};
  static const int dbg = [] {
    const char* v = getenv("EDL_KD_DEBUG");
    return v ? atoi(v) : 0;
  }();
  kp.debug = dbg;
  cudaError_t e = launch_kd_head(kmax, ta, tb, ty, B, K, Nw, D, kp, as_stream(stream));
  if (e == cudaSuccess) e = launch_loss_mean(row_loss, B, loss_out, status, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "linear_kd_loss");
}

int edl_kd_loss_fwd_bwd(const float* logits, long long ldz, const long long* labels,
                        const float* q_vals, const int* q_idx, int B, int K, int k, float alpha,
                        float beta, float T, float* row_loss, float* loss_out, unsigned* ticket,
                        void* dlogits, long long lddz, int* status, void* stream) {
  if (B < 1 || K < 1 || ldz < K || lddz < K) return fail(EDL_ERR_SHAPE, "kd_loss: bad shape B=%d K=%d", B, K);
  if (!(T > 0.f) || !std::isfinite(T)) return fail(EDL_ERR_PARAM, "kd_loss: temperature %g", T);
  if (alpha < 0.f || beta < 0.f || !(alpha + beta > 0.f)) return fail(EDL_ERR_PARAM, "kd_loss: alpha/beta");
  if (beta > 0.f && (k < 1 || k > K || !q_vals || !q_idx))
    return fail(EDL_ERR_SHAPE, "kd_loss: beta > 0 requires soft labels (k=%d)", k);
  cudaError_t e = launch_kd_loss(logits, ldz, reinterpret_cast<const int64_t*>(labels), q_vals, q_idx,
                                 B, K, beta > 0.f ? k : 0, alpha, beta, T, row_loss, loss_out, ticket,
                                 reinterpret_cast<__nv_bfloat16*>(dlogits), lddz, status,
                                 as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "kd_loss");
}

// Stream-ordered 32-bit flags: the split placement's soft-label handoff
// (pool.PeerSoftLabelRing). cuStreamWaitValue32 / cuStreamWriteValue32 keep
// the wait and the signal in the streams without holding an SM; a one-thread
// kernel pair stands in if the driver reports stream memory ops unsupported.
namespace {
using PFN_value32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_value32 driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<PFN_value32>(p);
  return nullptr;
}
PFN_value32 wait_value_fn() {
  static PFN_value32 fn = driver_fn("cuStreamWaitValue32");
  return fn;
}
PFN_value32 write_value_fn() {
  static PFN_value32 fn = driver_fn("cuStreamWriteValue32");
  return fn;
}
}  // namespace

int edl_stream_wait_geq(unsigned* addr, unsigned value, void* stream) {
  if (!addr) return fail(EDL_ERR_SHAPE, "stream_wait_geq: null address");
  PFN_value32 fn = wait_value_fn();
  if (fn) {
    const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value, 0);
    if (r == CUDA_SUCCESS) return 0;
    if (r != CUDA_ERROR_NOT_SUPPORTED) return fail(EDL_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", static_cast<int>(r));
  }
  cudaError_t e = launch_flag_wait(addr, value, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "stream_wait_geq");
}

int edl_stream_write_u32(unsigned* addr, unsigned value, void* stream) {
  if (!addr) return fail(EDL_ERR_SHAPE, "stream_write_u32: null address");
  PFN_value32 fn = write_value_fn();
  if (fn) {
    const CUresult r = fn(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value, 0);
    if (r == CUDA_SUCCESS) return 0;
    if (r != CUDA_ERROR_NOT_SUPPORTED) return fail(EDL_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", static_cast<int>(r));
  }
  cudaError_t e = launch_flag_write(addr, value, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "stream_write_u32");
}

int edl_nvls_allreduce_sgd(float* mc_grad, float* mc_param, void* mc_param_bf16, const float* param,
                           unsigned* const* pads, long long pad_bytes, unsigned* counter, int rank, int world,
                           long long n, float scale, unsigned epoch, void* stream) {
  if (world < 2 || world > 64 || rank < 0 || rank >= world || !pads || !counter)
    return fail(EDL_ERR_PARAM, "nvls_allreduce_sgd: bad rank %d / world %d", rank, world);
  if (n < 8 || n % (8LL * world) || !mc_grad || !mc_param || !mc_param_bf16 || !param)
    return fail(EDL_ERR_SHAPE, "nvls_allreduce_sgd: n=%lld must be a positive multiple of 8*world", n);
  const int max_blocks = nvls_max_blocks(world, pad_bytes);
  if (max_blocks < 1) return fail(EDL_ERR_PARAM, "nvls_allreduce_sgd: signal pad of %lld bytes too small", pad_bytes);
  // A small grid: it runs beside the co-located teacher's persistent GEMMs,
  // which leave only the stream reserve free (edl_set_stream_max_ctas);
  // blocks that cannot be resident would wait out a whole teacher GEMM.
  // EDL_NVLS_BLOCKS overrides (tuning runs).
  static const int env_blocks = [] {
    const char* v = getenv("EDL_NVLS_BLOCKS");
    return v ? atoi(v) : 0;
  }();
  const long long items = n / 8 / world;
  long long blocks = (items + 511) / 512;
  const long long want = env_blocks > 0 ? env_blocks : 24;
  if (blocks > want) blocks = want;
  if (blocks > num_sms()) blocks = num_sms();
  if (blocks > max_blocks) blocks = max_blocks;
  cudaError_t e = launch_nvls_allreduce_sgd(mc_grad, mc_param, mc_param_bf16, param,
                                            reinterpret_cast<uint32_t* const*>(pads), counter, n, scale, epoch,
                                            rank, world, static_cast<int>(blocks), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "nvls_allreduce_sgd");
}

int edl_sgd_step(float* p, void* p_bf16, const float* g, long long n, float scale, void* stream) {
  if (n < 0) return fail(EDL_ERR_SHAPE, "sgd_step: n=%lld", n);
  if ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g)) & 15)
    return fail(EDL_ERR_SHAPE, "sgd_step: buffers must be 16-byte aligned");
  if (n == 0) return 0;
  cudaError_t e = launch_sgd(p, reinterpret_cast<__nv_bfloat16*>(p_bf16), g, n, scale, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "sgd_step");
}

int edl_gather_rows(const void* src, long long ld_src, const long long* idx, void* dst,
                    long long ld_dst, int B, int D, const long long* src_labels,
                    long long* dst_labels, void* stream) {
  if (B < 1 || D < 1 || ld_src < D || ld_dst < D || (ld_src % 8) || (ld_dst % 8))
    return fail(EDL_ERR_SHAPE, "gather_rows: bad shape B=%d D=%d", B, D);
  cudaError_t e = launch_gather_rows(reinterpret_cast<const __nv_bfloat16*>(src), ld_src,
                                     reinterpret_cast<const int64_t*>(idx),
                                     reinterpret_cast<__nv_bfloat16*>(dst), ld_dst, B, D,
                                     reinterpret_cast<const int64_t*>(src_labels),
                                     reinterpret_cast<int64_t*>(dst_labels), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "gather_rows");
}

int edl_topk_hits(const float* logits, long long ld, const long long* labels, int B, int K, int k,
                  unsigned* hits, void* stream) {
  if (B < 1 || K < 1 || ld < K) return fail(EDL_ERR_SHAPE, "topk_hits: bad shape");
  if (k < 1 || k > K) return fail(EDL_ERR_PARAM, "topk_hits: k=%d", k);
  cudaError_t e = launch_topk_hits(logits, ld, reinterpret_cast<const int64_t*>(labels), B, K, k,
                                   hits, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "topk_hits");
}

int edl_cast_bf16(const float* src, long long ld_src, void* dst, long long ld_dst, int rows,
                  int cols, void* stream) {
  if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < cols) return fail(EDL_ERR_SHAPE, "cast_bf16: bad shape");
  if (rows == 0 || cols == 0) return 0;
  cudaError_t e = launch_cast_bf16(src, ld_src, reinterpret_cast<__nv_bfloat16*>(dst), ld_dst, rows,
                                   cols, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "cast_bf16");
}

int edl_cast_bf16_f64(const double* src, long long ld_src, void* dst, long long ld_dst, int rows, int cols,
                      void* stream) {
  if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < cols) return fail(EDL_ERR_SHAPE, "cast_bf16_f64: bad shape");
  if (rows == 0 || cols == 0) return 0;
  cudaError_t e = launch_cast_bf16_f64(src, ld_src, reinterpret_cast<__nv_bfloat16*>(dst), ld_dst, rows, cols,
                                       as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "cast_bf16_f64");
}

// ---- training-mode BatchNorm (cfg4 student)
static int bn_check(int M, int C, const char* what) {
  if (M < 1 || C < 8 || C % 8 || C > 2048) return fail(EDL_ERR_SHAPE, "%s: M=%d C=%d (C %% 8 == 0, <= 2048)", what, M, C);
  return 0;
}

long long edl_bn_workspace_floats(int M, int C) {
  return bn_partial_floats(M < 1 ? 1 : M, C < 8 ? 8 : C, num_sms());
}

int edl_bn_stats_nhwc(const void* z, int M, int C, float* workspace, long long ws_floats, float* mean, float* rstd,
                      float eps, void* stream) {
  if (int rc = bn_check(M, C, "bn_stats")) return rc;
  if (ws_floats < edl_bn_workspace_floats(M, C)) return fail(EDL_ERR_SHAPE, "bn_stats: workspace too small");
  if (!(eps > 0.f)) return fail(EDL_ERR_PARAM, "bn_stats: eps %g", eps);
  cudaError_t e = launch_bn_stats(static_cast<const __nv_bfloat16*>(z), M, C, workspace,
                                  stream_ticket(as_stream(stream)), mean, rstd, eps, num_sms(), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "bn_stats");
}

int edl_bn_apply_nhwc(const void* z, int M, int C, const float* mean, const float* rstd, const float* gamma,
                      const float* beta, const void* residual, int relu, void* y, void* stream) {
  if (int rc = bn_check(M, C, "bn_apply")) return rc;
  cudaError_t e = launch_bn_apply(static_cast<const __nv_bfloat16*>(z), M, C, mean, rstd, gamma, beta,
                                  static_cast<const __nv_bfloat16*>(residual), relu != 0,
                                  static_cast<__nv_bfloat16*>(y), num_sms(), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "bn_apply");
}

int edl_bn_bwd_nhwc(const void* g, const void* z, int M, int C, const float* mean, const float* rstd,
                    const float* gamma, float* workspace, long long ws_floats, float* dgamma, float* dbeta, void* dz,
                    void* stream) {
  if (int rc = bn_check(M, C, "bn_bwd")) return rc;
  if (ws_floats < edl_bn_workspace_floats(M, C)) return fail(EDL_ERR_SHAPE, "bn_bwd: workspace too small");
  const auto* gg = static_cast<const __nv_bfloat16*>(g);
  const auto* zz = static_cast<const __nv_bfloat16*>(z);
  cudaError_t e = launch_bn_bwd_reduce(gg, zz, M, C, mean, rstd, workspace, stream_ticket(as_stream(stream)), dbeta,
                                       dgamma, num_sms(), as_stream(stream));
  if (e == cudaSuccess)
    e = launch_bn_bwd_apply(gg, zz, M, C, mean, rstd, gamma, dbeta, dgamma, static_cast<__nv_bfloat16*>(dz),
                            num_sms(), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "bn_bwd");
}

int edl_memcpy_async(void* dst, const void* src, long long bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(EDL_ERR_SHAPE, "memcpy_async: bad arguments");
  if (bytes == 0) return 0;
  cudaError_t e = cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault, as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "memcpy_async");
}

int edl_host_register(void* ptr, long long bytes, void** dev_ptr) {
  if (!ptr || bytes <= 0 || !dev_ptr) return fail(EDL_ERR_SHAPE, "host_register: bad arguments");
  cudaError_t e = cudaHostRegister(ptr, static_cast<size_t>(bytes), cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) return cuda_fail(e, "host_register");
  e = cudaHostGetDevicePointer(dev_ptr, ptr, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(ptr);
    return cuda_fail(e, "host_register (device pointer)");
  }
  return 0;
}

int edl_host_unregister(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  return e == cudaSuccess ? 0 : cuda_fail(e, "host_unregister");
}

int edl_ipc_export(const void* ptr, void* handle, long long* offset) {
  if (!ptr || !handle || !offset) return fail(EDL_ERR_SHAPE, "ipc_export: bad arguments");
  // the handle names the whole cudaMalloc allocation (a caching allocator
  // sub-allocates); the importer adds the offset
  CUdeviceptr base = 0;
  size_t size = 0;
  using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    return (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess) ? reinterpret_cast<PFN_range>(p) : nullptr;
  }();
  if (!range) return fail(EDL_ERR_CUDA, "ipc_export: cuMemGetAddressRange unavailable");
  const CUresult r = range(&base, &size, reinterpret_cast<CUdeviceptr>(ptr));
  if (r != CUDA_SUCCESS) return fail(EDL_ERR_CUDA, "ipc_export: cuMemGetAddressRange failed (%d)", static_cast<int>(r));
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail(e, "ipc_export");
  std::memcpy(handle, &h, sizeof(h));
  *offset = static_cast<long long>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  return 0;
}

int edl_ipc_open(const void* handle, void** base) {
  if (!handle || !base) return fail(EDL_ERR_SHAPE, "ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : cuda_fail(e, "ipc_open");
}

int edl_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  return e == cudaSuccess ? 0 : cuda_fail(e, "ipc_close");
}

int edl_stream_delay_ns(long long ns, void* stream) {
  if (ns < 0) return fail(EDL_ERR_PARAM, "stream_delay_ns: negative delay");
  if (ns == 0) return 0;
  cudaError_t e = launch_stream_delay(static_cast<unsigned long long>(ns), as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "stream_delay_ns");
}

int edl_memcpy_peer_async(void* dst, int dst_device, const void* src, int src_device, long long bytes,
                          void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(EDL_ERR_SHAPE, "memcpy_peer_async: bad arguments");
  if (bytes == 0) return 0;
  cudaError_t e = cudaMemcpyPeerAsync(dst, dst_device, src, src_device, static_cast<size_t>(bytes),
                                      as_stream(stream));
  return e == cudaSuccess ? 0 : cuda_fail(e, "memcpy_peer_async");
}

}  // extern "C"
