// pnms_common.cuh — shared types, score keys, detection records and small device helpers.
//
// Exactness notes:
//  * Scores are never rounded: the gate s_i < s_j (engine.py:233) is evaluated on an
//    order-preserving 64-bit key of the float64 score.  NaN compares false with
//    everything, so NaN rows/columns are kept out of the ordered work entirely.
//  * The float64 threshold theta*(z_j+1)^2 (engine.py:197) becomes the integer
//    T_j = ceil(fl64(theta*(z_j+1)^2)); for integer w*h,  w*h < thr  <=>  w*h < T_j.
//  * Frames whose coordinates fit in 15 bits use packed s16x2 geometry (DPX VIADDMNMX);
//    anything else runs an exact emulation of the reference's int32/float64 arithmetic.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pnms {

// programmatic dependent launch as inline PTX (the runtime wrappers become calls in
// relocatable device code): wait for the preceding grid's completion and memory flush / let
// the dependent grid start launching.  Both are no-ops without a programmatic launch.
#ifdef PNMS_DEVICE_CHAIN
// pnms_devchain.cu: the list kernels there are only tail-launched by the binned kernel, after
// it completed; waiting on the launching grid from a tail launch would never return
__device__ __forceinline__ void pdl_wait() {}
#else
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#endif
#ifdef PNMS_DEVICE_CHAIN
// ... and a grid that tail-launches must not trigger its dependents early: measured on B200,
// griddepcontrol.launch_dependents in the parent keeps a tail launch from ever starting
__device__ __forceinline__ void pdl_trigger() {}
#else
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

constexpr int kSortMax = 4096;        // frames up to this many slots sort inside one CTA
constexpr int kSortThreads = 512;     // 16 warps
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kRecBytes = 32;         // per-slot record stride in the workspace
constexpr int kMapWarps = 4;          // warps per map CTA

// Per-frame arithmetic path, decided on the device from the frame's own values.
enum FrameMode : int {
  kNarrow7 = 0,   // 0<=x,y; 0<=z<=126; x+z+1, y+z+1 <= 32767  -> s16x2 geometry, 1-IMAD product
  kNarrow16 = 1,  // as above but z up to 32766                  -> s16x2 geometry, split product
  kWide = 2       // anything representable in int32            -> exact int32-wrap + fp64 emulation
};

struct FrameMeta {
  int n_active;       // valid, non-NaN detections; they occupy sorted positions [0, n_active)
  int mode;           // FrameMode
  int cnt_neg;        // valid non-NaN scores < 0   (padding gate terms of map_writes)
  int cnt_pos;        // valid non-NaN scores > 0
  int cnt_zero;       // valid scores == 0 (either sign)
  int pad_;
  unsigned long long lim_sum;  // sum over active rows of their column limit (= gate passes)
};
static_assert(sizeof(FrameMeta) == 32, "FrameMeta layout");

// Narrow record (16 B), one per sorted slot.  All geometry packed as two int16 halves
// (lo = x axis, hi = y axis).
//   a   = (x+z+1, y+z+1)         inclusive far edge + 1
//   nb  = (-x, -y)               negated near edge
//   zz  = (z+1, z+1)             side + 1
//   negT = -T * 2^17 (narrow7) or -T (narrow16), T = ceil(fl64(theta*(z+1)^2)) and T = 0
//          for z == 0 (engine.py:232)
struct __align__(16) RecNarrow {
  uint32_t a, nb, zz;
  int32_t negT;
};

// Wide record (32 B): the reference's own int32 working values and float64 threshold.
//   xe = x + z and ye = y + z with int32 wrap-around (engine.py:194-196)
//   thr = theta*(z+1)^2 in float64 (engine.py:197); -inf when z == 0 so keep is false
//   (engine.py:232).
struct __align__(16) RecWide {
  int32_t x, y, xe, ye;
  double thr;
  int32_t pad0, pad1;
};
static_assert(sizeof(RecWide) == kRecBytes, "RecWide layout");

// Order-preserving key: key(a) < key(b)  <=>  a < b for non-NaN doubles; -0.0 == +0.0.
// NaN maps to 0, below every other key (-inf maps to 0x000FFFFFFFFFFFFF).
__device__ __forceinline__ uint64_t score_key(double s) {
  if (s != s) return 0ull;
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(s));
  if (b == 0x8000000000000000ull) b = 0ull;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Sort key used by the ascending radix sort: descending score == ascending ~key.
__device__ __forceinline__ uint64_t sort_key(double s) { return ~score_key(s); }
constexpr uint64_t kNanSortKey = ~0ull;

// float64 threshold exactly as engine.py:197 computes it.
__device__ __forceinline__ double ref_threshold(double theta, int32_t z) {
  double zf = __dadd_rn(static_cast<double>(z), 1.0);
  return __dmul_rn(theta, __dmul_rn(zf, zf));
}

__device__ __forceinline__ int frame_mode_of(int32_t x, int32_t y, int32_t z) {
  if (x < 0 || y < 0 || z < 0) return kWide;
  long long xe1 = (long long)x + z + 1, ye1 = (long long)y + z + 1;
  if (xe1 > 32767 || ye1 > 32767) return kWide;
  return z <= 126 ? kNarrow7 : kNarrow16;
}

__device__ __forceinline__ RecNarrow make_rec_narrow(int32_t x, int32_t y, int32_t z, double theta, int mode) {
  RecNarrow r;
  uint32_t xe1 = static_cast<uint32_t>(x + z + 1), ye1 = static_cast<uint32_t>(y + z + 1);
  r.a = (xe1 & 0xFFFFu) | (ye1 << 16);
  r.nb = (static_cast<uint32_t>(-x) & 0xFFFFu) | (static_cast<uint32_t>(-y) << 16);
  r.zz = static_cast<uint32_t>(z + 1) * 0x10001u;
  uint32_t T = 0;
  if (z != 0) T = static_cast<uint32_t>(ceil(ref_threshold(theta, z)));
  r.negT = (mode == kNarrow7) ? -static_cast<int32_t>(T << 17) : -static_cast<int32_t>(T);
  return r;
}

__device__ __forceinline__ RecWide make_rec_wide(int32_t x, int32_t y, int32_t z, double theta) {
  RecWide r;
  r.x = x;
  r.y = y;
  r.xe = static_cast<int32_t>(static_cast<uint32_t>(x) + static_cast<uint32_t>(z));
  r.ye = static_cast<int32_t>(static_cast<uint32_t>(y) + static_cast<uint32_t>(z));
  r.thr = (z != 0) ? ref_threshold(theta, z) : -__longlong_as_double(0x7FF0000000000000ll);
  r.pad0 = r.pad1 = 0;
  return r;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024).
// `warp_sums` needs blockDim.x/32 + 1 slots.  Returns the exclusive prefix; *total gets the sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_sums[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < nwarps ? warp_sums[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nwarps) warp_sums[lane] = wi - w;
    if (lane == 31) warp_sums[nwarps] = wi;
  }
  __syncthreads();
  uint32_t excl = warp_sums[warp] + inc - v;
  if (total) *total = warp_sums[nwarps];
  __syncthreads();
  return excl;
}

// Block-wide exclusive max-scan (identity -1), same contract as block_exclusive_scan.
__device__ __forceinline__ int block_exclusive_max_scan(int v, int* warp_vals) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc = max(inc, t);
  }
  if (lane == 31) warp_vals[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nwarps ? warp_vals[lane] : -1;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi = max(wi, t);
    }
    int ex = __shfl_up_sync(0xFFFFFFFFu, wi, 1);
    if (lane < nwarps) warp_vals[lane] = lane == 0 ? -1 : ex;
  }
  __syncthreads();
  int prev = __shfl_up_sync(0xFFFFFFFFu, inc, 1);
  int excl = max(warp_vals[warp], lane == 0 ? -1 : prev);
  __syncthreads();
  return excl;
}

// ---- 1-D bulk async copy (TMA bulk engine, SASS UBLKCP) with an mbarrier -----------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar) {
  uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst));
  uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
      "l"(gmem_src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}

}  // namespace pnms
