// pnms_capi.cu — extern "C" entry points of libparnms_b200.so (declared in
// include/parnms_b200.h).  Host-side orchestration only: argument validation with the
// reference's ConfigError conditions, workspace carving, launch-shape heuristics, and the
// stream-ordered launch sequence
//     prep+sort  ->  map (+row reduce)  ->  compact
// No host synchronisation and no allocation happens here.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <utility>
#include <emmintrin.h>
#include <omp.h>

#include "../../include/parnms_b200.h"
#include "pnms_common.cuh"
#include "pnms_compact.cuh"
#include "pnms_map.cuh"
#include "pnms_reflayout.cuh"
#include "pnms_small.cuh"
#include "pnms_binned.cuh"
#include "pnms_binned2.cuh"
#include "pnms_coop.cuh"
#include "pnms_devchain.h"
#include "pnms_fallback.cuh"
#include "pnms_validate.cuh"
#include "pnms_binned_cluster.cuh"
#include "pnms_binned_tiles.cuh"
#include "pnms_gate.cuh"
#include "pnms_greedy.cuh"
#include "pnms_soft.cuh"
#include "pnms_sort.cuh"

using namespace pnms;

namespace pnms {
// int16 ingest planes -> the int32 planes the engine consumes (4 slots per thread, vectorised)
__global__ void __launch_bounds__(256) pnms_widen_i16_kernel(const int16_t* __restrict__ x16, const int16_t* __restrict__ y16,
                                                             const int16_t* __restrict__ z16, int32_t* __restrict__ x,
                                                             int32_t* __restrict__ y, int32_t* __restrict__ z, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 3 < n && ((reinterpret_cast<uintptr_t>(x16 + i) | reinterpret_cast<uintptr_t>(y16 + i) |
                       reinterpret_cast<uintptr_t>(z16 + i)) & 7) == 0 &&
        ((reinterpret_cast<uintptr_t>(x + i) | reinterpret_cast<uintptr_t>(y + i) | reinterpret_cast<uintptr_t>(z + i)) & 15) == 0) {
      const short4 a = *reinterpret_cast<const short4*>(x16 + i);
      const short4 b = *reinterpret_cast<const short4*>(y16 + i);
      const short4 c = *reinterpret_cast<const short4*>(z16 + i);
      *reinterpret_cast<int4*>(x + i) = make_int4(a.x, a.y, a.z, a.w);
      *reinterpret_cast<int4*>(y + i) = make_int4(b.x, b.y, b.z, b.w);
      *reinterpret_cast<int4*>(z + i) = make_int4(c.x, c.y, c.z, c.w);
    } else {
      for (long long k = i; k < min(i + 4, n); ++k) { x[k] = x16[k]; y[k] = y16[k]; z[k] = z16[k]; }
    }
  }
}

// packed 32-bit boxes (x | y << 12 | z << 24) -> the int32 planes the engine consumes
__global__ void __launch_bounds__(256) pnms_unpack_box32_kernel(const uint32_t* __restrict__ box,
                                                                int32_t* __restrict__ x, int32_t* __restrict__ y,
                                                                int32_t* __restrict__ z, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x * 4;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 3 < n && (reinterpret_cast<uintptr_t>(box + i) & 15) == 0 &&
        ((reinterpret_cast<uintptr_t>(x + i) | reinterpret_cast<uintptr_t>(y + i) | reinterpret_cast<uintptr_t>(z + i)) & 15) == 0) {
      const uint4 b = __ldcs(reinterpret_cast<const uint4*>(box + i));
      *reinterpret_cast<int4*>(x + i) = make_int4(b.x & 0xFFF, b.y & 0xFFF, b.z & 0xFFF, b.w & 0xFFF);
      *reinterpret_cast<int4*>(y + i) = make_int4((b.x >> 12) & 0xFFF, (b.y >> 12) & 0xFFF, (b.z >> 12) & 0xFFF, (b.w >> 12) & 0xFFF);
      *reinterpret_cast<int4*>(z + i) = make_int4(b.x >> 24, b.y >> 24, b.z >> 24, b.w >> 24);
    } else {
      for (long long k = i; k < min(i + 4, n); ++k) {
        const uint32_t v = box[k];
        x[k] = v & 0xFFF; y[k] = (v >> 12) & 0xFFF; z[k] = v >> 24;
      }
    }
  }
}
// y[i] = glibc_exp(x[i]): the device build of the libm restatement (diagnostics / tests)
__global__ void __launch_bounds__(256) pnms_exp_kernel(const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = glibc_exp(x[i]);
}
}  // namespace pnms

namespace {

thread_local int g_last_cuda_error = 0;
unsigned long long* g_pairs_counter = nullptr;  // diagnostics: binned pair tests (pnms_debug_count_pairs)
unsigned long long* g_trace = nullptr;          // diagnostics: phase timestamps (pnms_debug_trace)

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct Layout {
  size_t coop;
  size_t rec, perm, lim, supp, meta, sk, idx, dense, list, tiles, total;
};

Layout make_layout(int batch, int n_max) {
  Layout L;
  const size_t B = (size_t)batch, N = (size_t)n_max;
  const size_t W32 = (N + 31) / 32;
  size_t off = kSmallScratchBytes;  // [0, kSmallScratchBytes): persistent zeroed scratch
  L.rec = off;  off = align_up(off + B * N * kRecBytes, 256);
  L.perm = off; off = align_up(off + B * N * 4, 256);
  L.lim = off;  off = align_up(off + B * N * 4, 256);
  L.supp = off; off = align_up(off + B * W32 * 4, 256);
  L.meta = off; off = align_up(off + B * sizeof(FrameMeta), 256);
  L.dense = off; off = align_up(off + B, 256);
  L.list = off; off = align_up(off + (B + 1) * 4, 256);  // [0] = count, then frame ids
  if (n_max > kSortMax) {
    L.tiles = off; off = align_up(off + B * 4 + B * W32 * 4 + 16, 256);  // tile path: decline flags + masks
    L.sk = off;  off = align_up(off + B * N * 8, 256);
    L.idx = off; off = align_up(off + B * N * 4, 256);
  } else {
    L.sk = L.idx = L.tiles = 0;
  }
  // the cooperative latency path (batches of <= kCoopMaxFrames): tile lists
  L.coop = 0;
  if (batch <= kCoopMaxFrames) {
    L.coop = off; off = align_up(off + B * kCoopMaxTiles * kCoopCap * sizeof(uint4), 256);
  }
  L.total = off;
  return L;
}

// ---- per-device caches (attributes and properties are per device: a process may drive several)
constexpr int kMaxDevices = 64;

inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

// the largest dynamic shared memory a kernel has been opened up to, per device
struct SmemCache {
  std::atomic<size_t> v[kMaxDevices];
};

template <typename K>
cudaError_t ensure_smem(K kernel, size_t bytes, SmemCache& c) {
  std::atomic<size_t>& slot = c.v[current_device()];
  if (bytes <= 48 * 1024 || slot.load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) slot.store(bytes, std::memory_order_relaxed);
  return e;
}

// streaming multiprocessors of the current device
int sm_count() {
  static std::atomic<int> cached[kMaxDevices];
  const int dev = current_device();
  int v = cached[dev].load();
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  cached[dev].store(v);
  return v;
}

int fail_cuda(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return PNMS_ECUDA;
}

// launch `kernel` with programmatic stream serialization (PDL) when `pdl` is set: it may start
// while the previous kernel on the stream drains; it calls pdl_wait()
template <class... KArgs, class... Args>
cudaError_t launch_maybe_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&lc, kernel, std::forward<Args>(args)...);
}

SmemCache g_sort_frame_smem, g_sort_chunk_smem, g_compact_smem, g_sort_list_smem;
SmemCache g_map_smem[5], g_map_list_smem[5];
SmemCache g_small_smem[8];
SmemCache g_tiles_smem[2];

template <bool B, bool C, int P, int T>
cudaError_t launch_binned_t(const BinArgs& ba, int batch, size_t smem, cudaStream_t st, SmemCache& cfg) {
  cudaError_t e = ensure_smem(pnms_binned_frame<B, C, P, T>, smem, cfg);
  if (e != cudaSuccess) return e;
  pnms_binned_frame<B, C, P, T><<<batch, T, smem, st>>>(ba);
  return cudaGetLastError();
}

// input slots per cluster CTA (a multiple of 32) for cluster size cs, or 0 when too large
int cluster_slice(int n_max, int cs) {
  const int slice = ((n_max + cs - 1) / cs + 31) / 32 * 32;
  return slice <= kClMaxSlice ? slice : 0;
}

template <bool B, int CS, int P>
cudaError_t launch_cluster_t(const BinArgs& ba, int batch, int slice, cudaStream_t st) {
  static SmemCache cfg;
  static std::atomic<int> nonportable[kMaxDevices];
  const size_t smem = binned_cluster_smem_bytes();
  cudaError_t e = ensure_smem(pnms_binned_cluster<B, CS, P>, smem, cfg);
  if (e != cudaSuccess) return e;
  std::atomic<int>& np = nonportable[current_device()];
  if (CS > 8 && !np.load()) {
    e = cudaFuncSetAttribute(pnms_binned_cluster<B, CS, P>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    np.store(1);
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)batch * CS);
  lc.blockDim = dim3(kClThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, pnms_binned_cluster<B, CS, P>, ba, slice);
}

// whether the current device can co-schedule a 16-CTA cluster of the cluster kernel (probed
// once per device; benign if two threads race)
bool cluster16_ok() {
  static std::atomic<int> cached[kMaxDevices] = {};
  std::atomic<int>& c = cached[current_device()];
  int v = c.load();
  if (v == 0) {
    int n = 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(16);
    lc.blockDim = dim3(kClThreads);
    lc.dynamicSmemBytes = binned_cluster_smem_bytes();
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    const void* fn = (const void*)pnms_binned_cluster<false, 16, 1>;
    bool ok = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
              cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lc.dynamicSmemBytes) ==
                  cudaSuccess &&
              cudaOccupancyMaxActiveClusters(&n, fn, &lc) == cudaSuccess && n > 0;
    cudaGetLastError();
    v = ok ? 1 : 2;
    c.store(v);
  }
  return v == 1;
}

// cluster size: 16 CTAs (non-portable; one GPC) when the device can co-schedule them and the
// frame is large, else 8; `want` (8 or 16) pins it
int cluster_size_for(int n_max, int want) {
  const bool cs16 = cluster16_ok();
  if (want == 8 || want == 16) return (want == 16 && !cs16) ? 8 : want;
  return (cs16 && n_max > 8 * 1024) ? 16 : 8;
}

cudaError_t launch_cluster(const BinArgs& ba, int batch, int cs, int slice, bool by_index, cudaStream_t st) {
  const int per = slice <= kClThreads ? 1 : (slice <= 2 * kClThreads ? 2 : 4);
#define PNMS_CL(CS, P) (by_index ? launch_cluster_t<true, CS, P>(ba, batch, slice, st) \
                                 : launch_cluster_t<false, CS, P>(ba, batch, slice, st))
  if (cs == 16) return per == 1 ? PNMS_CL(16, 1) : (per == 2 ? PNMS_CL(16, 2) : PNMS_CL(16, 4));
  return per == 1 ? PNMS_CL(8, 1) : (per == 2 ? PNMS_CL(8, 2) : PNMS_CL(8, 4));
#undef PNMS_CL
}

// variant bits: 1 by_index, 2 count pairs; `wide` picks 1024-thread CTAs (one per SM, two
// boxes per thread) for batches that fit one wave.  impl 1 = the first-generation kernel
// (pnms_binned.cuh), kept for measurement; the default is pnms_binned2.cuh.
template <bool B, bool C, int P, int T, int M = (T == 512 ? 3 : 1)>
cudaError_t launch_binned2_t(const BinArgs& ba, int batch, size_t smem, cudaStream_t st, SmemCache& cfg) {
  cudaError_t e = ensure_smem(pnms_binned2_frame<B, C, P, T, M>, smem, cfg);
  if (e != cudaSuccess) return e;
  pnms_binned2_frame<B, C, P, T, M><<<batch, T, smem, st>>>(ba);
  return cudaGetLastError();
}

cudaError_t launch_binned(int impl, int variant, const BinArgs& ba, int batch, int n_max, cudaStream_t st, bool wide) {
  const int npad = binned_npad(n_max);
  if (impl == 1) {
    const size_t smem = binned_smem_bytes(npad);
    static SmemCache c1[12];
    const int per = binned_per_thread(n_max, kBinThreads);
#define PNMS_B1(P, T, I)                                                                        \
  switch (variant & 3) {                                                                        \
    case 0: return launch_binned_t<false, false, P, T>(ba, batch, smem, st, c1[I]);            \
    case 1: return launch_binned_t<true, false, P, T>(ba, batch, smem, st, c1[I + 1]);         \
    case 2: return launch_binned_t<false, true, P, T>(ba, batch, smem, st, c1[I + 2]);         \
    default: return launch_binned_t<true, true, P, T>(ba, batch, smem, st, c1[I + 3]);         \
  }
    if (wide) { PNMS_B1(2, 1024, 0) }
    if (per <= 4) { PNMS_B1(4, kBinThreads, 4) }
    PNMS_B1(8, kBinThreads, 8)
#undef PNMS_B1
  }
  const size_t smem = b2_smem_bytes(wide ? 2048 : npad);
  static SmemCache c2[16];
#define PNMS_B2(P, T, I)                                                                        \
  switch (variant & 3) {                                                                        \
    case 0: return launch_binned2_t<false, false, P, T>(ba, batch, smem, st, c2[I]);           \
    case 1: return launch_binned2_t<true, false, P, T>(ba, batch, smem, st, c2[I + 1]);        \
    case 2: return launch_binned2_t<false, true, P, T>(ba, batch, smem, st, c2[I + 2]);        \
    default: return launch_binned2_t<true, true, P, T>(ba, batch, smem, st, c2[I + 3]);        \
  }
  if (wide) { PNMS_B2(2, 1024, 0) }
  if (n_max <= 2 * kBinThreads) { PNMS_B2(2, kBinThreads, 12) }  // frames of <= 1024 slots: half the layout
  if (n_max <= 4 * kBinThreads) { PNMS_B2(4, kBinThreads, 4) }
  PNMS_B2(4, 1024, 8)
#undef PNMS_B2
}

template <bool B, bool C, int R>
cudaError_t launch_small_t(const SmallArgs& sa, long long grid, size_t smem, cudaStream_t st, SmemCache& cfg) {
  cudaError_t e = ensure_smem(pnms_small_kernel<B, C, R>, smem, cfg);
  if (e != cudaSuccess) return e;
  pnms_small_kernel<B, C, R><<<(unsigned)grid, kSmallThreads, smem, st>>>(sa);
  return cudaGetLastError();
}

// variant bits: 1 = count gate passes, 2 = by_index, 4 = one row per thread
cudaError_t launch_small(int v, const SmallArgs& sa, long long grid, size_t smem, cudaStream_t st) {
  switch (v) {
    case 0: return launch_small_t<false, false, kSmallRowsMax>(sa, grid, smem, st, g_small_smem[0]);
    case 1: return launch_small_t<false, true, kSmallRowsMax>(sa, grid, smem, st, g_small_smem[1]);
    case 2: return launch_small_t<true, false, kSmallRowsMax>(sa, grid, smem, st, g_small_smem[2]);
    case 3: return launch_small_t<true, true, kSmallRowsMax>(sa, grid, smem, st, g_small_smem[3]);
    case 4: return launch_small_t<false, false, 1>(sa, grid, smem, st, g_small_smem[4]);
    case 5: return launch_small_t<false, true, 1>(sa, grid, smem, st, g_small_smem[5]);
    case 6: return launch_small_t<true, false, 1>(sa, grid, smem, st, g_small_smem[6]);
    default: return launch_small_t<true, true, 1>(sa, grid, smem, st, g_small_smem[7]);
  }
}

// ---- path selection ---------------------------------------------------------------------
// Calls with little total work run the single-launch unsorted path (pnms_small.cuh): below
// 24 Mi slot pairs per call (measured: the single launch beats the sort/cull pipelines there)
constexpr long long kSmallPairs = 24LL << 20;
// calls of <= 2 frames above this many slots take the multi-CTA tile path (measured,
// tools/single_frame_paths.py: a 4096-box random frame 22 us on tiles against 52 us on one CTA)
constexpr int kTilesSmallSlots = 2048;
constexpr long long kCoopPairs = 12LL << 20;

bool small_fits(int batch, int n_max) {
  const int W32 = (n_max + 31) / 32;
  return n_max <= kSortMax && batch <= kSmallMaxFrames && (long long)batch * W32 <= kSmallMaxWords;
}

bool cluster_fits(int n_max, int cs) { return cluster_slice(n_max, 16) > 0 && cluster_slice(n_max, cs) > 0; }

// tile CTAs per frame of the cooperative path: ~128 boxes per tile, at most kCoopMaxTiles, and
// every CTA of the call co-resident (0 when the call cannot be)
int coop_tiles(int batch, int n_max, int want = 0) {
  static std::atomic<int> per_sm[kMaxDevices];
  const int dev = current_device();
  int b = per_sm[dev].load();
  if (b <= 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, pnms_coop<false>, kCoopThreads, 0) != cudaSuccess || b <= 0)
      b = 1;
    per_sm[dev].store(b);
  }
  int t = want > 0 ? std::min(want, kCoopMaxTiles) : std::min(kCoopMaxTiles, std::max(16, n_max / kCoopBoxesPerTile));
  const int resident = b * sm_count();
  while (t > 1 && (long long)batch * t > resident) t /= 2;
  // (each CTA stashes its slice of the frame in shared memory)
  return (long long)batch * t <= resident && (n_max + t - 1) / t <= kCoopCap ? t : 0;
}

bool path_fits(int path, int batch, int n_max, int cs) {
  switch (path) {
    case PNMS_PATH_SMALL: return small_fits(batch, n_max);
    case PNMS_PATH_BINNED: return n_max <= kBinMaxSlots;
    case PNMS_PATH_BINNED_WIDE: return n_max <= 2048;
    case PNMS_PATH_TILES: return n_max <= PNMS_MAX_SLOTS;
    case PNMS_PATH_CLUSTER: return cluster_fits(n_max, cs);
    case PNMS_PATH_DENSE: return true;
    case PNMS_PATH_COOP: return batch <= kCoopMaxFrames && n_max <= PNMS_MAX_SLOTS && coop_tiles(batch, n_max) > 0;
    default: return false;
  }
}

int auto_path(int batch, int n_max, int cs) {
  // one or two frames above 12 Mi slot pairs: the cooperative path (measured,
  // tools/single_frame_paths.py: 4096 clustered boxes 16.4 us against 18.4 on the small path,
  // a tie at 3584 random boxes; two frames of 3000: 17.3 against 20.5; 2 x 4096: 16.4 against 26.6)
  if (batch <= kCoopMaxFrames && (long long)batch * n_max * n_max > kCoopPairs && coop_tiles(batch, n_max) > 0)
    return PNMS_PATH_COOP;
  if (small_fits(batch, n_max) && (long long)batch * n_max * n_max <= kSmallPairs) return PNMS_PATH_SMALL;
  if (n_max <= kBinMaxSlots) {
    if (batch <= 2 && n_max > kTilesSmallSlots) return PNMS_PATH_TILES;
    // one wave of 1024-thread CTAs (two boxes per thread) when the batch fits the SMs
    return (n_max <= 2048 && batch <= sm_count()) ? PNMS_PATH_BINNED_WIDE : PNMS_PATH_BINNED;
  }
  if (batch <= 2 || !cluster_fits(n_max, cs)) return PNMS_PATH_TILES;
  return PNMS_PATH_CLUSTER;
}

struct MapShape {
  int R, RB, chunk;
};

int items_per_frame(int n_max, int RB, int chunk) {
  int ipf = 0;
  for (int rb = 0; rb * RB < n_max; ++rb) ipf += (std::min((rb + 1) * RB - 1, n_max) + chunk - 1) / chunk;
  return ipf;
}

// Work-item shape: the largest (rows-per-lane, chunk) whose item count still gives every SM
// a few items to balance the triangular work (measured on B200 with tools/tune_map.py).
MapShape choose_map_shape(int batch, int n_max, const pnms_launch_config& lc) {
  static const int cand[][2] = {{4, 1024}, {4, 512}, {2, 512}, {2, 256}, {1, 256}};
  MapShape m{1, kMapWarps * 32, 256};
  for (const auto& c : cand) {
    const long long items = (long long)batch * items_per_frame(n_max, kMapWarps * 32 * c[0], c[1]);
    m.R = c[0];
    m.chunk = c[1];
    if (items >= 512) break;
  }
  if (lc.map_rows == 1 || lc.map_rows == 2 || lc.map_rows == 4) m.R = lc.map_rows;
  if (lc.map_chunk >= 32 && lc.map_chunk <= 4096 && (lc.map_chunk % 32) == 0) m.chunk = lc.map_chunk;
  m.RB = kMapWarps * 32 * m.R;
  return m;
}

// when the host launches the fallback chain (profiled calls, host_chain): the declined
// count is snapshotted for the chain and zeroed for the next call, as the dispatcher does
__global__ void pnms_count_snapshot(int* count, int* snap, int batch) {
  pdl_wait();
  if (threadIdx.x == 0) {
    *snap = min(max(*count, 0), batch);
    *count = 0;
  }
}

// the binned path's declined-frame count lives in the persistent zeroed scratch
// (pnms_workspace_init), after the small path's words; every call leaves it zero
constexpr size_t kDeclCountOffset = kSmallMaxWords * 4 + kSmallMaxFrames * 4 + kSmallMaxFrames * 8;
static_assert(kDeclCountOffset + 4 <= kSmallScratchBytes, "scratch");
// the tile path's decline flags and survivor masks, re-zeroed by pnms_mask_compact
constexpr size_t kTilesScratchOffset = 32 * 1024;
static_assert(kDeclCountOffset + 4 <= kTilesScratchOffset, "scratch");
// the cooperative path's frame scratch and its double-buffered survivor masks (frames of up to
// PNMS_MAX_SLOTS): a region of its own, since a cooperative call leaves it non-zero
constexpr size_t kCoopScratchOffset = 64 * 1024;
static_assert(kCoopScratchOffset + kCoopScratchBytes <= kSmallScratchBytes, "scratch");

template <int R>
cudaError_t launch_map(const MapArgs& ma, long long grid, size_t smem, cudaStream_t st, bool list) {
  if (list) {
    cudaError_t e = ensure_smem(pnms_map_kernel_list<R>, smem, g_map_list_smem[R]);
    if (e != cudaSuccess) return e;
    return launch_maybe_pdl(true, pnms_map_kernel_list<R>, dim3((unsigned)grid), dim3(kMapWarps * 32), smem, st, ma);
  }
  cudaError_t e = ensure_smem(pnms_map_kernel<R>, smem, g_map_smem[R]);
  if (e != cudaSuccess) return e;
  pnms_map_kernel<R><<<(unsigned)grid, kMapWarps * 32, smem, st>>>(ma);
  return cudaGetLastError();
}

// WorkCounters.map_writes from the scores alone (pnms_gate.cuh), for the culling paths; runs
// after the call's other kernels and reuses the workspace from the record region on
cudaError_t launch_gate_pairs(const double* s, const int32_t* counts, int batch, int n_max, int d_max, int tie_break,
                              uint64_t* gate_pairs, uint8_t* ws, const Layout& L, cudaStream_t st) {
  GateArgs ga;
  ga.s = s; ga.counts = counts; ga.batch = batch; ga.n_max = n_max; ga.d_max = d_max; ga.tie_break = tie_break;
  ga.cap = 2 * n_max;
  const size_t keys_b = (size_t)batch * ga.cap * 8, mult_b = (size_t)batch * ga.cap * 4;
  ga.keys = reinterpret_cast<unsigned long long*>(ws + L.rec);
  ga.mult = reinterpret_cast<uint32_t*>(ws + L.rec + keys_b);
  ga.acc = reinterpret_cast<unsigned long long*>(ws + L.rec + keys_b + mult_b);  // 8 B aligned
  ga.gate_pairs = reinterpret_cast<unsigned long long*>(gate_pairs);
  // keys + multiplicities + accumulators: 24 B per slot + 16 B per frame <= the 40 B per slot
  // of the record, perm and lim regions that follow each other from L.rec
  cudaError_t e = cudaMemsetAsync(ws + L.rec, 0, keys_b + mult_b + (size_t)batch * 16, st);
  if (e != cudaSuccess) return e;
  pnms_gate_ties<<<dim3((unsigned)((n_max + kGateThreads - 1) / kGateThreads), (unsigned)batch), kGateThreads, 0, st>>>(ga);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  pnms_gate_finalize<<<(unsigned)((batch + kGateThreads - 1) / kGateThreads), kGateThreads, 0, st>>>(ga);
  return cudaGetLastError();
}

inline cudaError_t mark(void* const* events, int i, cudaStream_t st) {
  if (!events || !events[i]) return cudaSuccess;
  return cudaEventRecord((cudaEvent_t)events[i], st);
}

int run_impl(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
             int batch, int n_max, int d_max, double theta, int tie_break, int32_t* keep_idx,
             int32_t* keep_count, uint32_t* keep_mask, uint64_t* gate_pairs, void* workspace,
             size_t workspace_bytes, void* stream, const pnms_launch_config* config, pnms_run_info* info,
             void* const* events) {
  if (!(theta >= 0.0 && theta <= 1.0)) return PNMS_EINVAL_THETA;
  if (d_max < 1) return PNMS_EINVAL_DMAX;
  if (tie_break != PNMS_TIE_PAPER_FAITHFUL && tie_break != PNMS_TIE_BY_INDEX) return PNMS_EINVAL_TIE;
  if (batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (n_max > PNMS_MAX_SLOTS) return PNMS_ETOO_LARGE;
  const pnms_launch_config lc = config ? *config : pnms_launch_config{};
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (info) info->path = PNMS_PATH_AUTO;
  if (lc.declined && (e = cudaMemsetAsync(lc.declined, 0, sizeof(int32_t), st)) != cudaSuccess) return fail_cuda(e);
  if (batch == 0 || n_max == 0) {
    if (batch > 0 && keep_count) {
      e = cudaMemsetAsync(keep_count, 0, sizeof(int32_t) * batch, st);
      if (e != cudaSuccess) return fail_cuda(e);
    }
    if (batch > 0 && gate_pairs) {
      // all d_max slots are padding (0,0,0,0.0): only by_index gates equal-score pairs
      // (handled on the host side of the Python layer; here report zero work)
      e = cudaMemsetAsync(gate_pairs, 0, sizeof(uint64_t) * batch, st);
      if (e != cudaSuccess) return fail_cuda(e);
    }
    return PNMS_OK;
  }
  if (!x || !y || !z || !s) return PNMS_EINVAL_ARG;
  const Layout L = make_layout(batch, n_max);
  if (!workspace || workspace_bytes < L.total) return PNMS_EWORKSPACE;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int W32 = (n_max + 31) / 32;
  const int cs = cluster_size_for(n_max, lc.cluster_size);
  int path = lc.path;
  if (path != PNMS_PATH_AUTO && !path_fits(path, batch, n_max, cs)) path = PNMS_PATH_AUTO;
  if (path == PNMS_PATH_AUTO) path = auto_path(batch, n_max, cs);
  if (info) info->path = path;

  if (path == PNMS_PATH_SMALL) {
    SmallArgs sa;
    sa.x = x; sa.y = y; sa.z = z; sa.s = s; sa.counts = counts;
    sa.batch = batch; sa.n_max = n_max; sa.d_max = d_max; sa.tie_break = tie_break; sa.W32 = W32;
    sa.theta = theta;
    const int R = ((long long)batch * n_max <= 2048) ? 1 : kSmallRowsMax;  // tiny calls: more CTAs
    sa.n_rt = (n_max + kSmallThreads * R - 1) / (kSmallThreads * R);
    const int max_ct = (n_max + 31) / 32;
    int n_ct = (int)std::min<long long>(max_ct, std::max<long long>(1, (2LL * 148 + (long long)batch * sa.n_rt - 1) /
                                                                         ((long long)batch * sa.n_rt)));
    if (lc.small_col_tiles > 0) n_ct = std::min(lc.small_col_tiles, max_ct);
    sa.cols = ((n_max + n_ct - 1) / n_ct + 31) / 32 * 32;
    sa.n_ct = (n_max + sa.cols - 1) / sa.cols;
    sa.supp = reinterpret_cast<uint32_t*>(ws);
    sa.ticket = reinterpret_cast<unsigned int*>(ws + kSmallMaxWords * 4);
    sa.gacc = reinterpret_cast<unsigned long long*>(ws + kSmallMaxWords * 4 + kSmallMaxFrames * 4);
    sa.keep_idx = keep_idx; sa.keep_count = keep_count; sa.keep_mask = keep_mask;
    sa.gate_pairs = reinterpret_cast<unsigned long long*>(gate_pairs);
    const size_t smem = (size_t)sa.cols * (8 + sizeof(RecWide));
    const long long grid = (long long)batch * sa.n_rt * sa.n_ct;
    if ((e = mark(events, 0, st)) != cudaSuccess) return fail_cuda(e);
    if ((e = mark(events, 1, st)) != cudaSuccess) return fail_cuda(e);
    const int variant = (tie_break == PNMS_TIE_BY_INDEX ? 2 : 0) + (gate_pairs != nullptr ? 1 : 0) + (R == 1 ? 4 : 0);
    if ((e = launch_small(variant, sa, grid, smem, st)) != cudaSuccess) return fail_cuda(e);
    if ((e = mark(events, 2, st)) != cudaSuccess) return fail_cuda(e);
    if ((e = mark(events, 3, st)) != cudaSuccess) return fail_cuda(e);
    return PNMS_OK;
  }

  // arguments of the dense pipeline (prep+sort -> map -> compact) for frames [f0, f0 + nf)
  const MapShape ms = choose_map_shape(batch, n_max, lc);
  const bool culling = path != PNMS_PATH_DENSE;
  // the culling paths count map_writes from the scores (pnms_gate.cuh); the dense pipeline
  // counts the gate passes of its own sorted map
  uint64_t* dense_gate = culling ? nullptr : gate_pairs;
  auto chain_args = [&](int f0, int nf, const uint8_t* dense, const int32_t* list, const int* list_count,
                        PrepArgs& pa, MapArgs& ma, CompactArgs& ca) {
    const size_t fo = (size_t)f0 * n_max;
    pa.x = x + fo; pa.y = y + fo; pa.z = z + fo; pa.s = s + fo; pa.counts = counts ? counts + f0 : nullptr;
    pa.batch = nf; pa.n_max = n_max; pa.tie_break = tie_break; pa.W32 = W32;
    pa.theta = theta;
    pa.rec = ws + L.rec + fo * kRecBytes;
    pa.perm = reinterpret_cast<int32_t*>(ws + L.perm) + fo;
    pa.lim = reinterpret_cast<int32_t*>(ws + L.lim) + fo;
    pa.supp = reinterpret_cast<uint32_t*>(ws + L.supp) + (size_t)f0 * W32;
    pa.meta = reinterpret_cast<FrameMeta*>(ws + L.meta) + f0;
    pa.sk_scratch = L.sk ? reinterpret_cast<uint64_t*>(ws + L.sk) + fo : nullptr;
    pa.idx_scratch = L.idx ? reinterpret_cast<int32_t*>(ws + L.idx) + fo : nullptr;
    pa.dense = dense ? dense + f0 : nullptr;
    pa.list = list;
    pa.list_count = list_count;
    if (n_max <= kSortMax) {
      pa.npad = (n_max + kSortThreads - 1) / kSortThreads * kSortThreads;
      pa.nchunks = 1;
    } else {
      pa.npad = kSortMax;
      pa.nchunks = (n_max + kSortMax - 1) / kSortMax;
    }
    ma.rec = pa.rec; ma.lim = pa.lim; ma.supp = pa.supp; ma.meta = pa.meta;
    ma.batch = nf; ma.n_max = n_max; ma.W32 = W32;
    ma.rows_per_block = ms.RB;
    ma.chunk = ms.chunk;
    ma.n_rb = (n_max + ms.RB - 1) / ms.RB;
    ma.items_per_frame = items_per_frame(n_max, ms.RB, ms.chunk);
    ma.dense = pa.dense;
    ma.list = list;
    ma.list_count = list_count;
    ca.s = pa.s; ca.counts = pa.counts; ca.perm = pa.perm; ca.supp = pa.supp; ca.meta = pa.meta;
    ca.batch = nf; ca.n_max = n_max; ca.W32 = W32; ca.d_max = d_max; ca.tie_break = tie_break;
    ca.keep_idx = keep_idx ? keep_idx + fo : nullptr;
    ca.keep_count = keep_count ? keep_count + f0 : nullptr;
    ca.keep_mask = keep_mask ? keep_mask + (size_t)f0 * W32 : nullptr;
    ca.gate_pairs = dense_gate ? reinterpret_cast<unsigned long long*>(dense_gate) + f0 : nullptr;
    ca.dense = pa.dense;
    ca.list = list;
    ca.list_count = list_count;
  };
  const size_t compact_smem = ((size_t)W32 + 3) / 4 * 16 + 64 * 4;
  const size_t map_smem = (size_t)ms.chunk * kRecBytes;
  // one-CTA dispatcher behind a declining kernel (pnms_fallback.cuh): snapshots the declined
  // count into `snap`, zeroes it and, when frames were declined, tail-launches the dense chain
  // over them; `*host_chain` is set when the host must launch the chain itself (profiled calls)
  auto make_plan = [&](const int32_t* list, const int* snap) {
    FallbackPlan plan{};
    chain_args(0, batch, ws + L.dense, list, snap, plan.pa, plan.ma, plan.ca);
    plan.chunked = n_max > kSortMax;
    plan.map_R = ms.R;
    plan.sort_smem = (int)(plan.chunked ? sort_smem_bytes(kSortMax) : sort_frame_smem_bytes(plan.pa.npad));
    plan.map_smem = (int)map_smem;
    plan.compact_smem = (int)compact_smem;
    return plan;
  };
  auto dispatch_fallback = [&](const int32_t* list, int* count, int* snap, bool* host_chain) -> cudaError_t {
    FallbackPlan plan = make_plan(list, snap);
#ifdef PNMS_NO_DEVCHAIN  // diagnostic build without the relocatable unit (sanitizer tools)
    plan.enabled = 0;
#else
    plan.enabled = events == nullptr && lc.host_chain == 0;
#endif
    *host_chain = !plan.enabled;
    cudaError_t err;
    if (!plan.enabled) {  // snapshot + zero only; the host launches the chain over `snap`
      err = launch_maybe_pdl(true, pnms_count_snapshot, dim3(1), dim3(32), 0, st, count, snap, batch);
    } else {
#ifndef PNMS_NO_DEVCHAIN
      static const bool same_layout = pnms_devchain_plan_size() == sizeof(FallbackPlan);
      if (!same_layout) return cudaErrorInvalidValue;
      err = pnms_devchain_prepare(plan.chunked, ms.R, plan.sort_smem, map_smem, compact_smem);
      if (err == cudaSuccess) err = pnms_devchain_dispatch(&plan, count, snap, st);
#else
      err = cudaSuccess;
#endif
    }
    if (err == cudaSuccess && lc.declined)
      err = cudaMemcpyAsync(lc.declined, snap, sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
    return err;
  };
  // the counter runs behind everything else of the call (stream order includes the
  // dispatcher's tail launches)
  auto finish = [&]() -> int {
    if (culling && gate_pairs) {
      cudaError_t err = launch_gate_pairs(s, counts, batch, n_max, d_max, tie_break, gate_pairs, ws, L, st);
      if (err != cudaSuccess) return fail_cuda(err);
    }
    return PNMS_OK;
  };

  const uint8_t* dense_flags = nullptr;
  const int32_t* decl_list = nullptr;  // culling paths: the declined frames, read on the device
  const int* decl_count = nullptr;
  void* ev_local[4];
  BinArgs ba{};
  ba.x = x; ba.y = y; ba.z = z; ba.s = s; ba.counts = counts;
  ba.batch = batch; ba.n_max = n_max; ba.d_max = d_max; ba.tie_break = tie_break; ba.W32 = W32;
  ba.theta = theta;
  ba.fallback = ws + L.dense;
  ba.decl_count = reinterpret_cast<int*>(ws + kDeclCountOffset);  // zeroed scratch, left zero by the dispatcher
  ba.decl_list = reinterpret_cast<int32_t*>(ws + L.list) + 1;
  ba.keep_idx = keep_idx; ba.keep_count = keep_count; ba.keep_mask = keep_mask;
  ba.trace = g_trace;
  ba.cell_q8 = lc.cell_q8;
  ba.cell_sx = lc.cell_sx;
  if (culling) {
    if ((e = mark(events, 0, st)) != cudaSuccess) return fail_cuda(e);
    if (path == PNMS_PATH_COOP) {
      // ---- large single frames: one cooperative launch of T tile CTAs per frame (pnms_coop.cuh)
      ba.pairs_tested = nullptr;
      ba.meta = reinterpret_cast<FrameMeta*>(ws + L.meta);  // the chunked sort accumulates into it
      CoopArgs cargs;
      cargs.b = ba;
      cargs.b.trace = g_trace;
      cargs.scr = reinterpret_cast<CoopFrame*>(ws + kCoopScratchOffset);
      cargs.mask = reinterpret_cast<uint32_t*>(ws + kCoopScratchOffset + kCoopMaxFrames * sizeof(CoopFrame));
      cargs.lists = reinterpret_cast<uint4*>(ws + L.coop);
      cargs.tiles = coop_tiles(batch, n_max, lc.coop_tiles);
      cargs.cap = kCoopCap;
      cargs.count_fallback = lc.declined != nullptr;
      cudaLaunchConfig_t clc = {};
      clc.gridDim = dim3((unsigned)(batch * cargs.tiles));
      clc.blockDim = dim3(kCoopThreads);
      clc.dynamicSmemBytes = 0;
      clc.stream = st;
      cudaLaunchAttribute cattr[1];
      cattr[0].id = cudaLaunchAttributeCooperative;
      cattr[0].val.cooperative = 1;
      clc.attrs = cattr;
      clc.numAttrs = 1;
      e = cudaLaunchKernelEx(&clc, tie_break == PNMS_TIE_BY_INDEX ? pnms_coop<true> : pnms_coop<false>, cargs);
      if (e == cudaErrorCooperativeLaunchTooLarge) {
        // fewer SMs than the device reports (MPS / green contexts): the tile path instead
        (void)cudaGetLastError();
        path = PNMS_PATH_TILES;
        if (info) info->path = path;
      } else if (e != cudaSuccess) {
        return fail_cuda(e);
      }
    }
    if (path == PNMS_PATH_COOP) {
      // launched above
    } else if (path == PNMS_PATH_BINNED || path == PNMS_PATH_BINNED_WIDE) {
      // ---- exact spatial culling, one CTA per frame (pnms_binned.cuh)
      ba.pairs_tested = g_pairs_counter;
      ba.meta = nullptr;  // the frame-level sort rewrites FrameMeta of declined frames
      const int variant = (tie_break == PNMS_TIE_BY_INDEX ? 1 : 0) + (g_pairs_counter ? 2 : 0);
      // frames a CTA slot runs next: resident CTAs of the 512-thread kernel (3 per SM)
      ba.prefetch_ahead = path == PNMS_PATH_BINNED_WIDE ? sm_count() : 3 * sm_count();
      e = launch_binned(lc.binned_impl, variant, ba, batch, n_max, st, path == PNMS_PATH_BINNED_WIDE);
      if (e != cudaSuccess) return fail_cuda(e);
    } else if (path == PNMS_PATH_TILES) {
      // ---- large single frames: kTilesPerFrame independent tile CTAs per frame (pnms_binned_tiles.cuh)
      ba.pairs_tested = nullptr;
      ba.meta = reinterpret_cast<FrameMeta*>(ws + L.meta);  // the chunked sort accumulates into it
      TileArgs ta;
      ta.b = ba;
      // decline flags and survivor masks in the zeroed scratch (pnms_mask_compact re-zeroes
      // them) when they fit — the latency case, <= 2 frames — else zeroed per call
      const size_t fbytes = ((size_t)batch * 4 + 15) / 16 * 16;
      const size_t tbytes = fbytes + (size_t)batch * W32 * 4;
      const bool in_scratch = kTilesScratchOffset + tbytes <= kCoopScratchOffset;
      uint8_t* tbase = in_scratch ? ws + kTilesScratchOffset : (L.tiles ? ws + L.tiles : ws + L.rec);
      ta.decline = reinterpret_cast<int*>(tbase);
      ta.mask = reinterpret_cast<uint32_t*>(tbase + fbytes);
      if (!in_scratch && (e = cudaMemsetAsync(tbase, 0, tbytes, st)) != cudaSuccess) return fail_cuda(e);
      const size_t tsmem = binned_tiles_smem_bytes();
      const bool bi = tie_break == PNMS_TIE_BY_INDEX;
      if ((e = ensure_smem(bi ? pnms_binned_tiles<true> : pnms_binned_tiles<false>, tsmem, g_tiles_smem[bi])) != cudaSuccess)
        return fail_cuda(e);
      if ((e = launch_maybe_pdl(false, bi ? pnms_binned_tiles<true> : pnms_binned_tiles<false>,
                                dim3((unsigned)batch * kTilesPerFrame), dim3(kTileThreads), tsmem, st, ta)) != cudaSuccess)
        return fail_cuda(e);
      if ((e = launch_maybe_pdl(true, pnms_mask_compact, dim3((unsigned)batch), dim3(512), 0, st, ta)) != cudaSuccess)
        return fail_cuda(e);
    } else {
      // ---- large frames in batches: one thread-block cluster per frame (pnms_binned_cluster.cuh)
      ba.pairs_tested = nullptr;
      ba.meta = reinterpret_cast<FrameMeta*>(ws + L.meta);
      if ((e = launch_cluster(ba, batch, cs, cluster_slice(n_max, cs), tie_break == PNMS_TIE_BY_INDEX, st)) !=
          cudaSuccess)
        return fail_cuda(e);
    }
    // declined frames: the dense pipeline, tail-launched from the device by the dispatcher
    decl_list = ba.decl_list;
    int* snap = reinterpret_cast<int*>(ws + L.list);
    bool host_chain = false;
    if (path == PNMS_PATH_COOP) {
      // the cooperative kernel finishes the frames it declines itself (no fallback chain);
      // the count of those frames, when the caller asks for it, through the snapshot kernel
      if (lc.declined) {
        int* snap = reinterpret_cast<int*>(ws + L.list);
        if ((e = launch_maybe_pdl(true, pnms_count_snapshot, dim3(1), dim3(32), 0, st, ba.decl_count, snap, batch)) !=
                cudaSuccess ||
            (e = cudaMemcpyAsync(lc.declined, snap, sizeof(int32_t), cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
          return fail_cuda(e);
      }
      if ((e = mark(events, 3, st)) != cudaSuccess) return fail_cuda(e);
      return finish();
    }
    if ((e = dispatch_fallback(ba.decl_list, ba.decl_count, snap, &host_chain)) != cudaSuccess) return fail_cuda(e);
    if (!host_chain) {
      if ((e = mark(events, 3, st)) != cudaSuccess) return fail_cuda(e);
      return finish();
    }
    decl_count = snap;
    dense_flags = ws + L.dense;
    if (events) {
      // phases become: [0,1) culling kernel, [1,2) dense prep of declined frames, [2,3) their map+compact
      ev_local[0] = events[1]; ev_local[1] = events[2]; ev_local[2] = nullptr; ev_local[3] = events[3];
      events = ev_local;
    }
  }

  // ---- sorted pipeline: prep+sort -> map -> compact (every frame, or the declined list)
  {
    const int nf = batch;
    PrepArgs pa;
    MapArgs ma;
    CompactArgs ca;
    chain_args(0, nf, dense_flags, decl_list, decl_count, pa, ma, ca);
    if ((e = mark(events, 0, st)) != cudaSuccess) return fail_cuda(e);
    if (n_max <= kSortMax) {
      const size_t smem = sort_frame_smem_bytes(pa.npad);
      if (decl_list) {
        if ((e = ensure_smem(pnms_prep_sort_frame_list, smem, g_sort_list_smem)) != cudaSuccess) return fail_cuda(e);
        if ((e = launch_maybe_pdl(true, pnms_prep_sort_frame_list, dim3(std::min(nf, 148 * 2)), dim3(kSortThreads),
                                  smem, st, pa)) != cudaSuccess)
          return fail_cuda(e);
      } else {
        if ((e = ensure_smem(pnms_prep_sort_frame, smem, g_sort_frame_smem)) != cudaSuccess) return fail_cuda(e);
        pnms_prep_sort_frame<<<nf, kSortThreads, smem, st>>>(pa);
        if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e);
      }
    } else {
      // the declined-frame list path had each frame's FrameMeta zeroed by the decliner
      if (!decl_list && (e = cudaMemsetAsync(pa.meta, 0, sizeof(FrameMeta) * (size_t)nf, st)) != cudaSuccess)
        return fail_cuda(e);
      const size_t smem = sort_smem_bytes(kSortMax);
      if ((e = ensure_smem(pnms_prep_sort_chunk, smem, g_sort_chunk_smem)) != cudaSuccess) return fail_cuda(e);
      const long long cgrid = (long long)nf * pa.nchunks;
      if ((e = launch_maybe_pdl(decl_list != nullptr, pnms_prep_sort_chunk,
                                dim3((unsigned)(decl_list ? std::min<long long>(cgrid, 148 * 2) : cgrid)),
                                dim3(kSortThreads), smem, st, pa)) != cudaSuccess)
        return fail_cuda(e);
      const long long blocks = (long long)nf * ((n_max + 255) / 256);
      if ((e = launch_maybe_pdl(decl_list != nullptr, pnms_merge_rank,
                                dim3((unsigned)(decl_list ? std::min<long long>(blocks, 148 * 8) : blocks)), dim3(256), 0,
                                st, pa)) != cudaSuccess)
        return fail_cuda(e);
    }
    if ((e = mark(events, 1, st)) != cudaSuccess) return fail_cuda(e);
    const int ipf = ma.items_per_frame;
    const long long grid = decl_list ? std::min<long long>((long long)nf * ipf, 148 * 8) : (long long)nf * ipf;
    if (grid > 0x7FFFFFFFLL) return PNMS_ETOO_LARGE;
    const bool pdl = decl_list != nullptr;
    if (ms.R == 4) e = launch_map<4>(ma, grid, map_smem, st, pdl);
    else if (ms.R == 2) e = launch_map<2>(ma, grid, map_smem, st, pdl);
    else e = launch_map<1>(ma, grid, map_smem, st, pdl);
    if (e != cudaSuccess) return fail_cuda(e);
    if ((e = mark(events, 2, st)) != cudaSuccess) return fail_cuda(e);
    if ((e = ensure_smem(pnms_compact, compact_smem, g_compact_smem)) != cudaSuccess) return fail_cuda(e);
    if ((e = launch_maybe_pdl(decl_list != nullptr, pnms_compact, dim3(decl_list ? std::min(nf, 148 * 4) : nf),
                              dim3(kCompactThreads), compact_smem, st, ca)) != cudaSuccess)
      return fail_cuda(e);
  }
  if ((e = mark(events, 3, st)) != cudaSuccess) return fail_cuda(e);
  return finish();
}

}  // namespace

extern "C" {

const char* pnms_version(void) { return "parnms_b200 0.1.0 sm_100a"; }

int pnms_last_cuda_error(void) { return g_last_cuda_error; }

const char* pnms_strerror(int status) {
  switch (status) {
    case PNMS_OK: return "ok";
    case PNMS_EINVAL_THETA: return "theta must be in [0, 1]";
    case PNMS_EINVAL_DMAX: return "d_max must be positive and hold every frame's detections";
    case PNMS_EINVAL_TIE: return "tie_break must be paper_faithful (0) or by_index (1)";
    case PNMS_EINVAL_ARG: return "invalid argument (null pointer or negative size)";
    case PNMS_EWORKSPACE: return "workspace missing or smaller than pnms_workspace_bytes()";
    case PNMS_ETOO_LARGE: return "n_max exceeds PNMS_MAX_SLOTS";
    case PNMS_ECUDA: return "CUDA launch failed (see pnms_last_cuda_error)";
    case PNMS_EINVAL_K: return "k must be positive and divide d_max";
    default: return "unknown parnms_b200 status";
  }
}

int pnms_validate(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                  int batch, int n_max, int32_t* first_bad, int32_t* reason, void* stream) {
  if (batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (batch == 0) return PNMS_OK;
  if (!first_bad || !reason || (n_max > 0 && (!x || !y || !z || !s))) return PNMS_EINVAL_ARG;
  pnms_validate_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(x, y, z, s, counts, n_max, first_bad, reason);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PNMS_OK : fail_cuda(e);
}

int pnms_variant_workspace_bytes(int batch, int n_max, size_t* out_bytes) {
  if (!out_bytes || batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (n_max > PNMS_MAX_SLOTS) return PNMS_ETOO_LARGE;
  *out_bytes = n_max <= kGreedyMaxSlots ? 0 : (size_t)batch * std::max(greedy_smem_bytes(n_max), soft_smem_bytes(n_max));
  return PNMS_OK;
}

int pnms_greedy_run_ws(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                       int batch, int n_max, double theta, int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!(theta >= 0.0 && theta <= 1.0)) return PNMS_EINVAL_THETA;
  if (batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (n_max > PNMS_MAX_SLOTS) return PNMS_ETOO_LARGE;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (batch == 0) return PNMS_OK;
  if (n_max == 0) {
    if (keep_count && (e = cudaMemsetAsync(keep_count, 0, sizeof(int32_t) * batch, st)) != cudaSuccess) return fail_cuda(e);
    return PNMS_OK;
  }
  if (!x || !y || !z || !s) return PNMS_EINVAL_ARG;
  GreedyArgs ga;
  ga.x = x; ga.y = y; ga.z = z; ga.s = s; ga.counts = counts;
  ga.batch = batch; ga.n_max = n_max; ga.W32 = (n_max + 31) / 32; ga.theta = theta;
  ga.keep_idx = keep_idx; ga.keep_count = keep_count; ga.keep_mask = keep_mask;
  ga.scratch = static_cast<unsigned char*>(workspace);
  ga.scratch_stride = greedy_smem_bytes(n_max);
  if (n_max <= kGreedyMaxSlots) {  // per-slot state in shared memory
    static SmemCache cfg;
    const size_t smem = greedy_smem_bytes(n_max);
    if ((e = ensure_smem(pnms_greedy_frame<false>, smem, cfg)) != cudaSuccess) return fail_cuda(e);
    pnms_greedy_frame<false><<<batch, kGreedyThreads, smem, st>>>(ga);
  } else {                         // large frames: the same state in the caller's workspace
    if (!workspace || workspace_bytes < (size_t)batch * ga.scratch_stride) return PNMS_EWORKSPACE;
    pnms_greedy_frame<true><<<batch, kGreedyThreads, 0, st>>>(ga);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e);
  return PNMS_OK;
}

int pnms_greedy_run(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                    int batch, int n_max, double theta, int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask,
                    void* stream) {
  if (n_max > kGreedyMaxSlots) return PNMS_ETOO_LARGE;  // larger frames: pnms_greedy_run_ws
  return pnms_greedy_run_ws(x, y, z, s, counts, batch, n_max, theta, keep_idx, keep_count, keep_mask, nullptr, 0,
                            stream);
}

int pnms_soft_rescore_ws(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                         int batch, int n_max, int mode, double theta, double sigma, double* out_s, int32_t* status,
                         int32_t* rounds, void* workspace, size_t workspace_bytes, void* stream) {
  if (mode != 0 && mode != 1) return PNMS_EINVAL_ARG;
  if (!(sigma > 0.0)) return PNMS_EINVAL_ARG;
  if (batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (n_max > PNMS_MAX_SLOTS) return PNMS_ETOO_LARGE;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (batch == 0) return PNMS_OK;
  if (!status) return PNMS_EINVAL_ARG;
  if (n_max == 0) {
    if ((e = cudaMemsetAsync(status, 0, sizeof(int32_t) * batch, st)) != cudaSuccess) return fail_cuda(e);
    return PNMS_OK;
  }
  if (!x || !y || !z || !s || !out_s) return PNMS_EINVAL_ARG;
  SoftArgs sa;
  sa.x = x; sa.y = y; sa.z = z; sa.s = s; sa.counts = counts;
  sa.batch = batch; sa.n_max = n_max; sa.mode = mode; sa.theta = theta; sa.sigma = sigma;
  sa.out_s = out_s; sa.status = status; sa.rounds = rounds;
  sa.scratch = static_cast<unsigned char*>(workspace);
  sa.scratch_stride = soft_smem_bytes(n_max);
  if (n_max <= kSoftMaxSlots) {
    static SmemCache cfg;
    const size_t smem = soft_smem_bytes(n_max);
    if ((e = ensure_smem(pnms_soft_frame<false>, smem, cfg)) != cudaSuccess) return fail_cuda(e);
    pnms_soft_frame<false><<<batch, kSoftThreads, smem, st>>>(sa);
  } else {
    if (!workspace || workspace_bytes < (size_t)batch * sa.scratch_stride) return PNMS_EWORKSPACE;
    pnms_soft_frame<true><<<batch, kSoftThreads, 0, st>>>(sa);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e);
  return PNMS_OK;
}

int pnms_soft_rescore(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                      int batch, int n_max, int mode, double theta, double sigma, double* out_s, int32_t* status,
                      int32_t* rounds, void* stream) {
  if (n_max > kSoftMaxSlots) return PNMS_ETOO_LARGE;  // larger frames: pnms_soft_rescore_ws
  return pnms_soft_rescore_ws(x, y, z, s, counts, batch, n_max, mode, theta, sigma, out_s, status, rounds, nullptr, 0,
                              stream);
}

int pnms_widen_i16(const int16_t* x16, const int16_t* y16, const int16_t* z16, int32_t* x, int32_t* y, int32_t* z,
                   long long n, void* stream) {
  if (n < 0 || (n > 0 && (!x16 || !y16 || !z16 || !x || !y || !z))) return PNMS_EINVAL_ARG;
  if (n == 0) return PNMS_OK;
  const long long blocks = std::min<long long>((n + 1023) / 1024, 148LL * 16);
  pnms_widen_i16_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x16, y16, z16, x, y, z, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PNMS_OK : fail_cuda(e);
}

int pnms_unpack_box32(const uint32_t* box, int32_t* x, int32_t* y, int32_t* z, long long n, void* stream) {
  if (n < 0 || (n > 0 && (!box || !x || !y || !z))) return PNMS_EINVAL_ARG;
  if (n == 0) return PNMS_OK;
  const long long blocks = std::min<long long>((n + 1023) / 1024, 148LL * 16);
  pnms_unpack_box32_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(box, x, y, z, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PNMS_OK : fail_cuda(e);
}

int pnms_pack_box32_host(const int32_t* x, const int32_t* y, const int32_t* z, long long n, uint32_t* box,
                         int threads, int* packable) {
  if (!packable || n < 0 || (n > 0 && (!x || !y || !z || !box))) return PNMS_EINVAL_ARG;
  int bad = 0;
  // one streaming pass over 16 B per box (12 read, 4 written): memory-bound, so every core;
  // four boxes per step with SSE2, the words written with non-temporal stores (no read for
  // ownership of the output lines: the host memory bus is shared with the DMA reading them)
  const long long head = std::min<long long>(n, (long long)((16 - (reinterpret_cast<uintptr_t>(box) & 15)) & 15) / 4);
  const long long n4 = (n - head) / 4;
  for (long long i = 0; i < head; ++i) {
    const uint32_t xv = (uint32_t)x[i], yv = (uint32_t)y[i], zv = (uint32_t)z[i];
    bad |= (int)((xv > 4095u) | (yv > 4095u) | (zv > 255u));
    box[i] = xv | (yv << 12) | (zv << 24);
  }
#pragma omp parallel reduction(| : bad) num_threads(threads > 0 ? threads : omp_get_num_procs())
  {
#pragma omp for schedule(static) nowait
  for (long long q = 0; q < n4; ++q) {
    const long long i = head + 4 * q;
    const __m128i xv = _mm_loadu_si128(reinterpret_cast<const __m128i*>(x + i));
    const __m128i yv = _mm_loadu_si128(reinterpret_cast<const __m128i*>(y + i));
    const __m128i zv = _mm_loadu_si128(reinterpret_cast<const __m128i*>(z + i));
    // out of domain <=> any bit outside the field (as unsigned: negatives have the top bit)
    const __m128i over = _mm_or_si128(_mm_or_si128(_mm_andnot_si128(_mm_set1_epi32(4095), xv),
                                                   _mm_andnot_si128(_mm_set1_epi32(4095), yv)),
                                      _mm_andnot_si128(_mm_set1_epi32(255), zv));
    bad |= _mm_movemask_epi8(_mm_cmpeq_epi32(over, _mm_setzero_si128())) != 0xFFFF;
    const __m128i w = _mm_or_si128(_mm_or_si128(xv, _mm_slli_epi32(yv, 12)), _mm_slli_epi32(zv, 24));
    _mm_stream_si128(reinterpret_cast<__m128i*>(box + i), w);
  }
  _mm_sfence();  // this thread's streaming stores are globally visible before the region ends
  }
  for (long long i = head + 4 * n4; i < n; ++i) {
    const uint32_t xv = (uint32_t)x[i], yv = (uint32_t)y[i], zv = (uint32_t)z[i];
    bad |= (int)((xv > 4095u) | (yv > 4095u) | (zv > 255u));
    box[i] = xv | (yv << 12) | (zv << 24);
  }
  *packable = bad ? 0 : 1;
  return PNMS_OK;
}

int pnms_debug_exp(const double* x, double* y, long long n, void* stream) {
  if (n < 0 || (n > 0 && (!x || !y))) return PNMS_EINVAL_ARG;
  if (n == 0) return PNMS_OK;
  const long long blocks = std::min<long long>((n + 255) / 256, 148LL * 8);
  pnms_exp_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(x, y, n);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PNMS_OK : fail_cuda(e);
}

int pnms_debug_trace(uint64_t* device_buffer) {
  g_trace = reinterpret_cast<unsigned long long*>(device_buffer);
  return PNMS_OK;
}

int pnms_debug_count_pairs(uint64_t* device_counter) {
  g_pairs_counter = reinterpret_cast<unsigned long long*>(device_counter);
  return PNMS_OK;
}

int pnms_workspace_init(void* workspace, size_t workspace_bytes, void* stream) {
  if (!workspace || workspace_bytes < kSmallScratchBytes) return PNMS_EWORKSPACE;
  cudaError_t e = cudaMemsetAsync(workspace, 0, kSmallScratchBytes, (cudaStream_t)stream);
  return e == cudaSuccess ? PNMS_OK : fail_cuda(e);
}

int pnms_workspace_bytes(int batch, int n_max, size_t* out_bytes) {
  if (!out_bytes || batch < 0 || n_max < 0) return PNMS_EINVAL_ARG;
  if (n_max > PNMS_MAX_SLOTS) return PNMS_ETOO_LARGE;
  *out_bytes = make_layout(batch, n_max).total;
  return PNMS_OK;
}

}  // extern "C"

extern "C" {

int pnms_run(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
             int batch, int n_max, int d_max, double theta, int tie_break, int32_t* keep_idx,
             int32_t* keep_count, uint32_t* keep_mask, uint64_t* gate_pairs, void* workspace,
             size_t workspace_bytes, void* stream) {
  return run_impl(x, y, z, s, counts, batch, n_max, d_max, theta, tie_break, keep_idx, keep_count, keep_mask,
                  gate_pairs, workspace, workspace_bytes, stream, nullptr, nullptr, nullptr);
}

int pnms_run_profiled(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                      const int32_t* counts, int batch, int n_max, int d_max, double theta, int tie_break,
                      int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask, uint64_t* gate_pairs,
                      void* workspace, size_t workspace_bytes, void* stream, void* const* phase_events) {
  return run_impl(x, y, z, s, counts, batch, n_max, d_max, theta, tie_break, keep_idx, keep_count, keep_mask,
                  gate_pairs, workspace, workspace_bytes, stream, nullptr, nullptr, phase_events);
}

int pnms_run_ex(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, const int32_t* counts,
                int batch, int n_max, int d_max, double theta, int tie_break, int32_t* keep_idx, int32_t* keep_count,
                uint32_t* keep_mask, uint64_t* gate_pairs, void* workspace, size_t workspace_bytes, void* stream,
                const pnms_launch_config* config, pnms_run_info* info, void* const* phase_events) {
  return run_impl(x, y, z, s, counts, batch, n_max, d_max, theta, tie_break, keep_idx, keep_count, keep_mask,
                  gate_pairs, workspace, workspace_bytes, stream, config, info, phase_events);
}

int pnms_map_reference_layout(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, int d_max,
                              double theta, int tie_break, uint64_t* bits, uint64_t* gate_pairs, void* stream) {
  if (!(theta >= 0.0 && theta <= 1.0)) return PNMS_EINVAL_THETA;
  if (d_max < 1) return PNMS_EINVAL_DMAX;
  if (tie_break != PNMS_TIE_PAPER_FAITHFUL && tie_break != PNMS_TIE_BY_INDEX) return PNMS_EINVAL_TIE;
  if (!x || !y || !z || !s || !bits) return PNMS_EINVAL_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  RefMapArgs ra;
  ra.x = x; ra.y = y; ra.z = z; ra.s = s;
  ra.d_max = d_max; ra.W64 = (d_max + 63) / 64; ra.tie_break = tie_break; ra.theta = theta;
  ra.bits = bits;
  ra.gate_pairs = reinterpret_cast<unsigned long long*>(gate_pairs);
  if (gate_pairs && (e = cudaMemsetAsync(gate_pairs, 0, sizeof(uint64_t), st)) != cudaSuccess) return fail_cuda(e);
  const long long units = (long long)d_max * ra.W64;
  const long long blocks = (units + 7) / 8;
  if (blocks > 0x7FFFFFFFLL) return PNMS_ETOO_LARGE;
  pnms_ref_map<<<(unsigned)blocks, 256, 0, st>>>(ra);
  if ((e = cudaGetLastError()) != cudaSuccess) return fail_cuda(e);
  return PNMS_OK;
}

int pnms_reduce_rows(const uint64_t* bits, int d_max, int k, uint8_t* mask, void* stream) {
  if (d_max < 1) return PNMS_EINVAL_DMAX;
  if (k < 1 || d_max % k != 0) return PNMS_EINVAL_K;
  if (!bits || !mask) return PNMS_EINVAL_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int W64 = (d_max + 63) / 64;
  pnms_ref_reduce<<<(d_max + 7) / 8, 256, 0, st>>>(bits, d_max, W64, mask);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e);
  return PNMS_OK;
}

}  // extern "C"
