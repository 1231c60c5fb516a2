// pnms_fallback.cuh — the dense sorted pipeline for frames the single-CTA binned kernel
// declined, launched from the device only when there are such frames.
//
// The binned kernel appends declined frames to a list (binned_decline) and counts them in
// the caller's zeroed scratch (pnms_workspace_init).  A one-CTA dispatcher launched right
// behind it (programmatic dependent launch) snapshots the count, zeroes it for the next call —
// no per-call memset — and, only when it is non-zero, tail-launches the three list kernels
// (prep+sort, map, compact) with grids sized to it.  Tail launches run after the launching
// grid completes and in launch order, and the dispatcher counts as complete for the stream
// only once they are, so the caller's stream order is unchanged.  A batch without declined
// frames costs two launches (binned + dispatcher) instead of a memset and four (BASELINE
// config 4: 27.6 -> ~21 us per call).
//
// Device-side launches need relocatable device code, which costs the kernels compiled that
// way (measured: the map kernel 62 -> 102 registers; the binned kernel 3 % slower on config 5
// when it did the launching itself), so only pnms_devchain.cu — this dispatcher and the three
// list kernels, in namespace pnms_dc — is compiled with -rdc; everything else stays
// whole-program.
#pragma once
#include "pnms_common.cuh"
#include "pnms_compact.cuh"
#include "pnms_map.cuh"
#include "pnms_sort.cuh"

namespace pnms {

struct FallbackPlan {
  PrepArgs pa;      // list / list_count already point at the declined-frame list and snapshot
  MapArgs ma;
  CompactArgs ca;
  int map_R;        // 1, 2 or 4 rows per lane (choose_map_shape)
  int sort_smem, map_smem, compact_smem;
  int chunked;      // frames > kSortMax slots: chunk sorts + merge rank instead of the frame sort
  int enabled;      // 0: the host launches the chain itself (profiled calls), reading the snapshot
};

#ifdef PNMS_DEVICE_CHAIN  // relocatable unit only (pnms_devchain.cu)
// the chain over c declined frames (plan's list), as tail launches of the calling grid
__device__ __forceinline__ void launch_fallback_chain(const FallbackPlan& plan, int c) {
  if (plan.chunked) {
    const long long chunks = (long long)c * plan.pa.nchunks;
    pnms_prep_sort_chunk<<<(int)min(chunks, 148LL * 2), kSortThreads, plan.sort_smem, cudaStreamTailLaunch>>>(plan.pa);
    const long long blocks = (long long)c * ((plan.pa.n_max + 255) / 256);
    pnms_merge_rank<<<(int)min(blocks, 148LL * 8), 256, 0, cudaStreamTailLaunch>>>(plan.pa);
  } else {
    pnms_prep_sort_frame_list<<<min(c, 148 * 2), kSortThreads, plan.sort_smem, cudaStreamTailLaunch>>>(plan.pa);
  }
  const int map_grid = (int)min((long long)c * plan.ma.items_per_frame, 148LL * 8);
  if (plan.map_R == 4)
    pnms_map_kernel_list<4><<<map_grid, kMapWarps * 32, plan.map_smem, cudaStreamTailLaunch>>>(plan.ma);
  else if (plan.map_R == 2)
    pnms_map_kernel_list<2><<<map_grid, kMapWarps * 32, plan.map_smem, cudaStreamTailLaunch>>>(plan.ma);
  else
    pnms_map_kernel_list<1><<<map_grid, kMapWarps * 32, plan.map_smem, cudaStreamTailLaunch>>>(plan.ma);
  pnms_compact<<<min(c, 148 * 4), kCompactThreads, plan.compact_smem, cudaStreamTailLaunch>>>(plan.ca);
  // a chain that could not be launched would leave the declined frames without output: fail
  // loudly (the stream reports the fault at the caller's next synchronisation)
  if (cudaGetLastError() != cudaSuccess) __trap();
}

// One CTA, launched programmatically right after the binned kernel: waits for it, snapshots
// and zeroes the declined-frame count, and tail-launches the chain sized to it.  It must not
// trigger its own dependents (griddepcontrol.launch_dependents in a grid that tail-launches
// keeps the tail launch from ever starting — measured on B200).
__global__ void __launch_bounds__(32) pnms_fallback_dispatch(FallbackPlan plan, int* decl_count, int* count_snap) {
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the binned grid is complete and flushed
  if (threadIdx.x != 0) return;
  const int c = min(max(*decl_count, 0), plan.pa.batch);  // a workspace that was not zeroed
  *decl_count = 0;                                          // cannot send the chain out of range
  *count_snap = c;
  if (c == 0 || !plan.enabled) return;
  launch_fallback_chain(plan, c);
}
#endif

}  // namespace pnms
