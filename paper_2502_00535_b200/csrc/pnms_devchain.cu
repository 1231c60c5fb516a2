// pnms_devchain.cu — the relocatable-device-code unit: the one-CTA dispatcher and the list
// kernels of the dense pipeline it tail-launches for frames the binned kernel declined
// (pnms_fallback.cuh).  Compiled with -rdc=true and linked against cudadevrt; the
// namespace is renamed to pnms_dc so these kernels never collide with the whole-program
// copies in pnms_capi.cu (the host-launched chain of the large-frame paths).
#include <atomic>
#define PNMS_DEVICE_CHAIN 1
#define pnms pnms_dc
#include "pnms_fallback.cuh"
#undef pnms
#include "pnms_devchain.h"

namespace {

// the largest dynamic shared memory each list kernel has been opened up to, per device
// (function attributes are per device)
constexpr int kMaxDevices = 64;
struct SmemCache {
  std::atomic<size_t> v[kMaxDevices];
};

template <class Kernel>
cudaError_t ensure_smem_dc(Kernel kernel, size_t bytes, SmemCache& c) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  std::atomic<size_t>& slot = c.v[dev];
  if (bytes <= 48 * 1024 || slot.load(std::memory_order_relaxed) >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) slot.store(bytes, std::memory_order_relaxed);
  return e;
}

}  // namespace

size_t pnms_devchain_plan_size() { return sizeof(pnms_dc::FallbackPlan); }

cudaError_t pnms_devchain_prepare(int chunked, int map_R, int sort_smem, size_t map_smem, size_t compact_smem) {
  static SmemCache scfg, kcfg, mcfg[5], ccfg;
  cudaError_t e = chunked ? ensure_smem_dc(pnms_dc::pnms_prep_sort_chunk, (size_t)sort_smem, kcfg)
                          : ensure_smem_dc(pnms_dc::pnms_prep_sort_frame_list, (size_t)sort_smem, scfg);
  if (e != cudaSuccess) return e;
  if (map_R == 4) e = ensure_smem_dc(pnms_dc::pnms_map_kernel_list<4>, map_smem, mcfg[4]);
  else if (map_R == 2) e = ensure_smem_dc(pnms_dc::pnms_map_kernel_list<2>, map_smem, mcfg[2]);
  else e = ensure_smem_dc(pnms_dc::pnms_map_kernel_list<1>, map_smem, mcfg[1]);
  if (e != cudaSuccess) return e;
  return ensure_smem_dc(pnms_dc::pnms_compact, compact_smem, ccfg);
}

cudaError_t pnms_devchain_dispatch(const void* plan, int* decl_count, int* count_snap, cudaStream_t st) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(1);
  lc.blockDim = dim3(32);
  lc.dynamicSmemBytes = 0;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, pnms_dc::pnms_fallback_dispatch, *static_cast<const pnms_dc::FallbackPlan*>(plan),
                            decl_count, count_snap);
}

