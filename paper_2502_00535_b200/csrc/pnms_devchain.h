// pnms_devchain.h — host entry points of the relocatable unit pnms_devchain.cu (internal to
// libparnms_b200.so; the C ABI is include/parnms_b200.h).  Arguments are plain types: the
// FallbackPlan block is the same header-defined struct in both units (checked by size).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

#define PNMS_INTERNAL __attribute__((visibility("hidden")))

PNMS_INTERNAL size_t pnms_devchain_plan_size();
// dynamic shared memory limits of the list kernels the dispatcher may tail-launch
PNMS_INTERNAL cudaError_t pnms_devchain_prepare(int chunked, int map_R, int sort_smem, size_t map_smem,
                                                size_t compact_smem);
// pnms_fallback_dispatch<<<1, 32>>> behind the binned kernel (programmatic dependent launch);
// `plan` points at a FallbackPlan
PNMS_INTERNAL cudaError_t pnms_devchain_dispatch(const void* plan, int* decl_count, int* count_snap,
                                                 cudaStream_t stream);
