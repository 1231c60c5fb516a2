// pnms_validate.cuh — device-side ingest validation (detections.py:60-85).
//
// The reference validates every Detection on the host while building a DetectionVector
// (detections.py:125-127): integer coordinates in [0, COORD_LIMIT), side z >= 1, finite
// score s > 0.  This kernel applies the same invariants to device-resident planes and
// reports, per frame, the first offending slot and which check failed, so the host can raise
// the reference's ValidationError for that detection with a single small copy.
#pragma once
#include "pnms_common.cuh"
#include "pnms_sort.cuh"

namespace pnms {

constexpr int32_t kCoordLimit = 1 << 24;  // detections.py:22

// reason codes (match paper_2502_00535_b200/_lib.py)
enum ValidateReason : int {
  kValid = 0,
  kNegX = 1, kNegY = 2, kNegZ = 3,
  kBigX = 4, kBigY = 5, kBigZ = 6,
  kSideLt1 = 7,
  kScoreNotFinite = 8,
  kScoreNotPositive = 9
};

__device__ __forceinline__ int validate_one(int32_t x, int32_t y, int32_t z, double s) {
  // same order of checks as Detection.validate: x, y, z ranges, then side, then score
  if (x < 0) return kNegX;
  if (x >= kCoordLimit) return kBigX;
  if (y < 0) return kNegY;
  if (y >= kCoordLimit) return kBigY;
  if (z < 0) return kNegZ;
  if (z >= kCoordLimit) return kBigZ;
  if (z < 1) return kSideLt1;
  if (!isfinite(s)) return kScoreNotFinite;
  if (s <= 0.0) return kScoreNotPositive;
  return kValid;
}

// One CTA per frame: first_bad[f] = smallest invalid slot index (or -1), reason[f] its code.
__global__ void __launch_bounds__(256) pnms_validate_kernel(const int32_t* x, const int32_t* y, const int32_t* z,
                                                            const double* s, const int32_t* counts, int n_max,
                                                            int32_t* first_bad, int32_t* reason) {
  __shared__ int s_first;
  const int f = blockIdx.x;
  const long long fbase = (long long)f * n_max;
  const int cnt = frame_count(counts, f, n_max);
  if (threadIdx.x == 0) s_first = 0x7FFFFFFF;
  __syncthreads();
  // 16 B vector loads when the frame's slots are 16 B aligned (HBM streaming), else scalar
  const bool vec = ((fbase & 3) == 0) && ((((uintptr_t)x) | ((uintptr_t)y) | ((uintptr_t)z) | ((uintptr_t)s)) & 15) == 0;
  const int nv = vec ? cnt / 4 : 0;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    const long long g = fbase + 4LL * v;
    const int4 X = *reinterpret_cast<const int4*>(x + g), Y = *reinterpret_cast<const int4*>(y + g);
    const int4 Z = *reinterpret_cast<const int4*>(z + g);
    const double2 S0 = *reinterpret_cast<const double2*>(s + g), S1 = *reinterpret_cast<const double2*>(s + g + 2);
    // the smallest invalid slot of the four (atomicMin keeps the frame's smallest overall)
    int bad = 0x7FFFFFFF;
    if (validate_one(X.w, Y.w, Z.w, S1.y) != kValid) bad = 4 * v + 3;
    if (validate_one(X.z, Y.z, Z.z, S1.x) != kValid) bad = 4 * v + 2;
    if (validate_one(X.y, Y.y, Z.y, S0.y) != kValid) bad = 4 * v + 1;
    if (validate_one(X.x, Y.x, Z.x, S0.x) != kValid) bad = 4 * v;
    if (bad != 0x7FFFFFFF) atomicMin(&s_first, bad);
  }
  for (int e = 4 * nv + threadIdx.x; e < cnt; e += blockDim.x) {
    const long long g = fbase + e;
    if (validate_one(x[g], y[g], z[g], s[g]) != kValid) atomicMin(&s_first, e);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int e = s_first;
    first_bad[f] = e == 0x7FFFFFFF ? -1 : e;
    reason[f] = e == 0x7FFFFFFF ? kValid : validate_one(x[fbase + e], y[fbase + e], z[fbase + e], s[fbase + e]);
  }
}

}  // namespace pnms
