// pnms_reflayout.cuh — the reference's phase API on the device, in the reference's own
// bit layout: map_phase (engine.py:176-250) writes the full d_max x d_max SuppressionMatrix
// (engine.py:74-111) and reduce_phase (engine.py:253-281) folds its rows.  These are the
// parity/debug surface behind the drop-in `map_phase` / `reduce_phase`; the production path
// (pnms_run) never materialises the matrix.
//
// One warp produces one 64-bit matrix word: lane l evaluates columns 64w+l and 64w+32+l and
// two ballots assemble the word, which is bit-for-bit the little-endian packbits layout
// (bit j of a row = byte j/8 bit j%8 = uint64 word j/64 bit j%64).
#pragma once
#include "pnms_common.cuh"

namespace pnms {

struct RefMapArgs {
  const int32_t *x, *y, *z;
  const double* s;
  int d_max, W64, tie_break;
  double theta;
  uint64_t* bits;
  unsigned long long* gate_pairs;
};

// exact cell value of engine.py:219-239 for one ordered pair; *gate gets the score gate
__device__ __forceinline__ bool ref_cell(const RefMapArgs& a, int i, int j, int32_t xi, int32_t yi, int32_t zi,
                                         double si, bool* gate) {
  const int32_t xj = a.x[j], yj = a.y[j], zj = a.z[j];
  const double sj = a.s[j];
  const int32_t xei = (int32_t)((uint32_t)xi + (uint32_t)zi), yei = (int32_t)((uint32_t)yi + (uint32_t)zi);
  const int32_t xej = (int32_t)((uint32_t)xj + (uint32_t)zj), yej = (int32_t)((uint32_t)yj + (uint32_t)zj);
  int32_t w = (int32_t)((uint32_t)min(xei, xej) - (uint32_t)max(xi, xj) + 1u);
  int32_t h = (int32_t)((uint32_t)min(yei, yej) - (uint32_t)max(yi, yj) + 1u);
  w = max(w, 0);
  h = max(h, 0);
  const double prod = __dmul_rn((double)w, (double)h);
  const bool keep = (prod < ref_threshold(a.theta, zj)) && (zj != 0);
  bool g = si < sj;
  if (a.tie_break == 1) g = g || (si == sj && i > j);
  *gate = g;
  return keep || !g;
}

__global__ void __launch_bounds__(256) pnms_ref_map(RefMapArgs a) {
  __shared__ unsigned long long blk_gate;
  if (threadIdx.x == 0) blk_gate = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long unit = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  const long long n_units = (long long)a.d_max * a.W64;
  unsigned gcount = 0;
  if (unit < n_units) {
    const int i = (int)(unit / a.W64), w = (int)(unit % a.W64);
    const int32_t xi = a.x[i], yi = a.y[i], zi = a.z[i];
    const double si = a.s[i];
    const int j0 = w * 64 + lane, j1 = j0 + 32;
    bool g0 = false, g1 = false;
    const bool b0 = (j0 < a.d_max) ? ref_cell(a, i, j0, xi, yi, zi, si, &g0) : true;
    const bool b1 = (j1 < a.d_max) ? ref_cell(a, i, j1, xi, yi, zi, si, &g1) : true;
    const uint32_t lo = __ballot_sync(0xFFFFFFFFu, b0), hi = __ballot_sync(0xFFFFFFFFu, b1);
    gcount = __popc(__ballot_sync(0xFFFFFFFFu, g0)) + __popc(__ballot_sync(0xFFFFFFFFu, g1));
    if (lane == 0) {
      a.bits[unit] = ((uint64_t)hi << 32) | lo;
      if (gcount) atomicAdd(&blk_gate, (unsigned long long)gcount);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.gate_pairs && blk_gate) atomicAdd(a.gate_pairs, blk_gate);
}

// reduce: one warp per row, 8 rows (one output byte) per CTA
__global__ void __launch_bounds__(256) pnms_ref_reduce(const uint64_t* bits, int d_max, int W64, uint8_t* mask) {
  __shared__ uint32_t row_ok[8];
  const int lane = threadIdx.x & 31, wr = threadIdx.x >> 5;
  const int i = blockIdx.x * 8 + wr;
  bool ok = false;
  if (i < d_max) {
    bool all = true;
    for (int w = lane; w < W64; w += 32) {
      uint64_t v = bits[(long long)i * W64 + w];
      const int valid = d_max - w * 64;  // bits of this word that lie inside the row
      if (valid < 64) v |= ~0ull << valid;
      all &= (v == ~0ull);
    }
    ok = __all_sync(0xFFFFFFFFu, all);
  }
  if (lane == 0) row_ok[wr] = ok ? 1u : 0u;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t byte = 0;
    for (int r = 0; r < 8; ++r) byte |= row_ok[r] << r;
    mask[blockIdx.x] = (uint8_t)byte;
  }
}

}  // namespace pnms
