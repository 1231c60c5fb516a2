// pnms_gate.cuh — WorkCounters.map_writes (engine.py:134-153, 236-237) for every device path.
//
// The reference counts the ordered slot pairs (i, j) of the d_max x d_max map, padding slots
// included, that pass its gate (engine.py:233-235):
//     s_i < s_j   or   (tie_break == by_index  and  s_i == s_j  and  i > j)
// Every comparison with a NaN is false and a slot never gates itself.  Over the m non-NaN
// slots of a frame, an unordered pair of distinct scores therefore passes in exactly one
// direction, and a pair of equal scores in one direction under by_index, in none under
// paper_faithful:
//     map_writes = C(m, 2) - [paper_faithful] * sum over equal-score groups g of C(|g|, 2)
// The padding slots (0, 0, 0, 0.0) are one group together with the valid scores equal to
// zero (-0.0 == +0.0).  The culling paths never visit most pairs, so the count is computed
// here from the scores alone: each non-zero, non-NaN score is inserted into a per-frame
// open-addressing hash table in the workspace; the insert's previous multiplicity is the
// number of equal-score pairs it closes (sum_g C(|g|, 2) = sum over inserts of the count
// before the insert).  A second kernel adds the zero group and writes the counter.
#pragma once
#include "pnms_common.cuh"
#include "pnms_sort.cuh"  // frame_count

namespace pnms {

constexpr int kGateThreads = 256;

struct GateArgs {
  const double* s;
  const int32_t* counts;  // may be null: every frame has n_max valid slots
  int batch, n_max, d_max, tie_break;
  int cap;                          // hash slots per frame (2 * n_max)
  unsigned long long* keys;         // [batch][cap] zeroed: score_key of the score, 0 = empty
  uint32_t* mult;                   // [batch][cap] zeroed: inserts so far
  unsigned long long* acc;          // [batch][2] zeroed: equal-score pairs; NaN | zeros << 32
  unsigned long long* gate_pairs;   // [batch] out
};

__device__ __forceinline__ uint32_t gate_hash(uint64_t key, uint32_t cap) {
  const uint64_t h = key * 0x9E3779B97F4A7C15ull;
  return __umulhi((uint32_t)(h >> 32), cap);
}

// grid (ceil(n_max / kGateThreads), batch)
__global__ void __launch_bounds__(kGateThreads) pnms_gate_ties(GateArgs a) {
  const int f = blockIdx.y;
  const int e = blockIdx.x * kGateThreads + threadIdx.x;
  const int cnt = frame_count(a.counts, f, a.n_max);
  unsigned long long ties = 0, nz = 0;  // NaN count | zero count << 32
  if (e < cnt) {
    const double v = a.s[(long long)f * a.n_max + e];
    if (v != v) {
      nz = 1ull;
    } else if (v == 0.0) {
      nz = 1ull << 32;
    } else {
      const uint64_t key = score_key(v);  // > 0 for every non-NaN score
      unsigned long long* keys = a.keys + (long long)f * a.cap;
      uint32_t h = gate_hash(key, (uint32_t)a.cap);
      for (;;) {
        const unsigned long long old = atomicCAS(keys + h, 0ull, (unsigned long long)key);
        if (old == 0ull || old == key) {
          ties = atomicAdd(a.mult + (long long)f * a.cap + h, 1u);
          break;
        }
        h = h + 1 == (uint32_t)a.cap ? 0u : h + 1;  // load factor <= 1/2: short probes
      }
    }
  }
  ties = __reduce_add_sync(0xFFFFFFFFu, (unsigned)ties);
  const unsigned nan_c = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(nz & 0xFFFFFFFFu));
  const unsigned zero_c = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(nz >> 32));
  if ((threadIdx.x & 31) == 0 && (ties | nan_c | zero_c)) {
    if (ties) atomicAdd(a.acc + 2LL * f, ties);
    if (nan_c | zero_c) atomicAdd(a.acc + 2LL * f + 1, (unsigned long long)nan_c | ((unsigned long long)zero_c << 32));
  }
}

// grid ceil(batch / kGateThreads)
__global__ void __launch_bounds__(kGateThreads) pnms_gate_finalize(GateArgs a) {
  const int f = blockIdx.x * kGateThreads + threadIdx.x;
  if (f >= a.batch) return;
  const long long cnt = frame_count(a.counts, f, a.n_max);
  const unsigned long long ties = a.acc[2LL * f], nz = a.acc[2LL * f + 1];
  const long long nan_c = (long long)(nz & 0xFFFFFFFFull), zero_c = (long long)(nz >> 32);
  const long long pad = (long long)a.d_max - cnt;               // implicit padding slots
  const unsigned long long m = (unsigned long long)(cnt - nan_c + pad);
  const unsigned long long zeros = (unsigned long long)(zero_c + pad);
  unsigned long long writes = m * (m - (m > 0)) / 2;             // C(m, 2)
  if (a.tie_break == 0) writes -= ties + zeros * (zeros - (zeros > 0)) / 2;
  a.gate_pairs[f] = writes;
}

}  // namespace pnms
